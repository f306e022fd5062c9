"""Complement basis of the refined compression (reading G7'; P:L245-246 tail pass):
U (k x (k - kb)) must be an orthonormal basis of span(W)^perp, i.e. [W U] orthogonal. Checked
through the C ABI test hook for the LU-reconstruction kernel (k <= 96) and the column-by-column
Householder kernel (k > 96), including the degenerate kb = 0 and kb = k - 1 cases."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,kb", [(92, 35), (57, 20), (96, 95), (96, 1), (10, 0), (3, 1), (64, 63),
                                  (48, 24), (120, 50), (160, 20)])
def test_complement_orthonormal(k, kb):
    import paper_1805_08990_b200 as dme
    rng = np.random.default_rng(1000 + 7 * k + kb)
    W, _ = np.linalg.qr(rng.standard_normal((k, kb))) if kb else (np.zeros((k, 0)), None)
    # eigenvector-like columns: random signs and a few nearly axis-aligned ones
    if kb >= 3:
        W[:, 0] = 0.0
        W[:, 0] = np.eye(k)[:, 1] * 0.999999 + 1e-3 * rng.standard_normal(k) * 1e-3
        W, _ = np.linalg.qr(W)
    U = dme.complement_basis(W)
    assert U.shape == (k, k - kb)
    Q = np.hstack([W, U])
    assert np.abs(Q.T @ Q - np.eye(k)).max() < 1e-13
