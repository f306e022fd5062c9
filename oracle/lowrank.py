"""LDL^T factor algebra (oracle; test infrastructure only).

P ~ L D L^T, L in R^{n x r}, D in R^{r x r} symmetric (§2).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def concat(L1, D1, L2, D2, weight=1.0):
    """[L1, L2], blkdiag(D1, weight*D2) — the T2 factorisation (eq. after)."""
    L = np.hstack([L1, L2])
    D = sla.block_diag(D1, weight * D2) if (D1.size or D2.size) else np.zeros((0, 0))
    return L, D


def column_compression(L, D, tol=1e-16, rank_cap=None):
    """Column compression exactly as P:L245-246 states it:
    "we employ a reduced SVD factorization, followed by a diagonalization of the small
    resulting system".
      1. reduced SVD  L = U Sigma V^T                         (numpy LAPACK gesdd)
      2. small system M = Sigma V^T D V Sigma, diagonalise M = W Theta W^T  (eigh)
      3. keep |theta_i| > tol * max|theta|  (relative reading G7), sorted by |theta|
         descending (stable), at most `rank_cap` of them (reading G8)
      4. L <- U W_kept,  D <- diag(theta_kept)
    Rank-0 input returns rank-0 output.
    """
    n = L.shape[0]
    if L.shape[1] == 0:
        return np.zeros((n, 0)), np.zeros((0, 0))
    U, s, Vt = np.linalg.svd(L, full_matrices=False)
    M = (s[:, None] * (Vt @ D @ Vt.T)) * s[None, :]
    M = 0.5 * (M + M.T)
    theta, W = np.linalg.eigh(M)
    order = np.argsort(-np.abs(theta), kind="stable")
    theta, W = theta[order], W[:, order]
    top = abs(theta[0]) if theta.size else 0.0
    if top == 0.0:
        return np.zeros((n, 0)), np.zeros((0, 0))
    r = int(np.count_nonzero(np.abs(theta) > tol * top))
    if rank_cap is not None:
        r = min(r, int(rank_cap))
    return U @ W[:, :r], np.diag(theta[:r])


def to_dense(L, D):
    """P = L D L^T, symmetrised (test support)."""
    P = L @ D @ L.T
    return 0.5 * (P + P.T)


def rel_diff(L1, D1, L2, D2):
    """||L1 D1 L1^T - L2 D2 L2^T||_F / ||L2 D2 L2^T||_F without forming n x n matrices.

    QR of the stacked factor [L1, L2] = Q Rt; the difference is Q (Rt K Rt^T) Q^T with the
    core K = blkdiag(D1, -D2), so its Frobenius norm is ||Rt K Rt^T||_F (Q orthonormal).
    (the trace identity cancels catastrophically; this does not.)
    """
    n = L1.shape[0]
    if L2.shape[1] == 0:
        return float(np.linalg.norm(to_dense(L1, D1))) if L1.shape[1] else 0.0
    Ls = np.hstack([L1, L2])
    K = sla.block_diag(D1, -D2) if L1.shape[1] else -D2
    _, Rt = np.linalg.qr(Ls, mode="reduced")
    num = np.linalg.norm(Rt @ K @ Rt.T)
    _, R2 = np.linalg.qr(L2, mode="reduced")
    den = np.linalg.norm(R2 @ D2 @ R2.T)
    return float(num / den) if den > 0 else float(num)
