"""GPU: the Padé-13 denominator solve with partial pivoting (the paper's solves are
pivoted LU: MATLAB backslash, and a dense LU).

q13(X) for X = a J (J a skew 2x2 block, J^2 = -I) is alpha I + beta J: a normal matrix with
kappa = 1, but alpha -> 0 at a = pi (< theta_13 = 5.37, so no scaling applies). Without row
exchanges the elimination divides by alpha; with partial pivoting it swaps in the beta row.
A = omega (J (x) I_m) puts the partner row m rows away, so the pivot search must cross panels.
The reference is scipy.linalg.expm (Al-Mohy-Higham), independent of this build.
"""
import numpy as np
import pytest
import scipy.linalg as sla

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dme():
    import torch
    assert torch.cuda.is_available()
    import paper_1805_08990_b200 as m
    return m


def _skew_problem(m, omega, seed):
    J = np.array([[0.0, 1.0], [-1.0, 0.0]])
    A = omega * np.kron(J, np.eye(m))
    n = 2 * m
    rng = np.random.default_rng(seed)
    return dict(A=A, C=rng.uniform(size=(1, n)), L0=rng.uniform(size=(n, 2)),
                B=rng.uniform(size=(n, 1)), R=np.eye(1))


@pytest.mark.parametrize("m", [40, 300])
@pytest.mark.parametrize("delta", [1e-7, -1e-7, 1e-10, -1e-10])
@pytest.mark.parametrize("e_pass", ["auto", "dmma"])
def test_pade_skew_pivoting(dme, m, delta, e_pass):
    h = 0.01
    tau = h / 2
    omega = np.pi * (1 + delta) / tau            # ||tau A^T||_1 = pi (1 + delta): s = 0
    kw = _skew_problem(m, omega, seed=m)
    s = dme.Solver(**kw, h=h, expm="pade", e_pass=e_pass)
    st = s.stats()
    assert st["squarings"] == 0
    for which, t in ((0, tau), (1, h)):
        E = s.debug_get_exp(which)
        ref = sla.expm(t * kw["A"].T)
        err = np.abs(E - ref).max()
        assert err <= 1e-13, (which, err)
    s.close()


@pytest.mark.parametrize("n,seed", [(130, 1), (700, 2)])
def test_pade_random_nonsymmetric_needs_pivoting(dme, n, seed):
    """A dense random nonsymmetric A with a row permutation that puts tiny leading minors into
    q13(X): expm through the pivoted solve against scipy."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    A = rng.standard_normal((n, n)) / np.sqrt(n)
    A = 3.0 * A[perm]                         # nonsymmetric, rows shuffled
    h = 0.2
    kw = dict(A=A, C=rng.uniform(size=(1, n)), B=rng.uniform(size=(n, 1)), R=np.eye(1))
    s = dme.Solver(**kw, h=h, expm="pade")
    for which, t in ((0, h / 2), (1, h)):
        E = s.debug_get_exp(which)
        ref = sla.expm(t * A.T)
        assert np.abs(E - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
    s.close()


def _biharmonic(nx):
    from workloads import heat2d_matrix
    L = heat2d_matrix(nx)
    return -(L @ L)   # symmetric, 13 nonzeros per row, NOT diagonally dominant: Gershgorin b >> 0


@pytest.mark.parametrize("h", [2e-4, 2e-5])
def test_auto_expm_gate_non_diagonally_dominant(dme, h):
    """AUTO may build E by Chebyshev actions only when the expansion is accurate: for -L^2 the
    Gershgorin bound b >> lambda_max, the truncation error would be e^{tau (b - lambda_max)} times
    the tail (relative error 1e14 at tau = 1e-4); the gate sends it to Padé-13."""
    nx = 12
    A = _biharmonic(nx)
    n = A.shape[0]
    rng = np.random.default_rng(3)
    kw = dict(A=A, C=rng.uniform(size=(1, n)), B=rng.uniform(size=(n, 1)), R=np.eye(1))
    s = dme.Solver(**kw, h=h)
    for which, t in ((0, h / 2), (1, h)):
        E = s.debug_get_exp(which)
        ref = sla.expm(t * A.T)
        assert np.abs(E - ref).max() <= 1e-13 * np.abs(ref).max(), (which, np.abs(E - ref).max())
    s.close()
    import scipy.sparse as sps
    kw["A"] = sps.csr_matrix(A)
    with pytest.raises(dme.DmeError):
        dme.Solver(**kw, h=h)


def test_auto_expm_gate_keeps_heat_on_chebyshev(dme):
    from workloads import make_config
    prob = make_config(5, nx=20)
    s = dme.Solver(**dme.problem_kwargs(prob), h=0.005)
    assert s.stats()["expm_chebyshev"] == 1
    s.close()
