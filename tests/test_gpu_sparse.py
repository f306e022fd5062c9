"""Sparse-A path (include/dme.h A_rowptr): every E_tau L action is a Chebyshev
expansion of exp on the Gershgorin interval of tau A^T (csrc/cheb.cu), no dense exponential is
built. The result it approximates has a plain definition, exp(tau A^T) L, so the checks are:
  * one action against scipy.linalg.expm (small n, ragged column counts, substepped degrees);
  * whole schemes against the oracle (dense exponential, same quadrature rule) at 1e-10 (P-level)
    and against the dense GPU path;
  * invariants: A = 0 (empty CSR) gives exp(0) = I, so Strang F1F2 yields P0 + T Q exactly (P13);
  * the configuration errors of the boundary (a loose Gershgorin bound, M with a sparse A, bad CSR);
  * a nonsymmetric sparse A through the Taylor route of the same kernels.
"""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sps

pytestmark = pytest.mark.gpu

from oracle import lowrank  # noqa: E402
from oracle.schemes import OracleOptions, OracleSolver  # noqa: E402
from workloads import make_config  # noqa: E402

TOL_P = 1e-10


@pytest.fixture(scope="module")
def dme():
    import torch
    assert torch.cuda.is_available()
    import paper_1805_08990_b200 as m
    return m


def _kw(dme, prob):
    kw = dme.problem_kwargs(prob)
    kw["A"] = sps.csr_matrix(prob.A)
    return kw


@pytest.mark.parametrize("cfg,kw,k,which", [(5, dict(nx=20), 37, "half"), (5, dict(nx=20), 64, "full"),
                                            (2, dict(nx=23), 9, "full"), (1, dict(n=100), 1, "half")])
def test_action_vs_expm(dme, cfg, kw, k, which):
    prob = make_config(cfg, **kw)
    h = 0.005 if cfg != 1 else 1e-3
    tau = h if which == "full" else h / 2
    s = dme.Solver(A=sps.csr_matrix(prob.A), h=h)
    L = np.random.default_rng(k).random((prob.n, k))
    s.debug_set_factor(L)
    s.debug_apply("T1", tau)
    Y, _ = s.get_factor()
    st = s.stats()
    s.close()
    ref = sla.expm(tau * prob.A.T) @ L
    # absolute error per column relative to the column scale (||exp(tau A^T)||_2 <= 1 here)
    err = np.abs(Y - ref).max(axis=0) / np.abs(L).max(axis=0)
    assert err.max() <= 1e-13, err.max()
    assert st["e_passes"] >= 1


def test_action_substepped_degree(dme):
    """gamma beyond one substep's degree cap (1D heat, tau = 0.25: gamma ~ 5100): the kernel runs
    several substeps; still FP64-accurate against expm."""
    prob = make_config(1, n=100)
    h = 0.5
    s = dme.Solver(A=sps.csr_matrix(prob.A), h=h)
    L = np.random.default_rng(3).random((prob.n, 5))
    s.debug_set_factor(L)
    s.debug_apply("T1", h)
    Y, _ = s.get_factor()
    s.close()
    ref = sla.expm(h * prob.A.T) @ L
    assert np.abs(Y - ref).max() <= 1e-13 * np.abs(L).max()


SCHEME_CASES = [
    (1, dict(n=100), "lie", "F1F2", 0.1, 40, {}),
    (2, dict(nx=20), "strang", "F12", 0.5, 20, dict(quad_nodes=5, quad_subpanels=4)),
    (2, dict(nx=20), "strang", "F1F2", 0.5, 20, {}),
    (4, dict(nx=12), "strang", "F12F3F4", 0.5, 20, {}),
    (4, dict(nx=12, dle=True), "strang", "F1F4F2", 0.5, 20, {}),
    (5, dict(nx=24), "strang", "F12F3", 0.5, 20, dict(rank_cap=64)),
    (5, dict(nx=33), "strang", "F1F2F3", 0.5, 20, dict(rank_cap=64)),
]


@pytest.mark.parametrize("cfg,kw,scheme,comp,T,N,opts", SCHEME_CASES)
def test_scheme_vs_oracle(dme, cfg, kw, scheme, comp, T, N, opts):
    prob = make_config(cfg, **kw)
    h = T / N
    s = dme.Solver(**_kw(dme, prob), h=h, **opts)
    s.split_step(scheme, comp, N)
    Lg, Dg = s.get_factor()
    st = s.stats()
    s.close()
    oo = OracleOptions(rank_cap=opts.get("rank_cap"), quad_nodes=opts.get("quad_nodes", 14),
                       quad_subpanels=opts.get("quad_subpanels", 1))
    orc = OracleSolver(prob, h, oo)
    orc.step(scheme, comp, N)
    Lo, Do = orc.factor()
    d = lowrank.rel_diff(Lg, Dg, Lo, Do)
    assert d <= TOL_P, (d, Lg.shape[1], Lo.shape[1])
    assert st["ozaki_passes"] == 0 and st["cheb_degree"] > 0
    # same rule as the dense GPU path
    sd = dme.Solver(**dme.problem_kwargs(prob), h=h, **opts)
    sd.split_step(scheme, comp, N)
    Ld, Dd = sd.get_factor()
    sd.close()
    assert lowrank.rel_diff(Lg, Dg, Ld, Dd) <= TOL_P


def test_zero_A_strang_F1F2_exact(dme):
    """A = 0 (CSR with no entries): exp(0) = I, so Strang F1F2 gives P0 + T Q (P13)."""
    prob = make_config(2, nx=7, dle=True)
    n, T, N = prob.n, 0.5, 10
    kw = _kw(dme, prob)
    kw["A"] = sps.csr_matrix((n, n))
    s = dme.Solver(**kw, h=T / N)
    s.split_step("strang", "F1F2", N)
    Lg, Dg = s.get_factor()
    s.close()
    P0 = prob.L0 @ prob.L0.T
    ref = P0 + T * prob.C.T @ prob.C
    P = Lg @ Dg @ Lg.T
    assert np.linalg.norm(P - ref) <= 1e-13 * np.linalg.norm(ref)


def test_sparse_errors(dme):
    from workloads import heat2d_matrix
    L = heat2d_matrix(10)  # -L^2: symmetric, Gershgorin bound far above lambda_max (accuracy gate)
    with pytest.raises(dme.DmeError) as e:
        dme.Solver(A=sps.csr_matrix(-(L @ L)), h=2e-4)
    assert e.value.code == 3
    prob = make_config(5, nx=8)
    A = sps.csr_matrix(prob.A)
    s = dme.Solver(A=A, h=0.01)
    with pytest.raises(dme.DmeError) as e:
        s.debug_get_exp(0)
    assert e.value.code == 3
    s.close()
    with pytest.raises(dme.DmeError) as e:
        dme.Solver(A=A, M=np.eye(prob.n), h=0.01)
    assert e.value.code == 3
    bad = A.copy()
    bad.indices = bad.indices.copy()
    bad.indices[3] = prob.n + 5  # column index out of range
    with pytest.raises(dme.DmeError) as e:
        dme.Solver(A=bad, h=0.01)
    assert e.value.code == 1


@pytest.mark.slow
def test_fullsize_sparse_three_steps(dme):
    """BASELINE config 5 at full size (n = 10^4) through the sparse path: oracle parity (1e-10)."""
    prob = make_config(5)
    h = 0.005
    s = dme.Solver(**_kw(dme, prob), h=h, rank_cap=64)
    s.split_step("strang", "F12F3", 3)
    Lg, Dg = s.get_factor()
    s.close()
    orc = OracleSolver(prob, h, OracleOptions(rank_cap=64))
    orc.step("strang", "F12F3", 3)
    Lo, Do = orc.factor()
    d = lowrank.rel_diff(Lg, Dg, Lo, Do)
    assert d <= TOL_P, d


def test_action_wide_rows_fallback_kernel(dme):
    """Rows wider than 5 entries (w = 9..13) take the shared-memory kernel (vectors and accumulator in
    shared memory, halo pushes in a separate phase): against expm."""
    rng = np.random.default_rng(11)
    n = 300
    Wr = sps.random(n, n, density=4.0 / n, random_state=12, format="csr")
    Wg = Wr + Wr.T                                   # symmetric nonnegative weights, ~8 per row
    Wg.setdiag(0.0)
    Wg.eliminate_zeros()
    deg = np.asarray(Wg.sum(axis=1)).ravel()
    # minus a weighted graph Laplacian: symmetric, negative semidefinite and diagonally dominant
    # (Gershgorin b = 0: the Chebyshev accuracy gate of dme.cu accepts it)
    A = sps.csr_matrix(-(sps.diags(deg) - Wg) * 50.0)
    assert np.diff(A.indptr).max() > 5
    h = 0.01
    s = dme.Solver(A=A, h=h)
    L = rng.random((n, 11))
    s.debug_set_factor(L)
    s.debug_apply("T1", h / 2)
    Y, _ = s.get_factor()
    s.close()
    ref = sla.expm((h / 2) * A.toarray().T) @ L
    assert np.abs(Y - ref).max() <= 1e-13 * np.abs(L).max()


@pytest.mark.slow
def test_action_large_n_fallback_kernel(dme):
    """n = 110^2 > 8 x 1280 rows: the shared-memory kernel; sampled rows against the closed form of
    the 2D heat exponential (pin P5)."""
    from oracle import exact
    nx, h = 110, 0.005
    prob = make_config(5, nx=nx)
    s = dme.Solver(A=sps.csr_matrix(prob.A), h=h)
    L = np.random.default_rng(4).random((prob.n, 13))
    s.debug_set_factor(L)
    s.debug_apply("T1", h)
    Y, _ = s.get_factor()
    s.close()
    E1 = exact.heat_expm_closed_form(nx, h, 1)
    for i in np.random.default_rng(5).integers(0, prob.n, 40):
        Erow = np.kron(E1[i // nx], E1[i % nx])
        assert np.abs(Y[i] - Erow @ L).max() <= 1e-13 * np.abs(L).max()


@pytest.mark.parametrize("nx", [5, 20, 33])
def test_dense_A_chebyshev_E_matches_pade(dme, nx):
    """Dense input, sparse symmetric A: the default init builds E_{h/2} by Chebyshev actions
    (options.expm = AUTO; n >= 17, else Padé); both E against the DST closed form (pin P5)."""
    from oracle import exact
    prob = make_config(5, nx=nx)
    h = 0.005
    sa = dme.Solver(**dme.problem_kwargs(prob), h=h, rank_cap=64)
    sp = dme.Solver(**dme.problem_kwargs(prob), h=h, rank_cap=64, expm="pade")
    assert sa.stats()["expm_chebyshev"] == (1 if prob.n >= 17 else 0)
    assert sp.stats()["expm_chebyshev"] == 0
    for which, t in ((0, h / 2), (1, h)):
        ref = exact.heat_expm_closed_form(nx, t, 2)
        for s in (sa, sp):
            E = s.debug_get_exp(which)
            assert np.abs(E - ref).max() <= 2e-15 * np.abs(ref).sum(axis=1).max()
            assert np.array_equal(E, E.T)
    sa.close()
    sp.close()


@pytest.mark.parametrize("nx,comp", [(10, "F12F3"), (16, "F1F2F3")])
def test_nonsymmetric_sparse_taylor(dme, nx, comp):
    """Nonsymmetric sparse A (config 3's convection-diffusion operator, the paper's advection
    setting P:L343-348): the cluster kernels evaluate the truncated Taylor series with scaling
    (Al-Mohy & Higham); against the oracle at 1e-10."""
    prob = make_config(3, nx=nx)
    h, N = 0.005, 5
    kw = dme.problem_kwargs(prob)
    kw["A"] = sps.csr_matrix(prob.A)
    s = dme.Solver(**kw, h=h, rank_cap=64)
    s.split_step("strang", comp, N)
    Lg, Dg = s.get_factor()
    s.close()
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64))
    o.step("strang", comp, N)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10


def test_nonsymmetric_action_vs_expm(dme):
    n = 300
    rng = np.random.default_rng(7)
    R = sps.random(n, n, density=4.0 / n, random_state=8, format="csr")
    A = sps.csr_matrix(R * 30.0 - sps.eye(n) * 60.0)          # nonsymmetric, non-normal
    h = 0.02
    s = dme.Solver(A=A, h=h)
    L = rng.random((n, 7))
    s.debug_set_factor(L)
    s.debug_apply("T1", h)
    Y, _ = s.get_factor()
    s.close()
    ref = sla.expm(h * A.toarray().T) @ L
    assert np.abs(Y - ref).max() <= 1e-12 * np.abs(ref).max()


def _with_env(key, fn):
    import os
    old = os.environ.get(key)
    os.environ[key] = "1"
    try:
        return fn()
    finally:
        if old is None:
            del os.environ[key]
        else:
            os.environ[key] = old


@pytest.mark.parametrize("cfg,nx,comp", [(5, 14, "F12F3"), (3, 12, "F12F3"), (5, 10, "F1F2F3")])
def test_global_mode_forced_small(dme, cfg, nx, comp):
    """The grid-wide action (large-n layout) forced at small n (DME_CHEB_GLOBAL): Chebyshev for the
    symmetric heat operator, Taylor for convection-diffusion; against the oracle at 1e-10."""
    prob = make_config(cfg, nx=nx)
    h, N = 0.005, 4
    kw = dme.problem_kwargs(prob)
    kw["A"] = sps.csr_matrix(prob.A)
    s = _with_env("DME_CHEB_GLOBAL", lambda: dme.Solver(**kw, h=h, rank_cap=64))
    s.split_step("strang", comp, N)
    Lg, Dg = s.get_factor()
    s.close()
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64))
    o.step("strang", comp, N)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10


@pytest.mark.slow
def test_large_n_beyond_one_cluster(dme):
    """n = 190^2 = 36100 (> 3e4; one 8-CTA cluster's shared memory holds ~1.2e4 rows): the sparse
    action runs grid-wide. One T1 action against the closed-form heat eigenbasis (pin P5), and
    three Strang F1F2F3 DRE steps against the oracle (1e-10)."""
    from oracle import flows
    nx, h = 190, 0.005
    prob = make_config(5, nx=nx)
    kw = dme.problem_kwargs(prob)
    kw["A"] = sps.csr_matrix(prob.A)
    s = dme.Solver(**kw, h=h, rank_cap=64)
    L = np.random.default_rng(9).random((prob.n, 11))
    s.debug_set_factor(L)
    s.debug_apply("T1", h)
    Y, _ = s.get_factor()
    s.close()
    op = flows.Operator(prob.A, "heat", nx, 2)
    ref = op.apply(h, L)
    assert np.abs(Y - ref).max() <= 1e-13 * np.abs(L).max()
    s = dme.Solver(**kw, h=h, rank_cap=64)
    s.split_step("strang", "F1F2F3", 3)
    Lg, Dg = s.get_factor()
    s.close()
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64))
    o.step("strang", "F1F2F3", 3)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10
