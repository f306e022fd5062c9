"""GPU parity at BASELINE.json's full size (config 5: n = 10000, rank cap 64, h = 0.005, Strang F12F3,
the configuration bench.py times), on outputs the oracle can compute one by one:
  * sampled entries of E_{h/2} and E_h against the DST closed form (exact at any n, pin P5);
  * sampled rows of one T1 pass E_{h/2} L against closed-form rows of E_{h/2};
  * the quadrature factor L_I(h/2) against the oracle's direct composite rule (P-level metric);
  * three Strang F12F3 steps (FSAL merge on and off) against the oracle (1e-10).
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from oracle import exact, flows, lowrank, quadrature  # noqa: E402
from oracle.schemes import OracleOptions, OracleSolver  # noqa: E402
from workloads import make_config  # noqa: E402

H = 0.005
NX = 100


@pytest.fixture(scope="module")
def prob():
    return make_config(5)


@pytest.fixture(scope="module")
def solver(prob):
    import paper_1805_08990_b200 as dme
    s = dme.Solver(**dme.problem_kwargs(prob), h=H, rank_cap=64)
    yield s
    s.close()


def test_fullsize_expm_sampled(solver):
    assert solver.stats()["expm_chebyshev"] == 1  # sparse symmetric A: Chebyshev-built E_{h/2}
    rng = np.random.default_rng(0)
    n = NX * NX
    rows = np.concatenate([rng.integers(0, n, 3000), np.arange(0, n, 97)])
    cols = np.concatenate([rng.integers(0, n, 3000), np.arange(0, n, 97)])
    # near-diagonal entries carry the mass of a heat kernel
    rows = np.concatenate([rows, rng.integers(0, n, 2000)])
    cols = np.concatenate([cols, np.clip(rows[-2000:] + rng.integers(-NX - 2, NX + 3, 2000), 0, n - 1)])
    for which, t in ((0, H / 2), (1, H)):
        E = solver.debug_get_exp(which)
        ref = exact.heat_expm_entries(NX, t, rows, cols)
        # normwise FP64 accuracy: ||E||_inf = 1 (heat semigroup); the int8 digit-sliced init
        # products measure 4.8e-16 here, the FP64 DMMA products 1e-16
        err = np.abs(E[rows, cols] - ref).max()
        assert err <= 2e-15 * np.abs(E).sum(axis=1).max(), (which, err)
        # symmetry of the symmetric-A path
        assert np.array_equal(E[rows, cols], E[cols, rows])


def test_fullsize_expm_pade_sampled(prob):
    """The same sampled check for the Padé-13 scaling-and-squaring E (options.expm = PADE; the
    default builds E_{h/2} of this sparse symmetric A by Chebyshev actions)."""
    import paper_1805_08990_b200 as dme
    s = dme.Solver(**dme.problem_kwargs(prob), h=H, rank_cap=64, expm="pade")
    assert s.stats()["expm_chebyshev"] == 0
    rng = np.random.default_rng(7)
    n = NX * NX
    rows = rng.integers(0, n, 4000)
    cols = np.clip(rows + rng.integers(-NX - 2, NX + 3, 4000), 0, n - 1)
    for which, t in ((0, H / 2), (1, H)):
        E = s.debug_get_exp(which)
        ref = exact.heat_expm_entries(NX, t, rows, cols)
        assert np.abs(E[rows, cols] - ref).max() <= 2e-15 * np.abs(E).sum(axis=1).max()
    s.close()


def test_fullsize_T1_sampled_rows(prob):
    import paper_1805_08990_b200 as dme
    s = dme.Solver(A=prob.A, h=H)
    L = np.random.default_rng(1).random((prob.n, 64))
    s.debug_set_factor(L)
    s.debug_apply("T1", H / 2)
    Y, _ = s.get_factor()
    s.close()
    E1 = exact.heat_expm_closed_form(NX, H / 2, 1)
    for i in np.random.default_rng(2).integers(0, prob.n, 25):
        Erow = np.kron(E1[i // NX], E1[i % NX])  # row i of E = E1 (x) E1
        ref = Erow @ L
        assert np.abs(Y[i] - ref).max() <= 1e-13 * np.abs(Erow) @ np.abs(L).max(axis=1)


def test_fullsize_integral_factor(prob, solver):
    op = flows.Operator(prob.A, "heat", NX, 2)
    delta = quadrature.panel_width(prob.A, H)
    st = solver.stats()
    assert abs(st["panel_width"] - delta) <= 1e-15 * delta
    assert st["quad_panels"] == 64
    Lg = solver.debug_get_integral(0)
    Lo, Do = flows.build_integral(op, H / 2, delta, 14, prob.C.T, np.eye(2), 1e-16)
    assert lowrank.rel_diff(Lg, np.eye(Lg.shape[1]), Lo, Do) <= 1e-12


@pytest.mark.parametrize("fsal", [True, False])
def test_fullsize_three_steps(prob, fsal):
    import paper_1805_08990_b200 as dme
    s = dme.Solver(**dme.problem_kwargs(prob), h=H, rank_cap=64, fsal=fsal)
    s.split_step("strang", "F12F3", 3)
    Lg, Dg = s.get_factor()
    s.close()
    orc = OracleSolver(prob, H, OracleOptions(rank_cap=64))
    orc.step("strang", "F12F3", 3)
    Lo, Do = orc.factor()
    d = lowrank.rel_diff(Lg, Dg, Lo, Do)
    assert d <= 1e-10, (d, Lg.shape[1], Lo.shape[1])
