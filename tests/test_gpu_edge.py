"""GPU edge cases: tiny and ragged n, Q = 0, P0 = 0 and everything zero, m > 1 inputs (the tiny
m x m eigen path of the fused Riccati flow), rank collapse, configuration / validation errors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import lowrank  # noqa: E402
from oracle.schemes import OracleOptions, OracleSolver  # noqa: E402
from workloads import Problem, heat1d_matrix, heat2d_matrix, make_config  # noqa: E402


@pytest.fixture(scope="module")
def dme():
    import paper_1805_08990_b200 as m
    return m


def _run_both(dme, prob, h, scheme, comp, N, **kw):
    s = dme.Solver(**dme.problem_kwargs(prob), h=h, **kw)
    s.split_step(scheme, comp, N)
    Lg, Dg = s.get_factor()
    oo = OracleOptions(rank_cap=kw.get("rank_cap") or None)
    o = OracleSolver(prob, h, oo)
    o.step(scheme, comp, N)
    Lo, Do = o.factor()
    return Lg, Dg, Lo, Do


@pytest.mark.parametrize("n", [1, 2, 3, 17, 37])
def test_tiny_and_ragged_n(dme, n):
    rng = np.random.default_rng(n)
    prob = Problem(A=heat1d_matrix(n), C=rng.random((1, n)), L0=rng.random((n, min(2, n))),
                   D0=np.eye(min(2, n)), B=rng.random((n, 1)), R=np.eye(1), T=0.2)
    for comp in ("F12F3", "F1F3F2"):
        Lg, Dg, Lo, Do = _run_both(dme, prob, 0.02, "strang", comp, 10)
        assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10, (n, comp)


def test_two_inputs_m2(dme):
    """m = 2 columns of B with a non-diagonal R: the fused T3 evaluates g(F^T F) by the tiny
    m x m eigensolver (K^{-1/2} = I + F g(F^T F) F^T)."""
    prob = make_config(5, nx=9)
    rng = np.random.default_rng(3)
    prob.B = rng.random((prob.n, 2))
    prob.R = np.array([[2.0, 0.5], [0.5, 1.0]])
    for comp in ("F12F3", "F1F2F3"):
        Lg, Dg, Lo, Do = _run_both(dme, prob, 0.02, "strang", comp, 10)
        assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10, comp


def test_no_Q(dme):
    prob = make_config(2, nx=8)
    prob.C = None
    Lg, Dg, Lo, Do = _run_both(dme, prob, 0.02, "strang", "F1F2", 10)
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10
    Lg, Dg, Lo, Do = _run_both(dme, prob, 0.02, "strang", "F12", 10)
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10


def test_all_zero_and_P0_zero(dme):
    n = 16
    prob = Problem(A=heat1d_matrix(n), C=None, L0=None, D0=None, T=0.1)
    s = dme.Solver(**dme.problem_kwargs(prob), h=0.01)
    s.split_step("strang", "F12", 5)
    L, D = s.get_factor()
    assert L.shape == (n, 0) and D.shape == (0, 0)
    # P0 = 0 with Q != 0: the rank grows from zero
    prob.C = np.random.default_rng(0).random((1, n))
    Lg, Dg, Lo, Do = _run_both(dme, prob, 0.01, "strang", "F12", 5)
    assert Lg.shape[1] >= 1 and lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10


def test_errors(dme):
    prob = make_config(2, nx=6)
    s = dme.Solver(**dme.problem_kwargs(prob), h=0.01)
    with pytest.raises(dme.DmeError) as ei:
        s.split_step("strang", "F12F3", 1)  # F3 on a DLE
    assert ei.value.code == 3
    with pytest.raises(dme.DmeError) as ei:
        s.split_step("strang", "F12F4", 1)  # F4 without S
    assert ei.value.code == 3
    with pytest.raises(dme.DmeError) as ei:
        s.debug_apply("T1", 0.003)  # tau must be h or h/2
    assert ei.value.code == 3
    # the context stays usable after validation errors
    s.split_step("strang", "F12", 2)
    assert s.get_factor()[0].shape[1] > 0
    # non-finite A (checked on the device after the upload) and asymmetric/finite S
    badA = make_config(2, nx=6)
    badA.A = badA.A.copy()
    badA.A[3, 4] = np.nan
    with pytest.raises(dme.DmeError) as ei:
        dme.Solver(**dme.problem_kwargs(badA), h=0.01)
    assert ei.value.code == 1
    # indefinite D0 is rejected at init
    bad = make_config(2, nx=6)
    bad.D0 = np.diag([1.0, -1.0, 1.0, 1.0, 1.0])
    with pytest.raises(dme.DmeError) as ei:
        dme.Solver(**dme.problem_kwargs(bad), h=0.01)
    assert ei.value.code == 1


def test_determinism(dme):
    """Replicated compressions must be bitwise reproducible (multi-GPU replicas rely on it)."""
    prob = make_config(5, nx=20)
    out = []
    for _ in range(2):
        s = dme.Solver(**dme.problem_kwargs(prob), h=0.01, rank_cap=64)
        s.split_step("strang", "F12F3", 8)
        out.append(s.get_factor()[0])
        s.close()
    assert np.array_equal(out[0], out[1])


def test_device_resident_inputs(dme):
    """A (and S) passed as CUDA tensors (options.big_inputs_on_device) give the same result."""
    import torch
    prob = make_config(4, nx=10)
    a = dme.Solver(**dme.problem_kwargs(prob), h=0.02)
    kw = dme.problem_kwargs(prob)
    kw["A"] = torch.from_numpy(prob.A).cuda()
    kw["S"] = torch.from_numpy(prob.S).cuda()
    b = dme.Solver(**kw, h=0.02)
    for s in (a, b):
        s.split_step("strang", "F12F3F4", 5)
    La, Da = a.get_factor()
    Lb, Db = b.get_factor()
    assert np.array_equal(La, Lb)


@pytest.mark.parametrize("e_pass", ["auto", "dmma"])
def test_poisoned_workspace(dme, e_pass):
    """The workspace is caller memory with arbitrary contents (0xFF bytes here): every counter and
    scratch the kernels rely on is initialised by the library (regression: the int8 E pass's Stream-K
    fixup counters were once left uninitialised)."""
    prob = make_config(5, nx=30)
    out = []
    for poison in (False, True):
        s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64, e_pass=e_pass,
                       poison_workspace=poison)
        s.split_step("strang", "F12F3", 4)
        out.append(s.get_factor())
        s.close()
    (L1, D1), (L2, D2) = out
    assert L1.shape == L2.shape and np.array_equal(L1, L2) and np.array_equal(D1, D2)


@pytest.mark.parametrize("a,q,beta,p0", [(-1.0, 1.0, 1.0, 1.0), (-3.0, 0.5, 2.0, 0.2), (0.4, 2.0, 0.5, 1.5)])
def test_scalar_dre_scheme_closed_form(dme, a, q, beta, p0):
    """n = 1 through the whole GPU path against the paper's scalar recursions written out here
    (pin P3 of SURVEY §8(c), independent of the oracle): Strang F12F3 is
    p <- T12(h/2) T3(h) T12(h/2) p with T12(t) p = e^{2at} p + q (e^{2at} - 1) / (2a) (eq:full,
    P:L129) and T3(t) p = p / (1 + t beta p); Lie F1F2F3 is T1 T2 T3 with
    T1(t) p = e^{2at} p, T2(t) p = p + t q."""
    h, N = 0.01, 40
    prob = Problem(A=np.array([[a]]), C=np.array([[np.sqrt(q)]]), L0=np.array([[np.sqrt(p0)]]),
                   D0=np.eye(1), B=np.array([[1.0]]), R=np.array([[1.0 / beta]]), T=h * N)
    t12 = lambda p, t: np.exp(2 * a * t) * p + q * np.expm1(2 * a * t) / (2 * a)
    t3 = lambda p, t: p / (1 + t * beta * p)
    for scheme, comp, step in (("strang", "F12F3", lambda p: t12(t3(t12(p, h / 2), h), h / 2)),
                               ("lie", "F1F2F3", lambda p: t3(np.exp(2 * a * h) * p + h * q, h))):
        s = dme.Solver(**dme.problem_kwargs(prob), h=h)
        s.split_step(scheme, comp, N)
        L, D = s.get_factor()
        s.close()
        pg = float((L @ D @ L.T)[0, 0])
        p = p0
        for _ in range(N):
            p = step(p)
        assert abs(pg - p) <= 1e-12 * abs(p), (scheme, pg, p)
