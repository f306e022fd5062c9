"""GPU: the int8 digit-slicing (Ozaki) E pass.

Pins: integer operands whose digits are captured exactly give the exact product (bit-exact against
NumPy's exact integer sums); general operands satisfy the per-entry bound of DESIGN.md §5b,
|C - A B|_ij <= 2^-50 max_l|A_il| sum_l|B_lj| (the kernel's bound is ~2^-54; NumPy's own FP64
rounding is far below it); the solver with the Ozaki pass agrees with the FP64-DMMA pass and with
the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import lowrank  # noqa: E402
from oracle.schemes import OracleOptions, OracleSolver  # noqa: E402
from workloads import make_config  # noqa: E402


@pytest.fixture(scope="module")
def dme():
    import paper_1805_08990_b200 as m
    return m


def _bound(A, B):
    return 2.0 ** -50 * np.abs(A).max(axis=1)[:, None] * np.abs(B).sum(axis=0)[None, :]


@pytest.mark.parametrize("M,K,N", [(1, 1, 1), (130, 300, 5), (128, 128, 16), (257, 4099, 64),
                                   (1000, 1000, 48), (3000, 10000, 17), (64, 32768, 33)])
def test_ozaki_integer_exact(dme, M, K, N):
    rng = np.random.default_rng(M + K + N)
    A = rng.integers(-64, 65, (M, K)).astype(np.float64)
    B = rng.integers(-64, 65, (K, N)).astype(np.float64)
    C = dme.matmul_ozaki(A, B)
    assert np.array_equal(C, A @ B)


@pytest.mark.parametrize("M,K,N", [(130, 300, 5), (257, 4099, 64), (1000, 1000, 48),
                                   (3000, 10000, 17), (200, 32768, 16)])
def test_ozaki_random_bound(dme, M, K, N):
    rng = np.random.default_rng(7 * M + K + N)
    A = rng.standard_normal((M, K))
    B = rng.random((K, N))
    C = dme.matmul_ozaki(A, B)
    ref = A @ B
    assert np.all(np.abs(C - ref) <= _bound(A, B))


def test_ozaki_dynamic_range(dme):
    """Rows / columns scaled by 2^{+-300}, zero rows and columns, and entries spanning 1e-30..1
    within a row: the per-row / per-column exponents keep the per-entry bound."""
    rng = np.random.default_rng(11)
    M, K, N = 300, 2000, 40
    A = rng.standard_normal((M, K)) * np.logspace(-30, 0, K)[None, :]
    A *= np.ldexp(1.0, rng.integers(-300, 300, M))[:, None]
    B = rng.standard_normal((K, N)) * np.ldexp(1.0, rng.integers(-300, 300, N))[None, :]
    A[5] = 0.0
    B[:, 7] = 0.0
    C = dme.matmul_ozaki(A, B)
    ref = A @ B
    assert np.all(np.abs(C - ref) <= _bound(A, B))
    assert np.all(C[5] == 0.0) and np.all(C[:, 7] == 0.0)


def test_ozaki_matches_dmma_gemm(dme):
    rng = np.random.default_rng(3)
    A = rng.random((777, 5000))
    B = rng.random((5000, 64))
    C1 = dme.matmul_ozaki(A, B)
    C2 = dme.matmul(A, B)
    assert np.all(np.abs(C1 - C2) <= _bound(A, B))


@pytest.mark.parametrize("comp", ["F12F3", "F1F2F3"])
def test_solver_ozaki_vs_dmma_vs_oracle(dme, comp):
    prob = make_config(5, nx=30)
    out = {}
    for mode in ("auto", "dmma"):
        s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64, e_pass=mode)
        s.split_step("strang", comp, 8)
        out[mode] = s.get_factor()
        st = s.stats()
        if mode == "auto":
            assert st["ozaki_passes"] > 0
        else:
            assert st["ozaki_passes"] == 0
        s.close()
    (La, Da), (Lb, Db) = out["auto"], out["dmma"]
    assert lowrank.rel_diff(La, Da, Lb, Db) <= 1e-12
    orc = OracleSolver(prob, 0.005, OracleOptions(rank_cap=64))
    orc.step("strang", comp, 8)
    Lo, Do = orc.factor()
    assert lowrank.rel_diff(La, Da, Lo, Do) <= 1e-10


@pytest.mark.parametrize("cfg,kw", [(5, dict(nx=30)), (3, dict(nx=20)), (1, dict(n=300))])
def test_init_products_ozaki_vs_dmma(dme, cfg, kw):
    """The Padé products and squarings on the int8 tensor cores (square tiles, symmetric upper
    triangle or full) give the same E_{h/2}, E_h as the FP64 DMMA GEMMs to FP64 accuracy."""
    prob = make_config(cfg, **kw)
    E = {}
    for mode in ("auto", "dmma"):
        s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, e_pass=mode)
        E[mode] = (s.debug_get_exp(0), s.debug_get_exp(1))
        sq = s.stats()["squarings"]
        s.close()
    # normwise FP64 agreement: the digit-sliced products err by ~2^-55 of row max x column sum
    # (absolute, not per entry), and the squaring ladder doubles an absolute error per squaring
    # (||E||_inf = 1): bound 2^(s+2) u. Measured: 4.8e-16 (config 5, s = 6), 4.2e-15 (config 1,
    # s = 8); the FP64 DMMA products keep ~1e-16.
    tol = 2.0 ** (sq + 2) * 2.0 ** -53
    for w in (0, 1):
        a, b = E["auto"][w], E["dmma"][w]
        assert np.abs(a - b).max() <= tol * np.abs(b).sum(axis=1).max(), (w, sq, np.abs(a - b).max())
