"""GPU parity at BASELINE.json's sizes for configs 1-4 (SURVEY §8(d) recipe; the paper's tables run
n = 2500-22500, Tables 2-5): the same seeded problems through the C ABI and the oracle,
relative Frobenius error of P <= 1e-10 (north star).
  config 1: 1D heat n = 100, Lie F1F2, T = 0.1, all 100 steps
  config 2: 2D heat n = 1024, F12 with 5-node Gauss x 4 subpanels and Strang F1F2, all 100 steps
  config 3: convection-diffusion n = 2500 (nonsymmetric: Padé-13 with the pivoted LU), Strang
            F12F3, F1F2F3, F1F3F2, 6 steps each (oracle node actions by expm_multiply)
  config 4: Example-2 structure n = 4900 with dense S, Strang F12F3F4, Lie F12F3F4, Strang
            F1F2F3F4 and the generalized-DLE Strang F1F2F4, 4 steps each (oracle by eigh)
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

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


def _gpu(dme, prob, h, scheme, comp, N, **kw):
    s = dme.Solver(**dme.problem_kwargs(prob), h=h, rank_cap=64, **kw)
    s.split_step(scheme, comp, N)
    L, D = s.get_factor()
    st = s.stats()
    s.close()
    return L, D, st


def _orc(o, scheme, comp, N):
    o.step(scheme, comp, N)
    return o.factor()


def test_config1_full(dme):
    prob = make_config(1)
    h, N = 1e-3, 100
    Lg, Dg, _ = _gpu(dme, prob, h, "lie", "F1F2", N)
    Lo, Do = _orc(OracleSolver(prob, h, OracleOptions(rank_cap=64)), "lie", "F1F2", N)
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= TOL_P


@pytest.mark.parametrize("scheme,comp", [("strang", "F12"), ("strang", "F1F2")])
def test_config2_full(dme, scheme, comp):
    prob = make_config(2)
    h, N = 0.005, 100
    Lg, Dg, st = _gpu(dme, prob, h, scheme, comp, N, quad_nodes=5, quad_subpanels=4)
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64, quad_nodes=5, quad_subpanels=4))
    Lo, Do = _orc(o, scheme, comp, N)
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= TOL_P
    assert st["quad_panels"] == 4 * 2 ** st["squarings"]


@pytest.fixture(scope="module")
def orc3():
    prob = make_config(3)
    return prob, {}


@pytest.mark.parametrize("comp", ["F12F3", "F1F2F3", "F1F3F2"])
def test_config3_full_size(dme, orc3, comp):
    prob, _ = orc3
    h, N = 0.005, 6
    Lg, Dg, st = _gpu(dme, prob, h, "strang", comp, N)
    assert st["expm_chebyshev"] == 0      # nonsymmetric A: Padé-13
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64), method="action")
    Lo, Do = _orc(o, "strang", comp, N)
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= TOL_P


@pytest.fixture(scope="module")
def eig4():
    """One eigh of the n = 4900 symmetric A, shared by the config-4 oracle runs."""
    from oracle import flows
    prob = make_config(4)
    op = flows.Operator(prob.A, "eigh")
    return prob, op


@pytest.mark.parametrize("scheme,comp", [("strang", "F12F3F4"), ("lie", "F12F3F4"),
                                         ("strang", "F1F2F3F4"), ("strang", "F1F2F4")])
def test_config4_full_size(dme, eig4, scheme, comp):
    prob, op = eig4
    h, N = 0.005, 4
    Lg, Dg, _ = _gpu(dme, prob, h, scheme, comp, N)
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64), method="action")
    o.op = op                            # the shared eigendecomposition of the same A
    o._LI = {}
    Lo, Do = _orc(o, scheme, comp, N)
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= TOL_P


def test_config3_full_size_sparse_csr(dme, orc3):
    """Config 3 (nonsymmetric convection-diffusion, n = 2500) with A passed as CSR: the cluster
    kernels' Taylor route, no dense exponential; against the oracle at 1e-10."""
    import scipy.sparse as sps
    prob, _ = orc3
    h, N = 0.005, 4
    kw = dme.problem_kwargs(prob)
    kw["A"] = sps.csr_matrix(prob.A)
    s = dme.Solver(**kw, h=h, rank_cap=64)
    s.split_step("strang", "F12F3", N)
    Lg, Dg = s.get_factor()
    s.close()
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64), method="action")
    o.step("strang", "F12F3", N)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= TOL_P
