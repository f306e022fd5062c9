"""GPU: the bilinear flow T4 with S in CSR form ("S sparse"): the S L and
S (S L) products as sparse x skinny products instead of two 8 n^2-byte streams of a dense S.
Against the oracle (dense S) at 1e-10 and the dense-S GPU run at 1e-12."""
import numpy as np
import pytest
import scipy.sparse as sps

pytestmark = pytest.mark.gpu

from oracle import lowrank  # noqa: E402
from oracle.schemes import OracleOptions, OracleSolver  # noqa: E402
from workloads import make_config  # noqa: E402


@pytest.fixture(scope="module")
def dme():
    import torch
    assert torch.cuda.is_available()
    import paper_1805_08990_b200 as m
    return m


def _run(dme, prob, S, h, scheme, comp, N):
    kw = dme.problem_kwargs(prob)
    kw["S"] = S
    s = dme.Solver(**kw, h=h, rank_cap=64)
    s.split_step(scheme, comp, N)
    L, D = s.get_factor()
    s.close()
    return L, D


@pytest.mark.parametrize("scheme,comp", [("strang", "F12F3F4"), ("lie", "F12F3F4"),
                                         ("strang", "F1F2F4"), ("strang", "F1F4F2"),
                                         ("lie", "F1F2F3F4")])
def test_csr_s_small(dme, scheme, comp):
    prob = make_config(4, nx=12)
    h, N = 0.005, 5
    Ls, Ds = _run(dme, prob, sps.csr_matrix(prob.S), h, scheme, comp, N)
    Ld, Dd = _run(dme, prob, prob.S, h, scheme, comp, N)
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64))
    o.step(scheme, comp, N)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Ls, Ds, Lo, Do) <= 1e-10
    assert lowrank.rel_diff(Ls, Ds, Ld, Dd) <= 1e-12


def test_csr_s_general_pattern(dme):
    """A non-diagonal sparse S (random symmetric pattern, ~5 entries per row)."""
    prob = make_config(4, nx=10)
    n = prob.n
    R = sps.random(n, n, density=4.0 / n, random_state=5, format="csr")
    S = (R + R.T) * 3.0 + sps.diags(prob.S.diagonal())
    prob.S = S.toarray()
    h, N = 0.005, 4
    Ls, Ds = _run(dme, prob, sps.csr_matrix(S), h, "strang", "F12F3F4", N)
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64))
    o.step("strang", "F12F3F4", N)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Ls, Ds, Lo, Do) <= 1e-10


def test_csr_s_validation(dme):
    prob = make_config(4, nx=6)
    bad = sps.csr_matrix(prob.S)
    bad.data[0] = np.nan
    kw = dme.problem_kwargs(prob)
    kw["S"] = bad
    with pytest.raises(dme.DmeError):
        dme.Solver(**kw, h=0.005)
