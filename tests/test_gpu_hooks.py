"""GPU: the SURVEY §8(b) test hook dme_debug_set_exp (inject an oracle exponential: the "minimum
slice" of SURVEY §7.2) round-trips, and a run on the injected E_{h/2}, E_h matches the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import exact, lowrank  # noqa: E402
from oracle.schemes import OracleOptions, OracleSolver  # noqa: E402
from workloads import make_config  # noqa: E402


@pytest.fixture(scope="module")
def dme():
    import torch
    assert torch.cuda.is_available()
    import paper_1805_08990_b200 as m
    return m


@pytest.mark.parametrize("e_pass", ["auto", "dmma"])
def test_set_exp_roundtrip_and_step(dme, e_pass):
    nx, h, N = 12, 0.005, 6
    prob = make_config(5, nx=nx)
    s = dme.Solver(**dme.problem_kwargs(prob), h=h, rank_cap=64, e_pass=e_pass, fsal=False)
    for which, t in ((0, h / 2), (1, h)):
        E = exact.heat_expm_closed_form(nx, t, 2)   # the DST closed form (oracle/exact.py)
        s.debug_set_exp(which, E)
        assert np.array_equal(s.debug_get_exp(which), E)
    s.split_step("strang", "F1F2F3", N)
    Lg, Dg = s.get_factor()
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64))
    o.step("strang", "F1F2F3", N)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10
    s.close()


def test_set_exp_rejects_bad_which(dme):
    prob = make_config(5, nx=8)
    s = dme.Solver(**dme.problem_kwargs(prob), h=0.005)
    with pytest.raises(dme.DmeError):
        s.debug_set_exp(2, np.eye(prob.n))
    s.close()
