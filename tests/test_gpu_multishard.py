"""GPU: the row-sharded multi-GPU path executed on ONE GPU through
options.virtual_world = G: every E pass computes each of the G shards' rows with the per-shard
kernels into its staging block, runs the ncclAllGather (a real NCCL call on a one-rank
communicator) and unpacks the blocks, exactly as a G-rank run does; the init builds only the held
rows of E by the sharded method (Chebyshev column actions for symmetric A, held rows of the Padé E
otherwise). Compared with the oracle (1e-10) and with the unsharded run (1e-12)."""
import numpy as np
import pytest

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


def _run(dme, prob, h, N, scheme, comp, **kw):
    s = dme.Solver(**dme.problem_kwargs(prob), h=h, rank_cap=64, **kw)
    s.split_step(scheme, comp, N)
    L, D = s.get_factor()
    st = s.stats()
    s.close()
    return L, D, st


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("e_pass", ["auto", "dmma"])
def test_virtual_shards_config5(dme, G, e_pass):
    prob = make_config(5, nx=30)           # n = 900: ragged last shard for G = 8 (nloc = 128)
    h, N = 0.005, 8
    Lg, Dg, st = _run(dme, prob, h, N, "strang", "F12F3", virtual_world=G, e_pass=e_pass)
    L1, D1, _ = _run(dme, prob, h, N, "strang", "F12F3", e_pass=e_pass)
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64))
    o.step("strang", "F12F3", N)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10
    assert lowrank.rel_diff(Lg, Dg, L1, D1) <= 1e-12
    assert st["expm_chebyshev"] == 1


@pytest.mark.parametrize("G", [2, 5])
def test_virtual_shards_pade_nonsymmetric(dme, G):
    prob = make_config(3, nx=14)           # convection-diffusion: nonsymmetric A, Padé-13 init
    h, N = 0.005, 6
    Lg, Dg, st = _run(dme, prob, h, N, "strang", "F12F3", virtual_world=G)
    o = OracleSolver(prob, h, OracleOptions(rank_cap=64))
    o.step("strang", "F12F3", N)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10
    assert st["expm_chebyshev"] == 0


def test_virtual_shards_unmerged_and_lie(dme):
    prob = make_config(5, nx=16)
    h, N = 0.005, 5
    for scheme, comp in (("lie", "F1F2F3"), ("strang", "F1F3F2")):
        Lg, Dg, _ = _run(dme, prob, h, N, scheme, comp, virtual_world=4, fsal=False)
        o = OracleSolver(prob, h, OracleOptions(rank_cap=64))
        o.step(scheme, comp, N)
        Lo, Do = o.factor()
        assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10, (scheme, comp)
