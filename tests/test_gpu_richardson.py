"""GPU: Richardson-extrapolated Strang (dme_extrapolate) against the oracle's
extrapolation (pinned by observed order 4 in tests/test_oracle_richardson.py), P-level 1e-10."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import exact, lowrank  # noqa: E402
from oracle.schemes import OracleOptions, richardson  # noqa: E402
from workloads import make_config  # noqa: E402


@pytest.fixture(scope="module")
def dme():
    import paper_1805_08990_b200 as m
    return m


def _gpu_richardson(dme, prob, h, N, comp, **kw):
    fine = dme.Solver(**dme.problem_kwargs(prob), h=h / 2, **kw)
    coarse = dme.Solver(**dme.problem_kwargs(prob), h=h, **kw)
    fine.split_step("strang", comp, 2 * N)
    coarse.split_step("strang", comp, N)
    L, D = dme.extrapolate(fine, coarse)
    fine.close()
    coarse.close()
    return L, D


@pytest.mark.parametrize("cfg,kw,comp,h,N", [(5, dict(nx=8), "F12F3", 0.01, 10),
                                             (3, dict(nx=8), "F12F3", 0.01, 10),
                                             (5, dict(nx=6, dle=True), "F1F2", 0.02, 8),
                                             (4, dict(nx=6), "F12F3F4", 0.02, 8)])
def test_extrapolate_vs_oracle(dme, cfg, kw, comp, h, N):
    prob = make_config(cfg, **kw)
    Lg, Dg = _gpu_richardson(dme, prob, h, N, comp)
    Lo, Do = richardson(prob, h, N, comp, OracleOptions())
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10
    assert np.allclose(Lg.T @ Lg, np.eye(Lg.shape[1]), atol=1e-12)  # orthonormal columns


def test_extrapolate_order4(dme):
    p = make_config(5, nx=5)
    G = p.B @ np.linalg.solve(p.R, p.B.T)
    ref = exact.dre_moebius(p.A, p.C.T @ p.C, G, p.L0 @ p.L0.T, p.T, 2000)
    errs = []
    for N in (32, 64, 128):
        L, D = _gpu_richardson(dme, p, p.T / N, N, "F12F3")
        errs.append(np.linalg.norm(lowrank.to_dense(L, D) - ref) / np.linalg.norm(ref))
    o = np.log(errs[1] / errs[2]) / np.log(2.0)
    assert 3.5 <= o <= 4.5, (errs, o)


def test_extrapolate_errors(dme):
    prob = make_config(5, nx=6)
    a = dme.Solver(**dme.problem_kwargs(prob), h=0.01)
    b = dme.Solver(**dme.problem_kwargs(prob), h=0.01)
    a.split_step("strang", "F12F3", 2)
    b.split_step("strang", "F12F3", 1)
    with pytest.raises(dme.DmeError):
        dme.extrapolate(a, b)   # same step size: not a h/2, h pair
