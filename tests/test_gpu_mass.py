"""GPU: the mass-matrix equation of Example 4 against the oracle.

The library cancels M at init (A <- A M^-1, C <- C M^-1 by a dense LU of M); the
oracle does the same with numpy.linalg.solve and is pinned against the ORIGINAL M-form equation
in tests/test_oracle_mass.py. Synthetic P1 FEM pair (workloads.fem2d_matrices), symmetric and
nonsymmetric (transport) A, DRE and DLE."""
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


@pytest.mark.parametrize("nx,conv,dle,comp", [(8, 0.0, False, "F12F3"), (20, 0.0, False, "F12F3"),
                                              (12, 4.0, False, "F12F3"), (12, 4.0, False, "F1F3F2"),
                                              (10, 0.0, True, "F12")])
def test_mass_matrix_vs_oracle(dme, nx, conv, dle, comp):
    prob = make_config(6, nx=nx, conv=conv, dle=dle)
    h, N = 0.005, 12
    s = dme.Solver(**dme.problem_kwargs(prob), h=h)
    s.split_step("strang", comp, N)
    Lg, Dg = s.get_factor()
    s.close()
    o = OracleSolver(prob, h, OracleOptions())
    o.step("strang", comp, N)
    Lo, Do = o.factor()
    assert lowrank.rel_diff(Lg, Dg, Lo, Do) <= 1e-10


def test_mass_matrix_identity_and_errors(dme):
    prob = make_config(6, nx=8)
    kw = dme.problem_kwargs(prob)
    a = dme.Solver(**dict(kw, M=np.eye(prob.n)), h=0.005)
    kw0 = dict(kw)
    kw0.pop("M")
    b = dme.Solver(**kw0, h=0.005)
    for s in (a, b):
        s.split_step("strang", "F12F3", 5)
    assert lowrank.rel_diff(*a.get_factor(), *b.get_factor()) <= 1e-13
    with pytest.raises(dme.DmeError):
        dme.Solver(**dict(kw, S=np.eye(prob.n)), h=0.005)
