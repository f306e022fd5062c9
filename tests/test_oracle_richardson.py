"""Oracle pins for Richardson-extrapolated Strang: observed order 4 against the
brute-force references of the paper's n = 25 verification problem (pins P11/P12), and the
exact linear algebra of the signed combination."""
import numpy as np

from oracle import exact, lowrank
from oracle.schemes import OracleOptions, integrate, richardson
from workloads import make_config

NS = [32, 64, 128]


def _order(errs):
    e = np.asarray(errs)
    return np.log(e[:-1] / e[1:]) / np.log(2.0)


def test_richardson_order_dle():
    p = make_config(5, nx=5, dle=True)
    ref = exact.dle_kron(p.A, p.C.T @ p.C, p.L0 @ p.L0.T, p.T)
    errs = []
    for N in NS:
        L, D = richardson(p, p.T / N, N, "F1F2")
        errs.append(np.linalg.norm(lowrank.to_dense(L, D) - ref) / np.linalg.norm(ref))
    o = _order(errs)
    assert 3.5 <= o[-1] <= 4.5, (o, errs)
    # more accurate than plain Strang on the fine grid (h/2)
    Ls, Ds = integrate(p, "strang", "F1F2", 2 * NS[-1]).factor()
    es = np.linalg.norm(lowrank.to_dense(Ls, Ds) - ref) / np.linalg.norm(ref)
    assert errs[-1] < es / 10


def test_richardson_order_dre():
    p = make_config(5, nx=5)
    G = p.B @ np.linalg.solve(p.R, p.B.T)
    ref = exact.dre_moebius(p.A, p.C.T @ p.C, G, p.L0 @ p.L0.T, p.T, 2000)
    errs = []
    for N in NS:
        L, D = richardson(p, p.T / N, N, "F12F3")
        errs.append(np.linalg.norm(lowrank.to_dense(L, D) - ref) / np.linalg.norm(ref))
    o = _order(errs)
    assert 3.5 <= o[-1] <= 4.5, (o, errs)


def test_richardson_combination_is_exact_linear_algebra():
    """The compressed signed factor equals (4 P_fine - P_coarse)/3 to round-off."""
    p = make_config(5, nx=4)
    h, N = 0.05, 4
    L, D = richardson(p, h, N, "F12F3")
    Pf = lowrank.to_dense(*integrate(p, "strang", "F12F3", 2 * N, T=h * N).factor())
    Pc = lowrank.to_dense(*integrate(p, "strang", "F12F3", N, T=h * N).factor())
    Pr = (4 * Pf - Pc) / 3
    assert np.linalg.norm(lowrank.to_dense(L, D) - Pr) <= 1e-13 * np.linalg.norm(Pr)
