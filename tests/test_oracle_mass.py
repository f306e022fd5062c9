"""Oracle pins for the mass-matrix equation of Example 4.

The oracle cancels M (A -> A M^-1, Q -> M^-T Q M^-1). These tests check the
transformed run against the ORIGINAL equation M^T P' M = A^T P M + M^T P A + Q - M^T P B R^-1 B^T P M
 integrated directly as a vectorised ODE (DOP853), with a NONSYMMETRIC A so that the
reading A M^-1 (displayed equation) and the text's M^-1 A differ; and M = I reduces to the plain
oracle exactly.
"""
import numpy as np
from scipy.integrate import solve_ivp

from oracle import lowrank
from oracle.schemes import OracleOptions, OracleSolver, mass_transform
from workloads import Problem, make_config


def _mform_reference(M, A, C, B, R, P0, T):
    n = A.shape[0]
    Q = C.T @ C
    G = B @ np.linalg.solve(R, B.T)
    Mi = np.linalg.inv(M)

    def rhs(t, y):
        P = y.reshape(n, n)
        lhs = A.T @ P @ M + M.T @ P @ A + Q - M.T @ P @ G @ P @ M   # = M^T P' M
        return (Mi.T @ lhs @ Mi).ravel()

    sol = solve_ivp(rhs, (0.0, T), P0.ravel(), method="DOP853", rtol=1e-12, atol=1e-15)
    return sol.y[:, -1].reshape(n, n)


def test_mass_transform_vs_original_equation():
    prob = make_config(6, nx=3, conv=4.0)          # n = 9, nonsymmetric A
    assert not np.allclose(prob.A, prob.A.T)
    T = 0.05
    ref = _mform_reference(prob.M, prob.A, prob.C, prob.B, prob.R, np.zeros((9, 9)), T)
    errs = []
    for N in (20, 40):
        s = OracleSolver(prob, T / N, OracleOptions())
        s.step("strang", "F12F3", N)
        L, D = s.factor()
        errs.append(np.linalg.norm(L @ D @ L.T - ref) / np.linalg.norm(ref))
    assert errs[1] < 5e-5, errs
    assert 2.5 < errs[0] / errs[1] < 6.0, errs       # Strang: order 2 (ratio ~4)
    # the other reading (M^-1 A) solves a different equation
    At_wrong = np.linalg.solve(prob.M, prob.A)
    _, Ct = mass_transform(prob.M, prob.A, prob.C)
    wrong = Problem(A=At_wrong, C=Ct, L0=prob.L0, D0=prob.D0, B=prob.B, R=prob.R)
    s = OracleSolver(wrong, T / 40, OracleOptions())
    s.step("strang", "F12F3", 40)
    L, D = s.factor()
    assert np.linalg.norm(L @ D @ L.T - ref) / np.linalg.norm(ref) > 100 * errs[1]


def test_mass_identity_reduces_to_plain():
    prob = make_config(6, nx=4)
    plain = Problem(A=prob.A, C=prob.C, L0=prob.L0, D0=prob.D0, B=prob.B, R=prob.R)
    withI = Problem(A=prob.A, C=prob.C, L0=prob.L0, D0=prob.D0, B=prob.B, R=prob.R,
                    M=np.eye(prob.n))
    out = []
    for p in (plain, withI):
        s = OracleSolver(p, 0.01, OracleOptions())
        s.step("strang", "F12F3", 5)
        out.append(s.factor())
    assert lowrank.rel_diff(*out[0], *out[1]) < 1e-14
