"""Pins for oracle.flows / oracle.schemes (P1-P4, P8, P9, P11-P13 in DESIGN.md)."""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import exact, flows, lowrank, quadrature
from oracle.schemes import OracleOptions, OracleSolver, integrate, step_sequence
from workloads import Problem, heat2d_matrix, make_config

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scalar_cases.json")))


# ---------------------------------------------------------------- scalar golden values
def test_scalar_closed_forms_golden():
    g = GOLD["scalar_dle"]
    assert abs(exact.scalar_dle(g["a"], g["q"], g["p0"], g["t"]) - g["value"]) < 1e-15
    g = GOLD["scalar_dre"]
    assert abs(exact.scalar_dre(g["a"], g["q"], g["beta"], g["p0"], g["t"]) - g["value"]) < 1e-15


def test_scalar_dre_closed_form_vs_ivp():
    for a, q, beta, p0 in ((-1.0, 1.0, 1.0, 1.0), (0.5, 2.0, 3.0, 0.1), (-3.0, 0.0, 1.0, 2.0)):
        ref = exact.full_ivp(np.array([[a]]), np.array([[q]]), np.array([[p0]]), 0.7,
                             G=np.array([[beta]]))[0, 0]
        assert abs(exact.scalar_dre(a, q, beta, p0, 0.7) - ref) < 1e-12 * max(1, abs(ref))


def test_T3_golden_and_T12_golden():
    g = GOLD["T3"]
    L, D = flows.T3(g["h"], np.array([[1.0]]), np.array([[g["p0"]]]), np.array([[1.0]]),
                    np.array([[1.0]]))
    assert abs(lowrank.to_dense(L, D)[0, 0] - g["value"]) < 1e-15
    g = GOLD["T12"]
    A = np.array([[g["a"]]])
    op = flows.Operator(A, "expm")
    delta = quadrature.panel_width(A, 2 * g["h"])
    LI, DI = flows.build_integral(op, g["h"], delta, 14, np.array([[1.0]]), np.eye(1), 1e-16)
    L, D = flows.T12(op, g["h"], np.array([[1.0]]), np.eye(1), LI, DI, 1e-16, None)
    assert abs(lowrank.to_dense(L, D)[0, 0] - g["value"]) < 1e-15


# ---------------------------------------------------------------- T3 / T4 pins
def _rand_psd_factor(rng, n, r):
    return rng.random((n, r)), np.diag(rng.uniform(0.5, 1.5, r))


def test_T3_semigroup_and_dense():
    rng = np.random.default_rng(0)
    n = 12
    L, D = _rand_psd_factor(rng, n, 4)
    B, R = rng.random((n, 2)), np.diag([1.0, 2.0])
    G = B @ np.linalg.solve(R, B.T)
    La, Da = flows.T3(0.3, *flows.T3(0.2, L, D, B, R), B, R)
    Lb, Db = flows.T3(0.5, L, D, B, R)
    assert lowrank.rel_diff(La, Da, Lb, Db) < 1e-14
    # exact ODE solution of P' = -P G P from P0 (vectorised ODE, independent route)
    P0 = lowrank.to_dense(L, D)
    ref = exact.full_ivp(np.zeros((n, n)), np.zeros((n, n)), P0, 0.5, G=G)
    assert np.linalg.norm(lowrank.to_dense(Lb, Db) - ref) < 1e-11 * np.linalg.norm(ref)
    assert np.trace(lowrank.to_dense(Lb, Db)) <= np.trace(P0)


def _bilinear_exact(S, P0, tau):
    n = S.shape[0]
    return (sla.expm(tau * np.kron(S, S)) @ P0.reshape(-1, order="F")).reshape(n, n, order="F")


def test_T4_local_order():
    rng = np.random.default_rng(1)
    n = 8
    S = rng.standard_normal((n, n))
    L, D = _rand_psd_factor(rng, n, 3)
    P0 = lowrank.to_dense(L, D)
    errs = {1: [], 2: []}
    for tau in (0.02, 0.01, 0.005):
        ex = _bilinear_exact(S, P0, tau)
        for order in (1, 2):
            L2, D2 = flows.T4(tau, L, D, S, order, 1e-16, None)
            errs[order].append(np.linalg.norm(lowrank.to_dense(L2, D2) - ex))
    r2 = errs[2][1] / errs[2][2]
    r1 = errs[1][1] / errs[1][2]
    assert 7.0 < r2 < 9.0, r2   # midpoint: local error O(tau^3)
    assert 3.5 < r1 < 4.5, r1   # Euler:    local error O(tau^2)


def test_T4_S_zero_identity():
    rng = np.random.default_rng(2)
    L, D = _rand_psd_factor(rng, 10, 3)
    L2, D2 = flows.T4(0.1, L, D, np.zeros((10, 10)), 2, 1e-14, None)
    assert L2.shape[1] == 3 and lowrank.rel_diff(L2, D2, L, D) < 1e-14


# ---------------------------------------------------------------- composition tables
def test_step_sequences():
    assert step_sequence("lie", "F1F2", 1.0) == [("T1", 1.0), ("T2", 1.0)]
    assert step_sequence("strang", "F1F2", 1.0) == [("T1", .5), ("T2", 1.0), ("T1", .5)]
    assert step_sequence("strang", "F12", 1.0) == [("T12", 1.0)]
    assert step_sequence("strang", "F12F3", 1.0) == [("T12", .5), ("T3", 1.0), ("T12", .5)]
    assert step_sequence("strang", "F1F3F2", 1.0) == [("T1", .5), ("T3", .5), ("T2", 1.0),
                                                      ("T3", .5), ("T1", .5)]
    assert step_sequence("strang", "F12F3F4", 1.0) == [("T12", .5), ("T3", .5), ("T4", 1.0),
                                                       ("T3", .5), ("T12", .5)]


# ---------------------------------------------------------------- scalar recursion (P3)
def test_scalar_scheme_recursions():
    a, q, beta, p0, h, N = -1.3, 0.7, 2.0, 0.4, 0.05, 10
    prob = Problem(A=np.array([[a]]), C=np.array([[math.sqrt(q)]]), L0=np.array([[math.sqrt(p0)]]),
                   D0=np.eye(1), B=np.array([[math.sqrt(beta)]]), R=np.eye(1), T=h * N)
    t1 = lambda p, t: math.exp(2 * a * t) * p
    t2 = lambda p, t: p + t * q
    t3 = lambda p, t: p / (1 + t * beta * p)
    t12 = lambda p, t: exact.scalar_dle(a, q, p, t)
    cases = {("strang", "F1F2"): lambda p: t1(t2(t1(p, h / 2), h), h / 2),
             ("lie", "F1F2"): lambda p: t2(t1(p, h), h),
             ("strang", "F12F3"): lambda p: t12(t3(t12(p, h / 2), h), h / 2),
             ("strang", "F1F3F2"): lambda p: t1(t3(t2(t3(t1(p, h / 2), h / 2), h), h / 2), h / 2),
             ("lie", "F1F2F3"): lambda p: t3(t2(t1(p, h), h), h)}
    for (scheme, comp), f in cases.items():
        p = p0
        for _ in range(N):
            p = f(p)
        s = integrate(prob, scheme, comp, N)
        L, D = s.factor()
        assert abs(lowrank.to_dense(L, D)[0, 0] - p) < 1e-14, (scheme, comp)


# ---------------------------------------------------------------- diagonal A (P4)
def test_diagonal_A_dle_exact():
    rng = np.random.default_rng(3)
    n = 6
    a = -rng.uniform(1, 50, n)
    C = rng.random((2, n))
    L0 = rng.random((n, 2))
    prob = Problem(A=np.diag(a), C=C, L0=L0, D0=np.eye(2), T=0.3)
    s = integrate(prob, "strang", "F12", 7)
    Q, P0 = C.T @ C, L0 @ L0.T
    ss = a[:, None] + a[None, :]
    Pex = np.exp(ss * 0.3) * P0 + Q * np.expm1(ss * 0.3) / ss
    L, D = s.factor()
    assert np.linalg.norm(lowrank.to_dense(L, D) - Pex) < 1e-14 * np.linalg.norm(Pex)


# ---------------------------------------------------------------- invariants (P13)
def test_A_zero_strang_F1F2_exact():
    rng = np.random.default_rng(4)
    n = 9
    C, L0 = rng.random((2, n)), rng.random((n, 3))
    prob = Problem(A=np.zeros((n, n)), C=C, L0=L0, D0=np.eye(3), T=0.4)
    L, D = integrate(prob, "strang", "F1F2", 5).factor()
    assert np.allclose(lowrank.to_dense(L, D), L0 @ L0.T + 0.4 * C.T @ C, atol=1e-13)


def test_A_Q_zero_F12F3_exact_riccati():
    rng = np.random.default_rng(5)
    n = 9
    L0, B = rng.random((n, 3)), rng.random((n, 1))
    prob = Problem(A=np.zeros((n, n)), C=np.zeros((0, n)), L0=L0, D0=np.eye(3), B=B,
                   R=np.eye(1), T=0.4)
    L, D = integrate(prob, "strang", "F12F3", 4).factor()
    P0 = L0 @ L0.T
    ref = np.linalg.solve(np.eye(n) + 0.4 * P0 @ B @ B.T, P0)
    assert np.allclose(lowrank.to_dense(L, D), ref, atol=1e-13)


# ---------------------------------------------------------------- orders vs brute force (P11, P12)
def _example1(dre, rinv=1.0):
    return make_config(5, nx=5, rinv=rinv, dle=not dre)


def _fit(hs, es):
    return np.polyfit(np.log(hs), np.log(es), 1)[0]


@pytest.fixture(scope="module")
def ex1_dle_ref():
    p = _example1(False)
    # Kronecker/augmented expm (stable: K is negative definite) cross-checked against an
    # adaptive DOP853 integration of the vectorised equation (Van Loan's one-shot block
    # exponential overflows at T||A|| ~ 144, like the Hamiltonian formula)
    ref = exact.dle_kron(p.A, p.C.T @ p.C, p.L0 @ p.L0.T, p.T)
    ref2 = exact.full_ivp(p.A, p.C.T @ p.C, p.L0 @ p.L0.T, p.T)
    assert np.linalg.norm(ref - ref2) < 1e-11 * np.linalg.norm(ref)
    return p, ref


def _errs(p, ref, scheme, comp, Ns):
    out = []
    for N in Ns:
        L, D = integrate(p, scheme, comp, N).factor()
        out.append(np.linalg.norm(lowrank.to_dense(L, D) - ref) / np.linalg.norm(ref))
    return np.array(out)


NS = [64, 128, 256, 512]


def test_order_dle_lie_strang_quadrature(ex1_dle_ref):
    p, ref = ex1_dle_ref
    hs = p.T / np.array(NS)
    e_lie = _errs(p, ref, "lie", "F1F2", NS)
    e_str = _errs(p, ref, "strang", "F1F2", NS)
    e_q = _errs(p, ref, "strang", "F12", NS)
    assert 0.8 <= _fit(hs, e_lie) <= 1.2
    assert 1.7 <= _fit(hs, e_str) <= 2.3
    # P:L381 "constant but very low error": the quadrature error sits at round-off on the
    # whole grid (so a max/min flatness ratio would only measure noise)
    assert e_q.max() < 1e-12 and e_q.max() < e_str.min() / 100


@pytest.fixture(scope="module")
def ex1_dre_refs():
    out = {}
    for rinv in (1.0, 1e-3):
        p = _example1(True, rinv)
        G = p.B @ np.linalg.solve(p.R, p.B.T)
        ref = exact.dre_moebius(p.A, p.C.T @ p.C, G, p.L0 @ p.L0.T, p.T, 2000)
        out[rinv] = (p, ref)
    return out


def test_order_dre_three_schemes(ex1_dre_refs):
    for rinv, (p, ref) in ex1_dre_refs.items():
        hs = p.T / np.array(NS)
        es = {c: _errs(p, ref, "strang", c, NS) for c in ("F12F3", "F1F2F3", "F1F3F2")}
        for c, e in es.items():
            assert 1.7 <= _fit(hs, e) <= 2.3, (rinv, c, e)
        if rinv == 1e-3:   # P:L393 soft claim: two-term ~10x more accurate (tested at 3x)
            assert np.all(es["F12F3"] <= np.minimum(es["F1F2F3"], es["F1F3F2"]) / 3)
        e_lie = _errs(p, ref, "lie", "F12F3", NS)
        assert 0.8 <= _fit(hs, e_lie) <= 1.2


def test_moebius_vs_ivp():
    p = _example1(True)
    G = p.B @ np.linalg.solve(p.R, p.B.T)
    a = exact.dre_moebius(p.A, p.C.T @ p.C, G, p.L0 @ p.L0.T, 0.05, 400)
    b = exact.full_ivp(p.A, p.C.T @ p.C, p.L0 @ p.L0.T, 0.05, G=G)
    assert np.linalg.norm(a - b) < 1e-10 * np.linalg.norm(b)


def test_order_generalized(ex2=None):
    p = make_config(4, nx=5, dle=True)
    Q = p.C.T @ p.C
    n = p.n
    ref = exact.dle_kron(p.A, Q, np.zeros((n, n)), p.T, S=p.S)
    hs = p.T / np.array(NS)
    es = {c: _errs(p, ref, "strang", c, NS) for c in ("F12F4", "F1F2F4", "F1F4F2")}
    for c, e in es.items():
        assert 1.7 <= _fit(hs, e) <= 2.3, (c, e)
    pr = make_config(4, nx=5)
    G = pr.B @ pr.B.T
    ref = exact.full_ivp(pr.A, Q, np.zeros((n, n)), pr.T, S=pr.S, G=G)
    e = _errs(pr, ref, "strang", "F12F3F4", NS)
    assert 1.7 <= _fit(hs, e) <= 2.3, e


def test_symmetry_psd_config3_small():
    p = make_config(3, nx=6)
    s = integrate(p, "strang", "F12F3", 20)
    L, D = s.factor()
    P = L @ D @ L.T
    assert np.allclose(P, P.T, atol=1e-14 * np.abs(P).max())
    assert np.linalg.eigvalsh(0.5 * (P + P.T)).min() >= -1e-10 * np.linalg.norm(P, 2)
