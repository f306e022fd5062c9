"""Pins for the oracle's exponential actions and quadrature (P5, P6, P7 in DESIGN.md)."""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import exact, flows, lowrank, quadrature
from workloads import heat1d_matrix, heat2d_matrix, convdiff2d_matrix

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scalar_cases.json")))


def test_heat_closed_form_vs_scipy_expm():
    # P5: the DST closed form (any n) agrees with a library expm at small n
    for nx, dim in ((30, 1), (7, 2)):
        A = heat1d_matrix(nx) if dim == 1 else heat2d_matrix(nx)
        t = 2.5e-3
        assert np.allclose(exact.heat_expm_closed_form(nx, t, dim), sla.expm(t * A), rtol=0,
                           atol=1e-14)


@pytest.mark.parametrize("method", ["heat", "eigh", "expm"])
def test_operator_methods_agree(method):
    nx = 6
    A = heat2d_matrix(nx)
    op = flows.Operator(A, method, heat_nx=nx, heat_dim=2)
    X = np.random.default_rng(0).random((nx * nx, 3))
    E = exact.heat_expm_closed_form(nx, 1e-2, 2)
    assert np.allclose(op.apply(1e-2, X), E @ X, rtol=0, atol=1e-14)


def test_operator_transpose_guard():
    # reading G1: the factor is multiplied by exp(t A^T); nonsymmetric A must not use exp(tA)
    A = convdiff2d_matrix(5)
    assert not np.allclose(A, A.T)
    op = flows.Operator(A)
    X = np.random.default_rng(1).random((25, 2))
    Y = op.apply(1e-2, X)
    assert np.allclose(Y, sla.expm(1e-2 * A.T) @ X, atol=1e-14)
    assert not np.allclose(Y, sla.expm(1e-2 * A) @ X, atol=1e-6)


def test_scalar_T1_golden():
    g = GOLD["T1"]
    op = flows.Operator(np.array([[g["a"]]]), "expm")
    L, D = flows.T1(op, g["h"], np.array([[g["L"]]]), np.eye(1))
    assert abs(lowrank.to_dense(L, D)[0, 0] - g["value"]) < 1e-15


def test_gauss_legendre_golden():
    g = GOLD["gauss_legendre_5"]
    c, w = quadrature.gauss_legendre01(5)
    assert np.allclose(2 * c - 1, g["x"], atol=1e-15)
    assert np.allclose(2 * w, g["w"], atol=1e-15)


@pytest.mark.parametrize("q", [5, 14])
def test_gauss_exactness_polynomials(q):
    # q-point Gauss is exact for degree 2q-1 polynomials
    c, w = quadrature.gauss_legendre01(q)
    for deg in range(2 * q):
        assert abs(np.sum(w * c ** deg) - 1.0 / (deg + 1)) < 1e-14


def test_squarings_rule():
    A = heat2d_matrix(100)
    assert quadrature.squarings(A, 2.5e-3) == 6          # ||tau A||_1 = 204 -> s = 6
    assert quadrature.squarings(np.zeros((3, 3)), 1.0) == 0
    assert quadrature.squarings(np.eye(2) * quadrature.THETA13, 1.0) == 0
    assert quadrature.squarings(np.eye(2) * quadrature.THETA13 * 1.5, 1.0) == 1


def test_composite_rule_scalar_integral():
    # P7 scalar: int_0^tau e^{2 a s} ds = (e^{2a tau}-1)/(2a) with stiff a
    for a, tau in ((-1.0, 1.0), (-5000.0, 2.5e-3), (-40000.0, 5e-3)):
        A = np.array([[a]])
        delta = quadrature.panel_width(A, 2 * tau, 1) if tau < 1 else tau
        s, w = quadrature.composite_rule(tau, delta, 14)
        assert abs(np.sum(w) - tau) < 1e-15 * tau
        val = np.sum(w * np.exp(2 * a * s))
        ref = math.expm1(2 * a * tau) / (2 * a)
        assert abs(val - ref) <= 2e-15 * abs(ref)


def test_build_integral_vs_vanloan():
    # P7: the quadrature factor L_I D_I L_I^T equals Van Loan's exact integral
    nx = 5
    A = heat2d_matrix(nx)
    n = nx * nx
    C = np.random.default_rng(2).random((2, n))
    op = flows.Operator(A, "heat", heat_nx=nx, heat_dim=2)
    tau = 2.5e-3
    delta = quadrature.panel_width(A, 2 * tau)
    LI, DI = flows.build_integral(op, tau, delta, 14, C.T, np.eye(2), 1e-16)
    ref = exact.dle_vanloan(A, C.T @ C, np.zeros((n, n)), tau)
    assert np.linalg.norm(lowrank.to_dense(LI, DI) - ref) <= 1e-13 * np.linalg.norm(ref)


def test_build_integral_nonsymmetric_vanloan():
    A = convdiff2d_matrix(5)
    C = np.random.default_rng(3).random((1, 25))
    op = flows.Operator(A, "expm")
    tau = 5e-3
    delta = quadrature.panel_width(A, 2 * tau)
    LI, DI = flows.build_integral(op, tau, delta, 14, C.T, np.eye(1), 1e-16)
    ref = exact.dle_vanloan(A, C.T @ C, np.zeros((25, 25)), tau)
    assert np.linalg.norm(lowrank.to_dense(LI, DI) - ref) <= 1e-13 * np.linalg.norm(ref)


def test_integral_A_zero_is_tauQ():
    n = 4
    C = np.random.default_rng(4).random((1, n))
    op = flows.Operator(np.zeros((n, n)), "expm")
    LI, DI = flows.build_integral(op, 0.3, 0.3, 14, C.T, np.eye(1), 1e-16)
    assert np.allclose(lowrank.to_dense(LI, DI), 0.3 * C.T @ C, atol=1e-15)


def test_two_node_single_panel_is_inaccurate():
    # negative control: 2 nodes on a single panel must NOT reach 1e-8 here
    nx = 5
    A = heat2d_matrix(nx)
    C = np.random.default_rng(5).random((1, 25))
    op = flows.Operator(A, "heat", heat_nx=nx, heat_dim=2)
    tau = 2.5e-2
    LI, DI = flows.build_integral(op, tau, tau, 2, C.T, np.eye(1), 1e-16)
    ref = exact.dle_vanloan(A, C.T @ C, np.zeros((25, 25)), tau)
    assert np.linalg.norm(lowrank.to_dense(LI, DI) - ref) > 1e-8 * np.linalg.norm(ref)


@pytest.mark.parametrize("dim,nx,t", [(1, 60, 1e-3), (2, 14, 5e-3), (2, 20, 2.5e-3)])
def test_operator_action_method_vs_closed_form(dim, nx, t):
    """The 'action' method (expm_multiply on the sparse A^T) against the DST closed form of the
    heat exponential (pin P5): the oracle's route for large nonsymmetric A is pinned on an
    operator whose exponential is known exactly."""
    from workloads import heat1d_matrix, heat2d_matrix
    A = heat1d_matrix(nx) if dim == 1 else heat2d_matrix(nx)
    op = flows.Operator(A, "action")
    X = np.random.default_rng(nx).random((A.shape[0], 3))
    ref = exact.heat_expm_closed_form(nx, t, dim) @ X
    Y = op.apply(t, X)
    assert np.abs(Y - ref).max() <= 1e-13 * np.abs(ref).max()
