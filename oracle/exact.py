"""Brute-force exact solutions used to PIN the oracle (test infrastructure only).

None of these shares arithmetic with oracle.flows / oracle.schemes: they solve the full
equations (§2.4) by independent routes.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla
from scipy.integrate import solve_ivp


def scalar_dle(a, q, p0, t):
    """p' = 2 a p + q  =>  p(t) = e^{2at} p0 + q (e^{2at} - 1)/(2a)   (eq:full at n = 1)."""
    if a == 0.0:
        return p0 + q * t
    e = math.exp(2 * a * t)
    return e * p0 + q * (e - 1.0) / (2 * a)


def scalar_dre(a, q, beta, p0, t):
    """p' = 2 a p + q - beta p^2 (eq:ricc at n = 1, beta = b^2/r).
    gamma = sqrt(a^2 + beta q), th = tanh(gamma t):
    p(t) = (p0 (gamma + a th) + q th) / (gamma - (a - beta p0) th); gamma = 0 -> p0/(1+beta p0 t)."""
    g = math.sqrt(a * a + beta * q)
    if g == 0.0:
        return p0 / (1.0 + beta * p0 * t)
    th = math.tanh(g * t)
    return (p0 * (g + a * th) + q * th) / (g - (a - beta * p0) * th)


def dle_vanloan(A, Q, P0, t):
    """Exact DLE solution eq:full: e^{tA^T} P0 e^{tA} + int_0^t e^{sA^T} Q e^{sA} ds,
    the integral by Van Loan's block exponential: expm(t [[-A^T, Q], [0, A]]) =
    [[F11, F12], [0, F22]]  =>  integral = F22^T F12."""
    n = A.shape[0]
    M = np.zeros((2 * n, 2 * n))
    M[:n, :n] = -A.T
    M[:n, n:] = Q
    M[n:, n:] = A
    F = sla.expm(t * M)
    E = sla.expm(t * A.T)
    P = E @ P0 @ E.T + F[n:, n:].T @ F[:n, n:]
    return 0.5 * (P + P.T)


def dle_kron(A, Q, P0, t, S=None):
    """Exact (generalised) DLE by vectorisation: vec(P)' = K vec(P) + vec(Q),
    K = I (x) A^T + A^T (x) I [+ S (x) S] (column-major vec), solved with the augmented
    matrix exponential expm(t [[K, vecQ], [0, 0]])."""
    n = A.shape[0]
    I = np.eye(n)
    K = np.kron(I, A.T) + np.kron(A.T, I)
    if S is not None:
        K = K + np.kron(S, S)
    N = n * n
    M = np.zeros((N + 1, N + 1))
    M[:N, :N] = K
    M[:N, N] = Q.reshape(-1, order="F")
    v = sla.expm(t * M) @ np.concatenate([P0.reshape(-1, order="F"), [1.0]])
    P = v[:N].reshape(n, n, order="F")
    return 0.5 * (P + P.T)


def dre_moebius(A, Q, G, P0, t, substeps=2000):
    """Exact DRE P' = A^T P + P A + Q - P G P via the associated linear Hamiltonian system:
    [X; Y]' = [[-A, G], [Q, A^T]] [X; Y], P = Y X^{-1} (Radon's lemma), propagated over
    `substeps` substeps (the one-shot formula overflows)."""
    n = A.shape[0]
    H = np.block([[-A, G], [Q, A.T]])
    M = sla.expm((t / substeps) * H)
    P = P0.copy()
    for _ in range(substeps):
        X = M[:n, :n] + M[:n, n:] @ P
        Y = M[n:, :n] + M[n:, n:] @ P
        P = np.linalg.solve(X.T, Y.T).T
        P = 0.5 * (P + P.T)
    return P


def full_ivp(A, Q, P0, t, S=None, G=None, rtol=1e-13, atol=1e-16):
    """Vectorised full equation integrated by an adaptive DOP853 (the paper's own check uses
    a vectorised ode15s at rtol 2.22e-14)."""
    n = A.shape[0]

    def rhs(_, y):
        P = y.reshape(n, n)
        F = A.T @ P + P @ A + Q
        if S is not None:
            F = F + S @ P @ S.T
        if G is not None:
            F = F - P @ G @ P
        return F.ravel()

    sol = solve_ivp(rhs, (0.0, t), P0.ravel(), method="DOP853", rtol=rtol, atol=atol)
    assert sol.success, sol.message
    P = sol.y[:, -1].reshape(n, n)
    return 0.5 * (P + P.T)


def heat_expm_closed_form(nx, t, dim):
    """exp(t A) for the Dirichlet FD Laplacian (pin P5): 1D E = V diag(e^{t lam}) V with
    V_ij = sqrt(2/(n+1)) sin(ij pi/(n+1)), lam_i = -4 (n+1)^2 sin^2(i pi / (2(n+1)));
    2D (index i*nx + j) E = E_1D (x) E_1D."""
    j = np.arange(1, nx + 1)
    V = np.sqrt(2.0 / (nx + 1)) * np.sin(np.outer(j, j) * np.pi / (nx + 1))
    lam = -4.0 * (nx + 1) ** 2 * np.sin(j * np.pi / (2 * (nx + 1))) ** 2
    E1 = (V * np.exp(t * lam)[None, :]) @ V
    return E1 if dim == 1 else np.kron(E1, E1)


def heat_expm_entries(nx, t, rows, cols):
    """Sampled entries of the 2D heat exp(tA) at (rows[k], cols[k]) via E_1D (x) E_1D."""
    E1 = heat_expm_closed_form(nx, t, 1)
    rows, cols = np.asarray(rows), np.asarray(cols)
    return E1[rows // nx, cols // nx] * E1[rows % nx, cols % nx]
