"""Sub-flows T1, T2, T3, T4, T12 in LDL^T form (oracle; test infrastructure only).

Every flow follows the paper's formula in the paper's notation; compression
is applied after the rank-growing flows T2, T12, T4 and never after T1 or T3 (reading G10).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import lowrank, quadrature


class Operator:
    """Dense A with exponential actions exp(t A^T) X (eq:F_sol_LDL: the factor is
    multiplied by exp(h A^T); reading G1 — never exp(hA) for nonsymmetric A).

    method 'expm'   : scipy.linalg.expm(t A^T) (Al-Mohy & Higham), cached per t
    method 'eigh'   : symmetric A = V diag(lam) V^T, exp(tA^T) X = V diag(e^{t lam}) V^T X
    method 'heat'   : the Dirichlet FD Laplacian's closed-form sine eigenbasis (pin P5),
                      for 1D (n = nx) or 2D (n = nx^2, index i*nx+j) problems
    method 'action' : exp(t A^T) X by scipy.sparse.linalg.expm_multiply (Al-Mohy & Higham 2011,
                      truncated Taylor with scaling, double-precision tolerance) on A^T in CSR, the
                      a6 oracle form of SURVEY §8(c) for large nonsymmetric A (every quadrature
                      node action without a dense exponential); dense E(t) by expm when asked
    """

    def __init__(self, A, method="auto", heat_nx=None, heat_dim=None, dense_apply=False):
        self.A = np.asarray(A, dtype=np.float64)
        # dense_apply: T1/T12 actions multiply by the dense matrix exp(tau A^T) (the north star's
        # dense-E formulation); quadrature node actions keep the exact structured route.
        self.dense_apply = dense_apply
        n = self.A.shape[0]
        if method == "auto":
            if heat_nx is not None:
                method = "heat"
            elif n <= 3000 and np.array_equal(self.A, self.A.T):
                method = "eigh"
            else:
                method = "expm"
        self.method = method
        self._E = {}
        if method == "action":
            import scipy.sparse as sps
            self.At = sps.csr_matrix(self.A.T)
        if method == "eigh":
            self.lam, self.V = np.linalg.eigh(self.A)
        elif method == "heat":
            nx = heat_nx
            j = np.arange(1, nx + 1)
            self.Vx = np.sqrt(2.0 / (nx + 1)) * np.sin(np.outer(j, j) * np.pi / (nx + 1))
            lx = -4.0 * (nx + 1) ** 2 * np.sin(j * np.pi / (2 * (nx + 1))) ** 2
            self.dim = heat_dim
            self.nx = nx
            self.lam = lx if heat_dim == 1 else (lx[:, None] + lx[None, :]).ravel()

    def _to_eig(self, X):
        if self.method == "eigh":
            return self.V.T @ X
        if self.dim == 1:
            return self.Vx @ X
        nx = self.nx
        Y = X.T.reshape(-1, nx, nx)
        return np.matmul(np.matmul(self.Vx, Y), self.Vx).reshape(-1, nx * nx).T

    def _from_eig(self, Y):
        return self._to_eig(Y)  if self.method == "heat" else self.V @ Y

    def E(self, t):
        """Dense exp(t A^T)."""
        if t not in self._E:
            if self.method in ("expm", "action"):
                self._E[t] = sla.expm(t * self.A.T)
            else:
                self._E[t] = self._from_eig(np.exp(t * self.lam)[:, None] * self._to_eig(
                    np.eye(self.A.shape[0])))
        return self._E[t]

    def E_dense(self, t):
        """Dense exp(t A^T); for the 2D heat hint via the closed-form 1D factor E1 (x) E1."""
        if self.method == "heat" and self.dim == 2:
            if ("k", t) not in self._E:
                j = np.arange(1, self.nx + 1)
                lx = -4.0 * (self.nx + 1) ** 2 * np.sin(j * np.pi / (2 * (self.nx + 1))) ** 2
                E1 = (self.Vx * np.exp(t * lx)[None, :]) @ self.Vx
                self._E[("k", t)] = np.kron(E1, E1)
            return self._E[("k", t)]
        return self.E(t)

    def apply_step(self, t, X):
        """exp(t A^T) X for the step flows T1 / T12 (dense product when dense_apply)."""
        if self.dense_apply and X.shape[1]:
            return self.E_dense(t) @ X
        return self.apply(t, X)

    def apply(self, t, X):
        """exp(t A^T) X."""
        if X.shape[1] == 0:
            return X.copy()
        if self.method == "action":
            from scipy.sparse.linalg import expm_multiply
            return expm_multiply(t * self.At, X)
        if self.method == "expm":
            return self.E(t) @ X
        return self._from_eig(np.exp(t * self.lam)[:, None] * self._to_eig(X))


def T1(op, tau, L, D):
    """Linear flow F1(P) = A^T P + P A: T1(tau) P0 = e^{tau A^T} P0 e^{tau A}
    (P:L110); factorised as (e^{tau A^T} L) D (e^{tau A^T} L)^T (eq:F_sol_LDL)."""
    return op.apply_step(tau, L), D


def T2(tau, L, D, LQ, DQ, tol, cap):
    """Constant flow F2(P) = Q: T2(tau) P0 = P0 + tau Q = [L, L_Q]
    blkdiag(D, tau D_Q) [L, L_Q]^T; then column compression (Alg. 1 l.13)."""
    L2, D2 = lowrank.concat(L, D, LQ, DQ, tau)
    return lowrank.column_compression(L2, D2, tol, cap)


def T3(tau, L, D, B, R):
    """Riccati flow F3(P) = -P B R^-1 B^T P, exact (eq:nonlinear P:L152) in low-rank form
    (P:L156):  D <- (I + tau D L^T B R^-1 B^T L)^-1 D   (reading G2: Alg. 3 P:L257 drops
    B^T), an r x r linear solve, core re-symmetrised (reading G14)."""
    r = L.shape[1]
    if r == 0:
        return L, D
    U = L.T @ B
    K = np.eye(r) + tau * D @ U @ np.linalg.solve(R, U.T)
    Dn = np.linalg.solve(K, D)
    return L, 0.5 * (Dn + Dn.T)


def T4(tau, L, D, S, order, tol, cap):
    """Bilinear flow F4(P) = S P S^T.
    order 2 (Strang, midpoint rule P:L172, Alg. 4): L <- [L, sqrt(tau) S L, tau/sqrt(2) S^2 L]
        with S^2 L of the pre-step L (reading G3), D <- blkdiag(D, D, D);
    order 1 (Lie, explicit Euler P:L180): L <- [L, sqrt(tau) S L], D <- blkdiag(D, D);
    then column compression (Alg. 4 l.270)."""
    if L.shape[1] == 0:
        return L, D
    SL = S @ L
    if order == 2:
        Ln = np.hstack([L, np.sqrt(tau) * SL, tau / np.sqrt(2.0) * (S @ SL)])
        Dn = sla.block_diag(D, D, D)
    else:
        Ln = np.hstack([L, np.sqrt(tau) * SL])
        Dn = sla.block_diag(D, D)
    return lowrank.column_compression(Ln, Dn, tol, cap)


def build_integral(op, tau, delta, q, LQ, DQ, tol, cap=None):
    """Alg. 2 step 3: nodes s_k and weights w_k of the quadrature formula
    (composite reading G6), L_I = [exp(s_1 A^T) L_Q, ..., exp(s_N A^T) L_Q],
    D_I = blkdiag(w_1 D_Q, ..., w_N D_Q), then column compression."""
    s, w = quadrature.composite_rule(tau, delta, q)
    LI = np.hstack([op.apply(sk, LQ) for sk in s])
    DI = sla.block_diag(*[wk * DQ for wk in w])
    return lowrank.column_compression(LI, DI, tol, cap)


def T12(op, tau, L, D, LI, DI, tol, cap):
    """Affine flow F12(P) = A^T P + P A + Q, exact solution eq:full with the
    integral replaced by the precomputed quadrature factor: Alg. 2 loop
    L <- [exp(tau A^T) L, L_I], D <- blkdiag(D, D_I), column compression."""
    L2, D2 = lowrank.concat(op.apply_step(tau, L), D, LI, DI, 1.0)
    return lowrank.column_compression(L2, D2, tol, cap)
