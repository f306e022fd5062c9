"""Lie / Strang splitting compositions and the time-stepping loop (oracle; test infra only).

Composition names follow the paper's figure legends ("we identify the methods ... by
in which order the subproblems are solved"): F1F2, F12, F12F3, F1F2F3, F1F3F2, F12F4,
F1F2F4, F1F4F2, F12F3F4, plus the four-term F1F2F3F4 (beyond the paper, reading G19).

Lie:  apply the listed flows in order, each over h (reading G5).
Strang: flows f1..fm applied as
        f1(h/2) ... f_{m-1}(h/2) f_m(h) f_{m-1}(h/2) ... f1(h/2);  m = 1 -> f1(h).
T4 uses the midpoint rule under Strang and explicit Euler under Lie (reading G4).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import flows, lowrank, quadrature

COMPOSITIONS = {
    "F1F2": ["T1", "T2"], "F12": ["T12"], "F12F3": ["T12", "T3"],
    "F1F2F3": ["T1", "T2", "T3"], "F1F3F2": ["T1", "T3", "T2"],
    "F12F4": ["T12", "T4"], "F1F2F4": ["T1", "T2", "T4"], "F1F4F2": ["T1", "T4", "T2"],
    "F12F3F4": ["T12", "T3", "T4"], "F1F2F3F4": ["T1", "T2", "T3", "T4"],
}


def mass_transform(M, A, C):
    """Example 4: cancelling M^T and M in
        M^T P' M = A^T P M + M^T P A + Q - M^T P B R^-1 B^T P M
    gives  P' = M^-T A^T P + P A M^-1 + M^-T Q M^-1 - P B R^-1 B^T P,  i.e. the standard DRE
    with A replaced by A M^-1 (the displayed equation; the text's "M^-1 A" is the same
    matrix when A and M are symmetric -- reading G23) and Q = C^T C by (C M^-1)^T (C M^-1).
    B and R are unchanged. Returns (A M^-1, C M^-1)."""
    At = np.linalg.solve(M.T, A.T).T            # A M^-1
    Ct = None if C is None else np.linalg.solve(M.T, C.T).T   # C M^-1
    return At, Ct


def step_sequence(scheme, composition, h):
    """[(flow, tau), ...] in application order for one step."""
    fl = COMPOSITIONS[composition]
    if scheme == "lie":
        return [(f, h) for f in fl]
    if scheme != "strang":
        raise ValueError(scheme)
    if len(fl) == 1:
        return [(fl[0], h)]
    half = [(f, h / 2) for f in fl[:-1]]
    return half + [(fl[-1], h)] + half[::-1]


@dataclass
class OracleOptions:
    tol: float = 1e-16
    rank_cap: int | None = None
    quad_nodes: int = 14
    quad_subpanels: int = 1


class OracleSolver:
    """Runs a splitting scheme on a workloads.Problem in LDL^T form."""

    def __init__(self, prob, h, opts=OracleOptions(), method="auto", dense_apply=False):
        self.p = prob
        self.h = h
        self.o = opts
        A, C = prob.A, prob.C
        if getattr(prob, "M", None) is not None:
            A, C = mass_transform(prob.M, A, C)
        self.A = A
        self.op = flows.Operator(A, method, prob.heat_nx, prob.heat_dim, dense_apply)
        n = prob.n
        if C is not None and C.shape[0] > 0:
            self.LQ, self.DQ = C.T.copy(), np.eye(C.shape[0])   # Q = C^T C (G11)
        else:
            self.LQ, self.DQ = np.zeros((n, 0)), np.zeros((0, 0))
        self.delta = quadrature.panel_width(A, h, opts.quad_subpanels)
        self._LI = {}
        # P0 is compressed when loaded (reading G10)
        L0 = prob.L0 if prob.L0 is not None else np.zeros((n, 0))
        D0 = prob.D0 if prob.D0 is not None else np.zeros((0, 0))
        self.L, self.D = lowrank.column_compression(L0, D0, opts.tol, opts.rank_cap)
        self.t = 0.0

    def integral(self, tau):
        key = round(tau / self.delta)
        if key not in self._LI:
            self._LI[key] = flows.build_integral(self.op, tau, self.delta, self.o.quad_nodes,
                                                 self.LQ, self.DQ, self.o.tol, self.o.rank_cap)
        return self._LI[key]

    def apply_flow(self, f, tau, order=2):
        o, p = self.o, self.p
        if f == "T1":
            self.L, self.D = flows.T1(self.op, tau, self.L, self.D)
        elif f == "T2":
            self.L, self.D = flows.T2(tau, self.L, self.D, self.LQ, self.DQ, o.tol, o.rank_cap)
        elif f == "T3":
            self.L, self.D = flows.T3(tau, self.L, self.D, p.B, p.R)
        elif f == "T4":
            self.L, self.D = flows.T4(tau, self.L, self.D, p.S, order, o.tol, o.rank_cap)
        elif f == "T12":
            LI, DI = self.integral(tau)
            self.L, self.D = flows.T12(self.op, tau, self.L, self.D, LI, DI, o.tol, o.rank_cap)
        else:
            raise ValueError(f)

    def step(self, scheme, composition, nsteps=1):
        seq = step_sequence(scheme, composition, self.h)
        order = 2 if scheme == "strang" else 1
        for _ in range(nsteps):
            for f, tau in seq:
                self.apply_flow(f, tau, order)
            self.t += self.h
        return self.L, self.D

    def factor(self):
        """Canonical (L, D): compressed, L orthonormal, D diagonal sorted by |.| desc."""
        return lowrank.column_compression(self.L, self.D, self.o.tol, None)


def integrate(prob, scheme, composition, nsteps, T=None, opts=OracleOptions(), method="auto"):
    T = prob.T if T is None else T
    s = OracleSolver(prob, T / nsteps, opts, method)
    s.step(scheme, composition, nsteps)
    return s


def richardson(prob, h, nsteps, composition, opts=OracleOptions(), method="auto"):
    """Richardson extrapolation of the Strang composition (the paper cites
    higher-order splitting but restricts itself to Strang). Strang is symmetric,
    so its global error expands in even powers of h and
        P_R(t) = (4 P_{h/2}(t) - P_h(t)) / 3
    cancels the h^2 term: order 4 for smooth problems. Runs the fine (h/2, 2 nsteps) and coarse
    (h, nsteps) integrations and compresses the signed combination
        L = [L_fine, L_coarse],  D = blkdiag(4/3 D_fine, -1/3 D_coarse)
    with the same column compression (indefinite core). Returns (L, D)."""
    fine = OracleSolver(prob, h / 2, opts, method)
    fine.step("strang", composition, 2 * nsteps)
    coarse = OracleSolver(prob, h, opts, method)
    coarse.step("strang", composition, nsteps)
    Lf, Df = fine.factor()
    Lc, Dc = coarse.factor()
    L, D = lowrank.concat(Lf, (4.0 / 3.0) * Df, Lc, Dc, weight=-1.0 / 3.0)
    return lowrank.column_compression(L, D, opts.tol, None)
