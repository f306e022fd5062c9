"""Problem generators (problem data only; no method arithmetic).

Readings of the paper used here (all listed in DESIGN.md §Readings):
  * G13  FD scaling: n_x interior points per direction, dx = 1/(n_x+1),
         A = (n_x+1)^2 (T (x) I + I (x) T), T = tridiag(1,-2,1)   ("central second-order
         finite differences with n_x grid points").
  * G12  "randomly chosen" factors = uniform [0,1] entries (MATLAB `rand`), D = I,
         numpy PCG64 with seed 1000*config + role (1=C, 2=L0, 3=B, 4=S).
  * G17  convection-diffusion for config 3: A = Lap - 10 xi1 d/dxi1 - 100 xi2 d/dxi2, central FD.
  * G18  Example 2: Dirichlet on x=0 and y=0, control edge x=1 (x=u), stochastic
         Robin edge y=1 (n.grad x = 0.5(0.5 + dW) x) by a one-sided ghost-node elimination:
         A gets +0.25/dx on the y=1 row, S = diag(0.5/dx) on the y=1 row, B = (n_x+1)^2 on the
         x=1 column; C = (1/n)(1,...,1) (Q = C^T C, reading G11), P0 = 0.
All matrices are float64, C-contiguous numpy arrays; A is returned DENSE because the
north star's boundary takes a dense A (BASELINE.json north_star: "dle_init/dre_init with A").
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class Problem:
    """One differential matrix equation  P' = A^T P + P A + Q [+ S P S^T] [- P B R^-1 B^T P].

    Q = C^T C (C is p x n), P(0) = L0 D0 L0^T.  B, R, S optional (None).
    `heat_nx` / `heat_dim` are structure hints (the operator is the Dirichlet FD Laplacian)
    that let test code use the closed-form sine eigenbasis; they carry no arithmetic.
    """
    A: np.ndarray
    C: Optional[np.ndarray]
    L0: Optional[np.ndarray]
    D0: Optional[np.ndarray]
    B: Optional[np.ndarray] = None
    R: Optional[np.ndarray] = None
    S: Optional[np.ndarray] = None
    T: float = 0.5
    name: str = ""
    heat_nx: Optional[int] = None
    heat_dim: Optional[int] = None
    meta: dict = field(default_factory=dict)
    M: Optional[np.ndarray] = None   # mass matrix of  M^T P' M = A^T P M + M^T P A + ...

    @property
    def n(self) -> int:
        return self.A.shape[0]

    @property
    def is_dre(self) -> bool:
        return self.B is not None


def _tridiag(n: int) -> np.ndarray:
    T = np.zeros((n, n))
    i = np.arange(n)
    T[i, i] = -2.0
    T[i[:-1], i[:-1] + 1] = 1.0
    T[i[1:], i[1:] - 1] = 1.0
    return T


def heat1d_matrix(n: int) -> np.ndarray:
    """1D Dirichlet Laplacian on (0,1), n interior points, dx = 1/(n+1)."""
    return (n + 1) ** 2 * _tridiag(n)


def heat2d_matrix(nx: int) -> np.ndarray:
    """2D Dirichlet Laplacian on the unit square, nx^2 unknowns."""
    T = _tridiag(nx)
    I = np.eye(nx)
    return (nx + 1) ** 2 * (np.kron(T, I) + np.kron(I, T))


def convdiff2d_matrix(nx: int, c1: float = 10.0, c2: float = 100.0) -> np.ndarray:
    """A = Lap - c1*xi1*d/dxi1 - c2*xi2*d/dxi2, central differences (reading G17).

    Unknown ordering: index = i*nx + j with xi1 = (i+1)dx, xi2 = (j+1)dx.
    """
    n = nx * nx
    dx = 1.0 / (nx + 1)
    A = heat2d_matrix(nx)
    for i in range(nx):
        for j in range(nx):
            k = i * nx + j
            x1, x2 = (i + 1) * dx, (j + 1) * dx
            if i + 1 < nx:
                A[k, k + nx] -= c1 * x1 / (2 * dx)
            if i - 1 >= 0:
                A[k, k - nx] += c1 * x1 / (2 * dx)
            if j + 1 < nx:
                A[k, k + 1] -= c2 * x2 / (2 * dx)
            if j - 1 >= 0:
                A[k, k - 1] += c2 * x2 / (2 * dx)
    assert A.shape == (n, n)
    return A


def stochastic_heat_matrices(nx: int):
    """Example 2 structure (reading G18). Returns (A, B, S, C)."""
    n = nx * nx
    dx = 1.0 / (nx + 1)
    A = heat2d_matrix(nx)
    S = np.zeros((n, n))
    B = np.zeros((n, 1))
    for i in range(nx):          # i: x-index, j: y-index, index = i*nx + j
        for j in range(nx):
            k = i * nx + j
            if j == nx - 1:      # Robin edge y = 1
                A[k, k] += 0.25 / dx
                S[k, k] = 0.5 / dx
            if i == nx - 1:      # control edge x = 1: boundary value u enters the stencil
                B[k, 0] = (nx + 1) ** 2
    C = np.full((1, n), 1.0 / n)
    return A, B, S, C


def fem2d_matrices(nx: int, conv: float = 0.0):
    """Steel-cooling STRUCTURE (Example 4; the Oberwolfach data itself is not available):
    P1 finite elements on the unit square, uniform grid of spacing 1/nx, every square split into two
    triangles by its (0,0)-(1,1) diagonal; homogeneous Dirichlet on x = 0 and y = 0, Neumann on
    x = 1 and y = 1 (unknowns: nodes (i, j), i, j = 1..nx, index (i-1) nx + (j-1)).
    Returns (M, A, B, C): M consistent mass, A = -(stiffness) - conv * (x-derivative transport,
    element-wise, nonsymmetric when conv != 0), B = boundary mass of the Neumann edge x = 1 (boundary
    control, m = 1), C = 2 x n temperature differences between node pairs ("an operator that
    measures temperature differences between different points")."""
    n = nx * nx
    hh = 1.0 / nx
    M = np.zeros((n, n))
    A = np.zeros((n, n))

    def idx(i, j):
        return (i - 1) * nx + (j - 1) if i >= 1 and j >= 1 else -1

    Ke = 0.5 * np.array([[2.0, -1.0, -1.0], [-1.0, 1.0, 0.0], [-1.0, 0.0, 1.0]])  # right angle first
    Me = hh * hh / 24.0 * np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]])
    for i in range(nx):
        for j in range(nx):
            # lower triangle: right angle at (i+1, j), legs to (i, j) and (i+1, j+1)
            # upper triangle: right angle at (i, j+1), legs to (i+1, j+1) and (i, j)
            for tri, xs in (([(i + 1, j), (i, j), (i + 1, j + 1)], None),
                            ([(i, j + 1), (i + 1, j + 1), (i, j)], None)):
                g = [idx(a, b) for a, b in tri]
                # transport c d/dx: element matrix int phi_a d(phi_b)/dx = (area/3) d(phi_b)/dx
                xb = np.array([a for a, _ in tri], dtype=float) * hh
                yb = np.array([b for _, b in tri], dtype=float) * hh
                det = (xb[1] - xb[0]) * (yb[2] - yb[0]) - (xb[2] - xb[0]) * (yb[1] - yb[0])
                dphidx = np.array([yb[1] - yb[2], yb[2] - yb[0], yb[0] - yb[1]]) / det
                Ce = np.outer(np.full(3, abs(det) / 6.0), dphidx)
                for a in range(3):
                    if g[a] < 0:
                        continue
                    for b in range(3):
                        if g[b] < 0:
                            continue
                        M[g[a], g[b]] += Me[a, b]
                        A[g[a], g[b]] -= Ke[a, b] + conv * Ce[a, b]
    B = np.zeros((n, 1))
    for j in range(1, nx + 1):           # Neumann edge x = 1 (i = nx): boundary mass, lumped
        B[idx(nx, j), 0] = hh if j < nx else hh / 2
    C = np.zeros((2, n))
    C[0, idx(nx // 2, nx // 2)], C[0, idx(nx, nx)] = 1.0, -1.0
    C[1, idx(max(1, nx // 4), nx)], C[1, idx(nx, max(1, nx // 4))] = 1.0, -1.0
    return M, A, B, C


def _rng(config: int, role: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(1000 * config + role))


def uniform_factor(config: int, role: int, rows: int, cols: int) -> np.ndarray:
    return _rng(config, role).random((rows, cols))


# BASELINE.json configs (index 1..5), with the survey's §8(d) recipe.
CONFIGS = {
    1: dict(desc="DLE 1D heat n=100, C rank-1, Lie F1F2, T=0.1, 100 steps", kind="heat1d", n=100,
            p=1, r0=5, m=0, T=0.1, nsteps=100, scheme="lie", composition="F1F2"),
    2: dict(desc="DLE 2D heat n=1024, Strang F1F2 and F12 with 5-node Gauss", kind="heat2d", nx=32,
            p=1, r0=5, m=0, T=0.5, nsteps=100, scheme="strang", composition="F12",
            quad_nodes=5, quad_subpanels=4),
    3: dict(desc="DRE 2D convection-diffusion n=2500, Strang F12F3", kind="convdiff2d", nx=50,
            p=2, r0=5, m=1, T=0.5, nsteps=100, scheme="strang", composition="F12F3"),
    4: dict(desc="generalized DRE (S P S^T) n=4900, Lie/Strang F12F3F4 and F1F2F3F4",
            kind="stochastic", nx=70, p=1, r0=0, m=1, T=0.5, nsteps=100, scheme="strang",
            composition="F12F3F4"),
    5: dict(desc="DRE 2D heat n=10000 FP64, rank cap 64, Strang F12F3", kind="heat2d", nx=100,
            p=2, r0=5, m=1, T=0.5, nsteps=100, scheme="strang", composition="F12F3",
            rank_cap=64),
    # SURVEY §8(f3), beyond BASELINE.json's five: Example 4's mass-matrix DRE structure
    # on a synthetic P1 FEM pair, R^-1 = I, P0 = 0
    6: dict(desc="mass-matrix DRE (steel-cooling structure), P1 FEM n=nx^2, Strang F12F3",
            kind="fem2d", nx=40, p=2, r0=0, m=1, T=0.5, nsteps=100, scheme="strang",
            composition="F12F3"),
}


def make_config(config: int, nx: Optional[int] = None, n: Optional[int] = None,
                rinv: float = 1.0, dle: bool = False, conv: Optional[float] = None) -> Problem:
    """Build the problem of BASELINE.json config `config` (optionally at a smaller size).

    `nx`/`n` override the size (same recipe, e.g. the n=25 verification problems of P:L370).
    `rinv` sets R = (1/rinv) I (P:L384 uses R^-1 in {1, 1e-3}). `dle=True` drops B.
    """
    c = dict(CONFIGS[config])
    if conv is not None:
        c["conv"] = conv
    kind = c["kind"]
    heat_nx = heat_dim = None
    S = None
    if kind == "heat1d":
        nn = n or c["n"]
        A = heat1d_matrix(nn)
        heat_nx, heat_dim = nn, 1
    elif kind == "heat2d":
        nxx = nx or c["nx"]
        A = heat2d_matrix(nxx)
        heat_nx, heat_dim = nxx, 2
    elif kind == "convdiff2d":
        nxx = nx or c["nx"]
        A = convdiff2d_matrix(nxx)
    elif kind == "stochastic":
        nxx = nx or c["nx"]
        A, Bs, S, Cs = stochastic_heat_matrices(nxx)
    elif kind == "fem2d":
        nxx = nx or c["nx"]
        Mm, A, Bs, Cs = fem2d_matrices(nxx, conv=c.get("conv", 0.0))
    else:
        raise ValueError(kind)
    N = A.shape[0]
    if kind in ("stochastic", "fem2d"):
        C = Cs
        B = None if dle else Bs
    else:
        C = uniform_factor(config, 1, c["p"], N)
        B = None if (dle or c["m"] == 0) else uniform_factor(config, 3, N, c["m"])
    r0 = c["r0"]
    L0 = uniform_factor(config, 2, N, r0) if r0 > 0 else np.zeros((N, 0))
    D0 = np.eye(r0)
    R = None if B is None else np.eye(B.shape[1]) / rinv
    return Problem(A=np.ascontiguousarray(A), C=C, L0=L0, D0=D0, B=B, R=R, S=S, T=c["T"],
                   name=f"config{config}", heat_nx=heat_nx, heat_dim=heat_dim,
                   meta=dict(c, config=config), M=Mm if kind == "fem2d" else None)
