"""Quadrature rule for the integral term of eq:full (oracle; test infrastructure only).

PAPER.md gives only "high-order quadrature", "a quadrature formula" with nodes
s_k and weights w_k (Alg. 2) and "14 additional evaluations".
Reading G6: composite Gauss-Legendre with q nodes on each of N_p equal
panels of [0, tau]; the panel width is delta = (h/2) / (2^s * P0) where
s = max(0, ceil(log2(||(h/2) A^T||_1 / theta_13))) is the scaling exponent of the
Padé-13 expm of (h/2)A^T (Higham 2005, theta_13 = 5.371920351148152) and P0
(`subpanels`, a power of two) is 1 by default.
"""
from __future__ import annotations

import math

import numpy as np

THETA13 = 5.371920351148152


def gauss_legendre01(q):
    """Nodes c_i in (0,1) and weights w_i (sum 1) of the q-point Gauss-Legendre rule."""
    x, w = np.polynomial.legendre.leggauss(q)
    return (x + 1.0) / 2.0, w / 2.0


def squarings(A, tau):
    """s = max(0, ceil(log2(||tau A^T||_1 / theta_13)))."""
    nrm = float(np.abs(tau * A.T).sum(axis=0).max()) if A.size else 0.0
    if nrm <= THETA13:
        return 0
    return max(0, int(math.ceil(math.log2(nrm / THETA13))))


def panel_width(A, h, subpanels=1):
    return (h / 2.0) / (2 ** squarings(A, h / 2.0) * subpanels)


def composite_rule(tau, delta, q):
    """Nodes s_k and weights w_k of q-point Gauss-Legendre on each panel of width delta."""
    npan = int(round(tau / delta))
    assert npan >= 1 and abs(npan * delta - tau) <= 1e-12 * tau, (tau, delta)
    c, w = gauss_legendre01(q)
    s = (np.arange(npan)[:, None] + c[None, :]) * delta
    wk = np.broadcast_to(w[None, :] * delta, s.shape)
    return s.ravel(), np.array(wk).ravel()
