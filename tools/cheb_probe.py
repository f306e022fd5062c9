"""Timing probe of the sparse Chebyshev action (csrc/cheb.cu) through the public API:
per-launch time vs matrix (stencil / diagonal), column count k and degree (tau)."""
import sys
import time

import numpy as np
import scipy.sparse as sps
import torch

sys.path.insert(0, ".")
import paper_1805_08990_b200 as dme  # noqa: E402
from workloads import make_config  # noqa: E402


def t_action(A, k, h, which, reps=5):
    s = dme.Solver(A=A, h=h)
    L = np.random.default_rng(0).random((A.shape[0], k))
    s.debug_set_factor(L)
    s.debug_apply("T1", which)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s.debug_set_factor(L)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.debug_apply("T1", which)
        ts.append(time.perf_counter() - t0)
    deg = None
    s.close()
    return min(ts) * 1e6


prob = make_config(5)
A = sps.csr_matrix(prob.A)
D = sps.diags(prob.A.diagonal()).tocsr()
for name, M in (("stencil", A), ("diag", D)):
    for k in (5, 46, 64):
        for h in (0.005, 0.00125):
            us = t_action(M, k, h, h)
            g = h * 4 * 101 ** 2
            K = dme.cheb_coeffs(g).size - 1
            print(f"{name:8s} k={k:3d} tau={h:.5f} K={K:4d} {us:9.1f} us  {us / K:6.2f} us/degree", flush=True)
