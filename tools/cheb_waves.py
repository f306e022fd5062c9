"""Probe: Chebyshev action time vs column count k at a fixed columns-per-cluster C (DME_CHEB_C)."""
import os, sys, time
import numpy as np, scipy.sparse as sps, torch
sys.path.insert(0, ".")
import paper_1805_08990_b200 as dme
from workloads import make_config
A = sps.csr_matrix(make_config(5).A)
h = 0.005
K = dme.cheb_coeffs(h * 4 * 101 ** 2).size - 1
for k in [int(x) for x in sys.argv[1:]]:
    s = dme.Solver(A=A, h=h)
    L = np.random.default_rng(0).random((A.shape[0], k))
    ts = []
    for _ in range(4):
        s.debug_set_factor(L); torch.cuda.synchronize(); t0 = time.perf_counter()
        s.debug_apply("T1", h); ts.append(time.perf_counter() - t0)
    s.close()
    print(f"C={os.environ.get('DME_CHEB_C')} k={k:3d} {min(ts)*1e6:8.1f} us {min(ts)*1e6/K:6.2f} us/degree", flush=True)
