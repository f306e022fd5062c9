"""Scratch: exactly one fast eigen-compression at size k (for ncu: no compression during init)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import heat2d_matrix
k = int(sys.argv[1]) if len(sys.argv) > 1 else 90
A = heat2d_matrix(30)
s = dme.Solver(A=A, h=5e-3)
rng = np.random.default_rng(0)
L = rng.standard_normal((A.shape[0], k)) * np.logspace(0, -7, k)[None, :]
s.debug_set_factor(L)
s.debug_apply("compress", 0.0)
torch.cuda.synchronize()
print("done", s.get_factor()[0].shape)
