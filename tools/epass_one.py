"""Scratch: E_{h/2} L passes at n=10000 inside an NVTX range 'epass' (for ncu --set full)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import heat2d_matrix
k = int(sys.argv[1]) if len(sys.argv) > 1 else 56
A = heat2d_matrix(100)
s = dme.Solver(A=A, h=5e-3)
L = np.random.default_rng(0).random((A.shape[0], k))
s.debug_set_factor(L)
torch.cuda.synchronize()
for _ in range(2):
    torch.cuda.nvtx.range_push("epass")
    s.debug_apply("T1", 2.5e-3)
    torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
