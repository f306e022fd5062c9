"""Scratch: one fast eigen-compression at k=90 (for ncu)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(2, nx=30)
s = dme.Solver(**dme.problem_kwargs(prob), h=5e-3)
rng = np.random.default_rng(0)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 90
L = rng.standard_normal((prob.n, k)) * np.logspace(0, -7, k)[None, :]
s.debug_set_factor(L)
s.debug_apply("compress", 0.0)
torch.cuda.synchronize()
print("done", s.get_factor()[0].shape)
