"""Scratch: one isolated compression (k = 90) of L = rand * logspace(0, -g) for ncu (argv[1] = g)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import make_config
g = float(sys.argv[1])
prob = make_config(2, nx=30)
s = dme.Solver(**dme.problem_kwargs(prob), h=5e-3)
rng = np.random.default_rng(0)
L = rng.random((prob.n, 90)) * np.logspace(0, -g, 90)[None, :]
s.debug_set_factor(L)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("probe")
s.debug_apply("compress", 0.0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
