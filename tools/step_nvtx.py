"""Scratch: config 5 solver, 3 warm steps, then 2 pipelined steps inside an NVTX range 'step'
(for ncu --nvtx-include step/)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(5)
s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64)
s.split_step("strang", "F12F3", 3)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
s.split_step("strang", "F12F3", 3)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
