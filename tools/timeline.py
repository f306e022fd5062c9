"""Scratch: device timeline of a few pipelined steps (DME_TIMELINE=1)."""
import os, sys
os.environ["DME_TIMELINE"] = "1"
sys.path.insert(0, '.')
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(5)
s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64)
s.split_step("strang", "F12F3", 5)
torch.cuda.synchronize()
s.set_profiling(True)
s.split_step("strang", "F12F3", 6)
torch.cuda.synchronize()
s.stats()
