"""Scratch: eigen-kernel phase cycles of the LAST compression of a pipelined config-5 run
(the tail pass of the last step) -- compare with tools/eig_split_probe.py's isolated kernels."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(5)
s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64)
for it in range(3):
    s.split_step("strang", "F12F3", 6)
    torch.cuda.synchronize()
    ss = s.debug_small_stats()
    v = [x / 1e3 for x in [ss[6]] + list(ss[8:14])]
    print("pipeline last pass kcycles: tri-load %.1f tri %.1f tmax %.1f | vec load %.1f msec %.1f twist %.1f backtr %.1f" % tuple(v))
