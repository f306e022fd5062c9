"""Scratch timing of the end-to-end path (not the bench contract)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import make_config
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 100
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
prob = make_config(5, nx=nx)
t0 = time.time()
s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64)
torch.cuda.synchronize(); t1 = time.time()
st = s.stats(); print("init", t1 - t0, json.dumps(st))
for rep in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); s.split_step("strang", "F12F3", steps); e1.record(); torch.cuda.synchronize()
    print("steps", steps, "ms/step", e0.elapsed_time(e1) / steps, "rank", s.stats()["rank"])
