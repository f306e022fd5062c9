"""Scratch: init wall time of config 1 (n = 100) after the bench's tiny warm-up solve (lazy-loading
A/B of library builds via DME_LIB)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config
tiny = make_config(1, n=64)
w = dme.Solver(**dme.problem_kwargs(tiny), h=0.001, rank_cap=64)
w.split_step("lie", "F1F2", 3)
torch.cuda.synchronize()
w.close()
prob = make_config(1)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = dme.Solver(**dme.problem_kwargs(prob), h=0.001, rank_cap=64)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s.split_step("lie", "F1F2", 100)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("init %.4f s, 100 steps %.4f s" % (t1 - t0, t2 - t1))
    s.close()
