"""Scratch: config 6 (mass-matrix DRE) timing pieces."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 70
prob = make_config(6, nx=nx)
print("n", prob.n, flush=True)
t0 = time.time()
s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64)
torch.cuda.synchronize()
print("init", time.time() - t0, s.stats()["squarings"], s.stats()["q_full"], flush=True)
for N in (1, 5, 20):
    t0 = time.time()
    s.split_step("strang", "F12F3", N)
    torch.cuda.synchronize()
    print("steps", N, "ms/step", (time.time() - t0) / N * 1e3, "rank", s.stats()["rank"], flush=True)
