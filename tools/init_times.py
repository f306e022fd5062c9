import sys, time
sys.path.insert(0, '.')
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(5)
A = torch.from_numpy(prob.A).cuda()
for rep in range(3):
    kw = dict(dme.problem_kwargs(prob), A=A)
    torch.cuda.synchronize(); t0 = time.time()
    s = dme.Solver(**kw, h=0.005, rank_cap=64)
    torch.cuda.synchronize(); print("init wall", time.time() - t0, "lib", s.stats()["init_seconds"], flush=True)
    s.close(); del s
