"""Scratch: one dme_dre_init at config 5 (for an ncu launch list of the init phase)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(5)
s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64)
torch.cuda.synchronize()
print("init_seconds", s.stats()["init_seconds"])
