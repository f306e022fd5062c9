"""Scratch: eigen-kernel phase cycles vs the grading of the factor (is the pipelined tail pass slow
because of its values?). Isolated compressions of L = rand * logspace(0, -g) at k = 57 and 90."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(2, nx=30)
s = dme.Solver(**dme.problem_kwargs(prob), h=5e-3)
rng = np.random.default_rng(0)
for k in (57, 90):
    for g, dup in ((7, 0), (16, 0), (24, 0), (7, 20), (16, 20)):
        L = rng.random((prob.n, k)) * np.logspace(0, -g, k)[None, :]
        if dup:
            L[:, k - dup:] = L[:, :dup] @ rng.random((dup, dup)) * 1e-3  # exactly dependent columns
        for _ in range(3):
            s.debug_set_factor(L); s.debug_apply("compress", 0.0)
        torch.cuda.synchronize()
        ss = s.debug_small_stats()
        v = [x / 1e3 for x in [ss[6]] + list(ss[8:14]) + [ss[14], ss[15], ss[5]]]; print("tri kernel total kcyc %.1f" % (ss[7] / 1e3))
        print("k %d grade 1e-%d dup %d rank %d kcyc: tri-load %.1f tri %.1f tmax %.1f | vec load %.1f msec %.1f twist %.1f backtr %.1f | fin %.1f %.1f %.1f"
              % ((k, g, dup, s.get_factor()[0].shape[1]) + tuple(v)))
