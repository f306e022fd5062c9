"""Scratch: per-phase cycle counts of the split eigen-compression (TRI / VEC / FIN) at k = 64..96."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(2, nx=30)
s = dme.Solver(**dme.problem_kwargs(prob), h=5e-3)
rng = np.random.default_rng(0)
for k in (64, 90, 96):
    L = rng.random((prob.n, k)) * np.logspace(0, -7, k)[None, :]
    for _ in range(3):
        s.debug_set_factor(L); s.debug_apply("compress", 0.0)
    torch.cuda.synchronize()
    ss = s.debug_small_stats()
    print(k, "rank", s.get_factor()[0].shape[1], "tri-load %.1f" % (ss[6] / 1e3), "kcycles: tri %.1f tmax %.1f | vec load %.1f msec %.1f twist %.1f backtr %.1f"
          % tuple(ss[8:14] / 1e3))
    print("    fin kcycles: load %.1f check %.1f t3 %.1f" % (ss[14] / 1e3, ss[15] / 1e3, ss[5] / 1e3))
