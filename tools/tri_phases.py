"""Scratch (with a -DDME_TRI_PHASES build loaded through DME_LIB): per-phase cycle sums of the
Householder tridiagonalisation -- mat-vec phase (thread 0 view, incl. barrier), warp 0's phase-B work,
warp 0's barrier wait, warp 1's phase-B work and barrier wait, warp 2's phase-B work -- isolated
(k = 57, 90) and in the pipelined config-5 step (the last compression: pass 2, TRI on s x s)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import make_config
def show(tag, ss):
    print("%-20s kernel %6.0fk tri %6.0fk | sums (kcycles): A %6.1f  w0-work %6.1f  w0-bar %6.1f  w1-work %6.1f  w1-bar %6.1f  w2-work %6.1f"
          % (tag, ss[7] / 1e3, ss[8] / 1e3, ss[10] / 1e3, ss[11] / 1e3, ss[12] / 1e3, ss[13] / 1e3, ss[14] / 1e3, ss[15] / 1e3))
prob = make_config(2, nx=30)
s = dme.Solver(**dme.problem_kwargs(prob), h=5e-3, compression="gram")
rng = np.random.default_rng(0)
for k in (57, 90):
    L = rng.random((prob.n, k)) * np.logspace(0, -3, k)[None, :]
    for _ in range(2):
        s.debug_set_factor(L); s.debug_apply("compress", 0.0)
    torch.cuda.synchronize()
    show("isolated", s.debug_small_stats())
prob = make_config(5)
p = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64)
for _ in range(2):
    p.split_step("strang", "F12F3", 6)
    torch.cuda.synchronize()
    show("pipeline (pass 2)", p.debug_small_stats())
