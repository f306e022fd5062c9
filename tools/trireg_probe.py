"""Scratch: per-phase cycles of the register tridiagonalisation (eig_trireg_kernel) at k = 64..96."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(2, nx=30)
s = dme.Solver(**dme.problem_kwargs(prob), h=5e-3, compression="gram")
rng = np.random.default_rng(0)
for k in (64, 90, 96):
    L = rng.random((prob.n, k)) * np.logspace(0, -7, k)[None, :]
    for _ in range(3):
        s.debug_set_factor(L); s.debug_apply("compress", 0.0)
    torch.cuda.synchronize()
    ss = s.debug_small_stats()
    st = k - 2
    print(k, "tri total %.0f cyc/step | warp0: matvec %.0f bar2 %.0f update %.0f | refl (warp1, x16): norm %.0f scalars %.0f" % (
        ss[8] / st, ss[5] / st, ss[6] / st, ss[7] / st, ss[2] * 16 / st, ss[3] * 16 / st))
