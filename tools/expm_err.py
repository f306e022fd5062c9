"""Scratch: E_{h/2}, E_h error vs the DST closed form for the int8 and DMMA init products."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1805_08990_b200 as dme
from oracle import exact
from workloads import make_config
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 100
H = 0.005
prob = make_config(5, nx=nx)
n = nx * nx
rng = np.random.default_rng(0)
rows = rng.integers(0, n, 6000)
cols = np.concatenate([rng.integers(0, n, 3000), np.clip(rows[3000:] + rng.integers(-nx - 2, nx + 3, 3000), 0, n - 1)])
for mode in ("auto", "dmma"):
    s = dme.Solver(**dme.problem_kwargs(prob), h=H, rank_cap=64, e_pass=mode)
    for which, t in ((0, H / 2), (1, H)):
        E = s.debug_get_exp(which)
        ref = exact.heat_expm_entries(nx, t, rows, cols)
        scale = np.abs(np.diag(E)).max()
        err = np.abs(E[rows, cols] - ref)
        print(f"{mode:5s} E{which}: max err {err.max():.3e}  rel-to-diag {err.max()/scale:.3e}  median {np.median(err):.3e}  rowsum-max {np.abs(E).sum(1).max():.4f}")
    s.close()
