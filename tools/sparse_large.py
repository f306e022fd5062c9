"""Scratch: steps/s of the sparse-A path in cluster mode vs the grid-wide (large-n) mode, and at
n = 190^2 (beyond one cluster): Strang F12F3, rank cap 64."""
import os, sys, time
sys.path.insert(0, '.')
import scipy.sparse as sps
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config
for nx, force in ((100, False), (100, True), (190, False)):
    if force:
        os.environ["DME_CHEB_GLOBAL"] = "1"
    else:
        os.environ.pop("DME_CHEB_GLOBAL", None)
    prob = make_config(5, nx=nx)
    kw = dict(dme.problem_kwargs(prob), A=sps.csr_matrix(prob.A))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = dme.Solver(**kw, h=0.005, rank_cap=64)
    torch.cuda.synchronize(); init = time.perf_counter() - t0
    s.split_step("strang", "F12F3", 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream); s.split_step("strang", "F12F3", 20); e1.record(s.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"n={prob.n} global={force or nx > 110}: {1e3 / ms:.1f} steps/s ({ms:.3f} ms/step), init {init:.3f} s, "
          f"time-to-T {init + 100 * ms * 1e-3:.3f} s, degree {s.stats()['cheb_degree']}, rank {s.stats()['rank']}")
    s.close()
