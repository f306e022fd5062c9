"""Small workload touching every kernel family of libdme.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): int8 E pass (Stream-K fixup) and init products,
DMMA gemm_nt, pivoted LU (Padé path), eigen kernels (fast / split / Jacobi fallback), refined
compression (complement basis, tail assemble), Gram congruence pipeline, Chebyshev cluster
kernels (sparse A), T4 with S, virtual shards (staging + NCCL allgather)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import scipy.sparse as sps
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config

h = 0.005
which = sys.argv[1] if len(sys.argv) > 1 else "all"
def run(prob, scheme, comp, N, **kw):
    s = dme.Solver(**dme.problem_kwargs(prob), h=h, rank_cap=64, **kw)
    s.split_step(scheme, comp, N)
    L, D = s.get_factor()
    s.close()
    return L.shape[1]
if which in ("all", "dense"):
    print("heat dense F12F3", run(make_config(5, nx=12), "strang", "F12F3", 4))
    print("heat dmma", run(make_config(5, nx=12), "strang", "F12F3", 3, e_pass="dmma"))
    print("convdiff pade", run(make_config(3, nx=10), "strang", "F12F3", 3))
    print("config4 T4", run(make_config(4, nx=8), "strang", "F12F3F4", 2))
    print("virtual shards", run(make_config(5, nx=12), "strang", "F12F3", 3, virtual_world=3))
if which in ("all", "sparse"):
    prob = make_config(5, nx=12)
    kw = dme.problem_kwargs(prob)
    kw["A"] = sps.csr_matrix(prob.A)
    s = dme.Solver(**kw, h=h, rank_cap=64)
    s.split_step("strang", "F12F3", 3)
    print("sparse", s.get_factor()[0].shape)
    s.close()
torch.cuda.synchronize()
print("done")
