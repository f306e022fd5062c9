"""One E_h Chebyshev action at config 5 (n = 10^4, k columns) for ncu captures."""
import sys
import numpy as np, scipy.sparse as sps, torch
sys.path.insert(0, ".")
import paper_1805_08990_b200 as dme
from workloads import make_config
k = int(sys.argv[1]) if len(sys.argv) > 1 else 46
A = sps.csr_matrix(make_config(5).A)
s = dme.Solver(A=A, h=0.005)
s.debug_set_factor(np.random.default_rng(0).random((A.shape[0], k)))
s.debug_apply("T1", 0.005)
torch.cuda.synchronize()
s.close()
