"""Scratch: per-phase cycle counts of the fast eigen-compression at config-5-like sizes."""
import sys, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from workloads import make_config
prob = make_config(2, nx=30)
s = dme.Solver(**dme.problem_kwargs(prob), h=5e-3)
rng = np.random.default_rng(0)
for k in (40, 64, 90, 128, 160):
    L = rng.standard_normal((prob.n, k)) * np.logspace(0, -7, k)[None, :]
    s.debug_set_factor(L)
    s.set_profiling(True)
    for _ in range(3):
        s.debug_set_factor(L); s.debug_apply("compress", 0.0)
    st = s.stats()
    # read the per-phase counters from the stats scratch through a small ctypes peek is not exposed;
    print(k, "small_s per call %.1f us" % (st["prof_small_seconds"] / 3 * 1e6), "gram %.1f us" % (st["prof_gram_seconds"] / 3 * 1e6),
          "apply %.1f us" % (st["prof_apply_seconds"] / 3 * 1e6), "rank", s.get_factor()[0].shape[1], "fallbacks", st["eig_fallbacks"])
    ss = s.debug_small_stats()
    print("   phases (kcycles): tridiag %.1f  tmax %.1f  refine %.1f  vectors %.1f  backtr %.1f  check %.1f" % tuple(ss[8:14] / 1e3))
    s.set_profiling(False)
