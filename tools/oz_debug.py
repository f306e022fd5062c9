"""Scratch: locate the disagreement between the int8 (Ozaki) and DMMA E passes inside the solver."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1805_08990_b200 as dme
from oracle import lowrank
from workloads import make_config

for nx in [int(a) for a in sys.argv[1:]] or [10, 30]:
    prob = make_config(5, nx=nx)
    n = prob.n
    S = {m: dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64, e_pass=m) for m in ("auto", "dmma")}
    Ea = S["auto"].debug_get_exp(0); Ed = S["dmma"].debug_get_exp(0)
    print(nx, "E_half equal:", np.array_equal(Ea, Ed), "E_full eq:", np.array_equal(S["auto"].debug_get_exp(1), S["dmma"].debug_get_exp(1)))
    for w in (0, 1):
        Ia, Id = S["auto"].debug_get_integral(w), S["dmma"].debug_get_integral(w)
        print("  integral", w, Ia.shape, Id.shape, lowrank.rel_diff(Ia, np.eye(Ia.shape[1]), Id, np.eye(Id.shape[1])))
    La, Da = S["auto"].get_factor(); Ld, Dd = S["dmma"].get_factor()
    print("  initial factor", La.shape, Ld.shape, lowrank.rel_diff(La, Da, Ld, Dd))
    rng = np.random.default_rng(1)
    for k in (5, 20, 40, 60):
        L = rng.random((n, k))
        for m in S:
            S[m].debug_set_factor(L)
            S[m].debug_apply("T1", 0.0025)
        ref = Ea @ L
        for m in S:
            Z, _ = S[m].get_factor()
            print(f"  T1 k={k} {m}: max rel err {np.abs(Z - ref).max() / np.abs(ref).max():.3e}  shape {Z.shape}")
    for m in S:
        S[m].close()
    for steps in (1, 2, 3, 8):
        out = {}
        for m in ("auto", "dmma"):
            s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64, e_pass=m)
            for _ in range(steps):
                s.split_step("strang", "F12F3", 1)
            out[m + "_1by1"] = s.get_factor(); s.close()
            s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64, e_pass=m)
            s.split_step("strang", "F12F3", steps)
            out[m] = s.get_factor(); st = s.stats(); s.close()
        ref = out["dmma_1by1"]
        print(f"  steps={steps}", {k: f"{lowrank.rel_diff(*v, *ref):.2e}" for k, v in out.items()}, "ozpasses", st["ozaki_passes"])
