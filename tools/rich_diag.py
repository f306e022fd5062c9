"""Scratch: where the GPU/oracle Richardson difference comes from."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1805_08990_b200 as dme
from oracle import lowrank
from oracle.schemes import OracleOptions, OracleSolver, richardson
from workloads import make_config
prob = make_config(5, nx=8)
h, N = 0.01, 10
fine = dme.Solver(**dme.problem_kwargs(prob), h=h / 2)
coarse = dme.Solver(**dme.problem_kwargs(prob), h=h)
fine.split_step("strang", "F12F3", 2 * N)
coarse.split_step("strang", "F12F3", N)
Lf, Df = fine.get_factor(); Lc, Dc = coarse.get_factor()
Lg, Dg = dme.extrapolate(fine, coarse)
of = OracleSolver(prob, h / 2, OracleOptions()); of.step("strang", "F12F3", 2 * N)
oc = OracleSolver(prob, h, OracleOptions()); oc.step("strang", "F12F3", N)
print("fine parity", lowrank.rel_diff(Lf, Df, *of.factor()))
print("coarse parity", lowrank.rel_diff(Lc, Dc, *oc.factor()))
L, D = lowrank.concat(Lf, 4 / 3 * Df, Lc, Dc, weight=-1 / 3)
Lh, Dh = lowrank.column_compression(L, D, 1e-16)
print("gpu extrapolate vs host combination of gpu factors", lowrank.rel_diff(Lg, Dg, Lh, Dh))
Lo, Do = richardson(prob, h, N, "F12F3", OracleOptions())
print("host combination of gpu factors vs oracle richardson", lowrank.rel_diff(Lh, Dh, Lo, Do))
print("gpu vs oracle richardson", lowrank.rel_diff(Lg, Dg, Lo, Do))
Pf = lowrank.to_dense(Lf, Df); Pc = lowrank.to_dense(Lc, Dc); Pr = (4 * Pf - Pc) / 3
print("norms", np.linalg.norm(Pf), np.linalg.norm(Pc), np.linalg.norm(Pr), np.linalg.norm(Pf - Pc))
