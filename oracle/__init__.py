"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct float64 NumPy/SciPy implementation of what the hot path
computes, written from PAPER.md (arXiv 1805.08990) in the paper's notation (L, D, T_k, ...).
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it.  The CUDA product path (paper_1805_08990_b200/) never imports, links or
executes anything here, and this package never imports the product package: the two share
no code (only the seeded input generators in `workloads/`, which hold no method arithmetic).

Modules:
  lowrank     concat / column_compression / to_dense / parity metric
  quadrature  Gauss-Legendre rule and the composite-panel reading G6
  flows       T1, T2, T3, T4, T12 (Alg. 2-4)
  schemes     Lie / Strang compositions
  exact       brute-force exact references used to PIN the oracle (closed forms, Van Loan,
              Kronecker, Hamiltonian Moebius, vectorised ODE) — DESIGN.md §Pins
Parity status: every function above is pinned by tests/test_oracle_*.py (-m "not gpu");
none is "parity unpinned".
"""
