"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This package holds NO arithmetic of the method (no exponentials, flows, quadrature or
compression): only problem data (finite-difference operators, seeded random factors)
with the shapes and value distributions of the paper's workloads (§5.1,
P:L336-340). See DESIGN.md "Input recipe".
"""
from .generators import (Problem, heat1d_matrix, heat2d_matrix, convdiff2d_matrix,
                         stochastic_heat_matrices, fem2d_matrices, make_config, CONFIGS)

__all__ = ["Problem", "heat1d_matrix", "heat2d_matrix", "convdiff2d_matrix",
           "stochastic_heat_matrices", "fem2d_matrices", "make_config", "CONFIGS"]
