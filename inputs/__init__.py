"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NONE of the method's arithmetic (no weights, matching,
prolongators, Galerkin products, smoothing or Krylov steps).  It only builds the
model-problem matrices and right-hand sides the paper benchmarks on
(§4 Eq. 4.1; PAPER.md:537-549 SM anisotropic problem) and the
BASELINE.json config-5 jump-coefficient operator, plus a counter-free PCG64
raw-stream RNG.
"""
from .problems import (  # noqa: F401
    CSR,
    poisson7,
    jump27,
    random_spd,
    diagonal_spd,
    islands,
    uniform01,
    uniform_pm1,
    config_problem,
)
