"""hf_inputs -- seeded synthetic workloads for BASELINE.json's five configs.

This module is shared by the oracle side (tests, bench cpu_baseline) and the
CUDA side (tests, bench, smoke).  It holds none of the method's arithmetic:
it only builds the UNSCALED matrices Kbar and right-hand sides (scaling is
step a1 of the method and lives on each side separately).

Recipes (DESIGN.md section 4 states them in full):
  C0 planted  L=256,   4 hard u~U[-10,-8], rest U[-2,0], 30% negative
  C1 Neumann  64x64 5-point Laplacian, 3 inclusions (8x8) kappa=1e6, joined by 1e-8
  C2 planted  L=16384, 64 hard u~U[-12,-6]
  C3 saddle   [A B^T; B 0], A: 2-dof Laplacian 96x96, 1e4 jump across a seeded line
  C4 planted  L=65536, 256 hard u~U[-12,-6]
  NEXT-3 (nonsymmetric): stokes_ns [A B^T; -B delta D] (T8, T24, T96) and
          delta = 0 ([A B^T; -B 0], H8); colmajor() gives the column-major bytes
"""
from .configs import (  # noqa: F401
    CONFIGS, ConfigSpec, make_kbar, make_rhs, manufactured_x, planted, neumann_inclusions,
    saddle_point, config_seed, stokes_ns, colmajor,
)
