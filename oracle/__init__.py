"""oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of the hot path of
Suzuki, "A Hybrid Factorization Algorithm for Sparse Matrix with Mixed
Precision Arithmetic" (arXiv 2208.01907), written from the paper.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import, call, link or
execute anything in this package.  The product path
(``paper_2208_01907_b200``) never imports it, and the two share no code:
no kernels, headers, helpers, constants or pre/post-processing.  The seeded
input generators live in ``hf_inputs`` (no method arithmetic there).

Citations ``P:n`` are lines of the paper's LaTeX source; ``[Rn]``
are the readings listed in DESIGN.md section 3.

Parts and what pins them (tests/test_oracle_*.py):
  scale               -- closed form examples, idempotence  (pinned)
  factor_lowprec      -- exact-rational left-looking emulation (bitwise),
                         diagonal/special cases, ratio guarantee,
                         reconstruction, FP64 Schur argmax, planted count
                         (pinned)
  factor_lowprec_prefix -- the same body stopped after k pivots (output
                         interface only); pinned by equality with the first
                         k columns of the full run (test_oracle_lowprec.py)
  iterative_refinement -- exact factor converges in one step; the residual
                         ratio equals rho(I - A Q^{-1}) (pinned)
  precond_apply       -- exact factors of diagonal / triangular cases,
                         residual bound (pinned)
  block_gcr, gcr      -- constructed solutions, orthogonality, M=1 == GCR,
                         monotone residual (pinned)
  schur               -- dense Eq. (2) via LAPACK solve, long-double
                         Gaussian elimination for L <= 64 (pinned)
  factor_hard         -- constructed-rank kernels, 2x2 cases, eigen-count,
                         reconstruction (pinned)
  hybrid_solve        -- manufactured solution x_i = i mod 11,
                         dense solve (pinned)
Parity unpinned: the exact block-GCR iterate sequence and the
hard-factor permutation Pi_2 (both are graded by tolerance / kernel dimension,
not bitwise, because S22 carries FP64 cancellation noise).
"""
from .core import (  # noqa: F401
    LowFactor, HardFactor, Hybrid, GcrInfo, OracleBreakdown, OracleNotConverged,
    lib, scale, factor_lowprec, factor_lowprec_prefix, FactorPrefix, precond_apply, block_gcr, gcr,
    iterative_refinement, extract_blocks, schur, factor_hard, hard_solve,
    hybrid_factor, hybrid_solve, kernel_dimension,
)
