"""paper_2208_01907_b200 -- B200-native hot path of the hybrid mixed-precision
factorization of Suzuki (arXiv 2208.01907): libhf.so (hand-written CUDA for
sm_100a, C ABI in include/hf.h) and its thin Python binding ``hf``."""
from . import hf  # noqa: F401
from .hf import (  # noqa: F401
    Context, HFError, LowFactor, Hybrid, GcrInfo, hf_scale, hf_factor_lowprec, hf_schur_gcr,
    hf_factor_hard, hf_solve, nccl_unique_id,
)
