"""B200-native RSRS (randomized strong recursive skeletonization, arXiv 2311.01451).

The hot path -- the level-by-level batched per-box compress-and-eliminate
sweep -- lives in librsrs.so (hand-written sm_100a CUDA behind the C ABI
include/rsrs.h).  This package is a thin ctypes binding over it.
"""
from .rsrs import (Tree, Factorization, factor, RSRSError, version, sample_matvec, sample_matvec_rows, memory_info,  # noqa: F401
                   release_memory, NcclComm, factor_emulated, solve_emulated, apply_emulated,
                   RSRS_F64, RSRS_C128, EXPORTS, LIB_PATH, SAMPLER_PATH)
