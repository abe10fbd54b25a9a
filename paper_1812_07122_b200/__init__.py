"""paper_1812_07122_b200 -- B200-native (sm_100a) BLF-LS edge-preserving smoothing.

The hot path of arXiv 1812.07122 (circular gradients -> brute-force (joint)
bilateral filter of each gradient field -> periodic FFT least-squares solve)
as hand-written CUDA behind the C ABI in include/blfls/blfls.h.  This package
is the Python mirror of the reference's ``epls`` entry points
(see :mod:`paper_1812_07122_b200.blfls`).
"""
from .blfls import (CudaError, InvalidArgument, RangeSpatialParams, SmootherKind, SmootherSpec,
                    SolveParams, Unsupported, blf_ls, filter_gradients, flash_no_flash, generate,
                    get_plan, irfft2, ls_solve_fft, lsgrad_solve_fft, rfft2, smooth, sync_plans)
from .configs import CONFIGS, Config

__all__ = [
    "CudaError", "InvalidArgument", "RangeSpatialParams", "SmootherKind", "SmootherSpec",
    "SolveParams", "Unsupported", "blf_ls", "filter_gradients", "flash_no_flash", "generate",
    "get_plan", "irfft2", "ls_solve_fft", "lsgrad_solve_fft", "rfft2", "smooth", "sync_plans", "CONFIGS",
    "Config",
]
