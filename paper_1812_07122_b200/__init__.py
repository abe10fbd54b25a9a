"""paper_1812_07122_b200 -- B200-native (sm_100a) BLF-LS edge-preserving smoothing.

The hot path of arXiv 1812.07122 (circular gradients -> brute-force (joint)
bilateral filter of each gradient field -> periodic FFT least-squares solve)
as hand-written CUDA behind the C ABI in include/blfls/blfls.h, plus the
reference's other gradient filters on the same solve (bilateral grid,
domain-transform NC-LS, rolling guidance).  This package is the Python
mirror of the reference's ``epls`` entry points
(see :mod:`paper_1812_07122_b200.blfls`).
"""
from .blfls import (CudaError, DtParams, InvalidArgument, RangeSpatialParams, RollingParams,
                    SmootherKind, SmootherSpec, SolveParams, Unsupported, blf_brute, blf_ls, clipart_cleanup,
                    filter_gradients, flash_no_flash, forward_gradients, gaussian_blur, generate, get_plan, irfft2,
                    ls_solve_fft, lsgrad_solve_fft, nc_ls, rfft2, rolling_nc_ls, smooth, sync_plans,
                    texture_removal)
from .configs import CONFIGS, Config

__all__ = [
    "CudaError", "DtParams", "InvalidArgument", "RangeSpatialParams", "RollingParams",
    "SmootherKind", "SmootherSpec", "SolveParams", "Unsupported", "blf_brute", "blf_ls",
    "clipart_cleanup",
    "filter_gradients", "flash_no_flash", "forward_gradients", "gaussian_blur", "generate", "get_plan", "irfft2",
    "ls_solve_fft", "lsgrad_solve_fft", "nc_ls", "rfft2", "rolling_nc_ls", "smooth", "sync_plans",
    "texture_removal", "CONFIGS", "Config",
]
