"""paper_2102_08463_b200 -- B200-native (sm_100a) NUFFT, drop-in for nufftkit.

Hot path (CUDA, libnufft_b200.so): setpts bin sort (FP64 fold, histogram,
scan, stable radix permutation, subproblems), ES-kernel spreading (GM,
GM-sort, shared-memory SM) and interpolation, kernel-Fourier deconvolution
and its type-2 amplify/pad; the fine-grid FFT is cuFFT.

API (mirrors the reference nufftkit package and its SPEC):
  make_plan / set_points / execute / destroy, TransformPlan, Plan
  nufft2d1 / nufft2d2 / nufft3d1 / nufft3d2 one-shot calls
  kernel.*  (select_kernel_params, kernel_fourier, build_correction_factors, ...)
  stages.*  (bin_sort, build_subproblems, spread_gm/_gm_sort/_sm,
             interpolate, fft_fine, deconvolve_type1/2)
"""

from . import _lib
from .kernel import (KernelParams, build_correction_factors, centered_freqs, eval_kernel,
                     kernel_fourier, select_kernel_params, tolerance_to_width)
from .plan import GridSpec, Plan, TransformPlan, destroy, execute, make_plan, next_smooth, \
    set_points
from .oneshot import nufft2d1, nufft2d2, nufft3d1, nufft3d2

__all__ = ["KernelParams", "build_correction_factors", "centered_freqs", "eval_kernel",
           "kernel_fourier", "select_kernel_params", "tolerance_to_width", "GridSpec", "Plan",
           "TransformPlan", "destroy", "execute", "make_plan", "next_smooth", "set_points",
           "nufft2d1", "nufft2d2", "nufft3d1", "nufft3d2"]

# Fail loudly at import if the CUDA library is missing: there is no CPU path.
_lib.lib()
