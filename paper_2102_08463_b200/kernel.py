"""ES spreading kernel parameters and deconvolution factors.

Mirror of the reference ``nufftkit.kernel`` (kernel.py:1-205): same names,
argument meaning, return types and ValueError behaviour.  The plan-time
math runs in the C library (nk_tolerance_to_width, nk_kernel_fourier in
csrc/nk_host.cpp); the per-execute deconvolution is the CUDA kernel K8/K9
(csrc/nk_deconv.cu).
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["KernelParams", "select_kernel_params", "tolerance_to_width", "eval_kernel",
           "kernel_fourier", "centered_freqs", "build_correction_factors"]

MIN_WIDTH = 2            # kernel.py:27
MAX_WIDTH = 16           # kernel.py:28
SINGLE_EPS_FLOOR = 1e-6  # kernel.py:31
QUAD_NODES = 100         # kernel.py:36

_REAL_DTYPES = {"single": np.float32, "double": np.float64}
_COMPLEX_DTYPES = {"single": np.complex64, "double": np.complex128}


@dataclass(frozen=True)
class KernelParams:
    """kernel.py:42-72."""

    epsilon: float
    w: int
    beta: float
    alpha: tuple
    precision: str

    @property
    def real_dtype(self):
        return _REAL_DTYPES[self.precision]

    @property
    def complex_dtype(self):
        return _COMPLEX_DTYPES[self.precision]

    @property
    def halo(self) -> int:
        return (self.w + 1) // 2


def _check_precision(precision):
    if precision not in _REAL_DTYPES:
        raise ValueError(f"precision must be 'single' or 'double', got {precision!r}")
    return precision


def tolerance_to_width(epsilon, precision="double"):
    """kernel.py:83-103: (effective epsilon, w, beta = 2.30 w)."""
    _check_precision(precision)
    eps_eff, w, beta, cl = ctypes.c_double(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
    rc = _lib.lib().nk_tolerance_to_width(float(epsilon), _lib.PRECISIONS[precision],
                                          ctypes.byref(eps_eff), ctypes.byref(w),
                                          ctypes.byref(beta), ctypes.byref(cl))
    if rc:
        raise ValueError(f"tolerance must lie in (0, 1), got {float(epsilon)}")
    if cl.value:
        warnings.warn(f"tolerance {float(epsilon):g} is below single-precision rounding; "
                      f"clamping to {SINGLE_EPS_FLOOR:g}", stacklevel=2)
    return eps_eff.value, w.value, beta.value


def select_kernel_params(epsilon, grid, precision="double"):
    """kernel.py:106-118."""
    epsilon_eff, w, beta = tolerance_to_width(epsilon, precision)
    alpha = tuple(w * np.pi / n for n in grid.fine)
    return KernelParams(epsilon=epsilon_eff, w=w, beta=beta, alpha=alpha, precision=precision)


def eval_kernel(beta, z):
    """kernel.py:121-135: exp(beta (sqrt(1 - z^2) - 1)) on |z| <= 1, else 0."""
    z = np.asarray(z, dtype=np.float64)
    inside = np.abs(z) <= 1.0
    t = np.where(inside, 1.0 - z * z, 0.0)
    vals = np.where(inside, np.exp(beta * (np.sqrt(t) - 1.0)), 0.0)
    return float(vals) if vals.ndim == 0 else vals


def kernel_fourier(beta, xi):
    """kernel.py:149-173 (100-node Gauss-Legendre after z = sin theta)."""
    x = np.ascontiguousarray(np.asarray(xi, dtype=np.float64))
    flat = x.reshape(-1)
    out = np.empty_like(flat)
    rc = _lib.lib().nk_kernel_fourier(float(beta), flat.ctypes.data, flat.size, out.ctypes.data)
    _lib.check(rc)
    out = out.reshape(x.shape)
    return float(out) if out.ndim == 0 else out


def centered_freqs(n):
    """kernel.py:176-178."""
    return np.arange(n, dtype=np.int64) - n // 2


def build_correction_factors(grid, params):
    """kernel.py:181-205: (2/w)^d prod_i phi_hat(alpha_i k_i)^-1 over the
    centered mode grid, shaped (N_d, ..., N_1), in the plan's real dtype.
    Computed by the C library (nk_correction_factors, csrc/nk_host.cpp)."""
    d = grid.dim
    modes = (ctypes.c_int64 * d)(*[int(m) for m in grid.modes])
    alpha = (ctypes.c_double * d)(*[float(a) for a in params.alpha])
    out = np.empty(tuple(int(m) for m in grid.modes[::-1]), dtype=params.real_dtype)
    rc = _lib.lib().nk_correction_factors(float(params.beta), int(params.w), d, modes, alpha,
                                          _lib.PRECISIONS[params.precision], out.ctypes.data)
    _lib.check(rc)
    return out
