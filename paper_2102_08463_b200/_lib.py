"""ctypes binding of libnufft_b200.so (C-ABI: include/nufft_b200.h).

The CUDA library is the product; this module only loads it and maps its
error codes onto the reference's Python exceptions (ValueError for invalid
arguments, kernel.py:77,92-93; binsort.py:144,175; spread.py:138,156).
There is no CPU fallback: if the library is missing the import fails.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnufft_b200.so")

NK_OK, NK_ERR_VALUE, NK_ERR_NONFINITE, NK_ERR_STATE, NK_ERR_MEMORY, NK_ERR_CUDA = range(6)
NK_SINGLE, NK_DOUBLE = 0, 1
NK_METHOD_DEFAULT, NK_GM, NK_GMSORT, NK_SM = -1, 0, 1, 2

METHODS = {"default": NK_METHOD_DEFAULT, None: NK_METHOD_DEFAULT, "gm": NK_GM,
           "gmsort": NK_GMSORT, "sm": NK_SM}
METHOD_NAMES = {NK_GM: "gm", NK_GMSORT: "gmsort", NK_SM: "sm"}
PRECISIONS = {"single": NK_SINGLE, "double": NK_DOUBLE}


class NkOpts(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int), ("bin_dims", ctypes.c_int * 3),
                ("max_subproblem", ctypes.c_int), ("fine", ctypes.c_int64 * 3),
                ("device", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("timing", ctypes.c_int), ("n_trans", ctypes.c_int),
                ("deterministic", ctypes.c_int)]


class NkPlanInfo(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("dim", ctypes.c_int), ("precision", ctypes.c_int),
                ("method", ctypes.c_int), ("modes", ctypes.c_int64 * 3),
                ("fine", ctypes.c_int64 * 3), ("epsilon", ctypes.c_double),
                ("w", ctypes.c_int), ("beta", ctypes.c_double),
                ("alpha", ctypes.c_double * 3), ("eps_clamped", ctypes.c_int),
                ("bin_dims", ctypes.c_int * 3), ("bins_per_axis", ctypes.c_int64 * 3),
                ("nbins", ctypes.c_int64), ("max_subproblem", ctypes.c_int),
                ("halo", ctypes.c_int), ("num_points", ctypes.c_int64),
                ("num_subproblems", ctypes.c_int64), ("n_trans", ctypes.c_int)]


class NufftError(RuntimeError):
    """CUDA / cuFFT runtime failure inside libnufft_b200."""


class NonFiniteCoordinateError(ValueError):
    """set_points saw a NaN/Inf coordinate."""

    def __init__(self, msg, index):
        super().__init__(msg)
        self.index = index


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "nk_tolerance_to_width": (I, [D, I, ctypes.POINTER(D), ctypes.POINTER(I),
                                      ctypes.POINTER(D), ctypes.POINTER(I)]),
        "nk_next_smooth": (I64, [I64]),
        "nk_kernel_fourier": (I, [D, P, I64, P]),
        "nk_correction_factors": (I, [D, I, I, P, P, I, P]),
        "nk_default_opts": (None, [ctypes.POINTER(NkOpts)]),
        "nk_plan_create": (I, [I, I, P, D, I, ctypes.POINTER(NkOpts), PP]),
        "nk_plan_get_info": (I, [P, ctypes.POINTER(NkPlanInfo)]),
        "nk_set_stream": (I, [P, P]),
        "nk_setpts": (I, [P, I64, I, P, P, P, I64]),
        "nk_execute": (I, [P, P, P]),
        "nk_destroy": (I, [P]),
        "nk_last_error": (ctypes.c_char_p, []),
        "nk_error_index": (I64, []),
        "nk_get_layout": (I, [P, P, P, P, P]),
        "nk_get_subproblems": (I, [P, P, P, P, P, P]),
        "nk_spread": (I, [P, P, P]),
        "nk_interp": (I, [P, P, P]),
        "nk_fft": (I, [P, P, I]),
        "nk_deconv_type1": (I, [P, P, P]),
        "nk_deconv_type2": (I, [P, P, P]),
        "nk_fft_deconv_type1": (I, [P, P, P]),
        "nk_stage_times": (I, [P, ctypes.POINTER(ctypes.c_float), I]),
        "nk_last_launch_count": (I, [P]),
        "nk_set_timing": (I, [P, I]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ["nk_tolerance_to_width", "nk_next_smooth", "nk_kernel_fourier",
            "nk_correction_factors", "nk_default_opts",
            "nk_plan_create", "nk_plan_get_info", "nk_set_stream", "nk_setpts", "nk_execute",
            "nk_destroy", "nk_last_error", "nk_error_index", "nk_get_layout",
            "nk_get_subproblems", "nk_spread", "nk_interp", "nk_fft", "nk_deconv_type1",
            "nk_deconv_type2", "nk_fft_deconv_type1", "nk_stage_times", "nk_last_launch_count",
            "nk_set_timing"]


def check(rc):
    if rc == NK_OK:
        return
    L = lib()
    msg = L.nk_last_error().decode(errors="replace")
    if rc == NK_ERR_NONFINITE:
        raise NonFiniteCoordinateError(msg, int(L.nk_error_index()))
    if rc in (NK_ERR_VALUE, NK_ERR_STATE):
        raise ValueError(msg)
    if rc == NK_ERR_MEMORY:
        raise MemoryError(msg)
    raise NufftError(msg)
