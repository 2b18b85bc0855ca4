"""One-shot transforms nufft2d1 / nufft2d2 / nufft3d1 / nufft3d2.

Not in the reference (north_star requires them): each is make_plan +
set_points + execute + destroy.  Precision follows the
strength / mode dtype (complex64 -> single, else double).  Coordinates are
1-D arrays x, y[, z] (paper set_pts form).  A leading
batch axis on the strengths (type 1: (K, M)) or modes (type 2: (K, N_d, ...,
N_1)) runs K transforms on one set of points (plan n_trans = K).
"""

from __future__ import annotations

import numpy as np
import torch

from .plan import TransformPlan

__all__ = ["nufft2d1", "nufft2d2", "nufft3d1", "nufft3d2"]


def _precision(a):
    if isinstance(a, torch.Tensor):
        return "single" if a.dtype in (torch.complex64, torch.float32) else "double"
    return "single" if np.asarray(a).dtype in (np.complex64, np.float32) else "double"


def _type1(coords, c, n_modes, eps, method, out, kwargs):
    n_modes = tuple(int(n) for n in n_modes)
    if len(n_modes) != len(coords):
        raise ValueError(f"n_modes must have {len(coords)} entries")
    shape = tuple(c.shape)
    if len(shape) not in (1, 2):
        raise ValueError(f"strengths must be (M,) or (K, M), got shape {shape}")
    kwargs.setdefault("n_trans", shape[0] if len(shape) == 2 else 1)
    with TransformPlan(1, n_modes, eps, method, _precision(c), **kwargs) as p:
        p.set_points(*coords)
        return p.execute(c, out)


def _type2(coords, f, eps, method, out, kwargs):
    d = len(coords)
    shape = tuple(f.shape)
    if len(shape) == d + 1:
        kwargs.setdefault("n_trans", shape[0])
        shape = shape[1:]
    elif len(shape) != d:
        raise ValueError(f"mode array must be {d}-D (N_d, ..., N_1), got shape {shape}")
    with TransformPlan(2, shape[::-1], eps, method, _precision(f), **kwargs) as p:
        p.set_points(*coords)
        return p.execute(f, out)


def nufft2d1(x, y, c, n_modes, eps=1e-6, method="default", out=None, **kwargs):
    """f[k2, k1] = sum_j c_j exp(-i (k1 x_j + k2 y_j)); n_modes = (N1, N2)."""
    return _type1((x, y), c, n_modes, eps, method, out, kwargs)


def nufft2d2(x, y, f, eps=1e-6, method="default", out=None, **kwargs):
    """c_j = sum_k f[k2, k1] exp(+i (k1 x_j + k2 y_j)); f shaped (N2, N1)."""
    return _type2((x, y), f, eps, method, out, kwargs)


def nufft3d1(x, y, z, c, n_modes, eps=1e-6, method="default", out=None, **kwargs):
    """f[k3, k2, k1] = sum_j c_j exp(-i k.x_j); n_modes = (N1, N2, N3)."""
    return _type1((x, y, z), c, n_modes, eps, method, out, kwargs)


def nufft3d2(x, y, z, f, eps=1e-6, method="default", out=None, **kwargs):
    """c_j = sum_k f[k3, k2, k1] exp(+i k.x_j); f shaped (N3, N2, N1)."""
    return _type2((x, y, z), f, eps, method, out, kwargs)
