"""Stage-level operators with the reference's names and signatures.

Each function mirrors one reference operator (binsort.py / spread.py /
SPEC.md interp & pipeline) and runs it on the GPU through the C-ABI with a
cached internal plan.  Host (numpy) inputs give numpy outputs; CUDA tensor
inputs give CUDA tensors.  These exist for drop-in compatibility and parity
testing; the fused hot path is TransformPlan.execute.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _arrays, _lib
from .plan import GridSpec, TransformPlan

__all__ = ["BinLayout", "SubproblemSet", "default_bin_dims", "bin_index", "bin_sort",
           "build_subproblems", "spread_gm", "spread_gm_sort", "spread_sm", "interpolate",
           "fft_fine", "deconvolve_type1", "deconvolve_type2", "exec_type1", "exec_type2"]

DEFAULT_BIN_DIMS_2D = (32, 32)       # binsort.py:34
DEFAULT_BIN_DIMS_3D = (16, 16, 2)    # binsort.py:35
DEFAULT_MAX_SUBPROBLEM = 1024        # binsort.py:38

_CACHE: "OrderedDict[tuple, TransformPlan]" = OrderedDict()
_CACHE_MAX = 8


def _plan(nufft_type, modes, fine, epsilon, precision, method, bin_dims=None, msub=None):
    dev = torch.cuda.current_device()
    key = (nufft_type, tuple(modes), tuple(fine), float(epsilon), precision, method,
           tuple(bin_dims) if bin_dims else None, msub, dev)
    p = _CACHE.get(key)
    if p is None:
        p = TransformPlan(nufft_type, modes, epsilon, method, precision, fine=fine,
                          bin_dims=bin_dims, max_subproblem=msub, device=dev)
        _CACHE[key] = p
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.popitem(last=False)[1].destroy()
    else:
        _CACHE.move_to_end(key)
    return p


def _out(kind, t):
    """Device tensor -> caller's kind (numpy for host callers)."""
    return t if kind == "cuda" else t.cpu().numpy()


def _kind(x):
    return "cuda" if (_arrays.is_torch(x) and x.is_cuda) else "host"


def _points(points, dim):
    if _arrays.is_torch(points):
        t = points if points.is_cuda else points.cuda()
        if t.dtype not in (torch.float32, torch.float64):
            t = t.double()
        return t.reshape(-1, dim).contiguous()
    a = np.asarray(points)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    return torch.from_numpy(np.ascontiguousarray(a).reshape(-1, dim)).cuda()


def default_bin_dims(dim):
    return DEFAULT_BIN_DIMS_2D if dim == 2 else DEFAULT_BIN_DIMS_3D


@dataclass(frozen=True)
class BinLayout:
    """binsort.py:45-65."""

    fine: tuple
    bin_dims: tuple
    bins_per_axis: tuple
    nbins: int
    point_bins: object   # (M,) int64
    counts: object       # (nbins,) int64
    starts: object       # (nbins + 1,) int64
    perm: object         # (M,) int64
    _points: object = field(default=None, repr=False, compare=False)

    @property
    def num_points(self):
        return int(self.perm.shape[0])


@dataclass(frozen=True)
class SubproblemSet:
    """binsort.py:68-88."""

    max_size: int
    halo: int
    bin_ids: object
    slice_starts: object
    slice_stops: object
    offsets: object
    padded_dims: object

    def __len__(self):
        return int(self.bin_ids.shape[0])


def _check_dims(layout_dims, grid):
    if layout_dims is None:
        layout_dims = default_bin_dims(grid.dim)
    layout_dims = tuple(int(m) for m in layout_dims)
    if len(layout_dims) != grid.dim or any(m < 1 for m in layout_dims):
        raise ValueError(f"invalid bin dims {layout_dims} for dim {grid.dim}")
    return layout_dims


def bin_sort(points, grid, layout_dims=None):
    """binsort.py:134-163 on the GPU (K1 fold/key/histogram, K2 scan, K3
    stable radix sort).  Bit-exact with the reference."""
    layout_dims = _check_dims(layout_dims, grid)
    kind = _kind(points)
    pts = _points(points, grid.dim)
    p = _plan(1, grid.modes, grid.fine, 0.5, "double", "gmsort", layout_dims)
    p.set_points(pts)
    keys, counts, starts, perm = (t.long() for t in p.layout_tensors())
    nb = tuple(-(-n // m) for n, m in zip(grid.fine, layout_dims))
    return BinLayout(tuple(grid.fine), layout_dims, nb, int(np.prod(nb)), _out(kind, keys),
                     _out(kind, counts), _out(kind, starts), _out(kind, perm), pts)


def bin_index(points, grid, layout_dims=None):
    """binsort.py:114-131: bin key of one point (d,) -> int, or of (M, d)."""
    single = np.ndim(points) == 1 if not _arrays.is_torch(points) else points.dim() == 1
    lay = bin_sort(points, grid, layout_dims)
    return int(lay.point_bins[0]) if single else lay.point_bins


def build_subproblems(layout, params, max_size=DEFAULT_MAX_SUBPROBLEM):
    """binsort.py:166-219 on the GPU (K4).  Bit-exact with the reference."""
    max_size = int(max_size)
    if max_size < 1:
        raise ValueError(f"max subproblem size must be >= 1, got {max_size}")
    if layout._points is None:
        raise ValueError("layout was not produced by this package's bin_sort")
    kind = _kind(layout.perm)
    d = len(layout.fine)
    modes = tuple(max(1, n // 2) for n in layout.fine)
    p = _plan(1, modes, layout.fine, params.epsilon, params.precision, "sm", layout.bin_dims,
              max_size)
    p.set_points(layout._points)
    t = [x.long() for x in p.subproblem_tensors()]
    return SubproblemSet(max_size, params.halo, *[_out(kind, x) for x in t])


# ------------------------------------------------------------------ spread

def _strengths(strengths, m, cdt):
    n = _arrays.numel(strengths)
    if n != m:
        raise ValueError(f"expected {m} strengths, got {n}")   # spread.py:137-138
    if _arrays.is_torch(strengths):
        t = strengths.to(device="cuda", dtype=_arrays.torch_dtype(cdt))
    else:
        t = torch.from_numpy(np.ascontiguousarray(strengths, dtype=cdt).reshape(-1)).cuda()
    return t.reshape(-1).contiguous()


def _spread(points, strengths, params, grid, method, bin_dims=None, msub=None):
    kind = _kind(points)
    pts = _points(points, grid.dim)
    cdt = params.complex_dtype
    c = _strengths(strengths, pts.shape[0], cdt)
    p = _plan(1, grid.modes, grid.fine, params.epsilon, params.precision, method, bin_dims, msub)
    p.set_points(pts)
    out = torch.empty(grid.fine_shape, dtype=_arrays.torch_dtype(cdt), device=pts.device)
    p._sync_stream("cuda")
    _lib.check(p._lib.nk_spread(p._h, c.data_ptr(), out.data_ptr()))
    return _out(kind, out)


def spread_gm(points, strengths, params, grid, workers=1):
    """spread.py:142-149: unsorted global-memory spreading (K6a)."""
    return _spread(points, strengths, params, grid, "gm")


def spread_gm_sort(points, layout, strengths, params, grid, workers=1):
    """spread.py:152-163: bin-sorted global-memory spreading (K6b)."""
    m = _arrays.numel(points) // grid.dim
    if layout.num_points != m or tuple(layout.fine) != tuple(grid.fine):
        raise ValueError("bin layout does not match the supplied points/grid")
    return _spread(points, strengths, params, grid, "gmsort", layout.bin_dims)


def spread_sm(points, layout, subproblems, strengths, params, grid, workers=1):
    """spread.py:166-182: shared-memory padded-bin spreading (K6c)."""
    m = _arrays.numel(points) // grid.dim
    if layout.num_points != m or tuple(layout.fine) != tuple(grid.fine):
        raise ValueError("bin layout does not match the supplied points/grid")
    sizes = subproblems.slice_stops - subproblems.slice_starts
    if int(sizes.sum()) != m:
        raise ValueError("subproblem slices do not partition the point set")
    return _spread(points, strengths, params, grid, "sm", layout.bin_dims,
                   subproblems.max_size)


# ------------------------------------------------------------------ interp

def interpolate(points, layout, fine_values, params, grid, method=None):
    """out[j] = kernel-weighted gather at point j (K7).
    ``layout`` None visits in input order (GM), else bin-sorted (GM-sort);
    ``method="sm"`` uses the shared-memory staged gather."""
    kind = _kind(points)
    pts = _points(points, grid.dim)
    M = pts.shape[0]
    if layout is not None and layout.num_points != M:
        raise ValueError("bin layout does not match the supplied points/grid")
    cdt = params.complex_dtype
    if _arrays.is_torch(fine_values):
        g = fine_values.to(device="cuda", dtype=_arrays.torch_dtype(cdt)).contiguous()
    else:
        g = torch.from_numpy(np.ascontiguousarray(fine_values, dtype=cdt)).cuda()
    if tuple(g.shape) != tuple(grid.fine_shape):
        raise ValueError(f"fine grid must have shape {grid.fine_shape}, got {tuple(g.shape)}")
    method = method or ("gm" if layout is None else "gmsort")
    bd = layout.bin_dims if layout is not None else None
    p = _plan(2, grid.modes, grid.fine, params.epsilon, params.precision, method, bd)
    p.set_points(pts)
    out = torch.empty(M, dtype=_arrays.torch_dtype(cdt), device=pts.device)
    p._sync_stream("cuda")
    _lib.check(p._lib.nk_interp(p._h, g.data_ptr(), out.data_ptr()))
    return _out(kind, out)


# ---------------------------------------------------------------- pipeline

def fft_fine(b, direction, grid=None, params=None):
    """SPEC.md:398-406 with cuFFT: forward e^{-}, inverse unnormalised e^{+}."""
    if direction not in ("forward", "inverse"):
        raise ValueError("direction must be 'forward' or 'inverse'")
    kind = _kind(b)
    t = b if _arrays.is_torch(b) else torch.from_numpy(np.ascontiguousarray(b))
    if t.dtype not in (torch.complex64, torch.complex128):
        t = t.to(torch.complex128)
    t = t.cuda().clone().contiguous()
    if t.dim() not in (2, 3):
        raise ValueError("fine grid must be 2-D or 3-D")
    prec = "single" if t.dtype == torch.complex64 else "double"
    fine = tuple(t.shape[::-1])
    modes = tuple(max(1, n // 2) for n in fine)
    p = _plan(1, modes, fine, 0.5, prec, "gm")
    p._sync_stream("cuda")
    _lib.check(p._lib.nk_fft(p._h, t.data_ptr(), -1 if direction == "forward" else 1))
    return _out(kind, t)


def deconvolve_type1(spectrum, grid, params):
    """SPEC.md:408-416 (+ the (-1)^{sum k} phase), K8."""
    kind = _kind(spectrum)
    cdt = params.complex_dtype
    s = spectrum if _arrays.is_torch(spectrum) else torch.from_numpy(
        np.ascontiguousarray(spectrum, dtype=cdt))
    s = s.to(device="cuda", dtype=_arrays.torch_dtype(cdt)).contiguous()
    p = _plan(1, grid.modes, grid.fine, params.epsilon, params.precision, "gm")
    out = torch.empty(grid.mode_shape, dtype=s.dtype, device=s.device)
    p._sync_stream("cuda")
    _lib.check(p._lib.nk_deconv_type1(p._h, s.data_ptr(), out.data_ptr()))
    return _out(kind, out)


def deconvolve_type2(modes, grid, params):
    """SPEC.md:418-425 (+ phase), K9: amplify and zero-pad onto the fine grid."""
    kind = _kind(modes)
    cdt = params.complex_dtype
    f = modes if _arrays.is_torch(modes) else torch.from_numpy(
        np.ascontiguousarray(modes, dtype=cdt))
    f = f.to(device="cuda", dtype=_arrays.torch_dtype(cdt)).contiguous()
    if f.numel() != int(np.prod(grid.modes)):
        raise ValueError("mode array size mismatch")
    p = _plan(2, grid.modes, grid.fine, params.epsilon, params.precision, "gm")
    out = torch.empty(grid.fine_shape, dtype=f.dtype, device=f.device)
    p._sync_stream("cuda")
    _lib.check(p._lib.nk_deconv_type2(p._h, f.data_ptr(), out.data_ptr()))
    return _out(kind, out)


def exec_type1(plan, strengths):
    """spread -> FFT -> deconvolve."""
    if plan.type != 1:
        raise ValueError("exec_type1 needs a type-1 plan")
    return plan.execute(strengths)


def exec_type2(plan, modes):
    """pad -> inverse FFT -> interpolate."""
    if plan.type != 2:
        raise ValueError("exec_type2 needs a type-2 plan")
    return plan.execute(modes)
