"""CPU oracle for the nufftkit hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``cpu_baseline`` / ``--impl reference``) may import this module, and
only as the checker / the timed reference port.  The product package
``paper_2102_08463_b200`` never imports it.

Parity pin: every function here is checked against golden vectors produced
by the *real* reference package (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/nufftkit`` from a temp copy) in
``tests/test_oracle_golden.py``.  The FFT boundary is pinned only by DFT
identities ("parity unpinned at the FFT boundary"), because the
reference ships no pipeline module.

Restated reference functions (file:line under /root/reference/pkg/src/nufftkit):
  tolerance_to_width       kernel.py:83-103
  select_kernel_params     kernel.py:106-118
  eval_kernel              kernel.py:121-135
  kernel_fourier           kernel.py:149-173
  centered_freqs           kernel.py:176-178
  build_correction_factors kernel.py:181-205
  next_smooth / GridSpec / make_plan sizing   SPEC.md:105-140 (module missing)
  bin_sort / build_subproblems                binsort.py:134-219 (C: nufft_oracle.c)
  spread_gm / spread_gm_sort / spread_sm      spread.py:142-182 (C)
  interpolate                                 SPEC.md:358-366 over _kernels.py:150-198 (C)
  fft_fine / deconvolve_type1/2 / exec_type1/2 SPEC.md:398-443 + (-1)^{sum k} phase
  direct_type1 / direct_type2 / rel_l2_error  SPEC.md:473-500 (C, compensated)
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import warnings
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

TWO_PI = 2.0 * np.pi
MIN_WIDTH, MAX_WIDTH = 2, 16          # kernel.py:27-28
SINGLE_EPS_FLOOR = 1e-6               # kernel.py:31
QUAD_NODES = 100                      # kernel.py:36
DEFAULT_BIN_DIMS_2D = (32, 32)        # binsort.py:34
DEFAULT_BIN_DIMS_3D = (16, 16, 2)     # binsort.py:35
DEFAULT_MAX_SUBPROBLEM = 1024         # binsort.py:38
SERIAL_CUTOFF = 20_000                # _parallel.py:19
PRIVATE_GRID_BUDGET = 1 << 30         # spread.py:26

_REAL = {"single": np.float32, "double": np.float64}
_COMPLEX = {"single": np.complex64, "double": np.complex128}


def build():
    """Compile the C restatement (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.or_remainder.restype = D
        L.or_remainder.argtypes = [D, D]
        L.or_grid_coords.argtypes = [I64, I, P, P, P]
        L.or_bin_keys.argtypes = [I64, I, P, P, P, P]
        L.or_bin_sort.argtypes = [I64, I, P, P, P, P, P, P, P]
        L.or_build_subproblems.restype = I64
        L.or_build_subproblems.argtypes = [I, P, P, I64, P, P, I64, I64, P, P, P, P, P]
        L.or_spread_gm.argtypes = [I64, I, P, P, P, P, I, D, I, I, P]
        L.or_spread_sm.argtypes = [I64, I, P, P, P, P, I, D, I, I64, P, P, P, P, I, P]
        L.or_interp.argtypes = [I64, I, P, P, P, P, I, D, I, I, P]
        L.or_deconv_type1.argtypes = [I, P, P, P, P, I, P]
        L.or_deconv_type2.argtypes = [I, P, P, P, P, I, P]
        L.or_direct_type1.argtypes = [I64, I, P, P, P, I, P]
        L.or_direct_type2.argtypes = [I64, I, P, P, P, I, P]
        L.or_direct_type1_at.argtypes = [I64, I, P, P, I64, P, I, P]
        L.or_max_threads.restype = I
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def host_threads() -> int:
    return int(lib().or_max_threads())


# ----------------------------------------------------------------- kernel.py

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
        return _REAL[self.precision]

    @property
    def complex_dtype(self):
        return _COMPLEX[self.precision]

    @property
    def halo(self) -> int:
        return (self.w + 1) // 2


def tolerance_to_width(epsilon, precision="double"):
    """kernel.py:83-103."""
    if precision not in _REAL:
        raise ValueError(f"precision must be 'single' or 'double', got {precision!r}")
    epsilon = float(epsilon)
    if not np.isfinite(epsilon) or not (0.0 < epsilon < 1.0):
        raise ValueError(f"tolerance must lie in (0, 1), got {epsilon}")
    if precision == "single" and epsilon < SINGLE_EPS_FLOOR:
        warnings.warn(f"tolerance {epsilon:g} is below single-precision rounding; "
                      f"clamping to {SINGLE_EPS_FLOOR:g}", stacklevel=2)
        epsilon = SINGLE_EPS_FLOOR
    w = int(np.ceil(np.log10(1.0 / epsilon))) + 1
    w = min(max(w, MIN_WIDTH), MAX_WIDTH)
    return epsilon, w, 2.30 * w


def select_kernel_params(epsilon, grid, precision="double"):
    """kernel.py:106-118."""
    epsilon, w, beta = tolerance_to_width(epsilon, precision)
    alpha = tuple(w * np.pi / n for n in grid.fine)
    return KernelParams(epsilon=epsilon, w=w, beta=beta, alpha=alpha, precision=precision)


def eval_kernel(beta, z):
    """kernel.py:121-135."""
    z = np.asarray(z, dtype=np.float64)
    inside = np.abs(z) <= 1.0
    t = np.where(inside, 1.0 - z * z, 0.0)
    vals = np.where(inside, np.exp(beta * (np.sqrt(t) - 1.0)), 0.0)
    return float(vals) if vals.ndim == 0 else vals


_THETA, _WQ = np.polynomial.legendre.leggauss(QUAD_NODES)   # kernel.py:138-146
_THETA = _THETA * (np.pi / 2)
_WQ = _WQ * (np.pi / 2)


def kernel_fourier(beta, xi):
    """kernel.py:149-173."""
    xi = np.asarray(xi, dtype=np.float64)
    envelope = _WQ * np.cos(_THETA) * np.exp(beta * (np.cos(_THETA) - 1.0))
    vals = np.cos(np.multiply.outer(xi, np.sin(_THETA))) @ envelope
    if not np.all(np.isfinite(vals)) or np.max(np.abs(vals), initial=0.0) < (
            np.finfo(np.float64).tiny * 8):
        raise ValueError("kernel Fourier transform underflowed below the precision floor")
    return float(vals) if vals.ndim == 0 else vals


def centered_freqs(n):
    """kernel.py:176-178."""
    return np.arange(n, dtype=np.int64) - n // 2


def axis_factors(grid, params):
    """Per-axis (2/w)/phi_hat(alpha_i k_i) in float64 (factors of
    kernel.py:201-204's tensor product)."""
    out = []
    for i in range(grid.dim):
        xi = params.alpha[i] * centered_freqs(grid.modes[i])
        ft = np.atleast_1d(kernel_fourier(params.beta, xi))
        out.append((2.0 / params.w) / ft)
    return out


def build_correction_factors(grid, params):
    """kernel.py:181-205."""
    d = grid.dim
    floor = np.finfo(params.real_dtype).tiny * 100
    axis_ft = []
    for i in range(d):
        xi = params.alpha[i] * centered_freqs(grid.modes[i])
        ft = np.atleast_1d(kernel_fourier(params.beta, xi))
        if np.any(ft <= floor):
            raise ValueError("kernel Fourier transform underflowed on axis "
                             f"{i + 1}; correction factors would overflow")
        axis_ft.append(ft)
    prod = axis_ft[-1]
    for ft in axis_ft[-2::-1]:
        prod = np.multiply.outer(prod, ft)
    values = (2.0 / params.w) ** d / prod
    return values.astype(params.real_dtype)


# ------------------------------------------------------------ plan (SPEC)

def _is_smooth(m):
    for p in (2, 3, 5):
        while m % p == 0:
            m //= p
    return m == 1


def next_smooth(n):
    """smallest 2^q 3^p 5^r >= n."""
    n = int(n)
    if n < 1:
        raise ValueError("n must be >= 1")
    while not _is_smooth(n):
        n += 1
    return n


@dataclass(frozen=True)
class GridSpec:
    """SPEC.md:105-111 (duck-typed by kernel.py:115,189,193 and binsort.py:122-129)."""
    modes: tuple
    fine: tuple

    @property
    def dim(self):
        return len(self.modes)

    @property
    def fine_shape(self):
        return tuple(self.fine[::-1])

    @property
    def mode_shape(self):
        return tuple(self.modes[::-1])


def make_grid(modes, epsilon, precision="double"):
    """n_i = next_smooth(max(2 N_i, 2w))."""
    _, w, _ = tolerance_to_width(epsilon, precision)
    fine = tuple(next_smooth(max(2 * int(N), 2 * w)) for N in modes)
    return GridSpec(tuple(int(N) for N in modes), fine)


# -------------------------------------------------------------- binsort.py

@dataclass
class BinLayout:
    fine: tuple
    bin_dims: tuple
    bins_per_axis: tuple
    nbins: int
    point_bins: np.ndarray
    counts: np.ndarray
    starts: np.ndarray
    perm: np.ndarray


@dataclass
class SubproblemSet:
    max_size: int
    halo: int
    bin_ids: np.ndarray
    slice_starts: np.ndarray
    slice_stops: np.ndarray
    offsets: np.ndarray
    padded_dims: np.ndarray

    def __len__(self):
        return self.bin_ids.size


def default_bin_dims(dim):
    return DEFAULT_BIN_DIMS_2D if dim == 2 else DEFAULT_BIN_DIMS_3D


def _pts64(points, dim):
    return np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, dim))


def grid_coords(points, fine):
    """binsort.py:91-100 (C restatement of np.remainder semantics)."""
    d = len(fine)
    pts = _pts64(points, d)
    out = np.empty_like(pts)
    lib().or_grid_coords(pts.shape[0], d, _p(pts), _p(np.asarray(fine, np.int64)), _p(out))
    return out


def bin_sort(points, grid, layout_dims=None):
    """binsort.py:134-163."""
    if layout_dims is None:
        layout_dims = default_bin_dims(grid.dim)
    layout_dims = tuple(int(m) for m in layout_dims)
    if len(layout_dims) != grid.dim or any(m < 1 for m in layout_dims):
        raise ValueError(f"invalid bin dims {layout_dims} for dim {grid.dim}")
    d = grid.dim
    pts = _pts64(points, d)
    M = pts.shape[0]
    nb = tuple(-(-n // m) for n, m in zip(grid.fine, layout_dims))
    nbins = int(np.prod(nb))
    keys = np.empty(M, np.int64)
    counts = np.empty(nbins, np.int64)
    starts = np.empty(nbins + 1, np.int64)
    perm = np.empty(M, np.int64)
    fine = np.asarray(grid.fine, np.int64)
    lib().or_bin_sort(M, d, _p(pts), _p(fine), _p(np.asarray(layout_dims, np.int64)),
                      _p(keys), _p(counts), _p(starts), _p(perm))
    return BinLayout(tuple(grid.fine), layout_dims, nb, nbins, keys, counts, starts, perm)


def build_subproblems(layout, params, max_size=DEFAULT_MAX_SUBPROBLEM):
    """binsort.py:166-219."""
    max_size = int(max_size)
    if max_size < 1:
        raise ValueError(f"max subproblem size must be >= 1, got {max_size}")
    d = len(layout.fine)
    fine = np.asarray(layout.fine, np.int64)
    bd = np.asarray(layout.bin_dims, np.int64)
    counts = np.ascontiguousarray(layout.counts, np.int64)
    starts = np.ascontiguousarray(layout.starts, np.int64)
    L = lib()
    S = L.or_build_subproblems(d, _p(fine), _p(bd), layout.nbins, _p(counts), _p(starts),
                               max_size, params.halo, None, None, None, None, None)
    bin_ids = np.empty(S, np.int64)
    ss = np.empty(S, np.int64)
    se = np.empty(S, np.int64)
    offs = np.empty((S, d), np.int64)
    pad = np.empty((S, d), np.int64)
    L.or_build_subproblems(d, _p(fine), _p(bd), layout.nbins, _p(counts), _p(starts),
                           max_size, params.halo, _p(bin_ids), _p(ss), _p(se), _p(offs),
                           _p(pad))
    return SubproblemSet(max_size, params.halo, bin_ids, ss, se, offs, pad)


# --------------------------------------------------------------- spread.py

def _prec(params):
    return 1 if params.precision == "double" else 0


def _strengths(strengths, m, dtype):
    c = np.ascontiguousarray(strengths, dtype=dtype).reshape(-1)
    if c.size != m:
        raise ValueError(f"expected {m} strengths, got {c.size}")
    return c


def effective_workers(workers, nbytes, npoints):
    """spread.py:60-64."""
    if npoints < SERIAL_CUTOFF:
        return 1
    fit = max(1, int(PRIVATE_GRID_BUDGET // max(nbytes, 1)))
    return max(1, min(workers, fit))


def spread_gm(points, strengths, params, grid, workers=1, perm=None):
    """spread.py:142-163 (perm=None: GM input order; else GM-sort order)."""
    d = grid.dim
    pts = _pts64(points, d)
    M = pts.shape[0]
    c = _strengths(strengths, M, params.complex_dtype)
    out = np.zeros(grid.fine_shape, dtype=params.complex_dtype)
    eff = effective_workers(workers, out.nbytes, M)
    pr = None if perm is None else np.ascontiguousarray(perm, np.int64)
    lib().or_spread_gm(M, d, _p(pts), _p(pr), _p(c), _p(np.asarray(grid.fine, np.int64)),
                       params.w, params.beta, _prec(params), eff, _p(out))
    return out


def spread_gm_sort(points, layout, strengths, params, grid, workers=1):
    return spread_gm(points, strengths, params, grid, workers, perm=layout.perm)


def spread_sm(points, layout, subproblems, strengths, params, grid, workers=1):
    """spread.py:166-182."""
    d = grid.dim
    pts = _pts64(points, d)
    M = pts.shape[0]
    c = _strengths(strengths, M, params.complex_dtype)
    out = np.zeros(grid.fine_shape, dtype=params.complex_dtype)
    subs = subproblems
    eff = 1 if M < SERIAL_CUTOFF else max(1, workers)
    i64 = lambda a: np.ascontiguousarray(a, np.int64)
    lib().or_spread_sm(M, d, _p(pts), _p(i64(layout.perm)), _p(c),
                       _p(np.asarray(grid.fine, np.int64)), params.w, params.beta,
                       _prec(params), len(subs), _p(i64(subs.slice_starts)),
                       _p(i64(subs.slice_stops)), _p(i64(subs.offsets)),
                       _p(i64(subs.padded_dims)), eff, _p(out))
    return out


def interpolate(points, grid_values, params, grid, layout=None, workers=1):
    """SPEC.md:358-366 over _kernels.py:150-198; slot j gets point j."""
    d = grid.dim
    pts = _pts64(points, d)
    M = pts.shape[0]
    g = np.ascontiguousarray(grid_values, dtype=params.complex_dtype)
    out = np.empty(M, dtype=params.complex_dtype)
    pr = None if layout is None else np.ascontiguousarray(layout.perm, np.int64)
    lib().or_interp(M, d, _p(pts), _p(pr), _p(g), _p(np.asarray(grid.fine, np.int64)),
                    params.w, params.beta, _prec(params), max(1, workers), _p(out))
    return out


# --------------------------------------------------------- pipeline (SPEC)

def fft_fine(b, direction, workers=1):
    """forward e^{-}, inverse unnormalized e^{+}."""
    import scipy.fft as sfft
    axes = tuple(range(b.ndim))
    if direction == "forward":
        return sfft.fftn(b, axes=axes, workers=workers)
    return sfft.ifftn(b, axes=axes, norm="forward", workers=workers)


def _corr_flat(grid, params):
    return np.ascontiguousarray(np.concatenate(axis_factors(grid, params)), np.float64)


def deconvolve_type1(spec, grid, params, corr=None):
    """SPEC.md:408-416 with the (-1)^{sum k} phase."""
    corr = _corr_flat(grid, params) if corr is None else corr
    spec = np.ascontiguousarray(spec, dtype=params.complex_dtype)
    out = np.empty(grid.mode_shape, dtype=params.complex_dtype)
    lib().or_deconv_type1(grid.dim, _p(np.asarray(grid.modes, np.int64)),
                          _p(np.asarray(grid.fine, np.int64)), _p(corr), _p(spec),
                          _prec(params), _p(out))
    return out


def deconvolve_type2(modes, grid, params, corr=None):
    """SPEC.md:418-425 with the (-1)^{sum k} phase."""
    corr = _corr_flat(grid, params) if corr is None else corr
    f = np.ascontiguousarray(modes, dtype=params.complex_dtype).reshape(grid.mode_shape)
    out = np.empty(grid.fine_shape, dtype=params.complex_dtype)
    lib().or_deconv_type2(grid.dim, _p(np.asarray(grid.modes, np.int64)),
                          _p(np.asarray(grid.fine, np.int64)), _p(corr), _p(f),
                          _prec(params), _p(out))
    return out


class OraclePlan:
    """Composed CPU pipeline (plan/setpts/execute) -- the reference restated."""

    def __init__(self, nufft_type, modes, epsilon, method=None, precision="double",
                 workers=1, bin_dims=None, max_subproblem=DEFAULT_MAX_SUBPROBLEM):
        self.type = int(nufft_type)
        self.grid = make_grid(modes, epsilon, precision)
        self.params = select_kernel_params(epsilon, self.grid, precision)
        self.method = method or ("sm" if self.type == 1 else "gmsort")
        self.workers = workers
        self.bin_dims = bin_dims or default_bin_dims(self.grid.dim)
        self.max_subproblem = max_subproblem
        self.corr = _corr_flat(self.grid, self.params)
        self.points = None

    def set_points(self, points):
        self.points = _pts64(points, self.grid.dim)
        self.layout = bin_sort(self.points, self.grid, self.bin_dims)
        self.subs = build_subproblems(self.layout, self.params, self.max_subproblem)

    def spread(self, c):
        if self.method == "gm":
            return spread_gm(self.points, c, self.params, self.grid, self.workers)
        if self.method == "gmsort":
            return spread_gm_sort(self.points, self.layout, c, self.params, self.grid,
                                  self.workers)
        return spread_sm(self.points, self.layout, self.subs, c, self.params, self.grid,
                         self.workers)

    def execute(self, inp):
        g, p = self.grid, self.params
        if self.type == 1:
            b = self.spread(inp)
            bh = fft_fine(b, "forward", self.workers).astype(p.complex_dtype, copy=False)
            return deconvolve_type1(bh, g, p, self.corr).reshape(-1)
        bh = deconvolve_type2(inp, g, p, self.corr)
        b = fft_fine(bh, "inverse", self.workers).astype(p.complex_dtype, copy=False)
        lay = None if self.method == "gm" else self.layout
        return interpolate(self.points, b, p, g, lay, self.workers)


# ------------------------------------------------------------ oracle (SPEC)

def direct_type1(points, strengths, modes, workers=0):
    """f_k = sum_j c_j e^{-i k.x_j}, compensated."""
    d = len(modes)
    pts = _pts64(points, d)
    c = np.ascontiguousarray(strengths, np.complex128).reshape(-1)
    out = np.empty(tuple(modes[::-1]), np.complex128)
    lib().or_direct_type1(pts.shape[0], d, _p(pts), _p(c),
                          _p(np.asarray(modes, np.int64)), workers or host_threads(),
                          _p(out))
    return out.reshape(-1)


def direct_type1_at(points, strengths, kvecs, workers=0):
    """SPEC.md:473-481 at the integer wave vectors ``kvecs`` (n, d), axis 1
    first: f_k = sum_j c_j e^{-i k.x_j}, compensated."""
    kv = np.ascontiguousarray(kvecs, np.int64)
    d = kv.shape[1]
    pts = _pts64(points, d)
    c = np.ascontiguousarray(strengths, np.complex128).reshape(-1)
    out = np.empty(kv.shape[0], np.complex128)
    lib().or_direct_type1_at(pts.shape[0], d, _p(pts), _p(c), kv.shape[0], _p(kv),
                             workers or host_threads(), _p(out))
    return out


def direct_type2(points, fmodes, modes, workers=0):
    """c_j = sum_k f_k e^{+i k.x_j}, compensated."""
    d = len(modes)
    pts = _pts64(points, d)
    f = np.ascontiguousarray(fmodes, np.complex128).reshape(-1)
    out = np.empty(pts.shape[0], np.complex128)
    lib().or_direct_type2(pts.shape[0], d, _p(pts), _p(f),
                          _p(np.asarray(modes, np.int64)), workers or host_threads(),
                          _p(out))
    return out


def rel_l2_error(approx, exact):
    """SPEC.md:492-500."""
    a = np.asarray(approx).reshape(-1).astype(np.complex128)
    e = np.asarray(exact).reshape(-1).astype(np.complex128)
    if a.shape != e.shape:
        raise ValueError("length mismatch")
    den = np.linalg.norm(e)
    if den == 0:
        raise ValueError("exact vector is all zero")
    return float(np.linalg.norm(a - e) / den)


def gen_points(dist, M, grid, seed, dtype=np.float64):
    """SPEC.md:531-539 (rand / cluster) plus 'gauss' (builder's C3b choice,
    x_i ~ N(0, (pi/8)^2) folded into [-pi, pi))."""
    rng = np.random.default_rng(seed)
    d = grid.dim
    if dist == "rand":
        x = rng.uniform(-np.pi, np.pi, (M, d))
    elif dist == "cluster":
        h = np.array([TWO_PI / n for n in grid.fine])
        x = rng.uniform(0.0, 1.0, (M, d)) * (8 * h)
    elif dist == "gauss":
        x = np.remainder(rng.normal(0.0, np.pi / 8, (M, d)) + np.pi, TWO_PI) - np.pi
    else:
        raise ValueError(dist)
    return x.astype(dtype)


def gen_strengths(M, seed, dtype=np.complex128):
    rng = np.random.default_rng(seed + 1000003)
    return (rng.uniform(0, 1, M) + 1j * rng.uniform(0, 1, M)).astype(dtype)
