"""Plan lifecycle: make_plan / set_points / execute / destroy.

The reference package ships no plan module; its contract is SPEC.md:100-182
(plan), and the paper's GPU Python API is ``cufinufft(type, shape, eps,
gpu_device_id)`` / ``set_pts(X, Y, Z)`` / ``execute(c, fk)``
(PAPER.md:1603-1625).  Both are offered here over the C-ABI
(include/nufft_b200.h).

Buffers: numpy arrays (host) or torch CUDA tensors (device).  With CUDA
tensors the work is enqueued on torch's current stream and the output is a
CUDA tensor; with numpy arrays the C library stages through device memory,
synchronises and returns numpy.  There is no CPU compute path.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _arrays, _lib
from .kernel import KernelParams, SINGLE_EPS_FLOOR

__all__ = ["GridSpec", "next_smooth", "TransformPlan", "make_plan", "set_points", "execute",
           "destroy", "Plan"]

_COMPLEX = {"single": np.complex64, "double": np.complex128}
_REAL = {"single": np.float32, "double": np.float64}


def next_smooth(n):
    """smallest 2^q 3^p 5^r >= n."""
    n = int(n)
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    r = int(_lib.lib().nk_next_smooth(n))
    if r < 0:
        raise OverflowError("next_smooth overflowed")
    return r


@dataclass(frozen=True)
class GridSpec:
    """SPEC.md:105-111 (duck-typed by kernel.py:115,189,193, binsort.py:122-129)."""

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

    @property
    def spacing(self):
        return tuple(2 * np.pi / n for n in self.fine)

    sigma = 2.0


def _device_index(device):
    if device is None:
        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    if isinstance(device, torch.device):
        return device.index if device.index is not None else torch.cuda.current_device()
    if isinstance(device, str):
        d = torch.device(device)
        return d.index if d.index is not None else torch.cuda.current_device()
    return int(device)


class TransformPlan:
    """SPEC.md:113-119 TransformPlan over a libnufft_b200 handle.

    Args:
        nufft_type: 1 (nonuniform -> uniform) or 2 (uniform -> nonuniform).
        modes: (N_1, N_2[, N_3]) mode counts, axis 1 first.
        epsilon: tolerance in (0, 1).
        method: "gm", "gmsort", "sm" or "default".  "default" is SM for both
            types: type 1 as SPEC.md:170; for type 2 SPEC.md:170 names
            GM-sort, and this library deviates on purpose -- "sm" there is the
            shared-memory staged gather (same per-point arithmetic, measured
            1.4-2.5x faster than GM-sort on B200).
        precision: "single" or "double".
        workers: accepted for API compatibility with the CPU reference
            (SPEC.md:176); the GPU grid replaces the worker pool.
        bin_dims, max_subproblem: bin edge lengths (axis 1 first) and M_sub.
            Unset: GM-sort plans keep the reference defaults (binsort.py:34-38);
            SM plans use B200-tuned shapes (include/nufft_b200.h nk_opts).
        fine: explicit fine-grid sizes (default: the SPEC sizing rule).
        device: CUDA device (default: current).
        timing: record per-stage CUDA events (see stage_times()).
        n_trans: vectors per execute (cufinufft ``n_trans``; an extension --
            the reference has no batching).  Inputs and
            outputs then carry a leading axis of length n_trans; the sort and
            subproblems of one set_points serve every vector.
        deterministic: type-1 SM plans merge their subproblems in colour
            classes of non-overlapping bins (one launch each), so repeated
            executes are bit-identical.  Type 2 is always
            deterministic; GM / GM-sort type 1 is not.
    """

    def __init__(self, nufft_type, modes, epsilon, method="default", precision="double",
                 workers=0, *, bin_dims=None, max_subproblem=None, fine=None, device=None,
                 timing=False, n_trans=1, deterministic=False):
        if int(workers) < 0:
            raise ValueError(f"worker count must be >= 0, got {workers}")
        if precision not in _COMPLEX:
            raise ValueError(f"precision must be 'single' or 'double', got {precision!r}")
        if method not in _lib.METHODS:
            raise ValueError(f"method must be one of gm, gmsort, sm, got {method!r}")
        modes = tuple(int(m) for m in np.atleast_1d(modes))
        if len(modes) not in (2, 3):
            raise ValueError(f"dimension must be 2 or 3, got {len(modes)}")
        if any(m < 1 for m in modes):
            raise ValueError(f"mode counts must be >= 1, got {modes}")
        d = len(modes)
        self._lib = _lib.lib()
        self.device = _device_index(device)
        opts = _lib.NkOpts()
        self._lib.nk_default_opts(ctypes.byref(opts))
        opts.method = _lib.METHODS[method]
        opts.device = self.device
        opts.timing = 1 if timing else 0
        if int(n_trans) < 1:
            raise ValueError(f"n_trans must be >= 1, got {n_trans}")
        opts.n_trans = int(n_trans)
        opts.deterministic = 1 if deterministic else 0
        if bin_dims is not None:
            bin_dims = tuple(int(m) for m in bin_dims)
            if len(bin_dims) != d or any(m < 1 for m in bin_dims):
                raise ValueError(f"invalid bin dims {bin_dims} for dim {d}")
            for i, m in enumerate(bin_dims):
                opts.bin_dims[i] = m
        if max_subproblem is not None:
            if int(max_subproblem) < 1:
                raise ValueError(f"max subproblem size must be >= 1, got {max_subproblem}")
            opts.max_subproblem = int(max_subproblem)
        if fine is not None:
            for i, n in enumerate(fine):
                opts.fine[i] = int(n)
        with torch.cuda.device(self.device):
            opts.stream = _arrays.current_stream_ptr(self.device)
        self._stream = opts.stream
        N = (ctypes.c_int64 * 3)(*(list(modes) + [1] * (3 - d)))
        h = ctypes.c_void_p()
        _lib.check(self._lib.nk_plan_create(int(nufft_type), d, N, float(epsilon),
                                            _lib.PRECISIONS[precision], ctypes.byref(opts),
                                            ctypes.byref(h)))
        self._h = h
        info = self.info()
        if info.eps_clamped:   # kernel.py:94-100
            warnings.warn(f"tolerance {float(epsilon):g} is below single-precision rounding; "
                          f"clamping to {SINGLE_EPS_FLOOR:g}", stacklevel=2)
        self.type = int(nufft_type)
        self.precision = precision
        self.method = _lib.METHOD_NAMES[info.method]
        self.grid = GridSpec(modes, tuple(int(info.fine[i]) for i in range(d)))
        self.params = KernelParams(epsilon=info.epsilon, w=info.w, beta=info.beta,
                                   alpha=tuple(info.alpha[i] for i in range(d)),
                                   precision=precision)
        self.bin_dims = tuple(int(info.bin_dims[i]) for i in range(d))
        self.max_subproblem = int(info.max_subproblem)
        self.n_trans = int(info.n_trans)
        self.num_points = None
        self._points_kind = None

    # -- lifecycle ---------------------------------------------------------
    def info(self):
        self._check_alive()
        inf = _lib.NkPlanInfo()
        _lib.check(self._lib.nk_plan_get_info(self._h, ctypes.byref(inf)))
        return inf

    def _check_alive(self):
        if getattr(self, "_h", None) is None or not self._h:
            raise ValueError("plan has been destroyed")

    def _sync_stream(self, kind):
        if kind == "cuda":
            s = _arrays.current_stream_ptr(self.device)
            if s != self._stream:
                _lib.check(self._lib.nk_set_stream(self._h, s))
                self._stream = s

    def set_points(self, coords, y=None, z=None):
        """SPEC.md:142-150.  ``coords`` is an (M, d) array (reference form), or
        pass x, y[, z] as separate 1-D arrays (paper set_pts(X, Y, Z) form).
        Any finite coordinates are folded into [-pi, pi); a non-finite one
        raises ValueError naming its index."""
        self._check_alive()
        d = self.grid.dim
        if y is not None:
            axes = [coords, y] + ([z] if d == 3 else [])
            if len(axes) != d or (d == 2 and z is not None):
                raise ValueError(f"expected {d} coordinate arrays")
            bufs = []
            kinds = set()
            M = None
            for a in axes:
                dt = np.float32 if _dtype_of(a) == np.float32 else np.float64
                arr, ptr, kind = _arrays.as_buffer(a, dt, self.device)
                n = _arrays.numel(arr)
                if M is None:
                    M = n
                elif n != M:
                    raise ValueError("coordinate arrays differ in length")
                bufs.append((arr, ptr, dt))
                kinds.add(kind)
            if len({b[2] for b in bufs}) != 1:
                bufs = [_arrays.as_buffer(b[0], np.float64, self.device)[:2] + (np.float64,)
                        for b in bufs]
            dt = bufs[0][2]
            ptrs = [b[1] for b in bufs] + [None] * (3 - d)
            stride = 1
            kind = "cuda" if kinds == {"cuda"} else "host"
            keep = bufs
        else:
            dt = np.float32 if _dtype_of(coords) == np.float32 else np.float64
            arr, ptr, kind = _arrays.as_buffer(coords, dt, self.device)
            shape = tuple(arr.shape)
            if len(shape) == 1 and shape[0] % d == 0:
                M = shape[0] // d
            elif len(shape) == 2 and shape[1] == d:
                M = shape[0]
            elif len(shape) == 2 and shape[0] == 0:
                M = 0
            else:
                raise ValueError(f"points must have shape (M, {d}), got {shape}")
            es = np.dtype(dt).itemsize
            ptrs = [ptr + i * es for i in range(d)] + [None] * (3 - d)
            stride = d
            keep = arr
        self._sync_stream(kind)
        prec = _lib.NK_DOUBLE if dt == np.float64 else _lib.NK_SINGLE
        _lib.check(self._lib.nk_setpts(self._h, int(M), prec, ptrs[0], ptrs[1], ptrs[2],
                                       stride))
        del keep
        self.num_points = int(M)
        self._points_kind = kind
        return self

    setpts = set_points   # cufinufft spelling

    def _batch(self, shape):
        return shape if self.n_trans == 1 else (self.n_trans,) + tuple(shape)

    def _io_sizes(self):
        K = self.n_trans
        Ntot = int(np.prod(self.grid.modes))
        if self.type == 1:
            return (K * self.num_points, K * Ntot, self._batch((self.num_points,)),
                    self._batch(self.grid.mode_shape))
        return (K * Ntot, K * self.num_points, self._batch(self.grid.mode_shape),
                self._batch((self.num_points,)))

    def execute(self, inp, out=None):
        """type 1 maps M strengths to prod(N) modes shaped
        (N_d, ..., N_1); type 2 the reverse.  Returns ``out``."""
        self._check_alive()
        if self.num_points is None:
            raise ValueError("execute called before set_points")
        n_in, n_out, _, out_shape = self._io_sizes()
        cdt = _COMPLEX[self.precision]
        if _arrays.numel(inp) != n_in:
            what = "strengths" if self.type == 1 else "mode coefficients"
            raise ValueError(f"expected {n_in} {what}, got {_arrays.numel(inp)}")
        arr, ptr_in, kind = _arrays.as_buffer(inp, cdt, self.device)
        if out is None:
            out, ptr_out = _arrays.empty_like_kind(kind, out_shape, cdt, self.device)
        else:
            if _arrays.numel(out) != n_out:
                raise ValueError(f"output must hold {n_out} values, got {_arrays.numel(out)}")
            if _arrays.is_torch(out):
                if not out.is_cuda or out.dtype != _arrays.torch_dtype(cdt) or \
                        not out.is_contiguous():
                    raise ValueError("output tensor must be a contiguous CUDA tensor of "
                                     f"dtype {np.dtype(cdt).name}")
                ptr_out = out.data_ptr()
            else:
                if not isinstance(out, np.ndarray) or out.dtype != cdt or \
                        not out.flags.c_contiguous:
                    raise ValueError(f"output array must be C-contiguous {np.dtype(cdt).name}")
                ptr_out = out.ctypes.data
        self._sync_stream(kind)
        _lib.check(self._lib.nk_execute(self._h, ptr_in, ptr_out))
        del arr
        return out

    def destroy(self):
        h = getattr(self, "_h", None)
        if h is not None and h:
            self._lib.nk_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()

    # -- introspection / parity hooks ------------------------------------
    def stage_times(self):
        """Device ms of the last execute: dict(spread|interp, fft, deconv|pad, total)."""
        ms = (ctypes.c_float * 4)()
        _lib.check(self._lib.nk_stage_times(self._h, ms, 4))
        k0 = "spread" if self.type == 1 else "interp"
        k2 = "deconv" if self.type == 1 else "pad"
        return {k0: ms[0], "fft": ms[1], k2: ms[2], "total": ms[3]}

    def set_timing(self, on):
        """Per-stage CUDA-event timing (disables CUDA-graph replay while on)."""
        _lib.check(self._lib.nk_set_timing(self._h, 1 if on else 0))

    def last_launch_count(self):
        return int(self._lib.nk_last_launch_count(self._h))

    # -- device stage ops (CUDA tensors, torch current stream) ----------------
    # The pieces of execute() for callers that insert a collective between
    # them (dist.py: type-1 grid reduce, type-2 mode broadcast).
    def _dev(self, t, shape, what):
        import torch as _t
        cdt = _arrays.torch_dtype(_COMPLEX[self.precision])
        if not (_arrays.is_torch(t) and t.is_cuda and t.dtype == cdt and t.is_contiguous()):
            raise ValueError(f"{what} must be a contiguous CUDA {cdt} tensor")
        if shape is not None and t.numel() != int(np.prod(shape)):
            raise ValueError(f"{what} must have {int(np.prod(shape))} elements")
        return t

    def new_fine_grid(self):
        return torch.empty(self._batch(self.grid.fine_shape),
                           dtype=_arrays.torch_dtype(_COMPLEX[self.precision]),
                           device=torch.device("cuda", self.device))

    def spread_to(self, strengths, fine):
        """Step 1 of type 1: fine <- spread(strengths) (zeroed first)."""
        self._check_points()
        self._dev(strengths, self._batch((self.num_points,)), "strengths")
        self._dev(fine, self._batch(self.grid.fine_shape), "fine grid")
        self._sync_stream("cuda")
        _lib.check(self._lib.nk_spread(self._h, strengths.data_ptr(), fine.data_ptr()))
        return fine

    def fft_(self, fine, direction):
        """cuFFT in place: direction -1 forward, +1 inverse (unnormalised)."""
        self._dev(fine, self._batch(self.grid.fine_shape), "fine grid")
        self._sync_stream("cuda")
        _lib.check(self._lib.nk_fft(self._h, fine.data_ptr(), int(direction)))
        return fine

    def deconvolve_to(self, fine_spectrum, modes):
        """Step 3 of type 1: modes <- p_k (-1)^{sum k} bhat[k mod n]."""
        self._dev(fine_spectrum, self._batch(self.grid.fine_shape), "fine spectrum")
        self._dev(modes, self._batch(self.grid.mode_shape), "modes")
        self._sync_stream("cuda")
        _lib.check(self._lib.nk_deconv_type1(self._h, fine_spectrum.data_ptr(), modes.data_ptr()))
        return modes

    def fft_deconvolve_to(self, fine, modes):
        """Steps 2-3 of type 1 in one call: forward FFT of ``fine`` (in
        place) and the deconvolution / mode selection into ``modes`` (the
        fused row-FFT path where the plan has one)."""
        self._dev(fine, self._batch(self.grid.fine_shape), "fine grid")
        self._dev(modes, self._batch(self.grid.mode_shape), "modes")
        self._sync_stream("cuda")
        _lib.check(self._lib.nk_fft_deconv_type1(self._h, fine.data_ptr(), modes.data_ptr()))
        return modes

    def pad_to(self, modes, fine):
        """Step 1 of type 2: fine <- zero-padded p_k (-1)^{sum k} f_k."""
        self._dev(modes, self._batch(self.grid.mode_shape), "modes")
        self._dev(fine, self._batch(self.grid.fine_shape), "fine grid")
        self._sync_stream("cuda")
        _lib.check(self._lib.nk_deconv_type2(self._h, modes.data_ptr(), fine.data_ptr()))
        return fine

    def interp_to(self, fine, out):
        """Step 3 of type 2: out[j] <- gather at point j."""
        self._check_points()
        self._dev(fine, self._batch(self.grid.fine_shape), "fine grid")
        self._dev(out, self._batch((self.num_points,)), "output")
        self._sync_stream("cuda")
        _lib.check(self._lib.nk_interp(self._h, fine.data_ptr(), out.data_ptr()))
        return out

    def _check_points(self):
        self._check_alive()
        if self.num_points is None:
            raise ValueError("set_points has not been called")

    def layout_tensors(self):
        """Bin layout of the last set_points as int32 CUDA tensors:
        (point_bins, counts, starts, perm) -- binsort.py:45-65 fields."""
        inf = self.info()
        M, nb = self.num_points or 0, int(inf.nbins)
        dev = torch.device("cuda", self.device)
        t = [torch.empty(M, dtype=torch.int32, device=dev),
             torch.empty(nb, dtype=torch.int32, device=dev),
             torch.empty(nb + 1, dtype=torch.int32, device=dev),
             torch.empty(M, dtype=torch.int32, device=dev)]
        _lib.check(self._lib.nk_get_layout(self._h, *[x.data_ptr() for x in t]))
        return t

    def subproblem_tensors(self):
        """Subproblem table (binsort.py:68-88 fields) as int32 CUDA tensors:
        (bin_ids, slice_starts, slice_stops, offsets (S,d), padded_dims (S,d))."""
        inf = self.info()
        S, d = int(inf.num_subproblems), self.grid.dim
        dev = torch.device("cuda", self.device)
        t = [torch.empty(S, dtype=torch.int32, device=dev) for _ in range(3)] + \
            [torch.empty((S, d), dtype=torch.int32, device=dev) for _ in range(2)]
        if S:
            _lib.check(self._lib.nk_get_subproblems(self._h, *[x.data_ptr() for x in t]))
        return t


def _dtype_of(x):
    if _arrays.is_torch(x):
        return np.float32 if x.dtype == torch.float32 else np.float64
    return np.asarray(x).dtype.type


def make_plan(nufft_type, N, epsilon, method="default", precision="double", workers=0,
              **kwargs):
    """SPEC.md:132-140."""
    return TransformPlan(nufft_type, N, epsilon, method, precision, workers, **kwargs)


def set_points(plan, coords, y=None, z=None):
    """SPEC.md:142-150."""
    return plan.set_points(coords, y, z)


def execute(plan, input, output=None):
    """SPEC.md:152-160."""
    return plan.execute(input, output)


def destroy(plan):
    """SPEC.md:176."""
    plan.destroy()


class Plan(TransformPlan):
    """cufinufft-style constructor:
    ``Plan(nufft_type, n_modes, eps=1e-6, dtype="complex64", gpu_device_id=None)``
    with n_modes axis 1 first; then ``.setpts(x, y[, z])`` and ``.execute(c)``."""

    def __init__(self, nufft_type, n_modes, eps=1e-6, dtype="complex64", gpu_device_id=None,
                 method="default", **kwargs):
        precision = "single" if np.dtype(dtype) in (np.complex64, np.float32) else "double"
        super().__init__(nufft_type, n_modes, eps, method, precision, device=gpu_device_id,
                         **kwargs)
