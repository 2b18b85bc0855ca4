"""Generate golden vectors from the REAL reference package (nufftkit).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference is imported from a temporary COPY of
/root/reference/pkg/src (Numba's cache=True would otherwise write
__pycache__ into the read-only tree) with NUMBA_CACHE_DIR set
to a temp dir.  Outputs are small .npz fixtures committed next to this
script; nothing at test time reads /root/reference.

The shipped modules are kernel.py, binsort.py, spread.py, _kernels.py and
_parallel.py.  The pipeline/interp modules are missing from the reference;
the composed end-to-end fixtures below use the shipped spread/binsort/kernel
code plus numpy FFT and the SPEC.md:408-425 deconvolution with the
(-1)^{sum k} phase -- exactly the composition SURVEY.md
measured against direct sums.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


class Grid:
    """Duck-typed GridSpec (kernel.py:115,189,193; binsort.py:122-129)."""

    def __init__(self, modes, fine):
        self.modes = tuple(modes)
        self.fine = tuple(fine)
        self.dim = len(modes)
        self.fine_shape = tuple(fine[::-1])


def next_smooth(n):
    def ok(m):
        for p in (2, 3, 5):
            while m % p == 0:
                m //= p
        return m == 1
    while not ok(n):
        n += 1
    return n


def import_reference():
    tmp = tempfile.mkdtemp(prefix="nufftkit_ref_")
    shutil.copytree(REF_SRC, os.path.join(tmp, "src"))
    os.environ["NUMBA_CACHE_DIR"] = os.path.join(tmp, "numba_cache")
    sys.path.insert(0, os.path.join(tmp, "src"))
    from nufftkit import _kernels, binsort, kernel, spread  # noqa: E402
    return kernel, binsort, spread, _kernels


def grid_for(kernel, modes, eps, prec):
    _, w, _ = kernel.tolerance_to_width(eps, prec)
    return Grid(modes, [next_smooth(max(2 * N, 2 * w)) for N in modes])


def gen_points(rng, dist, M, grid):
    d = grid.dim
    if dist == "rand":
        return rng.uniform(-np.pi, np.pi, (M, d))
    if dist == "cluster":
        h = np.array([2 * np.pi / n for n in grid.fine])
        return rng.uniform(0, 1, (M, d)) * (8 * h)
    if dist == "wide":  # unfolded coordinates, exercises the fold
        return rng.uniform(-40.0, 40.0, (M, d))
    raise ValueError(dist)


def deconv_type1(spec, grid, pk):
    """SPEC.md:408-416 + phase."""
    d = grid.dim
    idx = np.ix_(*[np.mod(np.arange(N) - N // 2, n)
                   for N, n in zip(grid.modes[::-1], grid.fine[::-1])])
    sel = spec[idx]
    ks = np.meshgrid(*[np.arange(N) - N // 2 for N in grid.modes[::-1]], indexing="ij")
    phase = (-1.0) ** (sum(ks) % 2)
    return (pk * phase * sel).astype(spec.dtype)


def deconv_type2(f, grid, pk, dtype):
    d = grid.dim
    out = np.zeros(grid.fine_shape, dtype=dtype)
    idx = np.ix_(*[np.mod(np.arange(N) - N // 2, n)
                   for N, n in zip(grid.modes[::-1], grid.fine[::-1])])
    ks = np.meshgrid(*[np.arange(N) - N // 2 for N in grid.modes[::-1]], indexing="ij")
    phase = (-1.0) ** (sum(ks) % 2)
    out[idx] = (pk * phase * f.reshape(grid.modes[::-1])).astype(dtype)
    return out


def main():
    kernel, binsort, spread, _kernels = import_reference()
    rng = np.random.default_rng(20210217)
    out = {}

    # ---- kernel.py: widths, kernel values, Fourier transform, corrections
    eps_list = [1e-1, 1e-2, 1e-4, 1e-5, 1e-6, 1e-9, 1e-12, 1e-15, 1e-20, 0.5, 0.999]
    tw = []
    for prec in ("single", "double"):
        for e in eps_list:
            import warnings
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                ee, w, b = kernel.tolerance_to_width(e, prec)
            tw.append((e, 0 if prec == "single" else 1, ee, w, b))
    out["kernel_tw"] = np.array(tw, dtype=np.float64)
    zs = np.concatenate([np.linspace(-1.2, 1.2, 97), [0.0, 1.0, -1.0, 1.5, 1 + 1e-16]])
    out["kernel_eval_z"] = zs
    out["kernel_eval_v"] = np.stack([kernel.eval_kernel(2.30 * w, zs) for w in (2, 6, 13, 16)])
    xis = np.linspace(-25.0, 25.0, 201)
    out["kernel_ft_xi"] = xis
    out["kernel_ft_v"] = np.stack([kernel.kernel_fourier(2.30 * w, xis) for w in range(2, 17)])
    corr_cases = [((8, 8), 1e-5, "double"), ((16, 10), 1e-9, "double"),
                  ((6, 7, 5), 1e-6, "single"), ((64, 64), 1e-5, "single"),
                  ((4, 4), 1e-12, "double")]
    for ci, (modes, e, prec) in enumerate(corr_cases):
        g = grid_for(kernel, modes, e, prec)
        p = kernel.select_kernel_params(e, g, prec)
        out[f"corr{ci}_modes"] = np.array(modes)
        out[f"corr{ci}_fine"] = np.array(g.fine)
        out[f"corr{ci}_meta"] = np.array([e, 0 if prec == "single" else 1])
        out[f"corr{ci}_values"] = kernel.build_correction_factors(g, p)

    # ---- binsort.py: grid coords incl. seam/extreme values
    seam = [np.pi, -np.pi, np.nextafter(np.pi, 0), np.nextafter(-np.pi, 0),
            np.nextafter(-np.pi, -4), np.nextafter(np.pi, 4), 3 * np.pi, -3 * np.pi,
            0.0, -0.0, 1e30, -1e30, 1e-300, -1e-300, 2 * np.pi, -2 * np.pi,
            np.float32(np.pi), np.float32(-np.pi), np.nextafter(np.float32(-np.pi), np.float32(-4))]
    seam = np.array(seam, dtype=np.float64)
    rnd = rng.uniform(-10, 10, 4000)
    f32 = rng.uniform(-np.pi, np.pi, 4000).astype(np.float32).astype(np.float64)
    xs = np.concatenate([seam, rnd, f32])
    for n in (27, 128, 512, 2048, 256):
        out[f"gc_n{n}"] = binsort.grid_coords(xs.reshape(-1, 1), (n,))[:, 0]
    out["gc_x"] = xs

    # KAT cases: bin keys
    g128 = Grid((64, 64), (128, 128))
    h = 2 * np.pi / 128
    kat_pts = np.array([[-np.pi, -np.pi], [-np.pi + 33.5 * h, -np.pi + 0.5 * h],
                        [-np.pi + 0.5 * h, -np.pi + 32.5 * h]])
    out["kat_bins"] = binsort.bin_index(kat_pts, g128, (32, 32))

    # bin_sort + build_subproblems on several geometries
    sort_cases = [
        ("s2r", (32, 32), 1e-5, "single", "rand", 3000, None, 64),
        ("s2c", (32, 32), 1e-5, "single", "cluster", 3000, None, 100),
        ("s2w", (20, 24), 1e-9, "double", "wide", 2500, (8, 16), 37),
        ("s3r", (12, 12, 12), 1e-6, "single", "rand", 4000, None, 50),
        ("s3c", (10, 12, 8), 1e-12, "double", "cluster", 2000, (4, 4, 2), 128),
        ("s3w", (12, 10, 14), 1e-4, "double", "wide", 3000, (8, 4, 4), 1024),
    ]
    for name, modes, e, prec, dist, M, bd, msub in sort_cases:
        g = grid_for(kernel, modes, e, prec)
        p = kernel.select_kernel_params(e, g, prec)
        pts = gen_points(rng, dist, M, g)
        if prec == "single":
            pts = pts.astype(np.float32)
        lay = binsort.bin_sort(pts, g, bd)
        subs = binsort.build_subproblems(lay, p, msub)
        out[f"{name}_pts"] = pts
        out[f"{name}_meta"] = np.array([e, 0 if prec == "single" else 1, msub])
        out[f"{name}_modes"] = np.array(modes)
        out[f"{name}_fine"] = np.array(g.fine)
        out[f"{name}_bindims"] = np.array(lay.bin_dims)
        out[f"{name}_keys"] = lay.point_bins
        out[f"{name}_counts"] = lay.counts
        out[f"{name}_starts"] = lay.starts
        out[f"{name}_perm"] = lay.perm
        out[f"{name}_sub_bin"] = subs.bin_ids
        out[f"{name}_sub_start"] = subs.slice_starts
        out[f"{name}_sub_stop"] = subs.slice_stops
        out[f"{name}_sub_off"] = subs.offsets
        out[f"{name}_sub_pad"] = subs.padded_dims

        # spread (1 worker: deterministic order) GM, GM-sort, SM
        cdt = np.complex64 if prec == "single" else np.complex128
        c = (rng.uniform(-1, 1, M) + 1j * rng.uniform(-1, 1, M)).astype(cdt)
        out[f"{name}_c"] = c
        out[f"{name}_spread_gm"] = spread.spread_gm(pts, c, p, g, 1)
        out[f"{name}_spread_gmsort"] = spread.spread_gm_sort(pts, lay, c, p, g, 1)
        out[f"{name}_spread_sm"] = spread.spread_sm(pts, lay, subs, c, p, g, 1)
        # interp over a random fine grid (shipped numba kernels; the
        # interpolate wrapper itself is missing)
        fg = (rng.uniform(-1, 1, g.fine_shape) + 1j * rng.uniform(-1, 1, g.fine_shape)).astype(cdt)
        v = binsort.grid_coords(pts, g.fine)
        res = np.empty(M, dtype=cdt)
        if g.dim == 2:
            _kernels.interp_2d(np.ascontiguousarray(v[:, 0]), np.ascontiguousarray(v[:, 1]),
                               p.w, p.beta, fg, res)
        else:
            _kernels.interp_3d(np.ascontiguousarray(v[:, 0]), np.ascontiguousarray(v[:, 1]),
                               np.ascontiguousarray(v[:, 2]), p.w, p.beta, fg, res)
        out[f"{name}_interp_grid"] = fg
        out[f"{name}_interp"] = res

        # composed pipeline (shipped spread + numpy FFT + restated deconv)
        pk = kernel.build_correction_factors(g, p)
        b = out[f"{name}_spread_sm"]
        bh = np.fft.fftn(b).astype(cdt)
        out[f"{name}_type1"] = deconv_type1(bh, g, pk).reshape(-1)
        f = (rng.uniform(-1, 1, int(np.prod(modes))) +
             1j * rng.uniform(-1, 1, int(np.prod(modes)))).astype(cdt)
        bh2 = deconv_type2(f, g, pk, cdt)
        b2 = (np.fft.ifftn(bh2) * np.prod(g.fine)).astype(cdt)
        res2 = np.empty(M, dtype=cdt)
        if g.dim == 2:
            _kernels.interp_2d(np.ascontiguousarray(v[:, 0]), np.ascontiguousarray(v[:, 1]),
                               p.w, p.beta, b2, res2)
        else:
            _kernels.interp_3d(np.ascontiguousarray(v[:, 0]), np.ascontiguousarray(v[:, 1]),
                               np.ascontiguousarray(v[:, 2]), p.w, p.beta, b2, res2)
        out[f"{name}_f"] = f
        out[f"{name}_type2"] = res2

    # SPEC.md:232-234 subproblem KAT: counts (2500, 10), M_sub=1024
    g2 = Grid((32, 32), (64, 64))
    p2 = kernel.select_kernel_params(1e-5, g2, "double")
    hh = 2 * np.pi / 64
    pts = np.concatenate([np.full((2500, 2), -np.pi + 0.5 * hh),
                          np.tile([[-np.pi + 40.5 * hh, -np.pi + 0.5 * hh]], (10, 1))])
    lay = binsort.bin_sort(pts, g2, (32, 32))
    subs = binsort.build_subproblems(lay, p2, 1024)
    out["kat_sub_sizes"] = subs.slice_stops - subs.slice_starts
    out["kat_sub_off"] = subs.offsets
    out["kat_sub_pad"] = subs.padded_dims

    path = os.path.join(HERE, "golden_v1.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {os.path.getsize(path) / 1e6:.2f} MB, {len(out)} arrays")


if __name__ == "__main__":
    main()
