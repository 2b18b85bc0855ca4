#!/usr/bin/env python
"""Time the REAL reference (nufftkit's Numba loops, imported from
/root/reference the way tests/golden/make_golden.py does) beside the oracle
C port on the same sample and thread count, for the M-proportional stage of
each BASELINE config: SM spread (type 1, spread.py:166-182) and the GM-sort
interp (type 2; the reference ships _kernels.interp_2d/3d, its wrapper is
missing, so it is driven here over contiguous chunks of
the bin-sorted points on the reference's worker pool).

Run in the build container (where /root/reference exists):

    python scripts/time_numba_reference.py > profiles/r2/numba_vs_port.json

This is test / measurement infrastructure only (the product never imports
the reference or the oracle).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from make_golden import import_reference  # noqa: E402

from oracle import oracle as orc  # noqa: E402

CASES = [  # name, type, modes, M sample, dist, eps, precision
    ("C1", 1, (256, 256), 1_000_000, "rand", 1e-5, "single"),
    ("C2", 2, (1024, 1024), 2_000_000, "rand", 1e-5, "single"),
    ("C3a", 1, (128, 128, 128), 1_000_000, "cluster", 1e-6, "single"),
    ("C5t1", 1, (128, 128, 128), 300_000, "rand", 1e-12, "double"),
    ("C5t2", 2, (128, 128, 128), 300_000, "rand", 1e-12, "double"),
]


def best(f, reps=3):
    f()   # JIT / warm-up
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    kernel, binsort, spread, _kernels = import_reference()
    threads = os.cpu_count() or 1
    out = {"threads": threads, "host": os.uname().nodename, "cases": []}
    for name, t, modes, M, dist, eps, prec in CASES:
        grid = orc.make_grid(modes, eps, prec)
        rdt = np.float32 if prec == "single" else np.float64
        cdt = np.complex64 if prec == "single" else np.complex128
        pts = orc.gen_points(dist, M, grid, 1, rdt)
        c = orc.gen_strengths(M, 2).astype(cdt)
        rg = orc.GridSpec(modes, grid.fine)
        rparams = kernel.select_kernel_params(eps, rg, prec)
        lay = binsort.bin_sort(pts, rg)
        oparams = orc.select_kernel_params(eps, grid, prec)
        olay = orc.bin_sort(pts, grid)
        if t == 1:
            subs = binsort.build_subproblems(lay, rparams)
            osubs = orc.build_subproblems(olay, oparams)
            t_ref = best(lambda: spread.spread_sm(pts, lay, subs, c, rparams, rg,
                                                  workers=threads))
            t_port = best(lambda: orc.spread_sm(pts, olay, osubs, c, oparams, grid,
                                                workers=threads))
            stage = "SM spread"
        else:
            fine = (np.random.default_rng(3).standard_normal(grid.fine[::-1]) +
                    1j * np.random.default_rng(4).standard_normal(grid.fine[::-1])).astype(cdt)
            v = np.ascontiguousarray(binsort.grid_coords(pts, rg.fine)[lay.perm].T)
            from concurrent.futures import ThreadPoolExecutor
            interp = _kernels.interp_2d if len(modes) == 2 else _kernels.interp_3d
            res = np.empty(M, np.complex128)
            fine128 = fine.astype(np.complex128)

            def ref_interp():
                chunks = np.array_split(np.arange(M), threads)
                def run(ix):
                    interp(*[np.ascontiguousarray(r[ix]) for r in v], rparams.w, rparams.beta,
                           fine128, res[ix[0]:ix[-1] + 1])
                with ThreadPoolExecutor(threads) as ex:
                    list(ex.map(run, chunks))
            t_ref = best(ref_interp)
            t_port = best(lambda: orc.interpolate(pts, fine, oparams, grid, olay, threads))
            stage = "GM-sort interp"
        out["cases"].append({"config": name, "stage": stage, "M": M, "dist": dist,
                             "eps": eps, "precision": prec,
                             "numba_reference_s": t_ref, "oracle_port_s": t_port,
                             "numba_pts_per_s": M / t_ref, "port_pts_per_s": M / t_port,
                             "port_over_numba": t_ref / t_port})
        print(name, stage, f"numba {M / t_ref:.3e} pts/s, port {M / t_port:.3e} pts/s",
              file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
