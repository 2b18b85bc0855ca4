"""Pin the CPU oracle against golden vectors from the real reference.

Fixtures: tests/golden/golden_v1.npz, produced by tests/golden/make_golden.py
from the shipped nufftkit modules (kernel.py, binsort.py, spread.py,
_kernels.py).  Integer outputs must match bit-for-bit; floating point
within the stated tolerances.
"""

import warnings

import numpy as np
import pytest

SORT_CASES = ["s2r", "s2c", "s2w", "s3r", "s3c", "s3w"]


def _grid(orc, g, name):
    return orc.GridSpec(tuple(int(x) for x in g[f"{name}_modes"]),
                        tuple(int(x) for x in g[f"{name}_fine"]))


def _params(orc, g, name, grid):
    e, prec, _ = g[f"{name}_meta"]
    return orc.select_kernel_params(float(e), grid, "double" if prec else "single")


def test_tolerance_to_width(golden, orc):
    for e, prec, ee, w, b in golden["kernel_tw"]:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            got = orc.tolerance_to_width(e, "double" if prec else "single")
        assert got == (ee, int(w), b)


def test_tolerance_kats(orc):
    # SPEC.md:44-46
    assert orc.tolerance_to_width(1e-5)[1:] == (6, 2.30 * 6)
    assert orc.tolerance_to_width(1e-12)[1] == 13
    assert orc.tolerance_to_width(1e-2)[1] == 3
    for bad in (0.0, 1.0, -1e-3, float("nan"), float("inf")):
        with pytest.raises(ValueError):
            orc.tolerance_to_width(bad)
    with pytest.raises(ValueError):
        orc.tolerance_to_width(1e-3, "half")
    with pytest.warns(UserWarning):
        assert orc.tolerance_to_width(1e-8, "single")[0] == 1e-6


def test_eval_kernel(golden, orc):
    z = golden["kernel_eval_z"]
    for row, w in zip(golden["kernel_eval_v"], (2, 6, 13, 16)):
        np.testing.assert_array_equal(orc.eval_kernel(2.30 * w, z), row)


def test_kernel_fourier(golden, orc):
    xi = golden["kernel_ft_xi"]
    for row, w in zip(golden["kernel_ft_v"], range(2, 17)):
        np.testing.assert_allclose(orc.kernel_fourier(2.30 * w, xi), row, rtol=1e-14,
                                   atol=1e-14 * np.abs(row).max())


def test_correction_factors(golden, orc):
    for ci in range(5):
        modes = tuple(int(x) for x in golden[f"corr{ci}_modes"])
        e, prec = golden[f"corr{ci}_meta"]
        precision = "double" if prec else "single"
        grid = orc.make_grid(modes, e, precision)
        assert grid.fine == tuple(int(x) for x in golden[f"corr{ci}_fine"])
        p = orc.select_kernel_params(e, grid, precision)
        ref = golden[f"corr{ci}_values"]
        got = orc.build_correction_factors(grid, p)
        assert got.dtype == ref.dtype
        np.testing.assert_allclose(got, ref, rtol=1e-13 if prec else 1e-6)
        # tensor-product factors used by deconvolve_* reproduce the array
        ax = orc.axis_factors(grid, p)
        prod = ax[-1]
        for a in ax[-2::-1]:
            prod = np.multiply.outer(prod, a)
        np.testing.assert_allclose(prod, ref, rtol=1e-12 if prec else 1e-6)


def test_grid_coords_bitexact(golden, orc):
    xs = golden["gc_x"]
    for n in (27, 128, 512, 2048, 256):
        got = orc.grid_coords(xs.reshape(-1, 1), (n,))[:, 0]
        ref = golden[f"gc_n{n}"]
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), n


def test_bin_key_kats(golden, orc):
    g = orc.GridSpec((64, 64), (128, 128))
    h = 2 * np.pi / 128
    pts = np.array([[-np.pi, -np.pi], [-np.pi + 33.5 * h, -np.pi + 0.5 * h],
                    [-np.pi + 0.5 * h, -np.pi + 32.5 * h]])
    lay = orc.bin_sort(pts, g, (32, 32))
    assert list(lay.point_bins) == [0, 1, 4] == list(golden["kat_bins"])


def test_stable_perm_kat(orc):
    # bins (2,0,1,0,2) -> 1-based order (2,4,3,1,5)
    g = orc.GridSpec((32, 32), (64, 64))
    h = 2 * np.pi / 64
    xb = {0: 0.5, 1: 32.5, 2: 0.5}
    yb = {0: 0.5, 1: 0.5, 2: 32.5}
    bins = (2, 0, 1, 0, 2)
    pts = np.array([[-np.pi + xb[b] * h, -np.pi + yb[b] * h] for b in bins])
    lay = orc.bin_sort(pts, g, (32, 32))
    assert list(lay.point_bins) == [2, 0, 1, 0, 2]
    assert list(lay.perm + 1) == [2, 4, 3, 1, 5]


@pytest.mark.parametrize("name", SORT_CASES)
def test_bin_sort_and_subproblems_bitexact(golden, orc, name):
    grid = _grid(orc, golden, name)
    p = _params(orc, golden, name, grid)
    bd = tuple(int(x) for x in golden[f"{name}_bindims"])
    lay = orc.bin_sort(golden[f"{name}_pts"], grid, bd)
    for f, k in (("point_bins", "keys"), ("counts", "counts"), ("starts", "starts"),
                 ("perm", "perm")):
        np.testing.assert_array_equal(getattr(lay, f), golden[f"{name}_{k}"])
    subs = orc.build_subproblems(lay, p, int(golden[f"{name}_meta"][2]))
    np.testing.assert_array_equal(subs.bin_ids, golden[f"{name}_sub_bin"])
    np.testing.assert_array_equal(subs.slice_starts, golden[f"{name}_sub_start"])
    np.testing.assert_array_equal(subs.slice_stops, golden[f"{name}_sub_stop"])
    np.testing.assert_array_equal(subs.offsets, golden[f"{name}_sub_off"])
    np.testing.assert_array_equal(subs.padded_dims, golden[f"{name}_sub_pad"])


@pytest.mark.parametrize("name", SORT_CASES)
def test_spread_matches_reference(golden, orc, name):
    grid = _grid(orc, golden, name)
    p = _params(orc, golden, name, grid)
    bd = tuple(int(x) for x in golden[f"{name}_bindims"])
    pts, c = golden[f"{name}_pts"], golden[f"{name}_c"]
    lay = orc.bin_sort(pts, grid, bd)
    subs = orc.build_subproblems(lay, p, int(golden[f"{name}_meta"][2]))
    got = {
        "gm": orc.spread_gm(pts, c, p, grid, 1),
        "gmsort": orc.spread_gm_sort(pts, lay, c, p, grid, 1),
        "sm": orc.spread_sm(pts, lay, subs, c, p, grid, 1),
    }
    for m, g in got.items():
        ref = golden[f"{name}_spread_{m}"]
        assert g.dtype == ref.dtype and g.shape == ref.shape
        # serial loops restate the Numba loops operation for operation:
        # bit-identical to the reference
        np.testing.assert_array_equal(g, ref)


@pytest.mark.parametrize("name", SORT_CASES)
def test_interp_matches_reference(golden, orc, name):
    grid = _grid(orc, golden, name)
    p = _params(orc, golden, name, grid)
    pts = golden[f"{name}_pts"]
    ref = golden[f"{name}_interp"]
    got = orc.interpolate(pts, golden[f"{name}_interp_grid"], p, grid)
    np.testing.assert_array_equal(got, ref)     # bit-identical to the Numba loop
    lay = orc.bin_sort(pts, grid)
    got2 = orc.interpolate(pts, golden[f"{name}_interp_grid"], p, grid, lay)
    np.testing.assert_array_equal(got, got2)   # SPEC.md:364 GM == GM-sort


@pytest.mark.parametrize("name", SORT_CASES)
def test_composed_pipeline_matches_reference(golden, orc, name):
    grid = _grid(orc, golden, name)
    p = _params(orc, golden, name, grid)
    e = float(golden[f"{name}_meta"][0])
    modes = grid.modes
    bd = tuple(int(x) for x in golden[f"{name}_bindims"])
    prec = p.precision
    plan1 = orc.OraclePlan(1, modes, e, "sm", prec, 1, bd, int(golden[f"{name}_meta"][2]))
    plan1.set_points(golden[f"{name}_pts"])
    f1 = plan1.execute(golden[f"{name}_c"])
    ref1 = golden[f"{name}_type1"]
    tol = 1e-12 if prec == "double" else 2e-6
    assert orc.rel_l2_error(f1, ref1) < tol
    plan2 = orc.OraclePlan(2, modes, e, "gmsort", prec, 1, bd)
    plan2.set_points(golden[f"{name}_pts"])
    c2 = plan2.execute(golden[f"{name}_f"])
    assert orc.rel_l2_error(c2, golden[f"{name}_type2"]) < tol


def test_subproblem_kat(golden, orc):
    # SPEC.md:232-234
    assert list(golden["kat_sub_sizes"]) == [1024, 1024, 452, 10]
    g = orc.GridSpec((32, 32), (64, 64))
    p = orc.select_kernel_params(1e-5, g, "double")
    hh = 2 * np.pi / 64
    pts = np.concatenate([np.full((2500, 2), -np.pi + 0.5 * hh),
                          np.tile([[-np.pi + 40.5 * hh, -np.pi + 0.5 * hh]], (10, 1))])
    subs = orc.build_subproblems(orc.bin_sort(pts, g, (32, 32)), p, 1024)
    assert list(subs.slice_stops - subs.slice_starts) == [1024, 1024, 452, 10]
    np.testing.assert_array_equal(subs.offsets, golden["kat_sub_off"])
    np.testing.assert_array_equal(subs.padded_dims, golden["kat_sub_pad"])
    assert list(subs.padded_dims[0]) == [38, 38]
    assert list(subs.offsets[0]) == [-3, -3]


@pytest.mark.parametrize("dim,modes,eps", [(2, (24, 20), 1e-9), (3, (10, 8, 12), 1e-6)])
def test_oracle_accuracy_vs_direct(orc, dim, modes, eps):
    """rel l2 vs direct sum <= 10 eps (double)."""
    g = orc.make_grid(modes, eps, "double")
    M = 1500
    pts = orc.gen_points("rand", M, g, 3)
    c = orc.gen_strengths(M, 3)
    for method in ("gm", "gmsort", "sm"):
        pl = orc.OraclePlan(1, modes, eps, method, "double")
        pl.set_points(pts)
        assert orc.rel_l2_error(pl.execute(c), orc.direct_type1(pts, c, modes)) < 10 * eps
    f = orc.gen_strengths(int(np.prod(modes)), 4)
    pl = orc.OraclePlan(2, modes, eps, "gmsort", "double")
    pl.set_points(pts)
    assert orc.rel_l2_error(pl.execute(f), orc.direct_type2(pts, f, modes)) < 10 * eps


def test_direct_oracle_kats(orc):
    # SPEC.md:479-490
    f = orc.direct_type1(np.zeros((1, 2)), np.ones(1), (4, 4))
    np.testing.assert_allclose(f, np.ones(16), atol=1e-15)
    f = orc.direct_type1(np.array([[np.pi / 2, 0.0]]), np.ones(1), (4, 4))
    # k=(1,0) at i1 = 1 + 2, i2 = 0 + 2
    assert abs(f[2 * 4 + 3] - (-1j)) < 1e-15
    rng = np.random.default_rng(0)
    pts = rng.uniform(-np.pi, np.pi, (50, 3))
    c = rng.standard_normal(50) + 1j * rng.standard_normal(50)
    fm = rng.standard_normal(60) + 1j * rng.standard_normal(60)
    lhs = np.vdot(orc.direct_type2(pts, fm, (5, 4, 3)), c)
    rhs = np.vdot(fm, orc.direct_type1(pts, c, (5, 4, 3)))
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


def test_next_smooth(orc):
    assert [orc.next_smooth(n) for n in (2000, 254, 1)] == [2000, 256, 1]
    assert orc.make_grid((4, 4), 1e-12).fine == (27, 27)
    assert orc.make_grid((100, 100, 100), 1e-5).fine == (200, 200, 200)
