"""CPU-side checks of the product package (no GPU): the C-ABI library loads
and exports every symbol include/nufft_b200.h declares; its plan-time host
math matches the reference's golden vectors; argument validation raises the
reference's exceptions before any device work."""

import os
import re
import warnings

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def nk():
    import paper_2102_08463_b200 as nk
    return nk


def test_library_exports_every_header_symbol(nk):
    from paper_2102_08463_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "nufft_b200.h")).read()
    declared = set(re.findall(r"NK_API\s+[\w\s\*]*?\b(nk_\w+)\s*\(", hdr))
    assert len(declared) >= 20
    L = _lib.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(_lib.EXPORTED)


def test_tolerance_to_width_golden(golden, nk):
    for e, prec, ee, w, b in golden["kernel_tw"]:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            assert nk.tolerance_to_width(e, "double" if prec else "single") == (ee, int(w), b)
    with pytest.warns(UserWarning):
        nk.tolerance_to_width(1e-9, "single")
    for bad in (0.0, 1.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(ValueError):
            nk.tolerance_to_width(bad)
    with pytest.raises(ValueError):
        nk.tolerance_to_width(1e-3, "quad")


def test_kernel_fourier_golden(golden, nk):
    xi = golden["kernel_ft_xi"]
    for row, w in zip(golden["kernel_ft_v"], range(2, 17)):
        got = nk.kernel_fourier(2.30 * w, xi)
        assert np.abs(got - row).max() <= 1e-14 * np.abs(row).max()
    assert abs(nk.kernel_fourier(0.0, 0.0) - 2.0) < 1e-14
    assert nk.kernel_fourier(13.8, 5.0) == nk.kernel_fourier(13.8, -5.0)


def test_eval_kernel_golden(golden, nk):
    z = golden["kernel_eval_z"]
    for row, w in zip(golden["kernel_eval_v"], (2, 6, 13, 16)):
        np.testing.assert_array_equal(nk.eval_kernel(2.30 * w, z), row)


def test_correction_factors_golden(golden, nk, orc):
    for ci in range(5):
        modes = tuple(int(x) for x in golden[f"corr{ci}_modes"])
        e, prec = golden[f"corr{ci}_meta"]
        precision = "double" if prec else "single"
        fine = tuple(int(x) for x in golden[f"corr{ci}_fine"])
        grid = nk.GridSpec(modes, fine)
        assert orc.make_grid(modes, e, precision).fine == fine
        p = nk.select_kernel_params(e, grid, precision)
        got = nk.build_correction_factors(grid, p)
        ref = golden[f"corr{ci}_values"]
        assert got.dtype == ref.dtype
        np.testing.assert_allclose(got, ref, rtol=1e-13 if prec else 1e-6)


def test_next_smooth_exhaustive(nk):
    """SPEC.md:574 acceptance 4 (exhaustive 5-smooth enumeration)."""
    lim = 200_000
    smooth = set()
    p2 = 1
    while p2 <= 2 * lim:
        p3 = p2
        while p3 <= 2 * lim:
            p5 = p3
            while p5 <= 2 * lim:
                smooth.add(p5)
                p5 *= 5
            p3 *= 3
        p2 *= 2
    srt = sorted(smooth)
    import bisect
    for n in list(range(1, 3000)) + list(range(lim - 3000, lim)):
        assert nk.next_smooth(n) == srt[bisect.bisect_left(srt, n)]
    assert [nk.next_smooth(n) for n in (2000, 254, 1)] == [2000, 256, 1]
    with pytest.raises(ValueError):
        nk.next_smooth(0)


def test_plan_argument_validation(nk):
    with pytest.raises(ValueError):
        nk.make_plan(1, (16,), 1e-6)                 # dim 1
    with pytest.raises(ValueError):
        nk.make_plan(1, (4, 4, 4, 4), 1e-6)          # dim 4
    with pytest.raises(ValueError):
        nk.make_plan(1, (0, 4), 1e-6)                # zero modes
    with pytest.raises(ValueError):
        nk.make_plan(1, (4, 4), 1e-6, precision="half")
    with pytest.raises(ValueError):
        nk.make_plan(1, (4, 4), 1e-6, method="fast")
    with pytest.raises(ValueError):
        nk.make_plan(1, (4, 4), 1e-6, workers=-1)
    with pytest.raises(ValueError):
        nk.make_plan(1, (4, 4), 1e-6, bin_dims=(0, 4))
    with pytest.raises(ValueError):
        nk.make_plan(1, (4, 4), 1e-6, max_subproblem=0)


def test_no_cpu_fallback_in_product():
    """The product package must not import the oracle (the checker)."""
    pkg = os.path.join(ROOT, "paper_2102_08463_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "from oracle" not in src and "import oracle" not in src, fn
