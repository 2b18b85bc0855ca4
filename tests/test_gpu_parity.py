"""GPU parity: the CUDA path (through the C-ABI) against the reference's
golden vectors and the CPU oracle.

Bars:
  * bin keys, counts, starts, permutation, subproblem table: bit-exact;
  * spread / interp vs the reference's own loops: relative max error
    <= 2e-6 (single) / 1e-13 (double) -- kernel values are evaluated in
    the plan precision on the GPU, in FP64 by the reference;
  * transforms: rel l2 vs direct sums <= 10 eps and vs the
    oracle pipeline <= eps-level tolerances below.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SORT_CASES = ["s2r", "s2c", "s2w", "s3r", "s3c", "s3w"]


@pytest.fixture(scope="module")
def nk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2102_08463_b200 as nk
    return nk


@pytest.fixture(scope="module")
def st(nk):
    from paper_2102_08463_b200 import stages
    return stages


def _case(nk, g, name):
    grid = nk.GridSpec(tuple(int(x) for x in g[f"{name}_modes"]),
                       tuple(int(x) for x in g[f"{name}_fine"]))
    e, prec, msub = g[f"{name}_meta"]
    params = nk.select_kernel_params(float(e), grid, "double" if prec else "single")
    bd = tuple(int(x) for x in g[f"{name}_bindims"])
    return grid, params, bd, int(msub)


def _relmax(a, b):
    return float(np.abs(np.asarray(a) - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("name", SORT_CASES)
def test_bin_sort_bitexact_vs_reference(golden, nk, st, name):
    grid, params, bd, msub = _case(nk, golden, name)
    lay = st.bin_sort(golden[f"{name}_pts"], grid, bd)
    np.testing.assert_array_equal(lay.point_bins, golden[f"{name}_keys"])
    np.testing.assert_array_equal(lay.counts, golden[f"{name}_counts"])
    np.testing.assert_array_equal(lay.starts, golden[f"{name}_starts"])
    np.testing.assert_array_equal(lay.perm, golden[f"{name}_perm"])
    subs = st.build_subproblems(lay, params, msub)
    np.testing.assert_array_equal(subs.bin_ids, golden[f"{name}_sub_bin"])
    np.testing.assert_array_equal(subs.slice_starts, golden[f"{name}_sub_start"])
    np.testing.assert_array_equal(subs.slice_stops, golden[f"{name}_sub_stop"])
    np.testing.assert_array_equal(subs.offsets, golden[f"{name}_sub_off"])
    np.testing.assert_array_equal(subs.padded_dims, golden[f"{name}_sub_pad"])


def test_fold_seam_bitexact(golden, nk, st, orc):
    """x at +-pi, nextafter neighbours, 3pi, +-1e30, +-0 (binsort.py:98-100)."""
    xs = golden["gc_x"]
    for n in (128, 512, 2048):
        grid = nk.GridSpec((n // 2, n // 2), (n, n))
        pts = np.stack([xs, xs[::-1]], axis=1)
        lay = st.bin_sort(pts, grid, (1, 1))       # 1-cell bins: key = cell index
        ref = orc.bin_sort(pts, grid, (1, 1))
        np.testing.assert_array_equal(lay.point_bins, ref.point_bins)
        np.testing.assert_array_equal(lay.perm, ref.perm)


@pytest.mark.parametrize("M,dist,dims", [(200_000, "rand", 2), (300_000, "cluster", 3),
                                         (150_000, "gauss", 3), (500_000, "rand", 3)])
def test_bin_sort_bitexact_large(nk, st, orc, M, dist, dims):
    modes = (256, 256) if dims == 2 else (64, 64, 64)
    grid = orc.make_grid(modes, 1e-6, "single")
    pts = orc.gen_points(dist, M, grid, 11, np.float32)
    lay = st.bin_sort(pts, nk.GridSpec(modes, grid.fine))
    ref = orc.bin_sort(pts, grid)
    np.testing.assert_array_equal(lay.point_bins, ref.point_bins)
    np.testing.assert_array_equal(lay.counts, ref.counts)
    np.testing.assert_array_equal(lay.perm, ref.perm)
    p = orc.select_kernel_params(1e-6, grid, "single")
    subs = st.build_subproblems(lay, p, 1024)
    rs = orc.build_subproblems(ref, p, 1024)
    np.testing.assert_array_equal(subs.bin_ids, rs.bin_ids)
    np.testing.assert_array_equal(subs.slice_stops, rs.slice_stops)
    np.testing.assert_array_equal(subs.offsets, rs.offsets)


@pytest.mark.parametrize("name", SORT_CASES)
@pytest.mark.parametrize("method", ["gm", "gmsort", "sm"])
def test_spread_vs_reference(golden, nk, st, name, method):
    grid, params, bd, msub = _case(nk, golden, name)
    pts, c = golden[f"{name}_pts"], golden[f"{name}_c"]
    ref = golden[f"{name}_spread_sm"]
    if method == "gm":
        got = st.spread_gm(pts, c, params, grid)
    else:
        lay = st.bin_sort(pts, grid, bd)
        if method == "gmsort":
            got = st.spread_gm_sort(pts, lay, c, params, grid)
        else:
            got = st.spread_sm(pts, lay, st.build_subproblems(lay, params, msub), c, params,
                               grid)
    assert got.shape == ref.shape and got.dtype == ref.dtype
    tol = 1e-13 if params.precision == "double" else 2e-6
    assert _relmax(got, ref) < tol


@pytest.mark.parametrize("name", SORT_CASES)
@pytest.mark.parametrize("method", ["gm", "gmsort", "sm"])
def test_interp_vs_reference(golden, nk, st, name, method):
    grid, params, bd, msub = _case(nk, golden, name)
    pts = golden[f"{name}_pts"]
    ref = golden[f"{name}_interp"]
    lay = None if method == "gm" else st.bin_sort(pts, grid, bd)
    got = st.interpolate(pts, lay, golden[f"{name}_interp_grid"], params, grid, method=method)
    tol = 1e-13 if params.precision == "double" else 2e-6
    assert _relmax(got, ref) < tol


@pytest.mark.parametrize("name", SORT_CASES)
def test_transforms_vs_reference_composition(golden, nk, name):
    grid, params, bd, msub = _case(nk, golden, name)
    tol = 1e-12 if params.precision == "double" else 5e-6
    p1 = nk.make_plan(1, grid.modes, params.epsilon, "sm", params.precision, bin_dims=bd,
                      max_subproblem=msub)
    p1.set_points(golden[f"{name}_pts"])
    f = p1.execute(golden[f"{name}_c"])
    ref = golden[f"{name}_type1"]
    assert np.linalg.norm(f.reshape(-1) - ref) / np.linalg.norm(ref) < tol
    for method in ("gm", "gmsort", "sm"):
        p2 = nk.make_plan(2, grid.modes, params.epsilon, method, params.precision, bin_dims=bd)
        p2.set_points(golden[f"{name}_pts"])
        c = p2.execute(golden[f"{name}_f"])
        ref2 = golden[f"{name}_type2"]
        assert np.linalg.norm(c - ref2) / np.linalg.norm(ref2) < tol


ACC = [(2, "double", 1e-2), (2, "double", 1e-6), (2, "double", 1e-9), (2, "double", 1e-12),
       (3, "double", 1e-4), (3, "double", 1e-9), (3, "double", 1e-12),
       (2, "single", 1e-2), (2, "single", 1e-4), (2, "single", 1e-6),
       (3, "single", 1e-4), (3, "single", 1e-6)]


@pytest.mark.parametrize("dim,prec,eps", ACC)
@pytest.mark.parametrize("dist", ["rand", "cluster"])
def test_accuracy_vs_direct(nk, orc, dim, prec, eps, dist):
    """SPEC.md:571 acceptance 1 (N=(64,64) / (20,20,20), rho = 1): rel l2 vs
    the direct oracle <= 10 eps for every method."""
    modes = (64, 64) if dim == 2 else (20, 20, 20)
    grid = orc.make_grid(modes, eps, prec)
    M = min(int(np.prod(grid.fine)), 30000)    # rho = 1 in 2D; capped in 3D (oracle cost)
    rdt = np.float32 if prec == "single" else np.float64
    cdt = np.complex64 if prec == "single" else np.complex128
    pts = orc.gen_points(dist, M, grid, 5, rdt)
    c = orc.gen_strengths(M, 5, cdt)
    fm = orc.gen_strengths(int(np.prod(modes)), 6, cdt)
    d1 = orc.direct_type1(pts, c, modes)
    d2 = orc.direct_type2(pts, fm, modes)
    for method in ("gm", "gmsort", "sm"):
        p1 = nk.make_plan(1, modes, eps, method, prec)
        p1.set_points(pts)
        e1 = orc.rel_l2_error(p1.execute(c), d1)
        p2 = nk.make_plan(2, modes, eps, method, prec)
        p2.set_points(pts)
        e2 = orc.rel_l2_error(p2.execute(fm.reshape(modes[::-1])), d2)
        # The bar is 10 eps -- except where the reference itself
        # misses it: single-precision GM / GM-sort on clustered points
        # accumulates ~1e3 complex64 adds per cell (reference: 1.7e-5 at
        # eps=1e-6, 3D cluster).  There the bar is 2x the reference's error.
        bar1 = bar2 = 10 * eps
        if prec == "single" and dist == "cluster":
            op = orc.OraclePlan(1, modes, eps, method, prec)
            op.set_points(pts)
            bar1 = max(bar1, 2 * orc.rel_l2_error(op.execute(c), d1))
        assert e1 < bar1 and e2 < bar2, (method, e1, e2, bar1)


@pytest.mark.parametrize("dim,prec", [(2, "double"), (3, "double"), (2, "single")])
def test_adjointness(nk, orc, dim, prec):
    """<c, T2 f> == <T1 c, f>."""
    modes = (30, 26) if dim == 2 else (12, 10, 14)
    eps = 1e-6
    grid = orc.make_grid(modes, eps, prec)
    M = 5000
    rdt = np.float32 if prec == "single" else np.float64
    cdt = np.complex64 if prec == "single" else np.complex128
    pts = orc.gen_points("rand", M, grid, 9, rdt)
    rng = np.random.default_rng(1)
    for method in ("gmsort", "sm"):
        c = (rng.standard_normal(M) + 1j * rng.standard_normal(M)).astype(cdt)
        f = (rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])).astype(cdt)
        p1 = nk.make_plan(1, modes, eps, method, prec)
        p1.set_points(pts)
        p2 = nk.make_plan(2, modes, eps, method, prec)
        p2.set_points(pts)
        lhs = np.vdot(p2.execute(f).astype(np.complex128), c)
        rhs = np.vdot(f.astype(np.complex128), p1.execute(c).astype(np.complex128))
        tol = 1e-12 if prec == "double" else 1e-5
        assert abs(lhs - rhs) <= tol * (abs(lhs) + abs(rhs))


def test_c1_geometry_vs_oracle(nk, orc):
    """BASELINE C1 geometry (N=256^2, f32, eps 1e-5) at M=2e5: GPU SM and
    GM-sort vs the CPU oracle pipeline."""
    modes, eps = (256, 256), 1e-5
    grid = orc.make_grid(modes, eps, "single")
    M = 200_000
    pts = orc.gen_points("rand", M, grid, 1, np.float32)
    c = orc.gen_strengths(M, 1, np.complex64)
    op = orc.OraclePlan(1, modes, eps, "sm", "single", workers=orc.host_threads())
    op.set_points(pts)
    ref = op.execute(c)
    for method in ("sm", "gmsort", "gm"):
        p = nk.make_plan(1, modes, eps, method, "single")
        p.set_points(pts)
        assert orc.rel_l2_error(p.execute(c), ref) < 2e-6


def test_c2_geometry_type2_vs_oracle(nk, orc):
    """BASELINE C2 geometry (N=1024^2, n=2048^2, f32, eps 1e-5) at M=1e6."""
    modes, eps = (1024, 1024), 1e-5
    grid = orc.make_grid(modes, eps, "single")
    M = 1_000_000
    pts = orc.gen_points("rand", M, grid, 2, np.float32)
    f = orc.gen_strengths(int(np.prod(modes)), 2, np.complex64).reshape(modes[::-1])
    op = orc.OraclePlan(2, modes, eps, "gmsort", "single", workers=orc.host_threads())
    op.set_points(pts)
    ref = op.execute(f)
    for method in ("gmsort", "sm", "gm"):
        p = nk.make_plan(2, modes, eps, method, "single")
        p.set_points(pts)
        assert orc.rel_l2_error(p.execute(f), ref) < 2e-6


def test_torch_device_path(nk, orc):
    import torch
    modes, eps = (40, 36), 1e-9
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points("rand", 4096, grid, 3)
    c = orc.gen_strengths(4096, 3)
    dev = torch.device("cuda")
    p = nk.make_plan(1, modes, eps)
    p.set_points(torch.from_numpy(pts[:, 0]).to(dev), torch.from_numpy(pts[:, 1]).to(dev))
    out = p.execute(torch.from_numpy(c).to(dev))
    assert out.is_cuda and tuple(out.shape) == (36, 40)
    assert orc.rel_l2_error(out.cpu().numpy(), orc.direct_type1(pts, c, modes)) < 10 * eps
    # the one-shot API
    f2 = nk.nufft2d1(pts[:, 0], pts[:, 1], c, modes, eps=eps)
    np.testing.assert_allclose(f2, out.cpu().numpy(), rtol=0, atol=1e-12 * np.abs(f2).max())
    cj = nk.nufft2d2(pts[:, 0], pts[:, 1], f2, eps=eps)
    assert orc.rel_l2_error(cj, orc.direct_type2(pts, f2, modes)) < 10 * eps


def test_errors_and_edge_cases(nk, orc):
    p = nk.make_plan(1, (16, 16), 1e-6)
    with pytest.raises(ValueError):
        p.execute(np.zeros(4, np.complex128))          # before set_points
    bad = np.zeros((10, 2))
    bad[7, 1] = np.nan
    with pytest.raises(ValueError, match="7"):
        p.set_points(bad)
    p.set_points(np.zeros((0, 2)))                     # M = 0 is legal
    assert np.all(p.execute(np.zeros(0, np.complex128)) == 0)
    p.set_points(np.zeros((3, 2)))
    with pytest.raises(ValueError):
        p.execute(np.zeros(4, np.complex128))          # length mismatch
    with pytest.raises(ValueError):
        nk.make_plan(1, (16,), 1e-6)
    with pytest.raises(ValueError):
        nk.make_plan(1, (16, 16), 2.0)
    with pytest.raises(ValueError):
        nk.make_plan(3, (16, 16), 1e-3)
    with pytest.warns(UserWarning):
        nk.make_plan(1, (16, 16), 1e-9, precision="single")
    # single point at the origin -> all-ones.  The reference's
    # own max deviation here is 1.458e-8 (> 10 eps); the bar is parity with it.
    p = nk.make_plan(1, (32, 32), 1e-9)
    p.set_points(np.zeros((1, 2)))
    f = p.execute(np.ones(1, np.complex128))
    op = orc.OraclePlan(1, (32, 32), 1e-9, "sm", "double")
    op.set_points(np.zeros((1, 2)))
    ref = op.execute(np.ones(1, np.complex128))
    assert np.abs(f - 1).max() <= max(1e-8, 1.01 * np.abs(ref - 1).max())
    assert np.abs(f.reshape(-1) - ref).max() < 1e-13
    # constant-mode input -> all-ones
    p = nk.make_plan(2, (8, 10, 6), 1e-9)
    pts = np.random.default_rng(0).uniform(-7, 7, (100, 3))
    p.set_points(pts)
    fm = np.zeros((6, 10, 8), np.complex128)
    fm[3, 5, 4] = 1.0
    assert np.abs(p.execute(fm) - 1).max() < 1e-8


def test_repeat_execute_and_reuse(nk, orc):
    """Plan reuse without re-sorting and repeat determinism
    within eps (GPU atomics reorder sums)."""
    modes, eps = (64, 48), 1e-9
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points("rand", 20000, grid, 4)
    p = nk.make_plan(1, modes, eps)
    p.set_points(pts)
    c1, c2 = orc.gen_strengths(20000, 1), orc.gen_strengths(20000, 2)
    a = p.execute(c1)
    b = p.execute(c2)
    a2 = p.execute(c1)
    assert orc.rel_l2_error(a2, a) < 1e-14
    lin = p.execute(2 * c1 - 3j * c2)
    assert orc.rel_l2_error(lin, 2 * a - 3j * b) < 1e-12


@pytest.mark.parametrize("dim,nufft_type,prec,method", [
    (2, 1, "single", "sm"), (2, 2, "single", "sm"), (3, 1, "single", "sm"),
    (3, 2, "double", "sm"), (2, 1, "double", "gmsort"), (3, 2, "single", "gm")])
def test_batched_execute_matches_single(nk, dim, nufft_type, prec, method):
    """n_trans = K (cufinufft ntransf; PAPER.md:220-223 reuse of one setpts):
    vector k of a batched execute equals a single-vector execute on the same
    points (same kernels, same order of operations up to float atomics)."""
    import torch
    rng = np.random.default_rng(11 + dim + nufft_type)
    modes = (24, 20) if dim == 2 else (12, 10, 14)
    M, K, eps = 3000, 3, 1e-6 if prec == "double" else 1e-5
    cdt = np.complex64 if prec == "single" else np.complex128
    x = rng.uniform(-np.pi, np.pi, (M, dim))
    if nufft_type == 1:
        inp = (rng.standard_normal((K, M)) + 1j * rng.standard_normal((K, M))).astype(cdt)
    else:
        shp = (K,) + modes[::-1]
        inp = (rng.standard_normal(shp) + 1j * rng.standard_normal(shp)).astype(cdt)
    pb = nk.make_plan(nufft_type, modes, eps, method, prec, n_trans=K)
    pb.set_points(x)
    outb = pb.execute(inp)
    ps = nk.make_plan(nufft_type, modes, eps, method, prec)
    ps.set_points(x)
    tol = 1e-12 if prec == "double" else 2e-5
    for k in range(K):
        ref = ps.execute(np.ascontiguousarray(inp[k]))
        assert outb[k].shape == ref.shape
        assert np.linalg.norm(outb[k] - ref) / np.linalg.norm(ref) < tol
    # device tensors, batched one-shot
    xs = [torch.from_numpy(np.ascontiguousarray(x[:, a])).cuda() for a in range(dim)]
    fn = getattr(nk, f"nufft{dim}d{nufft_type}")
    if nufft_type == 1:
        got = fn(*xs, torch.from_numpy(inp).cuda(), modes, eps=eps, method=method)
    else:
        got = fn(*xs, torch.from_numpy(inp).cuda(), eps=eps, method=method)
    assert got.shape == outb.shape
    assert np.linalg.norm(got.cpu().numpy() - outb) / np.linalg.norm(outb) < tol
    pb.destroy()
    ps.destroy()


@pytest.mark.parametrize("nufft_type", [1, 2])
def test_graph_replay_on_fixed_buffers(nk, orc, nufft_type):
    """execute() on the same device (in, out) pair is captured once into a
    CUDA graph and replayed: replays must see new input contents, a new
    output buffer or new points (graph invalidated by set_points)."""
    import torch
    dev = torch.device("cuda")
    modes, eps = (48, 40), 1e-9
    grid = orc.make_grid(modes, eps, "double")
    rng = np.random.default_rng(5)
    pts = orc.gen_points("rand", 5000, grid, 5)
    p = nk.make_plan(nufft_type, modes, eps, "sm")
    p.set_points(torch.from_numpy(pts).to(dev))
    shape_in = (5000,) if nufft_type == 1 else modes[::-1]
    x = lambda: (rng.standard_normal(shape_in) + 1j * rng.standard_normal(shape_in))
    a = x()
    inp = torch.from_numpy(a).to(dev)
    out = p.execute(inp)
    ref = out.clone()
    for _ in range(3):                       # direct, capture, replay
        p.execute(inp, out)
        assert torch.allclose(out, ref, rtol=1e-12, atol=1e-12 * ref.abs().max().item())
    b = x()
    inp.copy_(torch.from_numpy(b))           # same buffer, new contents
    p.execute(inp, out)
    direct = orc.direct_type1(pts, b, modes) if nufft_type == 1 else \
        orc.direct_type2(pts, b, modes)
    assert orc.rel_l2_error(out.cpu().numpy(), direct) < 10 * eps
    out2 = torch.empty_like(out)             # new output buffer
    p.execute(inp, out2)
    assert torch.equal(out2, out) or torch.allclose(out2, out, rtol=1e-13, atol=0)
    pts2 = orc.gen_points("cluster", 5000, grid, 6)
    p.set_points(torch.from_numpy(pts2).to(dev))   # same M, new points
    p.execute(inp, out)
    direct2 = orc.direct_type1(pts2, b, modes) if nufft_type == 1 else \
        orc.direct_type2(pts2, b, modes)
    assert orc.rel_l2_error(out.cpu().numpy(), direct2) < 10 * eps
    p.set_timing(True)
    p.execute(inp, out)
    st = p.stage_times()
    assert st["total"] > 0 and st["fft"] > 0
    p.set_timing(False)
    p.destroy()


def test_method_equivalence_spec2(nk, orc):
    """SPEC.md:572 acceptance 2: on 20 random instances (M = 1e4, mixed
    dims / distributions, double) GM, GM-sort and SM agree pairwise within
    1e-10 relative, for type 1 and type 2."""
    rng = np.random.default_rng(2024)
    for inst in range(20):
        dim = 2 if inst % 2 == 0 else 3
        dist = "rand" if inst % 4 < 2 else "cluster"
        modes = (32, 24) if dim == 2 else (12, 16, 10)
        eps = [1e-6, 1e-9, 1e-12][inst % 3]
        grid = orc.make_grid(modes, eps, "double")
        pts = orc.gen_points(dist, 10_000, grid, 100 + inst)
        c = orc.gen_strengths(10_000, inst)
        f = rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])
        for t, inp in ((1, c), (2, f)):
            outs = []
            for method in ("gm", "gmsort", "sm"):
                p = nk.make_plan(t, modes, eps, method, "double")
                p.set_points(pts)
                outs.append(p.execute(inp))
                p.destroy()
            for a in range(3):
                for b in range(a + 1, 3):
                    assert orc.rel_l2_error(outs[a], outs[b]) < 1e-10, (inst, t, a, b)


def test_spreading_structure_spec5(nk, st, orc):
    """SPEC.md:575 acceptance 5: a single point spreads onto exactly w^d
    nonzero cells; translating the point by h_1 shifts the grid by one cell
    (1e-13); a point next to the seam wraps periodically like the explicit
    image sum (the oracle's wrapped spread, 1e-12)."""
    for dim, modes in ((2, (20, 16)), (3, (10, 12, 8))):
        eps = 1e-9
        grid = orc.make_grid(modes, eps, "double")
        params = nk.select_kernel_params(eps, nk.GridSpec(modes, grid.fine), "double")
        w = params.w
        gs = nk.GridSpec(modes, grid.fine)
        x0 = np.full((1, dim), 0.3)
        one = np.ones(1, np.complex128)
        for method in ("gm", "sm"):
            if method == "gm":
                b0 = st.spread_gm(x0, one, params, gs)
            else:
                lay = st.bin_sort(x0, gs)
                subs = st.build_subproblems(lay, params)
                b0 = st.spread_sm(x0, lay, subs, one, params, gs)
            b0 = np.asarray(b0)
            assert np.count_nonzero(np.abs(b0) > 0) == w ** dim
        h1 = 2 * np.pi / grid.fine[0]
        x1 = x0.copy()
        x1[0, 0] += h1
        b0 = np.asarray(st.spread_gm(x0, one, params, gs))
        b1 = np.asarray(st.spread_gm(x1, one, params, gs))
        assert np.abs(np.roll(b0, 1, axis=-1) - b1).max() <= 1e-13 * np.abs(b0).max()
        # seam: the point sits half a cell from -pi; its footprint wraps
        xs = np.full((1, dim), -np.pi + 0.5 * h1)
        got = np.asarray(st.spread_gm(xs, one, params, gs))
        oparams = orc.select_kernel_params(eps, grid, "double")
        ref = np.asarray(orc.spread_gm(xs, one, oparams, grid)).reshape(got.shape)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
        assert np.count_nonzero(np.abs(got) > 0) == w ** dim


def test_two_stage_start_order_fallback(nk, orc):
    """When bin << bits(padded cells) | start would exceed 32 bits (here
    256^3 unit bins: 24 + 10 bits) setpts falls back to two stable sorts
    (start, then bin); results must match the GM-sort plan and the exported
    layout must stay the reference's bin-stable one."""
    modes, eps, M = (128, 128, 128), 1e-5, 20001   # odd M: scratch alignment
    grid = orc.make_grid(modes, eps, "single")
    pts = orc.gen_points("rand", M, grid, 9, np.float32)
    c = orc.gen_strengths(M, 9).astype(np.complex64)
    a = nk.make_plan(1, modes, eps, "sm", "single", bin_dims=(1, 1, 1))
    a.set_points(pts)
    b = nk.make_plan(1, modes, eps, "gmsort", "single")
    b.set_points(pts)
    fa, fb = a.execute(c), b.execute(c)
    assert orc.rel_l2_error(fa, fb) < 1e-5
    keys, counts, starts, perm = (t.cpu().numpy() for t in a.layout_tensors())
    lay = orc.bin_sort(pts, orc.GridSpec(modes, a.grid.fine), (1, 1, 1))
    assert np.array_equal(perm, lay.perm) and np.array_equal(starts, lay.starts)


@pytest.mark.parametrize("dist,eps", [("rand", 1e-12), ("cluster", 1e-9), ("rand", 1e-11)])
def test_xwin_interp_matches_per_thread_gather(nk, orc, dist, eps, monkeypatch):
    """3D double type 2 with w > 8 gathers by x-window groups (K7x: a warp
    serves up to 4 start-adjacent points from one read of each window cell).
    Must match the per-thread staged gather (K7s, NK_INTERP_NO_XWIN=1) to
    rounding, in both its start and its non-start visit orders, and direct
    sums (10 eps)."""
    modes, M = (24, 20, 16), 6000
    monkeypatch.setenv("NK_INTERP_NO_TILE", "1")   # K7x, not the tiled K7t
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points(dist, M, grid, 31, np.float64)
    rng = np.random.default_rng(5)
    f = rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])
    p = nk.make_plan(2, modes, eps, "sm", "double")
    p.set_points(pts)
    got = p.execute(f)
    monkeypatch.setenv("NK_INTERP_NO_XWIN", "1")
    q = nk.make_plan(2, modes, eps, "sm", "double")
    q.set_points(pts)
    ref = q.execute(f)
    assert orc.rel_l2_error(got, ref) < 1e-14
    # K7x on the K7s visit order (set_points without, execute with K7x)
    monkeypatch.delenv("NK_INTERP_NO_XWIN")
    assert orc.rel_l2_error(q.execute(f), ref) < 1e-14
    assert orc.rel_l2_error(got, orc.direct_type2(pts, f, modes)) < 10 * eps


@pytest.mark.parametrize("dist,eps,bins", [("rand", 1e-12, None), ("cluster", 1e-9, None),
                                           ("rand", 1e-11, (5, 3, 7)), ("gauss", 1e-15, None),
                                           ("rand", 1e-8, (6, 6, 2))])
def test_tiled_spread_matches_plane_spread(nk, orc, dist, eps, bins, monkeypatch):
    """3D double type 1 with w >= 9 spreads through tile-group register
    windows (K6t: setpts orders each bin tile-major, a CTA of 16 plane warps
    accumulates every point of a start tile in registers).  Must match the
    plane-owned x-window spread (K6c, NK_SPREAD_NO_TILE=1) to rounding -- with
    odd user bins (partial tiles, edge bins), clustered points and w = 9 / 16
    (tile 8 / 1) -- and direct sums (10 eps)."""
    modes, M = (24, 20, 16), 7001
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points(dist, M, grid, 33, np.float64)
    c = orc.gen_strengths(M, 3)
    kw = {} if bins is None else {"bin_dims": bins}
    p = nk.make_plan(1, modes, eps, "sm", "double", **kw)
    p.set_points(pts)
    got = p.execute(c)
    monkeypatch.setenv("NK_SPREAD_NO_TILE", "1")
    q = nk.make_plan(1, modes, eps, "sm", "double", **kw)
    q.set_points(pts)
    ref = q.execute(c)
    assert orc.rel_l2_error(got, ref) < 1e-14
    # the exported layout stays the reference's bin-stable one
    keys, counts, starts, perm = (t.cpu().numpy() for t in p.layout_tensors())
    lay = orc.bin_sort(pts, orc.GridSpec(modes, p.grid.fine), p.bin_dims)
    assert np.array_equal(perm, lay.perm) and np.array_equal(starts, lay.starts)
    assert orc.rel_l2_error(got, orc.direct_type1(pts, c, modes)) < max(10 * eps, 1e-13)


@pytest.mark.parametrize("dist,eps,bins", [("rand", 1e-12, None), ("cluster", 1e-9, None),
                                           ("rand", 1e-11, (5, 3, 7)), ("gauss", 1e-15, None),
                                           ("rand", 1e-8, (6, 6, 2))])
def test_tiled_interp_matches_xwin(nk, orc, dist, eps, bins, monkeypatch):
    """3D double type 2 with w >= 9 interpolates per tile group on the FP64
    tensor cores (K7t: the adjoint of K6t).  Must match the x-window group
    gather (K7x, NK_INTERP_NO_TILE=1) to rounding, with odd user bins
    (partial tiles, edge bins), clustered points and w = 9 / 16, and direct
    sums (10 eps)."""
    modes, M = (24, 20, 16), 7001
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points(dist, M, grid, 35, np.float64)
    rng = np.random.default_rng(6)
    f = rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])
    kw = {} if bins is None else {"bin_dims": bins}
    p = nk.make_plan(2, modes, eps, "sm", "double", **kw)
    p.set_points(pts)
    got = p.execute(f)
    monkeypatch.setenv("NK_INTERP_NO_TILE", "1")
    q = nk.make_plan(2, modes, eps, "sm", "double", **kw)
    q.set_points(pts)
    ref = q.execute(f)
    assert orc.rel_l2_error(got, ref) < 1e-14
    assert orc.rel_l2_error(got, orc.direct_type2(pts, f, modes)) < max(10 * eps, 1e-13)


@pytest.mark.parametrize("modes", [(128, 96), (512, 300), (1024, 40)])
def test_fused_pad_rowfft_type2(nk, orc, modes, monkeypatch):
    """2D single-precision type 2 with n_1 = 2^L runs K9 fused with the row
    FFTs (own Stockham radix-8 kernel) + a cuFFT column plan.  Must match
    direct sums (10 eps) and the unfused pad + 2D cuFFT path."""
    eps, M = 1e-5, 4000
    grid = orc.make_grid(modes, eps, "single")
    assert grid.fine[0] & (grid.fine[0] - 1) == 0
    pts = orc.gen_points("rand", M, grid, 21, np.float32)
    rng = np.random.default_rng(3)
    f = (rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1]))
    f = f.astype(np.complex64)
    p = nk.make_plan(2, modes, eps, "sm", "single")
    p.set_points(pts)
    got = p.execute(f)
    monkeypatch.setenv("NK_FUSED_ROWS", "0")
    q = nk.make_plan(2, modes, eps, "sm", "single")
    q.set_points(pts)
    ref = q.execute(f)
    assert orc.rel_l2_error(got, ref) < 2e-6
    if int(np.prod(modes)) * M <= 4e8:
        assert orc.rel_l2_error(got, orc.direct_type2(pts.astype(np.float64), f, modes)) < 10 * eps


@pytest.mark.parametrize("modes", [(128, 96), (256, 256), (1024, 40)])
def test_fused_rowfft_deconv_type1(nk, orc, modes, monkeypatch):
    """2D single-precision type 1 with n_1 = 2^L: cuFFT column pass, then
    the forward row FFTs fused with K8 (own kernel).  Must match direct
    sums (10 eps) and the unfused 2D cuFFT + deconvolution path."""
    eps, M = 1e-5, 4000
    grid = orc.make_grid(modes, eps, "single")
    pts = orc.gen_points("rand", M, grid, 22, np.float32)
    c = orc.gen_strengths(M, 22).astype(np.complex64)
    p = nk.make_plan(1, modes, eps, "sm", "single")
    p.set_points(pts)
    got = p.execute(c)
    monkeypatch.setenv("NK_FUSED_ROWS", "0")
    q = nk.make_plan(1, modes, eps, "sm", "single")
    q.set_points(pts)
    ref = q.execute(c)
    assert orc.rel_l2_error(got, ref) < 2e-6
    if int(np.prod(modes)) * M <= 4e8:
        assert orc.rel_l2_error(got, orc.direct_type1(pts.astype(np.float64), c, modes)) < 10 * eps


@pytest.mark.parametrize("modes,prec", [((256, 200), "single"), ((48, 40), "double"),
                                         ((16, 12, 10), "single")])
def test_fft_deconvolve_stage_matches_execute(nk, orc, modes, prec):
    """The fused type-1 back half exposed for the sharded path
    (nk_fft_deconv_type1 / plan.fft_deconvolve_to) equals spread + FFT +
    deconvolution as separate stages and the plan's execute."""
    import torch
    eps = 1e-5 if prec == "single" else 1e-9
    grid = orc.make_grid(modes, eps, prec)
    rdt = np.float32 if prec == "single" else np.float64
    pts = orc.gen_points("rand", 3000, grid, 31, rdt)
    c = orc.gen_strengths(3000, 31).astype(np.complex64 if prec == "single" else np.complex128)
    p = nk.make_plan(1, modes, eps, "sm", prec)
    p.set_points(torch.from_numpy(pts).cuda())
    cd = torch.from_numpy(c).cuda()
    ref = p.execute(cd)
    fine = p.new_fine_grid()
    p.spread_to(cd, fine)
    out = torch.empty_like(ref)
    p.fft_deconvolve_to(fine, out)
    fine2 = p.new_fine_grid()
    p.spread_to(cd, fine2)
    p.fft_(fine2, -1)
    out2 = torch.empty_like(ref)
    p.deconvolve_to(fine2, out2)
    tol = 2e-6 if prec == "single" else 1e-13
    assert orc.rel_l2_error(out.cpu().numpy(), ref.cpu().numpy()) < tol
    assert orc.rel_l2_error(out2.cpu().numpy(), ref.cpu().numpy()) < tol


@pytest.mark.parametrize("modes,prec,eps,dist", [((24, 20, 16), "double", 1e-12, "rand"),
                                                 ((24, 20, 16), "double", 1e-12, "cluster"),
                                                 ((20, 20, 20), "single", 1e-6, "rand"),
                                                 ((64, 48), "single", 1e-5, "cluster"),
                                                 ((64, 48), "double", 1e-9, "rand")])
def test_deterministic_type1_bit_identical(nk, orc, modes, prec, eps, dist):
    """deterministic=True: SM type-1 plans merge their padded
    bins one colour class of non-overlapping bins per launch, so repeated
    executes -- and a second plan on the same points -- are bit-identical,
    and equal the default plan to rounding."""
    grid = orc.make_grid(modes, eps, prec)
    rdt = np.float32 if prec == "single" else np.float64
    cdt = np.complex64 if prec == "single" else np.complex128
    M = 40000
    pts = orc.gen_points(dist, M, grid, 61, rdt)
    c = orc.gen_strengths(M, 62, cdt)
    p = nk.make_plan(1, modes, eps, "sm", prec, deterministic=True)
    p.set_points(pts)
    outs = [np.asarray(p.execute(c)).copy() for _ in range(3)]
    q = nk.make_plan(1, modes, eps, "sm", prec, deterministic=True)
    q.set_points(pts)
    outs.append(np.asarray(q.execute(c)))
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint8), outs[0].view(np.uint8))
    r = nk.make_plan(1, modes, eps, "sm", prec)
    r.set_points(pts)
    tol = 1e-6 if prec == "single" else 1e-13
    assert orc.rel_l2_error(outs[0], r.execute(c)) < tol
