"""GPU parity at the BASELINE.json geometries (C1-C5) with the plans'
B200-tuned bins, plus odd mode counts and the widest fused row FFT.

Bars (binsort.py:134-219):
  * bin keys / counts / starts / perm / subproblem table bit-exact against
    the oracle's restatement of binsort.py at the plan's own bin dims;
  * transforms: rel l2 <= 10 eps against compensated direct sums (on
    sampled modes / points where the full sum is out of reach) and against
    the oracle pipeline at eps-level (1e-12 double; single precision is
    gated on the reference's own float32-accumulation error, see
    _single_gate).

The type-1 direct checks use the full point set for the plan (sort,
subproblems, spread all run at the BASELINE size) but strengths that are
zero outside the first ``m_direct`` points, so the compensated direct sum
over those points is the exact answer.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2102_08463_b200 as nk
    return nk


def _sorted_layout_matches(nk, orc, plan, pts, modes):
    """Bit-exact bin sort + subproblems of ``plan`` vs the oracle."""
    keys, counts, starts, perm = (t.cpu().numpy() for t in plan.layout_tensors())
    grid = orc.GridSpec(modes, plan.grid.fine)
    lay = orc.bin_sort(pts, grid, plan.bin_dims)
    assert np.array_equal(keys, lay.point_bins)
    assert np.array_equal(counts, lay.counts)
    assert np.array_equal(starts, lay.starts)
    assert np.array_equal(perm, lay.perm)
    if plan.method == "sm":
        b, s0, s1, off, pad = (t.cpu().numpy() for t in plan.subproblem_tensors())
        params = orc.select_kernel_params(plan.params.epsilon, grid, plan.precision)
        ref = orc.build_subproblems(lay, params, plan.max_subproblem)
        assert np.array_equal(b, ref.bin_ids)
        assert np.array_equal(s0, ref.slice_starts) and np.array_equal(s1, ref.slice_stops)
        assert np.array_equal(off, ref.offsets) and np.array_equal(pad, ref.padded_dims)


def _sample_kvecs(modes, n, seed):
    rng = np.random.default_rng(seed)
    cols = [rng.integers(-(N // 2), N - N // 2, n) for N in modes]
    kv = np.stack(cols, axis=1).astype(np.int64)
    # always include the corners (largest |k|, where the deconvolution is largest)
    corners = np.array([[-(N // 2) for N in modes], [N - N // 2 - 1 for N in modes]], np.int64)
    return np.concatenate([corners, kv])


def _modes_at(out, modes, kv):
    idx = tuple(kv[:, a] + modes[a] // 2 for a in range(len(modes) - 1, -1, -1))
    return np.asarray(out)[idx]


def _type1_direct_check(nk, orc, plan, pts, modes, cdt, m_direct, eps, n_modes=400, seed=1):
    M = pts.shape[0]
    c = np.zeros(M, cdt)
    c[:m_direct] = orc.gen_strengths(m_direct, seed, cdt)
    out = plan.execute(c)
    kv = _sample_kvecs(modes, n_modes, seed)
    ref = orc.direct_type1_at(pts[:m_direct].astype(np.float64), c[:m_direct], kv)
    return orc.rel_l2_error(_modes_at(out, modes, kv), ref)


def _type2_direct_check(nk, orc, plan, pts, modes, f, n_pts=64, seed=2):
    out = plan.execute(f)
    idx = np.random.default_rng(seed).choice(pts.shape[0], n_pts, replace=False)
    ref = orc.direct_type2(pts[idx].astype(np.float64), f, modes)
    return orc.rel_l2_error(np.asarray(out)[idx], ref)


# ---------------------------------------------------------------- C4

@pytest.mark.parametrize("nufft_type", [1, 2])
def test_c4_geometry_sort(nk, orc, nufft_type):
    """C4 (N=256^3, n=512^3, eps 1e-12, f64) with the default tuned bins and
    the tile-major start order of the tiled spread / interp.  1.5e6 uniform
    points; the exported layout must equal binsort.py's bit for bit."""
    modes, eps, M = (256, 256, 256), 1e-12, 1_500_001   # odd M on purpose
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points("rand", M, grid, 40 + nufft_type)
    p = nk.make_plan(nufft_type, modes, eps, "sm", "double")
    p.set_points(pts)
    _sorted_layout_matches(nk, orc, p, pts, modes)
    p.destroy()


@pytest.mark.parametrize("nufft_type", [1, 2])
def test_composite_key_uses_32_bits(nk, orc, nufft_type):
    """N=256^3 (n=512^3) single precision, eps 1e-6, bins 4 x 4 x 4: 2^21
    bins x 12^3 padded-bin start cells, so the composite (bin, start) sort
    key uses all 32 bits (sign bit included).  The exported layout must
    equal binsort.py's bit for bit and the transform the GM-sort plan's."""
    modes, eps, M = (256, 256, 256), 1e-6, 1_000_001
    grid = orc.make_grid(modes, eps, "single")
    pts = orc.gen_points("rand", M, grid, 50 + nufft_type, np.float32)
    p = nk.make_plan(nufft_type, modes, eps, "sm", "single", bin_dims=(4, 4, 4))
    nb = int(np.prod([(n + m - 1) // m for n, m in zip(p.grid.fine, p.bin_dims)]))
    cells = int(np.prod([m + 2 * p.params.halo for m in p.bin_dims]))
    assert (nb - 1).bit_length() + (cells - 1).bit_length() == 32
    p.set_points(pts)
    _sorted_layout_matches(nk, orc, p, pts, modes)
    q = nk.make_plan(nufft_type, modes, eps, "gmsort", "single")
    q.set_points(pts)
    rng = np.random.default_rng(nufft_type)
    if nufft_type == 1:
        inp = orc.gen_strengths(M, 3).astype(np.complex64)
    else:
        inp = (rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])
               ).astype(np.complex64)
    assert orc.rel_l2_error(p.execute(inp), q.execute(inp)) < 1e-5
    p.destroy()
    q.destroy()


def test_c4_geometry_transforms(nk, orc):
    """C4 geometry, 1e6 uniform points: type 1 (sampled modes) and type 2
    (sampled points) within 10 eps of compensated direct sums."""
    modes, eps, M = (256, 256, 256), 1e-12, 1_000_000
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points("rand", M, grid, 44)
    p1 = nk.make_plan(1, modes, eps, "sm", "double")
    p1.set_points(pts)
    e1 = _type1_direct_check(nk, orc, p1, pts, modes, np.complex128, 100_000, eps)
    p1.destroy()
    assert e1 < 10 * eps, e1
    rng = np.random.default_rng(3)
    f = rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])
    p2 = nk.make_plan(2, modes, eps, "sm", "double")
    p2.set_points(pts)
    e2 = _type2_direct_check(nk, orc, p2, pts, modes, f)
    p2.destroy()
    assert e2 < 10 * eps, e2


def test_c4_geometry_vs_oracle_pipeline(nk, orc):
    """C4 geometry (512^3 fine grid, w = 13), 2e5 points: type 1 and type 2
    against the oracle's full pipeline (reference SM spread / GM-sort
    interp + FFT + deconvolution) to 1e-12."""
    modes, eps, M = (256, 256, 256), 1e-12, 200_000
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points("rand", M, grid, 45)
    c = orc.gen_strengths(M, 45)
    op = orc.OraclePlan(1, modes, eps, "sm", "double", workers=orc.host_threads())
    op.set_points(pts)
    ref1 = op.execute(c)
    del op
    p1 = nk.make_plan(1, modes, eps, "sm", "double")
    p1.set_points(pts)
    assert orc.rel_l2_error(p1.execute(c), ref1) < 1e-12
    p1.destroy()
    del ref1
    rng = np.random.default_rng(4)
    f = rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])
    op = orc.OraclePlan(2, modes, eps, "gmsort", "double", workers=orc.host_threads())
    op.set_points(pts)
    ref2 = op.execute(f)
    del op
    p2 = nk.make_plan(2, modes, eps, "sm", "double")
    p2.set_points(pts)
    assert orc.rel_l2_error(p2.execute(f), ref2) < 1e-12
    p2.destroy()


# ---------------------------------------------------------------- C5

def test_c5_geometry(nk, orc):
    """C5 (N=128^3, n=256^3, w=13, f64), full M=1e7 uniform: sort and
    subproblems bit-exact for the type-1 and type-2 plans; type 2 then type
    1 (the M-TIP pair) within 10 eps of direct sums."""
    modes, eps, M = (128, 128, 128), 1e-12, 10_000_000
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points("rand", M, grid, 50)
    rng = np.random.default_rng(5)
    f = rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])
    p2 = nk.make_plan(2, modes, eps, "sm", "double")
    p2.set_points(pts)
    assert p2.params.w == 13
    _sorted_layout_matches(nk, orc, p2, pts, modes)
    e2 = _type2_direct_check(nk, orc, p2, pts, modes, f, n_pts=128)
    p2.destroy()
    assert e2 < 10 * eps, e2
    p1 = nk.make_plan(1, modes, eps, "sm", "double")
    p1.set_points(pts)
    _sorted_layout_matches(nk, orc, p1, pts, modes)
    e1 = _type1_direct_check(nk, orc, p1, pts, modes, np.complex128, 200_000, eps)
    p1.destroy()
    assert e1 < 10 * eps, e1


def test_c5_geometry_vs_oracle_pipeline(nk, orc):
    """C5 geometry at M=1e6: both transforms against the oracle pipeline."""
    modes, eps, M = (128, 128, 128), 1e-12, 1_000_000
    grid = orc.make_grid(modes, eps, "double")
    pts = orc.gen_points("rand", M, grid, 51)
    c = orc.gen_strengths(M, 51)
    rng = np.random.default_rng(6)
    f = rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])
    for t, inp, method in ((1, c, "sm"), (2, f, "gmsort")):
        op = orc.OraclePlan(t, modes, eps, method, "double", workers=orc.host_threads())
        op.set_points(pts)
        ref = op.execute(inp)
        p = nk.make_plan(t, modes, eps, "sm", "double")
        p.set_points(pts)
        assert orc.rel_l2_error(p.execute(inp), ref) < 1e-12, t
        p.destroy()


# ---------------------------------------------------------------- C3

def _single_gate(err_gpu, err_ref, eps):
    """Single precision: 10 eps, or -- where the reference's own
    float32 grid accumulation already misses it (clustered points pile
    ~1e3-1e6 float32 additions onto each cell) -- no worse than 2x the
    reference's error on the same inputs."""
    return err_gpu < max(10 * eps, 2 * err_ref)


@pytest.mark.parametrize("dist", ["cluster", "gauss"])
def test_c3_geometry_full_m(nk, orc, dist):
    """C3a / C3b (N=128^3, n=256^3, eps 1e-6, f32, the 4x4x4 tuned bins),
    full M=1e7: sort + subproblems bit-exact; type 1 vs the oracle pipeline
    and vs direct sums (strengths on the first 1e5 points)."""
    modes, eps, M = (128, 128, 128), 1e-6, 10_000_000
    grid = orc.make_grid(modes, eps, "single")
    pts = orc.gen_points(dist, M, grid, 30, np.float32)
    p = nk.make_plan(1, modes, eps, "sm", "single")
    assert p.bin_dims == (4, 4, 4)
    p.set_points(pts)
    _sorted_layout_matches(nk, orc, p, pts, modes)
    # against direct sums
    m_direct = 100_000
    c = np.zeros(M, np.complex64)
    c[:m_direct] = orc.gen_strengths(m_direct, 30, np.complex64)
    got = p.execute(c)
    kv = _sample_kvecs(modes, 400, 30)
    direct = orc.direct_type1_at(pts[:m_direct].astype(np.float64), c[:m_direct], kv)
    op = orc.OraclePlan(1, modes, eps, "sm", "single", workers=orc.host_threads())
    op.set_points(pts)
    ref = op.execute(c)
    e_gpu = orc.rel_l2_error(_modes_at(got, modes, kv), direct)
    e_ref = orc.rel_l2_error(_modes_at(np.asarray(ref).reshape(got.shape), modes, kv), direct)
    assert _single_gate(e_gpu, e_ref, eps), (e_gpu, e_ref)
    # against the oracle pipeline with strengths on every point
    call = orc.gen_strengths(M, 31, np.complex64)
    ref = op.execute(call)
    got = p.execute(call)
    assert orc.rel_l2_error(got, ref) < 10 * eps
    p.destroy()


@pytest.mark.parametrize("dist", ["rand", "gauss"])
def test_c3_geometry_type2_full_m(nk, orc, dist):
    """3D f32 type 2 at C3 size (128^3, M=1e7, eps 1e-6, 16x16x4 bins):
    sort bit-exact; sampled points within 10 eps of direct sums; full output
    vs the oracle's GM-sort interp pipeline."""
    modes, eps, M = (128, 128, 128), 1e-6, 10_000_000
    grid = orc.make_grid(modes, eps, "single")
    pts = orc.gen_points(dist, M, grid, 32, np.float32)
    rng = np.random.default_rng(7)
    f = (rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1]))
    f = f.astype(np.complex64)
    p = nk.make_plan(2, modes, eps, "sm", "single")
    p.set_points(pts)
    _sorted_layout_matches(nk, orc, p, pts, modes)
    assert _type2_direct_check(nk, orc, p, pts, modes, f, n_pts=128) < 10 * eps
    op = orc.OraclePlan(2, modes, eps, "gmsort", "single", workers=orc.host_threads())
    op.set_points(pts)
    assert orc.rel_l2_error(p.execute(f), op.execute(f)) < 10 * eps
    p.destroy()


# ---------------------------------------------------------------- C1 / C2 at full M

def test_c1_geometry_full_m(nk, orc):
    """C1 (N=256^2, f32, eps 1e-5) at the BASELINE M=1e6: every method vs
    the oracle pipeline; the SM plan's sort bit-exact."""
    modes, eps, M = (256, 256), 1e-5, 1_000_000
    grid = orc.make_grid(modes, eps, "single")
    pts = orc.gen_points("rand", M, grid, 1, np.float32)
    c = orc.gen_strengths(M, 1, np.complex64)
    op = orc.OraclePlan(1, modes, eps, "sm", "single", workers=orc.host_threads())
    op.set_points(pts)
    ref = op.execute(c)
    for method in ("sm", "gmsort", "gm"):
        p = nk.make_plan(1, modes, eps, method, "single")
        p.set_points(pts)
        if method != "gm":
            _sorted_layout_matches(nk, orc, p, pts, modes)
        assert orc.rel_l2_error(p.execute(c), ref) < 2e-6, method
        p.destroy()
    p = nk.make_plan(1, modes, eps, "sm", "single")
    p.set_points(pts)
    assert _type1_direct_check(nk, orc, p, pts, modes, np.complex64, 50_000, eps) < 10 * eps


def test_c2_geometry_full_m(nk, orc):
    """C2 (N=1024^2, n=2048^2, f32, eps 1e-5) at the BASELINE M=1e7: SM,
    GM-sort and GM vs the oracle's GM-sort interp pipeline; sampled points
    vs direct sums."""
    modes, eps, M = (1024, 1024), 1e-5, 10_000_000
    grid = orc.make_grid(modes, eps, "single")
    pts = orc.gen_points("rand", M, grid, 2, np.float32)
    f = orc.gen_strengths(int(np.prod(modes)), 2, np.complex64).reshape(modes[::-1])
    op = orc.OraclePlan(2, modes, eps, "gmsort", "single", workers=orc.host_threads())
    op.set_points(pts)
    ref = op.execute(f)
    for method in ("sm", "gmsort", "gm"):
        p = nk.make_plan(2, modes, eps, method, "single")
        p.set_points(pts)
        if method == "sm":
            _sorted_layout_matches(nk, orc, p, pts, modes)
            assert _type2_direct_check(nk, orc, p, pts, modes, f, n_pts=64) < 10 * eps
        assert orc.rel_l2_error(p.execute(f), ref) < 2e-6, method
        p.destroy()


# ---------------------------------------------------------------- odd N, wide fused rows

@pytest.mark.parametrize("modes", [(33, 17), (9, 11, 7), (31, 1), (1, 5, 3)])
@pytest.mark.parametrize("prec", ["single", "double"])
@pytest.mark.parametrize("method", ["gm", "gmsort", "sm"])
def test_odd_mode_counts(nk, orc, modes, prec, method):
    """Odd N: the centered ordering -floor(N/2) .. ceil(N/2)-1 (
    kernel.py:176-178) for both types and every method, vs direct sums."""
    eps = 1e-5 if prec == "single" else 1e-10
    grid = orc.make_grid(modes, eps, prec)
    rdt = np.float32 if prec == "single" else np.float64
    cdt = np.complex64 if prec == "single" else np.complex128
    M = 2001
    pts = orc.gen_points("rand", M, grid, 60 + len(modes), rdt)
    c = orc.gen_strengths(M, 60, cdt)
    rng = np.random.default_rng(61)
    f = (rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1])).astype(cdt)
    p1 = nk.make_plan(1, modes, eps, method, prec)
    p1.set_points(pts)
    fk = p1.execute(c)
    assert fk.shape == tuple(modes[::-1])
    assert orc.rel_l2_error(fk, orc.direct_type1(pts, c, modes)) < 10 * eps
    p2 = nk.make_plan(2, modes, eps, method, prec)
    p2.set_points(pts)
    assert orc.rel_l2_error(p2.execute(f), orc.direct_type2(pts, f, modes)) < 10 * eps


@pytest.mark.parametrize("nufft_type", [1, 2])
def test_fused_rows_n1_4096(nk, orc, nufft_type, monkeypatch):
    """The widest fused row FFT (n_1 = 4096: N_1 = 2048): matches direct sums
    (10 eps) and the unfused cuFFT path."""
    modes, eps, M = (2048, 40), 1e-5, 3000
    grid = orc.make_grid(modes, eps, "single")
    assert grid.fine[0] == 4096
    pts = orc.gen_points("rand", M, grid, 70, np.float32)
    rng = np.random.default_rng(71)
    if nufft_type == 1:
        inp = orc.gen_strengths(M, 70, np.complex64)
        direct = orc.direct_type1(pts, inp, modes)
    else:
        inp = (rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1]))
        inp = inp.astype(np.complex64)
        direct = orc.direct_type2(pts, inp, modes)
    p = nk.make_plan(nufft_type, modes, eps, "sm", "single")
    p.set_points(pts)
    got = p.execute(inp)
    monkeypatch.setenv("NK_FUSED_ROWS", "0")
    q = nk.make_plan(nufft_type, modes, eps, "sm", "single")
    q.set_points(pts)
    ref = q.execute(inp)
    assert orc.rel_l2_error(got, ref) < 2e-6
    assert orc.rel_l2_error(got, direct) < 10 * eps
