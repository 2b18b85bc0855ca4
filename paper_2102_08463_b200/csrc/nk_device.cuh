// Device helpers: the exact FP64 fold, the ES kernel, complex atomics.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "nk_es_poly.h"
#include "nk_internal.cuh"

// binsort.py:98-100 grid_coords with numpy remainder semantics, bit-exact:
// r = fmod(x + pi, 2 pi); r < 0 -> r + 2 pi; r == 0 -> +0.0; v = r * (n / 2 pi).
// Explicit _rn intrinsics keep nvcc from contracting into FMAs.
__device__ __forceinline__ double nk_fold(double x, double scale) {
    double a = __dadd_rn(x, NK_PI);
    double r;
    // fast paths, bit-identical to fmod: fmod(a, 2 pi) == a for 0 <= a < 2 pi;
    // for 2 pi <= a < 4 pi it is a - 2 pi, exact by Sterbenz's lemma; for
    // -2 pi <= a < 0 it is a and numpy adds 2 pi (rounded, like below)
    if (a >= 0.0 && a < NK_TWO_PI) {
        r = a;
    } else if (a >= NK_TWO_PI && a < 2.0 * NK_TWO_PI) {
        r = __dsub_rn(a, NK_TWO_PI);
    } else {
        r = fmod(a, NK_TWO_PI);
    }
    if (r != 0.0) {
        if (r < 0.0) r = __dadd_rn(r, NK_TWO_PI);
    } else {
        r = 0.0;
    }
    return __dmul_rn(r, scale);
}

// binsort.py:126-128: cell = clamp(floor(v), 0, n-1).  v is finite here.
__device__ __forceinline__ int nk_cell(double v, int n) {
    double f = floor(v);
    int c = f >= (double)(n - 1) ? n - 1 : (int)f;
    return c < 0 ? 0 : c;
}

// ES kernel exp(beta (sqrt(1 - z^2) - 1)) on |z| <= 1 (_kernels.py:20-26).
// Single precision uses exp2 with beta*log2(e) folded in (one MUFU.EX2);
// double uses the accurate libdevice exp.
// Single precision: MUFU.SQRT / MUFU.EX2 directly (sqrt.approx, ex2.approx:
// ~1-2 ulp, no slow-path branches); the exponent lies in [-beta log2 e, 0].
__device__ __forceinline__ float nk_sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float nk_ex2_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float nk_es(float z, const Geom &g) {
    // |z| <= 1 on every footprint cell (start = ceil(u - w/2)); the clamp
    // only absorbs rounding at z = +-1, where the value is exp(-beta).
    const float t = fmaxf(fmaf(-z, z, 1.0f), 0.0f);
    return nk_ex2_approx(fmaf(g.betaf_log2e, nk_sqrt_approx(t), -g.betaf_log2e));
}
__device__ __forceinline__ double nk_es(double z, const Geom &g) {
    double t = 1.0 - z * z;
    return t >= 0.0 ? exp(g.beta * (sqrt(t) - 1.0)) : 0.0;
}

template <typename T> __device__ __forceinline__ T nk_ceil(T x);
template <> __device__ __forceinline__ float nk_ceil<float>(float x) { return ceilf(x); }
template <> __device__ __forceinline__ double nk_ceil<double>(double x) { return ceil(x); }

// Kernel row for one axis: local coordinate u (relative to the bin corner),
// returns the local start cell ceil(u - w/2) (_kernels.py:43-46) and fills
// ker[r] = phi((start + r - u) * 2/w) (_kernels.py:29-33).
// Single precision: the interior pieces r = 1..w-2 are Horner polynomials in
// s = 2 (start - u) + w - 1 with compile-time coefficients (nk_es_poly.h,
// FFMA with immediate operands, no MUFU); the two edge pieces, which touch
// the sqrt branch point at z = -1 / +1, keep the exact exp/sqrt path.
template <typename T, int W>
__device__ __forceinline__ int nk_kernel_row(T u, const Geom &g, T *ker) {
    const T st = nk_ceil<T>(u - (T)(0.5 * W));
    if constexpr (sizeof(T) == 4 && W >= 3) {
        const float d = st - u;
        const float z0 = d * (2.0f / W);
        ker[0] = nk_es(z0, g);
        ker[W - 1] = nk_es(z0 + (float)(2.0 * (W - 1) / W), g);
        const float s = fmaf(2.0f, d, (float)(W - 1));
        typedef EsPoly<W> P;
#pragma unroll
        for (int r = 1; r < W - 1; ++r) {
            float p = P::c(r - 1, P::D);
#pragma unroll
            for (int k = P::D - 1; k >= 0; --k) p = fmaf(p, s, P::c(r - 1, k));
            ker[r] = p;
        }
    } else {
        const T z0 = (st - u) * (T)(2.0 / W);
#pragma unroll
        for (int r = 0; r < W; ++r) ker[r] = nk_es(z0 + (T)(2.0 * r / W), g);
    }
    return (int)st;
}

// Double-precision kernel row from the degree-14 interior pieces
// (EsPoly64, nk_es_poly.h: max abs error 6e-15 against the exact kernel)
// and the exact exp/sqrt path for the two edge pieces.  Same contract as
// nk_kernel_row: returns the local start cell ceil(u - w/2).
template <int W>
__device__ __forceinline__ int nk_kernel_row_poly(double u, const Geom &g, double *ker) {
    const double st = ceil(u - 0.5 * W);
    const double d = st - u;
    const double z0 = d * (2.0 / W);
    ker[0] = nk_es(z0, g);
    ker[W - 1] = nk_es(z0 + (2.0 * (W - 1) / W), g);
    const double s = fma(2.0, d, (double)(W - 1));
    typedef EsPoly64<W> P;
#pragma unroll
    for (int r = 1; r < W - 1; ++r) {
        double p = P::c(r - 1, P::D);
#pragma unroll
        for (int k = P::D - 1; k >= 0; --k) p = fma(p, s, P::c(r - 1, k));
        ker[r] = p;
    }
    return (int)st;
}

// FP64 tensor-core MMA (DMMA.8x8x4): C[8x8] += A[8x4] B[4x8], row-major A,
// column-major B.  Lane l holds A[l / 4][l % 4], B[l % 4][l / 4] and
// C[l / 4][2 (l % 4) + {0, 1}].  B200 runs it at the FP64 peak (63 FMA / clk /
// SM measured, scripts/dmma_peak.cu) for 1/8 of the issue slots of DFMA.
__device__ __forceinline__ void nk_dmma(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// ---- TMA bulk copies + mbarriers (sm_90+/sm_100 async proxy) ----------
__device__ __forceinline__ uint32_t nk_smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void nk_mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(nk_smem_u32(bar)), "r"(count)
                 : "memory");
}
// make the initialised barriers visible to the async (TMA) proxy
__device__ __forceinline__ void nk_fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order this thread's earlier generic-proxy shared accesses (made visible to
// it by a barrier) before its subsequent async-proxy (TMA) writes
__device__ __forceinline__ void nk_fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void nk_mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(nk_smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// 1D TMA bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completion counted in bytes on the mbarrier (UBLKCP)
__device__ __forceinline__ void nk_bulk_g2s(void *dst, const void *src, unsigned bytes,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            nk_smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(nk_smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void nk_mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "NK_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra NK_WAIT_%=;\n\t}" ::"r"(nk_smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// TMA bulk reduction shared -> global: dst[i] += src[i] for n complex
// doubles (UBLKRED.G.S.ADD.F64), tracked in this thread's bulk group
__device__ __forceinline__ void nk_bulk_red_add(double2 *dst, const double2 *src, int n) {
    if (n <= 0) return;
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(
                     dst),
                 "r"(nk_smem_u32(src)), "r"(16 * n)
                 : "memory");
}
// commit this thread's bulk operations and wait until their shared-memory
// sources have been read (before the CTA may exit or reuse them)
__device__ __forceinline__ void nk_bulk_wait_read() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// 4D TMA tensor copy global -> shared (box of the tensor map at
// coordinates c0..c3, innermost first), completion on the mbarrier (UTMALDG)
__device__ __forceinline__ void nk_tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1,
                                               int c2, int c3, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(nk_smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(nk_smem_u32(bar))
        : "memory");
}

// Packed FMA with a broadcast constant addend: (a.x, a.y) * (b.x, b.y) + (c, c)
// (sm_100 FFMA2 with a 32-bit immediate when c is a compile-time constant).
__device__ __forceinline__ float2 nk_fma2_cc(float2 a, float2 b, float c) {
    unsigned long long r;
    asm("{\n\t.reg .b64 cc;\n\tmov.b64 cc, {%3, %3};\n\tfma.rn.f32x2 %0, %1, %2, cc;\n\t}"
        : "=l"(r)
        : "l"(*reinterpret_cast<unsigned long long *>(&a)),
          "l"(*reinterpret_cast<unsigned long long *>(&b)), "f"(c));
    return *reinterpret_cast<float2 *>(&r);
}

// Kernel rows of two axes at once (the 2D footprint, or axes 1-2 in 3D):
// single precision evaluates both axes' interior Horner pieces as one
// packed FFMA2 chain per piece (same coefficients, s = (s1, s2)).
template <typename T, int W>
__device__ __forceinline__ void nk_kernel_rows2(T u1, T u2, const Geom &g, T *k1, T *k2,
                                                int &st1, int &st2) {
    if constexpr (sizeof(T) == 4 && W >= 3) {
        const float a1 = ceilf(u1 - 0.5f * W), a2 = ceilf(u2 - 0.5f * W);
        const float d1 = a1 - u1, d2 = a2 - u2;
        const float z1 = d1 * (2.0f / W), z2 = d2 * (2.0f / W);
        constexpr float zl = (float)(2.0 * (W - 1) / W);
        k1[0] = nk_es(z1, g);
        k2[0] = nk_es(z2, g);
        k1[W - 1] = nk_es(z1 + zl, g);
        k2[W - 1] = nk_es(z2 + zl, g);
        const float2 s = make_float2(fmaf(2.0f, d1, (float)(W - 1)), fmaf(2.0f, d2, (float)(W - 1)));
        typedef EsPoly<W> P;
#pragma unroll
        for (int r = 1; r < W - 1; ++r) {
            float2 p = make_float2(P::c(r - 1, P::D), P::c(r - 1, P::D));
#pragma unroll
            for (int k = P::D - 1; k >= 0; --k) p = nk_fma2_cc(p, s, P::c(r - 1, k));
            k1[r] = p.x;
            k2[r] = p.y;
        }
        st1 = (int)a1;
        st2 = (int)a2;
    } else {
        st1 = nk_kernel_row<T, W>(u1, g, k1);
        st2 = nk_kernel_row<T, W>(u2, g, k2);
    }
}

// Packed single-precision FMA (sm_100 FFMA2): (a.x, a.y) * b + (c.x, c.y).
__device__ __forceinline__ float2 nk_fma2(float2 a, float b, float2 c) {
    unsigned long long r;
    asm("{\n\t.reg .b64 bb;\n\tmov.b64 bb, {%2, %2};\n\tfma.rn.f32x2 %0, %1, bb, %3;\n\t}"
        : "=l"(r)
        : "l"(*reinterpret_cast<unsigned long long *>(&a)), "f"(b),
          "l"(*reinterpret_cast<unsigned long long *>(&c)));
    return *reinterpret_cast<float2 *>(&r);
}
__device__ __forceinline__ double2 nk_fma2(double2 a, double b, double2 c) {
    return make_double2(fma(a.x, b, c.x), fma(a.y, b, c.y));
}

__device__ __forceinline__ int nk_wrap(int l, int n) {
    l = l < 0 ? l + n : l;
    return l >= n ? l - n : l;
}

// Complex accumulation into global memory: native REDG.E.ADD.F32x2 / F64.
__device__ __forceinline__ void nk_red(float2 *p, float re, float im) {
    atomicAdd(p, make_float2(re, im));
}
__device__ __forceinline__ void nk_red(double2 *p, double re, double im) {
    atomicAdd(&p->x, re);
    atomicAdd(&p->y, im);
}

// Footprint-start visit code of a point in its bin's padded frame (setpts
// K4d sorts by bin, then this code): lexicographic (t3 p2 + t2) p1 + t1, or
// for tiled plans tile-major -- all starts of one 2^L x 2^L x 2^L tile are
// adjacent, so the tiled f64 spread (K6t) accumulates them in one register
// window.
// Tiles start at the smallest footprint start, t0 = halo - floor(w / 2)
// (u >= 0 in the bin): a bin of m cells has starts t0 .. t0 + m, so bins
// with m + 1 a multiple of the tile size are covered by whole tiles.
__device__ __forceinline__ int nk_tile_t0(const Geom &g) { return g.halo - g.w / 2; }
__device__ __forceinline__ int nk_start_code(int t1, int t2, int t3, int p1, int p2,
                                             const Geom &g) {
    if (!g.tiled) return (t3 * p2 + t2) * p1 + t1;
    const int o = nk_tile_t0(g);
    t1 -= o;
    t2 -= o;
    t3 -= o;
    // starts t - t0 lie in [0, bin width] (p - 2 halo + 1 values per axis)
    const int L = g.tile_lg, m = (1 << L) - 1;
    const int nt1 = (p1 - 2 * g.halo + 1 + m) >> L, nt2 = (p2 - 2 * g.halo + 1 + m) >> L;
    const int tile = ((t3 >> L) * nt2 + (t2 >> L)) * nt1 + (t1 >> L);
    return (tile << (3 * L)) | ((((t3 & m) << L) | (t2 & m)) << L) | (t1 & m);
}

// Decode a bin key into its corner cells (axis 1 fastest, binsort.py:103-111).
__device__ __forceinline__ void nk_bin_corner(int key, const Geom &g, int *corner) {
    int b0 = key % g.nb[0];
    int r = key / g.nb[0];
    corner[0] = b0 * g.m[0];
    if (g.dim == 2) {
        corner[1] = r * g.m[1];
        corner[2] = 0;
    } else {
        corner[1] = (r % g.nb[1]) * g.m[1];
        corner[2] = (r / g.nb[1]) * g.m[2];
    }
}

// L2 eviction-priority hints (PTX createpolicy / st.global.L2::cache_hint):
// scattered output stores keep their lines resident so partially written
// sectors are completed in L2 instead of read-modify-written from HBM.
__device__ __forceinline__ uint64_t nk_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void nk_st_keep(float2 *ptr, float2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(ptr), "f"(v.x),
                 "f"(v.y), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void nk_st_keep(double2 *ptr, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(v.x),
                 "d"(v.y), "l"(pol)
                 : "memory");
}

// i / d and i % d for 0 <= i < 2^31, 1 <= d < 2^16 with one IMAD.HI:
// magic = ceil(2^32 / d) (exact for i * d < 2^32).
struct nk_divmod {
    unsigned d, magic;
    __device__ __forceinline__ explicit nk_divmod(unsigned dd)
        : d(dd), magic((unsigned)((0x100000000ull + dd - 1) / dd)) {}
    __device__ __forceinline__ unsigned div(unsigned i) const { return __umulhi(i, magic); }
};

// Ampere-style asynchronous global -> shared copies (LDGSTS): no register
// staging, completion tracked per commit group.
__device__ __forceinline__ void nk_cp_async(float2 *smem, const float2 *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void nk_cp_async(double2 *smem, const double2 *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void nk_cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N> __device__ __forceinline__ void nk_cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
