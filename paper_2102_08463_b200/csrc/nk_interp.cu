// Type-2 step 3: ES-kernel interpolation (the adjoint gather).
//
//  K7  GM / GM-sort (_kernels.py:150-198; wrapper SPEC.md:358-366): one
//      thread per point in input / bin-sorted order gathers its w^d
//      footprint from the fine grid and writes slot perm[j] (output keeps
//      the input indexing).
//  K7s staged ("sm" for type 2): one CTA per subproblem copies its padded
//      bin (with periodic wrap) from HBM into shared memory once, then its
//      points gather from shared memory.  Same per-point arithmetic.
#include <algorithm>

#include "nk_device.cuh"

namespace {

#ifndef NK_XWIN_EU
#define NK_XWIN_EU 1
#endif
constexpr int kXwinEU = NK_XWIN_EU;   // K7x plane-loop unroll

template <typename T, int D, int W>
__device__ __forceinline__ typename cplx<T>::t
gather_global(const typename cplx<T>::t *__restrict__ fine, const Geom &g, int s1, int s2,
              int s3, const T *k1, const T *k2, T u3, T st3) {
    typedef typename cplx<T>::t C;
    const int n1 = g.n[0], n2 = g.n[1], n3 = g.n[2];
    int l1[W];
#pragma unroll
    for (int a = 0; a < W; ++a) l1[a] = nk_wrap(s1 + a, n1);
    T accr = 0, acci = 0;
#pragma unroll 1
    for (int e = 0; e < (D == 3 ? W : 1); ++e) {
        int64_t plane = D == 3 ? (int64_t)nk_wrap(s3 + e, n3) * n2 : 0;
        T mr = 0, mi = 0;
#pragma unroll
        for (int b = 0; b < W; ++b) {
            const C *row = fine + (plane + nk_wrap(s2 + b, n2)) * (int64_t)n1;
            T ir = 0, ii = 0;
#pragma unroll
            for (int a = 0; a < W; ++a) {
                C v = __ldg(row + l1[a]);
                ir += v.x * k1[a];
                ii += v.y * k1[a];
            }
            mr += ir * k2[b];
            mi += ii * k2[b];
        }
        if (D == 3) {
            const T k3 = nk_es((st3 + (T)e - u3) * (T)(2.0 / W), g);
            accr += mr * k3;
            acci += mi * k3;
        } else {
            accr = mr;
            acci = mi;
        }
    }
    C out;
    out.x = accr;
    out.y = acci;
    return out;
}

template <typename T, int D, int W>
__global__ void __launch_bounds__(256)
k_interp_gm(int M, const int32_t *__restrict__ perm, const int32_t *__restrict__ keys,
            const T *__restrict__ pts, int64_t pitch,
            const typename cplx<T>::t *__restrict__ fine, Geom g,
            typename cplx<T>::t *__restrict__ out) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    fine += blockIdx.y * g.ntot;   // batched execute: vector blockIdx.y
    out += blockIdx.y * g.M;
    int corner[3];
    nk_bin_corner(keys[j], g, corner);
    T k1[W], k2[W];
    int s1, s2;
    nk_kernel_rows2<T, W>(pts[j], pts[pitch + j], g, k1, k2, s1, s2);
    s1 += corner[0];
    s2 += corner[1];
    T u3 = 0, st3 = 0;
    if (D == 3) {
        u3 = pts[2 * pitch + j];
        st3 = nk_ceil<T>(u3 - (T)(0.5 * W));
    }
    const int s3 = corner[2] + (int)st3;
    const int dst = perm ? perm[j] : j;
    out[dst] = gather_global<T, D, W>(fine, g, s1, s2, s3, k1, k2, u3, st3);
}

// Copy subproblem s's padded bin (Eq. (16), periodic wrap) from the fine
// grid into shared memory with cp.async (no register round trip; all of a
// thread's copies are in flight at once).  Division-free index decode.
template <typename T, int D>
__device__ __forceinline__ void stage_padded_bin(typename cplx<T>::t *buf,
                                                 const typename cplx<T>::t *__restrict__ fine,
                                                 const Geom &g, int key) {
    int corner[3];
    nk_bin_corner(key, g, corner);
    const int h = g.halo;
    const int p1 = min(g.m[0], g.n[0] - corner[0]) + 2 * h;
    const int p2 = min(g.m[1], g.n[1] - corner[1]) + 2 * h;
    const int p3 = D == 3 ? min(g.m[2], g.n[2] - corner[2]) + 2 * h : 1;
    const int P = p1 * p2 * p3;
    const int o1 = corner[0] - h, o2 = corner[1] - h, o3 = corner[2] - h;
    const nk_divmod dm1(p1), dm2(p2);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int r = dm1.div(i);
        const int q1 = i - r * p1;
        const int q3 = D == 3 ? dm2.div(r) : 0;
        const int q2 = r - q3 * p2;
        int64_t l = nk_wrap(o1 + q1, g.n[0]) +
                    (int64_t)g.n[0] * (nk_wrap(o2 + q2, g.n[1]) +
                                       (D == 3 ? (int64_t)g.n[1] * nk_wrap(o3 + q3, g.n[2]) : 0));
        nk_cp_async(buf + i, fine + l);
    }
}

// K7s: persistent CTAs stride over the subproblems.  With NBUF = 2 the next
// subproblem's padded bin streams into the second shared-memory buffer
// (cp.async group) while the points of the current one gather, so the HBM
// latency of the staging is hidden behind the gather arithmetic.  Points
// are visited in footprint-start order (K4c), so a warp's 32 gathers from
// one padded-bin row hit adjacent words (one shared-memory wavefront).
template <typename T, int D, int W, int NBUF>
__global__ void __launch_bounds__(NBUF == 1 ? 512 : 256)
k_interp_staged(int S, const int32_t *__restrict__ sub_bin, const int32_t *__restrict__ sub_start,
                const int32_t *__restrict__ sub_stop, const int32_t *__restrict__ perm,
                const T *__restrict__ pts, int64_t pitch,
                const typename cplx<T>::t *__restrict__ fine, Geom g,
                typename cplx<T>::t *__restrict__ out, int buf_cells, int *__restrict__ work,
                const __grid_constant__ CUtensorMap tmap, int use_tma) {
    typedef typename cplx<T>::t C;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // buffers at 128-byte aligned strides (TMA destinations), then the two
    // buffers' mbarriers and the work-counter slot
    const int bstride = (buf_cells * (int)sizeof(C) + 127) / 128 * 128 / (int)sizeof(C);
    C *bufs = reinterpret_cast<C *>(smem_raw);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(bufs + NBUF * bstride);
    int &sh_next = *reinterpret_cast<int *>(mbar + 2);
    const int h = g.halo;
    const uint64_t keep = nk_policy_evict_last();
    fine += blockIdx.y * g.ntot;   // batched execute: vector blockIdx.y
    out += blockIdx.y * g.M;
    work += blockIdx.y;
    // dynamic scheduling: after its first subproblem a CTA takes the next
    // unclaimed one from a counter (balanced tails for uneven subproblems)
    int s = blockIdx.x;
    int cur = 0;
    // a full, non-wrapping padded bin arrives as one TMA box (mbarrier of its
    // buffer, phase bit per buffer); other bins by cp.async per cell
    unsigned tma_used = 0, phase = 0;   // bit b: buffer b's pending load is TMA / its parity
    // the descriptor's address in parameter space, taken outside the lambda
    // (a by-reference capture would copy the parameter to local memory,
    // which TMA cannot read)
    const CUtensorMap *tm = &tmap;
    auto load = [&, tm](int b, int ss) {
        int corner[3];
        nk_bin_corner(sub_bin[ss], g, corner);
        const int o1 = corner[0] - h, o2 = corner[1] - h, o3 = D == 3 ? corner[2] - h : 0;
        const bool full = corner[0] + g.m[0] <= g.n[0] && corner[1] + g.m[1] <= g.n[1] &&
                          (D == 2 || corner[2] + g.m[2] <= g.n[2]);
        // (single-buffered instantiations only: the double-buffered ones
        // raised illegal-instruction faults at the TMA issue on B200)
        const bool tma = NBUF == 1 && use_tma && full && o1 >= 0 && o2 >= 0 && o3 >= 0 &&
                         o1 + g.m[0] + 2 * h <= g.n[0] && o2 + g.m[1] + 2 * h <= g.n[1] &&
                         (D == 2 || o3 + g.m[2] + 2 * h <= g.n[2]);
        if (tma) {
            tma_used |= 1u << b;
            if (threadIdx.x == 0) {
                const int cells = (g.m[0] + 2 * h) * (g.m[1] + 2 * h) * (D == 3 ? g.m[2] + 2 * h : 1);
                nk_fence_proxy_async();
                nk_mbar_expect_tx(mbar + b, (unsigned)(cells * (int)sizeof(C)));
                nk_tma_load_4d(bufs + b * bstride, tm, 2 * o1, o2, o3, blockIdx.y, mbar + b);
            }
        } else {
            tma_used &= ~(1u << b);
            stage_padded_bin<T, D>(bufs + b * bstride, fine, g, sub_bin[ss]);
        }
    };
    auto wait_tma = [&](int b) {
        if (tma_used >> b & 1u) {
            nk_mbar_wait(mbar + b, (phase >> b) & 1u);
            phase ^= 1u << b;
        }
    };
    if (threadIdx.x == 0) {
        nk_mbar_init(mbar, 1);
        nk_mbar_init(mbar + 1, 1);
        nk_fence_mbar_init();
        sh_next = atomicAdd(work, 1) + gridDim.x;
    }
    if (s < S) load(0, s);
    nk_cp_async_commit();
    __syncthreads();
    int sn = sh_next;
    while (s < S) {
        if (NBUF == 2) {
            if (sn < S) load(cur ^ 1, sn);
            nk_cp_async_commit();
            nk_cp_async_wait<1>();
        } else {
            nk_cp_async_wait<0>();
        }
        wait_tma(cur);
        __syncthreads();
        const C *buf = bufs + cur * bstride;
        int corner[3];
        nk_bin_corner(sub_bin[s], g, corner);
        const int p1 = min(g.m[0], g.n[0] - corner[0]) + 2 * h;
        const int p2 = min(g.m[1], g.n[1] - corner[1]) + 2 * h;
        const int j0 = sub_start[s], j1 = sub_stop[s];
        // software pipeline: the next point's coordinates and output slot
        // load while this point gathers
        int j = j0 + threadIdx.x;
        T u1n = 0, u2n = 0, u3n = 0;
        int dstn = 0;
        if (j < j1) {
            u1n = __ldcs(pts + j);
            u2n = __ldcs(pts + pitch + j);
            if (D == 3) u3n = __ldcs(pts + 2 * pitch + j);
            dstn = __ldcs(perm + j);
        }
        for (; j < j1; j += blockDim.x) {
            const T u1 = u1n, u2 = u2n, u3 = u3n;
            const int dst = dstn;
            const int jn = j + blockDim.x;
            if (jn < j1) {
                u1n = __ldcs(pts + jn);
                u2n = __ldcs(pts + pitch + jn);
                if (D == 3) u3n = __ldcs(pts + 2 * pitch + jn);
                dstn = __ldcs(perm + jn);
            }
            T k1[W], k2[W];
            int t1, t2;
            nk_kernel_rows2<T, W>(u1, u2, g, k1, k2, t1, t2);
            t1 += h;
            t2 += h;
            T st3 = 0;
            if (D == 3) st3 = nk_ceil<T>(u3 - (T)(0.5 * W));
            const int t3 = (int)st3 + (D == 3 ? h : 0);
            C acc;
            acc.x = 0;
            acc.y = 0;
#pragma unroll 1
            for (int e = 0; e < (D == 3 ? W : 1); ++e) {
                C m;
                m.x = 0;
                m.y = 0;
#pragma unroll
                for (int b = 0; b < W; ++b) {
                    const C *row = buf + ((t3 + e) * p2 + (t2 + b)) * p1 + t1;
                    C ir;
                    ir.x = 0;
                    ir.y = 0;
#pragma unroll
                    for (int a = 0; a < W; ++a) ir = nk_fma2(row[a], k1[a], ir);
                    m = nk_fma2(ir, k2[b], m);
                }
                if (D == 3) {
                    const T k3 = nk_es((st3 + (T)e - u3) * (T)(2.0 / W), g);
                    acc = nk_fma2(m, k3, acc);
                } else {
                    acc = m;
                }
            }
            nk_st_keep(out + dst, acc, keep);
        }
        __syncthreads();   // buffer cur is free for the prefetch after next
        if (NBUF == 2) {
            cur ^= 1;
        } else if (sn < S) {
            load(0, sn);
            nk_cp_async_commit();
        }
        s = sn;
        if (threadIdx.x == 0) sh_next = atomicAdd(work, 1) + gridDim.x;
        __syncthreads();
        sn = sh_next;
    }
    nk_cp_async_wait<0>();
}

// One K7x group of exactly GN points (staged rows at wk[q..q+GN)): every
// lane reads its window cells (x, bs + 2 i) of all w planes once and
// accumulates the GN points' k2 k3 weighted sums; k1 and a warp butterfly
// finish each point.  Cells past the padded row carry k1 = 0 for all points.
template <typename T, int W, int GN>
__device__ __forceinline__ void xwin_group(const typename cplx<T>::t *buf, int p1, int p2,
                                           const int4 *wt, const T *wk, int q, int4 ta, int x,
                                           int bs, int lane, typename cplx<T>::t *out,
                                           const int32_t *perm, uint64_t keep) {
    typedef typename cplx<T>::t C;
    constexpr int NI = (W + 1) / 2;
    T kx[GN], k2r[GN][NI];
#pragma unroll
    for (int p = 0; p < GN; ++p) {
        const int sx = x - (wt[q + p].x - ta.x);   // lane's x in point p's row
        const T *kp = wk + (q + p) * 3 * W;
        kx[p] = (sx >= 0 && sx < W) ? kp[min(max(sx, 0), W - 1)] : (T)0;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int b = bs + 2 * i;
            k2r[p][i] = b < W ? kp[W + min(b, W - 1)] : (T)0;
        }
    }
    C acc[GN];
#pragma unroll
    for (int p = 0; p < GN; ++p) acc[p].x = acc[p].y = 0;
    const C *col = buf + (ta.z * p2 + ta.y) * p1 + min(ta.x + x, p1 - 1);
    const T *k3 = wk + q * 3 * W + 2 * W;
#pragma unroll kXwinEU
    for (int e = 0; e < W; ++e) {
        const C *pl = col + e * p2 * p1;
        C t[GN];
#pragma unroll
        for (int p = 0; p < GN; ++p) t[p].x = t[p].y = 0;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const C c = pl[min(bs + 2 * i, W - 1) * p1];
#pragma unroll
            for (int p = 0; p < GN; ++p) t[p] = nk_fma2(c, k2r[p][i], t[p]);
        }
#pragma unroll
        for (int p = 0; p < GN; ++p) acc[p] = nk_fma2(t[p], k3[p * 3 * W + e], acc[p]);
    }
#pragma unroll
    for (int p = 0; p < GN; ++p) {
        T vr = acc[p].x * kx[p], vi = acc[p].y * kx[p];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            vr += __shfl_xor_sync(0xffffffffu, vr, o);
            vi += __shfl_xor_sync(0xffffffffu, vi, o);
        }
        if (lane == p) {
            C v;
            v.x = vr;
            v.y = vi;
            nk_st_keep(out + __ldcs(perm + q + p), v, keep);
        }
    }
}

// exact-size group instantiation for gn in [GN, XG]
template <typename T, int W, int GN, int XG>
__device__ __forceinline__ void xwin_dispatch(int gn, const typename cplx<T>::t *buf, int p1,
                                              int p2, const int4 *wt, const T *wk, int q,
                                              int4 ta, int x, int bs, int lane,
                                              typename cplx<T>::t *out, const int32_t *perm,
                                              uint64_t keep) {
    if constexpr (GN == XG) {
        xwin_group<T, W, GN>(buf, p1, p2, wt, wk, q, ta, x, bs, lane, out, perm, keep);
    } else {
        if (gn == GN)
            xwin_group<T, W, GN>(buf, p1, p2, wt, wk, q, ta, x, bs, lane, out, perm, keep);
        else
            xwin_dispatch<T, W, GN + 1, XG>(gn, buf, p1, p2, wt, wk, q, ta, x, bs, lane, out,
                                            perm, keep);
    }
}

// K7x: 3D wide-footprint (f64, w > 8) staged interpolation with x-window
// groups -- the gather counterpart of the f64 spread's register windows.
// The per-thread gather of K7s reads w^3 x 16 B of shared memory per point
// (35 KB at w = 13: shared-bandwidth bound, L1 85 %, 22 % bank conflicts).
// Here a warp takes a GROUP of up to XG consecutive points with the same
// (t2, t3) footprint start and t1 within 16 - w of the group's first point
// (footprint-start visit order, K4c, makes them neighbours): its lanes cover
// a 16-cell x window x 2 rows, read each window cell ONCE per group (one
// contiguous 256-B row segment per half-warp, no bank conflicts) and
// accumulate every group point's k2[b] k3[e] weighted sums in registers;
// the k1[x - t1] factor and a butterfly reduction over the warp finish each
// point.  Kernel rows are staged per warp, one (point, axis) row per lane.
template <typename T, int W>
__global__ void __launch_bounds__(32 * NK_XWIN_WARPS)
k_interp_xwin(int S, const int32_t *__restrict__ sub_bin, const int32_t *__restrict__ sub_start,
              const int32_t *__restrict__ sub_stop, const int32_t *__restrict__ perm,
              const T *__restrict__ pts, int64_t pitch,
              const typename cplx<T>::t *__restrict__ fine, Geom g,
              typename cplx<T>::t *__restrict__ out, int buf_cells, int *__restrict__ work) {
    typedef typename cplx<T>::t C;
    constexpr int XW = 16, NB = NK_XWIN_NB, XG = NK_XWIN_G, NWARP = NK_XWIN_WARPS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ int sh_next;
    C *buf = reinterpret_cast<C *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int4 *wt = reinterpret_cast<int4 *>(buf + buf_cells) + warp * NB;   // (t1, t2, t3)
    T *wk = reinterpret_cast<T *>(reinterpret_cast<int4 *>(buf + buf_cells) + NWARP * NB) +
            warp * NB * 3 * W;                                          // k rows [q][axis][r]
    const int h = g.halo;
    const uint64_t keep = nk_policy_evict_last();
    fine += blockIdx.y * g.ntot;
    out += blockIdx.y * g.M;
    work += blockIdx.y;
    const int x = lane & (XW - 1), bs = lane >> 4;
    int s = blockIdx.x;
    if (threadIdx.x == 0) sh_next = atomicAdd(work, 1) + gridDim.x;
    if (s < S) stage_padded_bin<T, 3>(buf, fine, g, sub_bin[s]);
    nk_cp_async_commit();
    __syncthreads();
    int sn = sh_next;
    while (s < S) {
        nk_cp_async_wait<0>();
        __syncthreads();
        int corner[3];
        nk_bin_corner(sub_bin[s], g, corner);
        const int p1 = min(g.m[0], g.n[0] - corner[0]) + 2 * h;
        const int p2 = min(g.m[1], g.n[1] - corner[1]) + 2 * h;
        const int j0 = sub_start[s], j1 = sub_stop[s];
        const int chunk = (j1 - j0 + NWARP - 1) / NWARP;
        const int a0 = j0 + warp * chunk, a1 = min(j1, a0 + chunk);
        for (int base = a0; base < a1; base += NB) {
            const int nb = min(NB, a1 - base);
            __syncwarp();
            for (int v = lane; v < 3 * nb; v += 32) {
                const int q = v / 3, ax = v - 3 * q;
                T k[W];
                const int t = nk_kernel_row<T, W>(__ldcs(pts + ax * pitch + base + q), g, k) + h;
#pragma unroll
                for (int r = 0; r < W; ++r) wk[(q * 3 + ax) * W + r] = k[r];
                reinterpret_cast<int *>(wt)[q * 4 + ax] = t;
            }
            __syncwarp();
            for (int q = 0; q < nb;) {   // warp-uniform group walk
                const int4 ta = wt[q];
                int gn = 1;
                while (gn < XG && q + gn < nb) {
                    const int4 tb = wt[q + gn];
                    if (tb.y != ta.y || tb.z != ta.z || (unsigned)(tb.x - ta.x) > XW - W) break;
                    ++gn;
                }
                xwin_dispatch<T, W, 1, XG>(gn, buf, p1, p2, wt, wk, q, ta, x, bs, lane, out,
                                            perm + base, keep);
                q += gn;
            }
        }
        __syncthreads();   // buffer free
        if (sn < S) {
            stage_padded_bin<T, 3>(buf, fine, g, sub_bin[sn]);
            nk_cp_async_commit();
        }
        s = sn;
        if (threadIdx.x == 0) sh_next = atomicAdd(work, 1) + gridDim.x;
        __syncthreads();
        sn = sh_next;
    }
    nk_cp_async_wait<0>();
}

// K7t: tiled f64 3D interpolation on the FP64 tensor cores -- the adjoint
// of K6t (nk_spread.cu) on the same tile groups (setpts: tile-major
// footprint-start order).  The padded bin is copied into shared memory
// (cp.async, periodic wrap) while warp 0 cuts the subproblem into chunks:
// runs of <= 8 consecutive points of one start tile.  Interpolation only
// reads the bin, so warps then work independently (no barriers): a warp
// takes a chunk, evaluates its points' kernel rows into a private table
// (pre-shifted into the tile's 16 x 16 x 16 window, zeros outside the
// footprint), and for each window plane e runs one small GEMM on the DMMA
// units,
//   V[(x, c)][p] += sum_y G[e][y][x]_c (k2_p[y] k3_p[e])   (16 DMMA m8n8k4)
// (y as the reduction index: a half-warp's A fragment is 2 x-cells x 4 rows
// x re|im, conflict-free for the 22-cell padded rows of the default bins;
// k3 folded into B so all planes share the accumulators), then contracts
// x with k1_p[x] in registers and sums
// over its lanes (2 shuffles) and stores each point's value to its input
// slot.  Planes outside every chunk point's footprint (k3 = 0) are skipped.
template <int W>
__global__ void __launch_bounds__(512, 1)
k_interp_tiled(const int32_t *__restrict__ sub_bin, const int32_t *__restrict__ sub_start,
               const int32_t *__restrict__ sub_stop, const int32_t *__restrict__ perm,
               const double *__restrict__ pts, int64_t pitch,
               const double2 *__restrict__ fine, Geom g, double2 *__restrict__ out,
               int64_t stage_off, const __grid_constant__ CUtensorMap tmap, int use_tma,
               const int32_t *__restrict__ sched) {
    constexpr int WIN = kTileWin, L = nk_tile_lg(W), TM = (1 << L) - 1, NWARP = 16;
    // staged rows: [3 axes][16 cells][8 points], point slot swizzled by cell
    // bit 1 (conflict-free B fragment and epilogue reads)
    constexpr int CS = 8;
    auto pos = [](int c, int q) { return c * CS + (q ^ (((c >> 1) & 1) << 2)); };
    static_assert(W + TM <= WIN, "window too small for the tile");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *buf = reinterpret_cast<double2 *>(smem_raw);
    // per warp: k1 / k2 / k3 rows [3][16 cells][CS]; chunk starts
    double *wst = reinterpret_cast<double *>(smem_raw + stage_off) +
                  (threadIdx.x >> 5) * (3 * WIN * CS);
    int *cstart = reinterpret_cast<int *>(smem_raw + stage_off) + 2 * NWARP * 3 * WIN * CS;
    int &sh_nchunk = cstart[kTileMsub + 1];
    uint64_t *mbar = reinterpret_cast<uint64_t *>(cstart + kTileMsub + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = sched ? sched[blockIdx.x] : (int)blockIdx.x;
    fine += blockIdx.y * g.ntot;
    out += blockIdx.y * g.M;
    int corner[3];
    nk_bin_corner(sub_bin[s], g, corner);
    const int h = g.halo;
    const int p1 = min(g.m[0], g.n[0] - corner[0]) + 2 * h;
    const int p2 = min(g.m[1], g.n[1] - corner[1]) + 2 * h;
    const int p3 = min(g.m[2], g.n[2] - corner[2]) + 2 * h;
    const int pstride = p1 * p2;
    // the padded bin: one TMA box when it is full-size and does not wrap,
    // else cp.async per cell with periodic wrap
    const int o1 = corner[0] - h, o2 = corner[1] - h, o3 = corner[2] - h;
    const bool tma = use_tma && p1 == g.m[0] + 2 * h && p2 == g.m[1] + 2 * h &&
                     p3 == g.m[2] + 2 * h && o1 >= 0 && o2 >= 0 && o3 >= 0 &&
                     o1 + p1 <= g.n[0] && o2 + p2 <= g.n[1] && o3 + p3 <= g.n[2];
    if (tma) {
        if (threadIdx.x == 0) {
            nk_mbar_init(mbar, 1);
            nk_fence_mbar_init();
            nk_mbar_expect_tx(mbar, (unsigned)(p1 * p2 * p3) * 16u);
            nk_tma_load_4d(buf, &tmap, 2 * o1, o2, o3, blockIdx.y, mbar);
        }
    } else {
        stage_padded_bin<double, 3>(buf, fine, g, sub_bin[s]);
        nk_cp_async_commit();
    }
    const double half = 0.5 * W;
    const int j0 = sub_start[s], j1 = sub_stop[s];
    auto tile_of = [&](int j) {
        const int t1 = (int)ceil(__ldg(pts + j) - half) + h;
        const int t2 = (int)ceil(__ldg(pts + pitch + j) - half) + h;
        const int t3 = (int)ceil(__ldg(pts + 2 * pitch + j) - half) + h;
        return nk_start_code(t1, t2, t3, p1, p2, g) >> (3 * L);
    };
    if (warp == 0) {
        // chunks: a point starts one if its tile differs from its
        // predecessor's or it is 8 points past its group's start
        int gs = j0, nc = 0, prev = -1;
        for (int base = j0; base < j1; base += 32) {
            const int j = base + lane;
            const int tl = j < j1 ? tile_of(j) : -2;
            const int tp = __shfl_up_sync(0xffffffffu, tl, 1);
            const bool f = j < j1 && (lane == 0 ? tl != prev : tl != tp);
            const unsigned fm = __ballot_sync(0xffffffffu, f);
            // latest group start at or below this lane
            const unsigned below = fm & (0xffffffffu >> (31 - lane));
            const int g_at = below ? base + 31 - __clz(below) : gs;
            const bool cst = j < j1 && ((j - g_at) & 7) == 0;
            const unsigned cm = __ballot_sync(0xffffffffu, cst);
            if (cst) cstart[nc + __popc(cm & ((1u << lane) - 1u))] = j;
            nc += __popc(cm);
            gs = fm ? base + 31 - __clz(fm) : gs;
            prev = __shfl_sync(0xffffffffu, tl, 31);
        }
        if (lane == 0) {
            cstart[nc] = j1;
            sh_nchunk = nc;
        }
    }
    if (tma) {
        __syncthreads();   // the mbarrier is initialised
        nk_mbar_wait(mbar, 0);
    } else {
        nk_cp_async_wait<0>();
    }
    __syncthreads();   // padded bin and chunk list ready
    const int nchunk = sh_nchunk;
    const int kx = lane & 3, prow = lane >> 2, ylane = lane >> 3, cpart = (lane >> 2) & 1;
    double *sk1 = wst, *sk2 = wst + WIN * CS, *sk3 = wst + 2 * WIN * CS;
    for (int ch = warp; ch < nchunk; ch += NWARP) {
        const int cs = cstart[ch], n = cstart[ch + 1] - cs;   // 1..8 points, one tile
        // kernel rows: lane (q, axis) for q < n, window-shifted, transposed
        int t0 = 0;
        if (lane < 3 * n) {
            const int q = lane / 3, ax = lane - 3 * q;
            double k[W];
            const int t = nk_kernel_row_poly<W>(__ldg(pts + ax * pitch + cs + q), g, k) + h;
            const int sh = (t - nk_tile_t0(g)) & TM;
            double *dst = wst + ax * WIN * CS;
#pragma unroll
            for (int i = 0; i < WIN - W; ++i) dst[pos(i < sh ? i : i + W, q)] = 0.0;
#pragma unroll
            for (int r = 0; r < W; ++r) dst[pos(sh + r, q)] = k[r];
            t0 = nk_tile_t0(g) + ((t - nk_tile_t0(g)) & ~TM);
        }
        // the chunk's window anchor (any point's tile corner: lanes 0-2)
        const int a1 = __shfl_sync(0xffffffffu, t0, 0);
        const int a2 = __shfl_sync(0xffffffffu, t0, 1);
        const int a3 = __shfl_sync(0xffffffffu, t0, 2);
        // zero rows of the unused point columns (n..7) so B / k2 / k3 are 0
        for (int v = lane; v < 3 * WIN * (8 - n); v += 32) {
            const int c = v / (8 - n), q = n + (v - c * (8 - n));
            wst[(c / WIN) * WIN * CS + pos(c % WIN, q)] = 0.0;
        }
        __syncwarp();
        // B_e[y][p] = k2_p[y] k3_p[e] (y = ks * 4 + lane % 4, p = lane / 4):
        // with k3 folded into B every plane accumulates into the same DMMA
        // tiles, V[(x, c)][p] = sum_e sum_y G[e][y][x]_c k2_p[y] k3_p[e]
        double bf[4];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) bf[ks] = sk2[pos(ks * 4 + kx, prow)];
        double cacc[4][2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) cacc[mt][0] = cacc[mt][1] = 0.0;
        const double *plane0 = reinterpret_cast<const double *>(buf) + cpart;
        const int e_end = min(WIN, p3 - a3);
#pragma unroll 1
        for (int e = 0; e < e_end; ++e) {
            const double k3v = sk3[pos(e, prow)];
            if (!__any_sync(0xffffffffu, k3v != 0.0)) continue;   // outside every footprint
            // A[(x, c)][y] = G[a3 + e][a2 + y][a1 + x]_c, row (x, c) = mt * 8 +
            // lane / 4, column y = ks * 4 + lane % 4
            const double *pl = plane0 + 2 * (a3 + e) * pstride;
            double af[4][4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const int xx = a1 + mt * 4 + ylane, yy = a2 + ks * 4 + kx;
                    af[mt][ks] = (xx < p1 && yy < p2) ? pl[2 * (yy * p1 + xx)] : 0.0;
                }
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const double bv = bf[ks] * k3v;
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
                    nk_dmma(cacc[mt][0], cacc[mt][1], af[mt][ks], bv);
            }
        }
        // C[(x, c)][p]: lane rows x = mt * 4 + lane / 8 (component c), points
        // 2 (lane % 4) + {0, 1}; contract x with k1_p[x]
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            acc0 = fma(cacc[mt][0], sk1[pos(mt * 4 + ylane, 2 * kx)], acc0);
            acc1 = fma(cacc[mt][1], sk1[pos(mt * 4 + ylane, 2 * kx + 1)], acc1);
        }
        acc0 += __shfl_xor_sync(0xffffffffu, acc0, 8);
        acc1 += __shfl_xor_sync(0xffffffffu, acc1, 8);
        acc0 += __shfl_xor_sync(0xffffffffu, acc0, 16);
        acc1 += __shfl_xor_sync(0xffffffffu, acc1, 16);
        if (ylane == 0) {   // lanes 0-7: points 2 (lane % 4) + {0, 1}, component c
            const int pa = 2 * kx;
            if (pa < n) reinterpret_cast<double *>(out + __ldcs(perm + cs + pa))[cpart] = acc0;
            if (pa + 1 < n)
                reinterpret_cast<double *>(out + __ldcs(perm + cs + pa + 1))[cpart] = acc1;
        }
        __syncwarp();   // the staged rows are reused by the warp's next chunk
    }
}

template <typename T, int D, int W>
int launch_w(nk_plan *p, const void *fine, void *out, int *launches) {
    typedef typename cplx<T>::t C;
    const int M = (int)p->M;
    if (M == 0) return NK_OK;
    if (p->method == NK_SM) {
        if (p->S == 0) return NK_OK;
        int nsm = 0;
        NK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device));
        const size_t one = (size_t)p->max_sub_smem;   // padded bin, 16-B rounded
        if constexpr (D == 3 && sizeof(T) == 8 && W >= 9) {
            if (p->geom.tiled) {
                auto kern = k_interp_tiled<W>;
                NK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)one));
                const int64_t stage_off = (p->max_pad_cells * 16 + 15) / 16 * 16;
                // TMA box loads only from the plan's own grid (the tensor map
                // describes p->d_fine); stage-level calls pass other grids
                const int use_tma = p->tmap_ok && fine == p->d_fine && !getenv("NK_NO_TMA");
                kern<<<dim3((unsigned)p->S, p->ntrans), 512, one, p->stream>>>(
                    p->d_sub_bin, p->d_sub_start, p->d_sub_stop, p->d_vperm,
                    (const double *)p->d_pts, p->cap_M, (const double2 *)fine, p->geom,
                    (double2 *)out, stage_off, p->tmap_fine, use_tma, p->d_sub_sched);
                NK_LAUNCH_CHECK();
                ++*launches;
                return NK_OK;
            }
        }
        if constexpr (D == 3 && sizeof(T) == 8 && W > 8) {
            const size_t xsm = one + nk_xwin_smem_bytes(W);
            if (nk_interp_xwin(p->type, p->dim, p->prec, p->w, p->method, p->max_sub_smem)) {
                auto kern = k_interp_xwin<T, W>;
                NK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)xsm));
                int per_sm = 0;
                NK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * NK_XWIN_WARPS, xsm));
                const int64_t grid =
                    std::min<int64_t>(p->S, (int64_t)std::max(per_sm, 1) * nsm);
                NK_CUDA(cudaMemsetAsync(p->d_work, 0, sizeof(int) * p->ntrans, p->stream));
                kern<<<dim3((unsigned)grid, p->ntrans), 32 * NK_XWIN_WARPS, xsm, p->stream>>>(
                    (int)p->S, p->d_sub_bin, p->d_sub_start, p->d_sub_stop, p->d_vperm,
                    (const T *)p->d_pts, p->cap_M, (const C *)fine, p->geom, (C *)out,
                    (int)(one / sizeof(C)), p->d_work);
                NK_LAUNCH_CHECK();
                ++*launches;
                return NK_OK;
            }
        }
        // double-buffer when two padded bins leave room for a useful occupancy
        const bool two = 2 * one <= 100 * 1024;
        const size_t smem = (two ? 2 * (one + 128) : one + 128) + 64;   // + alignment, mbarriers
        auto kern = two ? k_interp_staged<T, D, W, 2> : k_interp_staged<T, D, W, 1>;
        NK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        // single-buffer (large padded bin: one CTA per SM) -> 512 threads
        // share it for latency hiding
        const int threads = two ? 256 : 512;
        int per_sm = 0;
        NK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
        const int64_t grid = std::min<int64_t>(p->S, (int64_t)std::max(per_sm, 1) * nsm);
        NK_CUDA(cudaMemsetAsync(p->d_work, 0, sizeof(int) * p->ntrans, p->stream));
        const int use_tma = p->tmap_ok && fine == p->d_fine && !getenv("NK_NO_TMA");
        kern<<<dim3((unsigned)grid, p->ntrans), threads, smem, p->stream>>>(
            (int)p->S, p->d_sub_bin, p->d_sub_start, p->d_sub_stop, p->d_vperm,
            (const T *)p->d_pts, p->cap_M, (const C *)fine, p->geom, (C *)out,
            (int)(one / sizeof(C)), p->d_work, p->tmap_fine, use_tma);
    } else {
        const int32_t *perm = p->method == NK_GM ? nullptr : p->d_vperm;
        k_interp_gm<T, D, W><<<dim3((M + 255) / 256, p->ntrans), 256, 0, p->stream>>>(
            M, perm, p->d_keys, (const T *)p->d_pts, p->cap_M, (const C *)fine, p->geom,
            (C *)out);
    }
    NK_LAUNCH_CHECK();
    ++*launches;
    return NK_OK;
}

template <typename T, int D>
int launch_d(nk_plan *p, const void *fine, void *out, int *launches) {
    switch (p->w) {
#define NK_W(W) \
    case W: return launch_w<T, D, W>(p, fine, out, launches);
        NK_W(2) NK_W(3) NK_W(4) NK_W(5) NK_W(6) NK_W(7) NK_W(8) NK_W(9) NK_W(10) NK_W(11)
        NK_W(12) NK_W(13) NK_W(14) NK_W(15) NK_W(16)
#undef NK_W
    }
    nk_set_error("unsupported kernel width");
    return NK_ERR_VALUE;
}

}  // namespace

int nk_launch_interp(nk_plan *p, const void *fine, void *out, int *launches) {
    if (p->prec == NK_DOUBLE)
        return p->dim == 2 ? launch_d<double, 2>(p, fine, out, launches)
                           : launch_d<double, 3>(p, fine, out, launches);
    return p->dim == 2 ? launch_d<float, 2>(p, fine, out, launches)
                       : launch_d<float, 3>(p, fine, out, launches);
}
