// Type-1 step 1: ES-kernel spreading onto the fine grid.
//
//  K6a/K6b  GM / GM-sort (spread.py:142-163 -> _kernels.py:36-79): one thread
//           per point in input / bin-sorted order, w^d native global
//           REDG.E.ADD.F32x2 (single) or F64 (double) reductions.
//  K6c      SM (spread.py:166-182 -> _kernels.py:82-147): each subproblem's
//           padded bin (Eq. (16)) is accumulated in shared memory without
//           atomics (one warp per subproblem in 2D, plane-owned warps in 3D),
//           then merged into the grid with periodic wrap (Eq. (17)).
#include <algorithm>

#include "nk_device.cuh"

namespace {

template <typename T, int D, int W>
__global__ void __launch_bounds__(256)
k_spread_gm(int M, const int32_t *__restrict__ perm, const int32_t *__restrict__ keys,
            const T *__restrict__ pts, int64_t pitch, const typename cplx<T>::t *__restrict__ c,
            Geom g, typename cplx<T>::t *__restrict__ fine) {
    typedef typename cplx<T>::t C;
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    c += blockIdx.y * g.M;
    fine += blockIdx.y * g.ntot;
    int corner[3];
    nk_bin_corner(keys[j], g, corner);
    const int src = perm ? perm[j] : j;
    const C cv = c[src];
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
    const int n1 = g.n[0], n2 = g.n[1], n3 = g.n[2];
    int l1[W];
#pragma unroll
    for (int a = 0; a < W; ++a) l1[a] = nk_wrap(s1 + a, n1);
    // 3D: the axis-3 loop stays rolled (compile size), its kernel value is
    // evaluated per iteration
#pragma unroll 1
    for (int e = 0; e < (D == 3 ? W : 1); ++e) {
        T t3r = cv.x, t3i = cv.y;
        int64_t plane = 0;
        if (D == 3) {
            const T k3 = nk_es((st3 + (T)e - u3) * (T)(2.0 / W), g);
            t3r *= k3;
            t3i *= k3;
            plane = (int64_t)nk_wrap(s3 + e, n3) * n2;
        }
#pragma unroll
        for (int b = 0; b < W; ++b) {
            const T t2r = t3r * k2[b], t2i = t3i * k2[b];
            C *row = fine + (plane + nk_wrap(s2 + b, n2)) * (int64_t)n1;
#pragma unroll
            for (int a = 0; a < W; ++a) nk_red(row + l1[a], t2r * k1[a], t2i * k1[a]);
        }
    }
}

// K6c-3D: plane-owned shared-memory spreading with run accumulation, no
// atomics.  A CTA of NW warps owns one subproblem's padded bin (p1 x p2 x
// p3 cells, Eq. (16)).  Points are staged in batches: each thread evaluates
// one point's three kernel rows (c folded into the axis-3 row) into shared
// memory.  Every warp walks the whole batch; warp w only touches padded-bin
// planes z == w (mod NW), its lanes covering distinct cells of a plane, so
// plain read-modify-write replaces the CAS loops that atomicAdd(float /
// double) compiles to on shared memory.  Points arrive in (bin, t3, t2, t1)
// footprint-start order (setpts K4d) and a lane keeps its cells' sums in
// registers while consecutive points fit the warp's register window:
//  * single precision: window = the point's w x w footprint (lane idx =
//    it * 32 + lane); runs of identical starts (clustered points) write
//    shared memory once per run.
//  * double precision (w = 13, uniform density): window = 16 x-cells x w
//    rows anchored at the first point of a group; points with the same
//    (t2, t3) and t1 within 16 - w of the anchor join the group, each lane
//    adding k1[x - t1] k2[b] c k3[e] for its (x, b).  One shared
//    read-modify-write per group instead of per point and footprint cell
//    (the f64 kernel is shared-bandwidth bound: 13 x 13 x 16 B x 2 per
//    point and plane otherwise).
// The finished bin is merged with native global vector reductions (Eq. 17).
template <typename T, int W, int NW>
__global__ void __launch_bounds__(NW * 32)
k_spread_sm3(const int32_t *__restrict__ sub_bin, const int32_t *__restrict__ sub_start,
             const int32_t *__restrict__ sub_stop, const int32_t *__restrict__ perm,
             const T *__restrict__ pts, int64_t pitch, const typename cplx<T>::t *__restrict__ c,
             Geom g, typename cplx<T>::t *__restrict__ fine, int64_t stage_off, int nbatch,
             const int32_t *__restrict__ sched, int sched_base) {
    typedef typename cplx<T>::t C;
    constexpr bool XWIN = sizeof(T) == 8 && W <= 16;
    constexpr int XW = 16;                      // x-window width (XWIN)
    constexpr int NIT = XWIN ? (W + 1) / 2 : (W * W + 31) / 32;
    constexpr int NE = (W + NW - 1) / NW;       // planes per warp per footprint
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *buf = reinterpret_cast<C *>(smem_raw);
    int4 *sst = reinterpret_cast<int4 *>(smem_raw + stage_off);   // t1, t2, t3
    // XWIN: each point's k1 row sits at offset XW of a zero-padded 2 XW row,
    // so the window gather k1[x - shift] needs no bounds test
    constexpr int K1P = XWIN ? 2 * XW : W;
    T *sk1 = reinterpret_cast<T *>(sst + nbatch);
    T *sk2 = sk1 + nbatch * K1P;
    C *sck3 = reinterpret_cast<C *>(sk2 + nbatch * W);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = sched ? sched[sched_base + blockIdx.x] : (int)blockIdx.x;
    c += blockIdx.y * g.M;          // batched execute: vector blockIdx.y
    fine += blockIdx.y * g.ntot;
    int corner[3];
    nk_bin_corner(sub_bin[s], g, corner);
    const int h = g.halo;
    const int p1 = min(g.m[0], g.n[0] - corner[0]) + 2 * h;
    const int p2 = min(g.m[1], g.n[1] - corner[1]) + 2 * h;
    const int p3 = min(g.m[2], g.n[2] - corner[2]) + 2 * h;
    const int P = p1 * p2 * p3, pstride = p1 * p2;
    // lane -> window cell (a = x, b) of each pass
    int la[NIT], lb[NIT], lofs[NIT];
    bool lok[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        if (XWIN) {
            la[it] = lane & (XW - 1);
            lb[it] = (lane >> 4) + 2 * it;
            lok[it] = lb[it] < W;
        } else {
            const int idx = it * 32 + lane;
            lb[it] = idx / W;
            la[it] = idx - lb[it] * W;
            lok[it] = idx < W * W;
        }
        la[it] = XWIN ? la[it] : min(la[it], W - 1);
        lb[it] = min(lb[it], W - 1);
        lofs[it] = lb[it] * p1 + la[it];
    }
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        C zero;
        zero.x = 0;
        zero.y = 0;
        buf[i] = zero;
    }
    C acc[NE][NIT];
#pragma unroll
    for (int k = 0; k < NE; ++k)
#pragma unroll
        for (int it = 0; it < NIT; ++it) acc[k][it].x = acc[k][it].y = 0;
    // current window: origin offset in the padded bin, its row offset and
    // x (XWIN), the warp's first plane
    int run_off = -1, run_row = -1, run_x0 = 0, e0 = 0;
    // add the register sums of the window to its planes, then clear
    // (lanes outside the footprint / window never write)
    auto flush = [&]() {
        __syncwarp();   // lanes' cells moved with the window: order the accesses
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int e = e0 + k * NW;
            if (e < W) {   // warp-uniform
                C *plane = buf + run_off + e * pstride;
#pragma unroll
                for (int it = 0; it < NIT; ++it) {
                    const bool ok = XWIN ? (lok[it] && run_x0 + la[it] < p1)
                                         : ((it < NIT - 1) || lok[it]);
                    if (ok) {
                        C *cell = plane + lofs[it];
                        C v = *cell;
                        v.x += acc[k][it].x;
                        v.y += acc[k][it].y;
                        *cell = v;
                    }
                    acc[k][it].x = acc[k][it].y = 0;
                }
            }
        }
    };
    const int j0 = sub_start[s], j1 = sub_stop[s];
    for (int base = j0; base < j1; base += nbatch) {
        const int nb = min(nbatch, j1 - base);
        __syncthreads();   // previous batch consumed (and buffer zeroed)
        if constexpr (sizeof(T) == 8) {
            // double: one kernel row (point, axis) per thread -- 3 nb rows
            // of FP64 exp/sqrt spread over the CTA instead of nb threads
            int *stt = reinterpret_cast<int *>(sst);
            for (int v = threadIdx.x; v < 3 * nb; v += blockDim.x) {
                const int q = v / 3, ax = v - 3 * q;
                const int j = base + q;
                T k[W];
                const int t = nk_kernel_row<T, W>(pts[ax * pitch + j], g, k) + h;
                if (ax == 2) {
                    const C cv = c[perm[j]];
#pragma unroll
                    for (int r = 0; r < W; ++r) {
                        C cvk;
                        cvk.x = cv.x * k[r];
                        cvk.y = cv.y * k[r];
                        sck3[q * W + r] = cvk;
                    }
                } else {
                    if (ax == 0 && XWIN) {
                        T *dstk = sk1 + q * K1P;
#pragma unroll
                        for (int r = 0; r < K1P; ++r)
                            dstk[r] = (r >= XW && r < XW + W) ? k[(r - XW) % W] : (T)0;
                    } else {
                        T *dstk = (ax == 0 ? sk1 : sk2) + q * (ax == 0 ? K1P : W);
#pragma unroll
                        for (int r = 0; r < W; ++r) dstk[r] = k[r];
                    }
                }
                stt[q * 4 + ax] = t;
            }
        } else {
            for (int q = threadIdx.x; q < nb; q += blockDim.x) {
                const int j = base + q;
                const C cv = c[perm[j]];
                T k[W], kb[W];
                int t1, t2;
                nk_kernel_rows2<T, W>(pts[j], pts[pitch + j], g, k, kb, t1, t2);
#pragma unroll
                for (int r = 0; r < W; ++r) {
                    sk1[q * K1P + r] = k[r];
                    sk2[q * W + r] = kb[r];
                }
                const int t3 = nk_kernel_row<T, W>(pts[2 * pitch + j], g, k) + h;
#pragma unroll
                for (int r = 0; r < W; ++r) {
                    C v;
                    v.x = cv.x * k[r];
                    v.y = cv.y * k[r];
                    sck3[q * W + r] = v;
                }
                sst[q] = make_int4(t1 + h, t2 + h, t3, 0);
            }
        }
        __syncthreads();
        for (int q = 0; q < nb; ++q) {
            const int4 st = sst[q];   // (t1, t2, t3) in the padded frame
            const int row = (st.z * p2 + st.y) * p1;
            // uniform across the CTA: does point q fit the current window?
            const bool fits = XWIN ? (row == run_row && st.x - run_x0 <= XW - W)
                                   : (row + st.x == run_off);
            if (!fits) {
                if (run_off >= 0) flush();
                run_row = row;
                run_x0 = st.x;
                run_off = row + st.x;
                e0 = ((warp - st.z) % NW + NW) % NW;
            }
            const T *k1q = sk1 + q * K1P;
            const T *k2q = sk2 + q * W;
            T kk[NIT];
            if (XWIN) {
                const int sh = st.x - run_x0;   // point's x offset in the window
#pragma unroll
                for (int it = 0; it < NIT; ++it) {
                    const int kx = la[it] - sh;
                    kk[it] = k2q[lb[it]] * k1q[XW + kx];   // zero padding outside [0, W)
                }
            } else {
#pragma unroll
                for (int it = 0; it < NIT; ++it) kk[it] = k2q[lb[it]] * k1q[la[it]];
            }
#pragma unroll
            for (int k = 0; k < NE; ++k) {
                const int e = e0 + k * NW;
                if (e < W) {
                    const C ck = sck3[q * W + e];
#pragma unroll
                    for (int it = 0; it < NIT; ++it) acc[k][it] = nk_fma2(ck, kk[it], acc[k][it]);
                }
            }
        }
    }
    if (run_off >= 0) flush();
    __syncthreads();
    const int o1 = corner[0] - h, o2 = corner[1] - h, o3 = corner[2] - h;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const C v = buf[i];
        if (v.x == (T)0 && v.y == (T)0) continue;
        const int q1 = i % p1;
        const int r = i / p1;
        const int q2 = r % p2;
        const int q3 = r / p2;
        int64_t l = nk_wrap(o1 + q1, g.n[0]) +
                    (int64_t)g.n[0] * (nk_wrap(o2 + q2, g.n[1]) +
                                       (int64_t)g.n[1] * nk_wrap(o3 + q3, g.n[2]));
        nk_red(fine + l, v.x, v.y);
    }
}

// Strengths in visit order for the tiled spread: cv[t][j] = c[t][perm[j]]
// (one pass per execute; the spread then streams contiguous slices by TMA).
// GV_PPT points per thread, every load issued before the first store
// (memory-level parallelism for the random 16-byte reads).
constexpr int GV_PPT = 4;
__global__ void __launch_bounds__(256)
k_gather_visit(int M, const int32_t *__restrict__ perm, const double2 *__restrict__ c,
               int64_t cpitch, double2 *__restrict__ cv, int64_t vpitch) {
    const int j0 = blockIdx.x * (256 * GV_PPT) + threadIdx.x;
    c += blockIdx.y * cpitch;
    cv += blockIdx.y * vpitch;
    int src[GV_PPT];
#pragma unroll
    for (int k = 0; k < GV_PPT; ++k) {
        const int j = j0 + k * 256;
        src[k] = j < M ? __ldg(perm + j) : -1;
    }
    double2 v[GV_PPT];
#pragma unroll
    for (int k = 0; k < GV_PPT; ++k) v[k] = src[k] >= 0 ? __ldg(c + src[k]) : make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < GV_PPT; ++k)
        if (src[k] >= 0) cv[j0 + k * 256] = v[k];
}
inline int64_t g_M(const nk_plan *p) { return p->M; }

// K6t: tiled f64 3D spread on the FP64 tensor cores (w >= 9; C4 / C5).
// The padded bin sits in shared memory as in K6c.  setpts orders each bin's
// points tile-major (nk_start_code): every point whose footprint start lies
// in one tile of 2^L start values per axis (w + 2^L - 1 <= 16) fits the
// 16 x 16 x 16-cell window anchored at the tile corner, and the group of
// all of them (C4 density: ~12 points) is spread as one small GEMM per
// window plane: warp = plane (absolute plane z == warp mod 16, so warps own
// disjoint planes and read-modify-write shared memory without atomics),
//   C[x][(y, re|im)] += sum_p k1_p[x] * (k2_p[y] (c k3_p[z]))_{re|im},
// 2 x-tiles x 4 y-tiles of DMMA m8n8k4 (K = 4 points per step) -- 1/8 of
// the issue slots of the equivalent DFMAs, at the same FP64 peak.  A lane's
// accumulator pair is one complex cell (x, y), so the group's flush is 8
// 16-byte read-modify-writes per lane.  Kernel rows are staged pre-shifted
// into the window frame (zeros outside the footprint, so planes outside a
// point's footprint contribute nothing and all-zero steps are skipped) by
// one thread per (point, axis) with degree-14 polynomial pieces (EsPoly64),
// double-buffered: batch b + 1 is staged between the barrier that retires
// batch b - 1 and the DMMAs of batch b.  Flush = native f64 reductions, one
// padded-bin row per warp pass (Eq. 17).
template <int W, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
k_spread_tiled(const int32_t *__restrict__ sub_bin, const int32_t *__restrict__ sub_start,
               const int32_t *__restrict__ sub_stop, const double *__restrict__ pts,
               int64_t pitch, const double2 *__restrict__ cvis, Geom g,
               double2 *__restrict__ fine, int64_t stage_off,
               const int32_t *__restrict__ sched, int sched_base) {
    constexpr int WIN = kTileWin, NB = kTileBatch, L = nk_tile_lg(W), TM = (1 << L) - 1;
    // NW warps; warp w owns the window planes z == w (mod NW): PL planes per
    // warp and group (16 warps x 1 plane, or 8 warps x 2 planes sharing the
    // A / k2 operand loads)
    constexpr int NWARP = NW, PL = WIN / NW;
    static_assert(WIN % NW == 0, "planes per warp");
    static_assert(W + TM <= WIN, "window too small for the tile");
    static_assert(NB <= 32, "one boundary mask word per batch");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *buf = reinterpret_cast<double2 *>(smem_raw);
    // two staging buffers: info [NB], k1 rows [NB][16], k2 rows [NB][16],
    // c k3 rows [NB][16] (complex)
    unsigned char *stg = smem_raw + stage_off;
    // rows stored transposed, [window cell][point]: a DMMA step's 4
    // consecutive points are adjacent words; k rows are padded to NB + 4
    // points so that 4 cells x 4 points of a half-warp hit distinct banks
    constexpr int KS = NB + 4;
    constexpr int SB = NB * 16 + 2 * WIN * KS * 8 + WIN * NB * 16;
    auto sinfo_of = [&](int bi) { return reinterpret_cast<int4 *>(stg + bi * SB); };
    auto sk1_of = [&](int bi) { return reinterpret_cast<double *>(stg + bi * SB + NB * 16); };
    auto sk2_of = [&](int bi) { return sk1_of(bi) + WIN * KS; };
    auto sck3_of = [&](int bi) { return reinterpret_cast<double2 *>(sk2_of(bi) + WIN * KS); };
    // raw inputs ring (3 slots, TMA bulk copies): u_axis [NB + 2] x 3, c [NB]
    constexpr int RU = NB + 2, RB = 3 * RU * 8 + NB * 16;
    unsigned char *raw = stg + 2 * SB;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(raw + 3 * RB);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = sched ? sched[sched_base + blockIdx.x] : (int)blockIdx.x;
    cvis += blockIdx.y * pitch;
    fine += blockIdx.y * g.ntot;
    int corner[3];
    nk_bin_corner(sub_bin[s], g, corner);
    const int h = g.halo;
    const int p1 = min(g.m[0], g.n[0] - corner[0]) + 2 * h;
    const int p2 = min(g.m[1], g.n[1] - corner[1]) + 2 * h;
    const int p3 = min(g.m[2], g.n[2] - corner[2]) + 2 * h;
    const int P = p1 * p2 * p3, pstride = p1 * p2;
    const double half = 0.5 * W;
    const int j0 = sub_start[s], j1 = sub_stop[s];
    // stage window rows of points [b, b + nb) into buffer bi: row v = (point
    // q, axis) runs on lane v / 16 of warp v % 16 (every warp gets its share,
    // no barrier); entry i = k[i - sh] (c folded into axis 3); the axis-1
    // thread also records the point's tile
    // TMA: batch k's coordinates and strengths into raw slot k % 3
    auto issue = [&](int k) {
        const int b = j0 + k * NB, nb = min(NB, j1 - b);
        if (nb <= 0) return;
        unsigned char *slot = raw + (k % 3) * RB;
        const int b0 = b & ~1;                           // 16-byte aligned start
        const unsigned ub = (unsigned)(((b + nb - b0) + 1) & ~1) * 8u;
        nk_fence_proxy_async();
        nk_mbar_expect_tx(mbar + k % 3, 3 * ub + 16u * nb);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax)
            nk_bulk_g2s(slot + ax * RU * 8, pts + ax * pitch + b0, ub, mbar + k % 3);
        nk_bulk_g2s(slot + 3 * RU * 8, cvis + b, 16u * nb, mbar + k % 3);
    };
    auto stage = [&](int k, int bi) {
        const int b = j0 + k * NB, nb = min(NB, j1 - b);
        int4 *sinfo = sinfo_of(bi);
        double *sk1 = sk1_of(bi), *sk2 = sk2_of(bi);
        double2 *sck3 = sck3_of(bi);
        const unsigned char *slot = raw + (k % 3) * RB;
        const double *ru = reinterpret_cast<const double *>(slot) + (b - (b & ~1));
        const double2 *rc = reinterpret_cast<const double2 *>(slot + 3 * RU * 8);
        nk_mbar_wait(mbar + k % 3, (k / 3) & 1);
        // a row's W values are split over 4 warps (pieces [part PP, part PP +
        // PP)), each warp covering 32 rows, so the staging lag of a warp is a
        // quarter of a row
        constexpr int NPART = NW == 16 ? 4 : 2, PP = (W + NPART - 1) / NPART;
        const int v = (int)threadIdx.x;
        const int part = (v >> 5) & (NPART - 1);
        const int rowi = (((v >> 5) / NPART) << 5) | (v & 31);
        if (rowi < nb * 3) {
            const int q = rowi / 3, ax = rowi - 3 * q;
            const double u = ru[ax * RU + q];
            const double st = ceil(u - half);
            const int t = (int)st + h;
            const int sh = (t - nk_tile_t0(g)) & TM;
            const double d = st - u;
            const double z0 = d * (2.0 / W), sp = fma(2.0, d, (double)(W - 1));
            double2 cv = make_double2(0.0, 0.0);
            if (ax == 2) cv = rc[q];
            double *dst = (ax == 0 ? sk1 : sk2) + q;
            double2 *dstc = sck3 + q;
            typedef EsPoly64<W> P;
#pragma unroll
            for (int r = 0; r < W; ++r) {
                if (r / PP != part) continue;   // warp-uniform
                double kv;
                if (r == 0 || r == W - 1) {
                    kv = nk_es(z0 + (2.0 * r / W), g);
                } else {
                    kv = P::c(r - 1, P::D);
#pragma unroll
                    for (int kk = P::D - 1; kk >= 0; --kk) kv = fma(kv, sp, P::c(r - 1, kk));
                }
                if (ax == 2) dstc[(sh + r) * NB] = make_double2(cv.x * kv, cv.y * kv);
                else dst[(sh + r) * KS] = kv;
            }
            if (part == NPART - 1) {   // zeros outside the footprint
#pragma unroll
                for (int i = 0; i < WIN - W; ++i) {
                    const int c0 = i < sh ? i : i + W;
                    if (ax == 2) dstc[c0 * NB] = make_double2(0.0, 0.0);
                    else dst[c0 * KS] = 0.0;
                }
            }
            if (part == 0 && ax == 0) {
                const double u2 = ru[RU + q], u3 = ru[2 * RU + q];
                const int t2 = (int)ceil(u2 - half) + h, t3 = (int)ceil(u3 - half) + h;
                // tile corner (window anchor) per axis, t3's offset in its tile
                const int o = nk_tile_t0(g);
                sinfo[q] = make_int4(nk_start_code(t, t2, t3, p1, p2, g) >> (3 * L),
                                     (o + ((t - o) & ~TM)) | ((o + ((t2 - o) & ~TM)) << 8) |
                                         ((o + ((t3 - o) & ~TM)) << 16),
                                     (t3 - o) & TM, 0);
            }
        }
    };
    // batch state: batch kb = [j0 + kb NB, +nb) in staging buffer kb & 1;
    // batch kb + 1 is staged, batch kb + 2's raw inputs are in flight.  The
    // first three batches' copies start before the bin is zeroed
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i) nk_mbar_init(mbar + i, 1);
        nk_fence_mbar_init();
        issue(0);
        issue(1);
        issue(2);
    }
    for (int i = threadIdx.x; i < P; i += blockDim.x) buf[i] = make_double2(0.0, 0.0);
    // staged rows are read up to 3 points past a segment (operands of the
    // points beyond it are multiplied by a zeroed c k3): keep them finite
    for (int i = threadIdx.x; i < 2 * SB / 16; i += blockDim.x)
        reinterpret_cast<double2 *>(stg)[i] = make_double2(0.0, 0.0);
    __syncthreads();   // barriers initialised (and the bin zeroed)
    int kb = 0;
    int nb = min(NB, j1 - j0);
    if (nb > 0) stage(0, 0);
    __syncthreads();   // batch 0 staged, bin zeroed
    if (j1 - j0 > NB) stage(1, 1);
    const int4 *sinfo = sinfo_of(0);
    const double *sk1 = sk1_of(0), *sk2 = sk2_of(0);
    const double2 *sck3 = sck3_of(0);
    // group boundaries of the current batch as a bit mask (bit q: point q
    // starts a new group), so the chunk loop knows its segment [q, qe)
    unsigned bnd = 0;
    auto boundaries = [&]() {
        const int ga = lane < nb ? sinfo[lane].x : -1;
        const int pa = __shfl_up_sync(0xffffffffu, ga, 1);
        bnd = __ballot_sync(0xffffffffu, lane < nb && (lane == 0 || ga != pa));
    };
    // retire the current batch, switch to the staged one, stage the next
    auto advance = [&]() {
        __syncthreads();   // every warp is done with batch kb; kb + 1 is staged
        ++kb;
        nb = min(NB, j1 - (j0 + kb * NB));
        if (threadIdx.x == 0) issue(kb + 2);   // into the slot batch kb - 1 used
        if (j1 - (j0 + (kb + 1) * NB) > 0) stage(kb + 1, (kb + 1) & 1);
        sinfo = sinfo_of(kb & 1);
        sk1 = sk1_of(kb & 1);
        sk2 = sk2_of(kb & 1);
        sck3 = sck3_of(kb & 1);
        if (nb > 0) boundaries();
    };
    if (nb > 0) boundaries();
    const int kp = lane & 3, row = lane >> 2, ycol = lane >> 3, cpart = (lane >> 2) & 1;
    int q = 0;
    while (nb > 0) {
        if (q == nb) {
            advance();
            q = 0;
            continue;
        }
        // a tile group (CTA-uniform control flow)
        const int4 g0 = sinfo[q];
        const int grp = g0.x;
        const int a1 = g0.y & 0xff, a2 = (g0.y >> 8) & 0xff, a3 = g0.y >> 16;
        const int e = (warp - a3) & (NW - 1);    // the warp's first window plane
        // lane (row lane / 4, column pair lane % 4) holds cell (x, y) as (re, im)
        double acc[PL][2][4][2];
#pragma unroll
        for (int pl = 0; pl < PL; ++pl)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) acc[pl][mt][nt][0] = acc[pl][mt][nt][1] = 0.0;
        for (;;) {
            // the group's segment of this batch: [q, qe)
            const unsigned rest = q + 1 < 32 ? bnd >> (q + 1) : 0u;
            const int qe = rest ? min(nb, q + __ffs(rest)) : nb;
            // chunks of 4 points (lane k-index = point cq + kp); the next
            // chunk's operands load while the current chunk's DMMAs issue
            struct Ops {
                double2 ck[PL];
                double a0, a8, k2[4], bv[PL][4];
                bool act[PL];
            };
            // lane operand pointers at point q + kp (rows padded to NB + 4
            // points; advance by 4 points per chunk)
            const double2 *pck = sck3 + e * NB + q + kp;
            const double *pa = sk1 + row * KS + q + kp;
            const double *pb = sk2 + ycol * KS + q + kp;
            auto load = [&](int cq, Ops &o) {
                const int d = cq - q;
#pragma unroll
                for (int pl = 0; pl < PL; ++pl)
                    o.ck[pl] = cq + kp < qe ? pck[pl * NW * NB + d] : make_double2(0.0, 0.0);
                o.a0 = pa[d];
                o.a8 = pa[8 * KS + d];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) o.k2[nt] = pb[nt * 4 * KS + d];
            };
            // B operands k2[y] (c k3[e]) and the plane-activity votes, one
            // pipeline stage before the DMMAs that consume them
            auto prep = [&](Ops &o) {
#pragma unroll
                for (int pl = 0; pl < PL; ++pl) {
                    // plane outside every chunk point's footprint: c k3 = 0
                    o.act[pl] = __any_sync(0xffffffffu, o.ck[pl].x != 0.0 ||
                                                                         o.ck[pl].y != 0.0);
                    const double ckc = cpart ? o.ck[pl].y : o.ck[pl].x;
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) o.bv[pl][nt] = o.k2[nt] * ckc;
                }
            };
            auto mma = [&](const Ops &o) {
#pragma unroll
                for (int pl = 0; pl < PL; ++pl) {
                    if (o.act[pl]) {
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) {
                            nk_dmma(acc[pl][0][nt][0], acc[pl][0][nt][1], o.a0, o.bv[pl][nt]);
                            nk_dmma(acc[pl][1][nt][0], acc[pl][1][nt][1], o.a8, o.bv[pl][nt]);
                        }
                    }
                }
            };
            Ops A, B;
            load(q, A);
            prep(A);
            int cq = q;
            for (;;) {
                if (cq + 4 >= qe) {
                    mma(A);
                    break;
                }
                load(cq + 4, B);
                mma(A);
                prep(B);
                cq += 4;
                if (cq + 4 >= qe) {
                    mma(B);
                    break;
                }
                load(cq + 4, A);
                mma(B);
                prep(A);
                cq += 4;
            }
            q = qe;
            if (q < nb) break;   // a new group starts inside the batch
            advance();           // the group may continue into the next batch
            q = 0;
            if (nb <= 0 || sinfo[0].x != grp) break;
        }
        // flush the warp's plane of the window; cells outside the padded bin
        // carry zero sums (footprints lie inside)
        // (all 8 loads first: the lane's cells are distinct, so no store can
        // alias a later load, which the compiler cannot prove)
        // (the window moved since the warp's last flush: a cell another lane
        // wrote then may be this lane's now -- order the warp's accesses)
        __syncwarp();
#pragma unroll
        for (int pl = 0; pl < PL; ++pl) {
            const int zpl = a3 + e + pl * NW;
            if (zpl < p3) {
                double2 *pp = buf + zpl * pstride + (a2 + kp) * p1 + a1 + row;
                bool ok[2][4];
                double2 v[2][4];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) {
                        ok[mt][nt] = a1 + mt * 8 + row < p1 && a2 + nt * 4 + kp < p2;
                        v[mt][nt] = ok[mt][nt] ? pp[nt * 4 * p1 + mt * 8] : make_double2(0.0, 0.0);
                    }
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt)
                        if (ok[mt][nt])
                            pp[nt * 4 * p1 + mt * 8] =
                                make_double2(v[mt][nt].x + acc[pl][mt][nt][0],
                                             v[mt][nt].y + acc[pl][mt][nt][1]);
            }
        }
    }
    // merge with periodic wrap (Eq. 17): one padded-bin row per thread as
    // TMA bulk reductions (UBLKRED.ADD.F64) of its 1-2 contiguous segments
    nk_fence_proxy_async();   // the flushes' generic stores before the async reads
    __syncthreads();
    const int o1 = corner[0] - h, o2 = corner[1] - h, o3 = corner[2] - h;
    bool issued = false;
    for (int r = threadIdx.x; r < p2 * p3; r += blockDim.x) {
        const int zz = r / p2, yy = r - zz * p2;
        double2 *rowp = fine + ((int64_t)nk_wrap(o3 + zz, g.n[2]) * g.n[1] +
                                nk_wrap(o2 + yy, g.n[1])) * (int64_t)g.n[0];
        const double2 *src = buf + r * p1;
        // x = o1 + k wraps periodically: contiguous segments up to the seam
        for (int k = 0; k < p1;) {
            int x = (o1 + k) % g.n[0];
            x += x < 0 ? g.n[0] : 0;
            const int seg = min(p1 - k, g.n[0] - x);
            nk_bulk_red_add(rowp + x, src + k, seg);
            k += seg;
        }
        issued = true;
    }
    if (issued) nk_bulk_wait_read();
}

// K6c-2D: one warp per subproblem.  The warp owns the whole padded bin, so
// its lanes can cover one point's w x w footprint with plain shared-memory
// read-modify-writes (distinct cells per pass, points in sequence): no
// atomics and no inter-warp conflicts.  Each lane first evaluates one
// point's kernel rows into shared memory (c folded into the axis-2 row).
// Runs of points with the same footprint start accumulate in registers.
template <typename T, int W>
__global__ void __launch_bounds__(32)
k_spread_sm2(const int32_t *__restrict__ sub_bin, const int32_t *__restrict__ sub_start,
             const int32_t *__restrict__ sub_stop, const int32_t *__restrict__ perm,
             const T *__restrict__ pts, int64_t pitch, const typename cplx<T>::t *__restrict__ c,
             Geom g, typename cplx<T>::t *__restrict__ fine, int64_t stage_off,
             const int32_t *__restrict__ sched, int sched_base) {
    typedef typename cplx<T>::t C;
    constexpr int NIT = (W * W + 31) / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *buf = reinterpret_cast<C *>(smem_raw);
    int *sbase = reinterpret_cast<int *>(smem_raw + stage_off);
    T *sk1 = reinterpret_cast<T *>(sbase + 32);
    C *sck2 = reinterpret_cast<C *>(smem_raw + stage_off + 128 + ((32 * W * sizeof(T) + 15) / 16) * 16);
    const int lane = threadIdx.x;
    const int s = sched ? sched[sched_base + blockIdx.x] : (int)blockIdx.x;
    c += blockIdx.y * g.M;          // batched execute: vector blockIdx.y
    fine += blockIdx.y * g.ntot;
    int corner[3];
    nk_bin_corner(sub_bin[s], g, corner);
    const int h = g.halo;
    const int p1 = min(g.m[0], g.n[0] - corner[0]) + 2 * h;
    const int p2 = min(g.m[1], g.n[1] - corner[1]) + 2 * h;
    const int P = p1 * p2;
    int la[NIT], lb[NIT], lofs[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const int idx = min(it * 32 + lane, W * W - 1);
        lb[it] = idx / W;
        la[it] = idx - lb[it] * W;
        lofs[it] = lb[it] * p1 + la[it];
    }
    const bool last_ok = (NIT - 1) * 32 + lane < W * W;
    for (int i = lane; i < P; i += 32) {
        C zero;
        zero.x = 0;
        zero.y = 0;
        buf[i] = zero;
    }
    C acc[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) acc[it].x = acc[it].y = 0;
    int run = -1;
    auto flush = [&]() {
        if (run < 0) return;
        __syncwarp();   // lanes' cells moved with the run start: order the accesses
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            if (it < NIT - 1 || last_ok) {
                C *cell = buf + run + lofs[it];
                C v = *cell;
                v.x += acc[it].x;
                v.y += acc[it].y;
                *cell = v;
            }
            acc[it].x = acc[it].y = 0;
        }
    };
    const int j0 = sub_start[s], j1 = sub_stop[s];
    for (int base = j0; base < j1; base += 32) {
        const int nb = min(32, j1 - base);
        __syncwarp();
        if (lane < nb) {
            const int j = base + lane;
            const C cv = c[perm[j]];
            T ka[W], k[W];
            int t1, t2;
            nk_kernel_rows2<T, W>(pts[j], pts[pitch + j], g, ka, k, t1, t2);
            t1 += h;
            t2 += h;
#pragma unroll
            for (int r = 0; r < W; ++r) sk1[lane * W + r] = ka[r];
#pragma unroll
            for (int r = 0; r < W; ++r) {
                C v;
                v.x = cv.x * k[r];
                v.y = cv.y * k[r];
                sck2[lane * W + r] = v;
            }
            sbase[lane] = t2 * p1 + t1;
        }
        __syncwarp();
        // points arrive in (bin, footprint start) order (setpts K4d): while
        // the start stays the same the lane's cells accumulate in registers;
        // a start change writes them back (read-modify-write, no atomics:
        // the warp owns the padded bin)
        for (int q = 0; q < nb; ++q) {
            const int org = sbase[q];
            if (org != run) {   // warp-uniform
                flush();
                run = org;
            }
#pragma unroll
            for (int it = 0; it < NIT; ++it)
                acc[it] = nk_fma2(sck2[q * W + lb[it]], sk1[q * W + la[it]], acc[it]);
        }
        __syncwarp();
    }
    flush();
    __syncwarp();
    const int o1 = corner[0] - h, o2 = corner[1] - h;
    for (int i = lane; i < P; i += 32) {
        const C v = buf[i];
        if (v.x == (T)0 && v.y == (T)0) continue;
        const int q1 = i % p1;
        const int q2 = i / p1;
        nk_red(fine + nk_wrap(o1 + q1, g.n[0]) + (int64_t)g.n[0] * nk_wrap(o2 + q2, g.n[1]),
               v.x, v.y);
    }
}

template <typename T, int D, int W>
int launch_w(nk_plan *p, const void *c, void *fine, int *launches) {
    typedef typename cplx<T>::t C;
    const int M = (int)p->M;
    if (M == 0) return NK_OK;
    if constexpr (D == 3 && sizeof(T) == 8 && W >= 9) {
        if (p->method == NK_SM && p->geom.tiled) {
            if (p->S == 0) return NK_OK;
            size_t smem = (size_t)p->max_sub_smem;
            // 16 warps x one window plane (default; NK_SPREAD_WARPS=8: 8 warps
            // x 2 planes sharing the A / k2 loads, measured 3 % slower)
            const char *ew = getenv("NK_SPREAD_WARPS");
            const int nw = (ew && atoi(ew) == 8) ? 8 : 16;
            auto kern = nw == 16 ? k_spread_tiled<W, 16> : k_spread_tiled<W, 8>;
            NK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
            int64_t stage_off = (p->max_pad_cells * (int64_t)sizeof(C) + 15) / 16 * 16;
            // strengths in visit order (the kernel streams them by TMA)
            const int64_t need = p->cap_M * p->ntrans;
            if (need > p->cap_cvis || !p->d_cvis) {
                if (p->d_cvis) cudaFree(p->d_cvis);
                p->d_cvis = nullptr;
                NK_CUDA(cudaMalloc(&p->d_cvis, 16 * (size_t)need));
                p->cap_cvis = need;
            }
            k_gather_visit<<<dim3((M + 256 * GV_PPT - 1) / (256 * GV_PPT), p->ntrans), 256, 0,
                             p->stream>>>(
                M, p->d_vperm, (const double2 *)c, g_M(p), (double2 *)p->d_cvis, p->cap_M);
            NK_LAUNCH_CHECK();
            ++*launches;
            for (int gi = 0; gi < std::max(p->n_det, 1); ++gi) {
                const int b0 = p->n_det ? p->h_det_off[gi] : 0;
                const int cnt = p->n_det ? p->h_det_off[gi + 1] - b0 : (int)p->S;
                kern<<<dim3((unsigned)cnt, p->ntrans), nw * 32, smem, p->stream>>>(
                    p->d_sub_bin, p->d_sub_start, p->d_sub_stop, (const double *)p->d_pts,
                    p->cap_M, (const double2 *)p->d_cvis, p->geom, (double2 *)fine, stage_off,
                    p->d_sub_sched, b0);
                NK_LAUNCH_CHECK();
                ++*launches;
            }
            return NK_OK;
        }
    }
    if (p->method == NK_SM && D == 3) {
        if (p->S == 0) return NK_OK;
        size_t smem = (size_t)p->max_sub_smem;
        constexpr int NW = nk_sm3_warps(W);
        auto kern = k_spread_sm3<T, W, NW>;
        NK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        int64_t stage_off = (p->max_pad_cells * (int64_t)sizeof(C) + 15) / 16 * 16;
        for (int gi = 0; gi < std::max(p->n_det, 1); ++gi) {
            const int b0 = p->n_det ? p->h_det_off[gi] : 0;
            const int cnt = p->n_det ? p->h_det_off[gi + 1] - b0 : (int)p->S;
            kern<<<dim3((unsigned)cnt, p->ntrans), NW * 32, smem, p->stream>>>(
                p->d_sub_bin, p->d_sub_start, p->d_sub_stop, p->d_vperm, (const T *)p->d_pts,
                p->cap_M, (const C *)c, p->geom, (C *)fine, stage_off, nk_sm3_batch(p->prec),
                p->n_det ? p->d_sub_sched : nullptr, b0);
            if (gi + 1 < p->n_det) ++*launches;
        }
    } else if (p->method == NK_SM && D == 2) {
        if (p->S == 0) return NK_OK;
        size_t smem = (size_t)p->max_sub_smem;
        auto kern = k_spread_sm2<T, W>;
        NK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        int64_t stage_off = (p->max_pad_cells * (int64_t)sizeof(C) + 15) / 16 * 16;
        for (int gi = 0; gi < std::max(p->n_det, 1); ++gi) {
            const int b0 = p->n_det ? p->h_det_off[gi] : 0;
            const int cnt = p->n_det ? p->h_det_off[gi + 1] - b0 : (int)p->S;
            kern<<<dim3((unsigned)cnt, p->ntrans), 32, smem, p->stream>>>(
                p->d_sub_bin, p->d_sub_start, p->d_sub_stop, p->d_vperm, (const T *)p->d_pts,
                p->cap_M, (const C *)c, p->geom, (C *)fine, stage_off,
                p->n_det ? p->d_sub_sched : nullptr, b0);
            if (gi + 1 < p->n_det) ++*launches;
        }
    } else {
        const int32_t *perm = p->method == NK_GM ? nullptr : p->d_vperm;
        k_spread_gm<T, D, W><<<dim3((M + 255) / 256, p->ntrans), 256, 0, p->stream>>>(
            M, perm, p->d_keys, (const T *)p->d_pts, p->cap_M, (const C *)c, p->geom, (C *)fine);
    }
    NK_LAUNCH_CHECK();
    ++*launches;
    return NK_OK;
}

template <typename T, int D>
int launch_d(nk_plan *p, const void *c, void *fine, int *launches) {
    switch (p->w) {
#define NK_W(W) \
    case W: return launch_w<T, D, W>(p, c, fine, launches);
        NK_W(2) NK_W(3) NK_W(4) NK_W(5) NK_W(6) NK_W(7) NK_W(8) NK_W(9) NK_W(10) NK_W(11)
        NK_W(12) NK_W(13) NK_W(14) NK_W(15) NK_W(16)
#undef NK_W
    }
    nk_set_error("unsupported kernel width");
    return NK_ERR_VALUE;
}

}  // namespace

int nk_launch_spread(nk_plan *p, const void *c, void *fine, int *launches) {
    NK_CUDA(cudaMemsetAsync(fine, 0, p->n_tot * p->csize * p->ntrans, p->stream));
    if (p->prec == NK_DOUBLE)
        return p->dim == 2 ? launch_d<double, 2>(p, c, fine, launches)
                           : launch_d<double, 3>(p, c, fine, launches);
    return p->dim == 2 ? launch_d<float, 2>(p, c, fine, launches)
                       : launch_d<float, 3>(p, c, fine, launches);
}
