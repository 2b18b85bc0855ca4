// setpts hot path: FP64 fold + bin key + histogram (K1), exclusive scans
// (K2), stable LSD radix sort of bin keys -> permutation (K3), subproblem
// table (K4) and the sorted local-coordinate gather (K5).
//
// Bit-exact targets: binsort.py:91-131 (fold, cells, keys), :149-153
// (bincount, cumsum, stable argsort), :166-219 (build_subproblems).
#include <limits.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "nk_device.cuh"

namespace {

constexpr int SORT_BLOCK = 256;
constexpr int SORT_ITEMS = 16;
constexpr int SORT_TILE = SORT_BLOCK * SORT_ITEMS;  // keys per tile
constexpr int SORT_WARPS = SORT_BLOCK / 32;
constexpr int RADIX_BITS = 8;
constexpr int RADIX = 1 << RADIX_BITS;

constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_CHUNK = SCAN_BLOCK * SCAN_ITEMS;

// ---------------------------------------------------------------- K1
// One thread per input point: fold each axis in FP64 exactly like
// grid_coords, clamp the cell, flatten the bin key (axis 1 fastest).  Only
// unsorted (GM) plans count here (warp-aggregated atomics); sorted plans
// derive counts/starts from the sorted keys (K2b), free of the same-address
// atomic contention (2.4k increments per bin at C2).
// Each thread folds FOLD_PPT points (256-strided, coalesced): every point's
// coordinate loads are issued before the first fold, so a warp keeps
// FOLD_PPT x the bytes in flight (C2: one point per thread ran at ~2.5 TB/s,
// latency bound).
constexpr int FOLD_PPT = 4;

template <typename TC, typename T>
__global__ void __launch_bounds__(256)
k_fold_keys(int M, const TC *__restrict__ x, const TC *__restrict__ y,
            const TC *__restrict__ z, int64_t stride, Geom g, int32_t *__restrict__ keys,
            int32_t *__restrict__ counts, unsigned long long *__restrict__ bad,
            int32_t *__restrict__ ckeys, int sb, T *__restrict__ rec) {
    const int i0 = blockIdx.x * (256 * FOLD_PPT) + threadIdx.x;
    const TC *ax[3] = {x, y, z};
    const T halfw = (T)(0.5 * g.w);
    double xin[FOLD_PPT][3];
#pragma unroll
    for (int k = 0; k < FOLD_PPT; ++k)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int i = i0 + k * 256;
            xin[k][a] = a < g.dim && i < M ? (double)ax[a][(int64_t)i * stride] : 0.0;
        }
#pragma unroll
    for (int k = 0; k < FOLD_PPT; ++k) {
        const int i = i0 + k * 256;
        const bool in = i < M;
        const unsigned mask = __ballot_sync(0xffffffffu, in);
        if (!in) continue;   // every lane still reaches the next point's ballot
        int key = 0, kstride = 1;
        int t[3] = {0, 0, 0}, pd[3] = {1, 1, 1};
        T u[3] = {0, 0, 0};
        bool ok = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (a < g.dim) {
                const double xv = xin[k][a];
                if (!isfinite(xv)) ok = false;
                double v = ok ? nk_fold(xv, g.scale[a]) : 0.0;
                // cell = clamp(floor(v), 0, n - 1) (nk_cell; v is finite and in
                // [0, n] here) with one conversion; bin by multiply-high
                const int c = min(max(__double2int_rd(v), 0), g.n[a] - 1);
                const int b = g.mdiv[a] ? (int)__umulhi((unsigned)c, g.mdiv[a]) : c / g.m[a];
                key += kstride * b;
                kstride *= g.nb[a];
                // local coordinate in plan precision (K5: the visit-order
                // gather copies these records) and, for SM plans, the
                // footprint start in the bin's padded frame from the same value
                const int corner = b * g.m[a];
                u[a] = (T)(v - (double)corner);
                if (ckeys) {
                    t[a] = (int)nk_ceil<T>(u[a] - halfw) + g.halo;
                    pd[a] = min(g.m[a], g.n[a] - corner) + 2 * g.halo;
                }
            }
        }
        if (!ok) {
            atomicMin(bad, (unsigned long long)i);
            key = 0;
            t[0] = t[1] = t[2] = 0;
            u[0] = u[1] = u[2] = 0;
        }
        keys[i] = key;
        // record (u1, u2[, u3, 0]): one aligned 8/16/32-byte vector per point
        if (g.dim == 3) {
            if constexpr (sizeof(T) == 8) {
                double2 *r = reinterpret_cast<double2 *>(rec) + 2 * (int64_t)i;
                r[0] = make_double2(u[0], u[1]);
                r[1] = make_double2(u[2], 0.0);
            } else {
                reinterpret_cast<float4 *>(rec)[i] = make_float4(u[0], u[1], u[2], 0.0f);
            }
        } else {
            if constexpr (sizeof(T) == 8)
                reinterpret_cast<double2 *>(rec)[i] = make_double2(u[0], u[1]);
            else
                reinterpret_cast<float2 *>(rec)[i] = make_float2(u[0], u[1]);
        }
        if (ckeys)
            ckeys[i] = (int32_t)(((unsigned)key << sb) |
                                 (unsigned)nk_start_code(t[0], t[1], t[2], pd[0], pd[1], g));
        if (counts) {
            unsigned peers = __match_any_sync(mask, key);
            if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&counts[key], __popc(peers));
        }
    }
}

// ---------------------------------------------------------------- K2b
// starts[b] = first sorted position with key >= b (length nbins + 1, so
// starts[nbins] = M) from the bin-sorted keys; counts = adjacent
// differences.  Identical to bincount + exclusive cumsum (binsort.py:149-151).
// One thread per bin, lower_bound over the sorted keys: O(nbins log M),
// independent of how the points cluster (empty-bin runs cost nothing).
__global__ void __launch_bounds__(256)
k_bin_starts(int M, int nbins, const int32_t *__restrict__ skeys, int sb,
             int32_t *__restrict__ starts) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nbins) return;
    // (composite keys carry the bin in the bits above sb; sorted as unsigned)
    int lo = 0, hi = M;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int)((unsigned)__ldg(skeys + mid) >> sb) < b) lo = mid + 1;
        else hi = mid;
    }
    starts[b] = lo;
}

// sum_b counts[b]^2 (point-weighted bin density for the visit-order choice)
__global__ void __launch_bounds__(256)
k_sum_sq(int nbins, const int32_t *__restrict__ counts, unsigned long long *__restrict__ out) {
    unsigned long long acc = 0;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nbins; b += gridDim.x * blockDim.x) {
        const unsigned long long c = (unsigned)counts[b];
        acc += c * c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

__global__ void __launch_bounds__(256)
k_counts_from_starts(int nbins, const int32_t *__restrict__ starts, int32_t *__restrict__ counts) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nbins) counts[b] = starts[b + 1] - starts[b];
}

// ---------------------------------------------------------------- K2
// Three-phase exclusive scan of int32: out[0..n] with out[n] = total.
__device__ __forceinline__ int pad_idx(int i) { return i + (i >> 4); }

__device__ __forceinline__ int warp_incl_scan(int v) {
    int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ int block_excl_scan(int v, int *total) {
    __shared__ int wsum[33];
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = warp_incl_scan(v);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int nw = blockDim.x >> 5;
        int s = lane < nw ? wsum[lane] : 0;
        int si = warp_incl_scan(s);
        if (lane < nw) wsum[lane] = si - s;
        if (lane == nw - 1) wsum[32] = si;
    }
    __syncthreads();
    int res = inc - v + wsum[warp];
    *total = wsum[32];
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_reduce(const int32_t *__restrict__ in, int64_t n, int32_t *__restrict__ partials) {
    int64_t base = (int64_t)blockIdx.x * SCAN_CHUNK;
    int s = 0;
    for (int it = 0; it < SCAN_ITEMS; ++it) {
        int64_t i = base + it * SCAN_BLOCK + threadIdx.x;
        if (i < n) s += in[i];
    }
    int tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_partials(int32_t *partials, int np) {
    int carry = 0;
    for (int base = 0; base < np; base += blockDim.x) {
        int i = base + threadIdx.x;
        int v = i < np ? partials[i] : 0;
        int tot;
        int ex = block_excl_scan(v, &tot);
        if (i < np) partials[i] = ex + carry;
        carry += tot;
    }
}

__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_down(const int32_t *in, int64_t n, const int32_t *__restrict__ partials,
            int32_t *out) {   // in may alias out
    __shared__ int buf[SCAN_CHUNK + SCAN_CHUNK / 16];
    int64_t base = (int64_t)blockIdx.x * SCAN_CHUNK;
    for (int it = 0; it < SCAN_ITEMS; ++it) {
        int li = it * SCAN_BLOCK + threadIdx.x;
        int64_t i = base + li;
        buf[pad_idx(li)] = i < n ? in[i] : 0;
    }
    __syncthreads();
    int loc[SCAN_ITEMS];
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        loc[k] = s;
        s += buf[pad_idx(threadIdx.x * SCAN_ITEMS + k)];
    }
    int tot;
    int ex = block_excl_scan(s, &tot) + partials[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) buf[pad_idx(threadIdx.x * SCAN_ITEMS + k)] = loc[k] + ex;
    __syncthreads();
    for (int it = 0; it < SCAN_ITEMS; ++it) {
        int li = it * SCAN_BLOCK + threadIdx.x;
        int64_t i = base + li;
        if (i < n) out[i] = buf[pad_idx(li)];
    }
    // in may alias out: the grand total comes from the scanned partials
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = partials[blockIdx.x] + tot;
}

// ---------------------------------------------------------------- K3
// Stable LSD radix sort, 8-bit digits, 4096-key tiles.  Upsweep: per-tile
// digit histogram stored digit-major; the (digit, tile) matrix is
// exclusive-scanned; downsweep ranks each key stably inside its tile
// (warp-striped order, __match_any_sync peers + per-warp digit counters)
// and scatters (key, value) to its global slot.
__global__ void __launch_bounds__(SORT_BLOCK)
k_radix_hist(const int32_t *__restrict__ keys, int M, int shift, int dmask, int ntiles,
             int32_t *__restrict__ hist) {
    // per-warp digit histograms with native shared integer atomics (no
    // match.any: ranks are not needed here), 16-byte key loads
    __shared__ int h[SORT_WARPS][RADIX];
    for (int i = threadIdx.x; i < SORT_WARPS * RADIX; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const int base = blockIdx.x * SORT_TILE + threadIdx.x * SORT_ITEMS;
    if (base + SORT_ITEMS <= M) {
        const int4 *k4 = reinterpret_cast<const int4 *>(keys + base);
#pragma unroll
        for (int v = 0; v < SORT_ITEMS / 4; ++v) {
            const int4 q = __ldg(k4 + v);
            atomicAdd(&h[warp][(q.x >> shift) & dmask], 1);
            atomicAdd(&h[warp][(q.y >> shift) & dmask], 1);
            atomicAdd(&h[warp][(q.z >> shift) & dmask], 1);
            atomicAdd(&h[warp][(q.w >> shift) & dmask], 1);
        }
    } else {
        for (int it = 0; it < SORT_ITEMS; ++it)
            if (base + it < M) atomicAdd(&h[warp][(keys[base + it] >> shift) & dmask], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < RADIX; i += blockDim.x) {
        int t = 0;
#pragma unroll
        for (int w = 0; w < SORT_WARPS; ++w) t += h[w][i];
        hist[(int64_t)i * ntiles + blockIdx.x] = t;
    }
}

template <int DB>
__global__ void __launch_bounds__(SORT_BLOCK)
k_radix_scatter(const int32_t *__restrict__ keys_in, const int32_t *__restrict__ vals_in,
                int M, int shift, int ntiles, const int32_t *__restrict__ offs,
                int32_t *__restrict__ keys_out, int32_t *__restrict__ vals_out) {
    // 1) stable ranks inside each warp's slice (8 ballots per item, per-warp
    //    digit counters); 2) the tile is reordered by digit in shared memory;
    //    3) written out in that order, so consecutive threads store
    //    consecutive slots of each digit's run (coalesced; a 4096-key tile
    //    gives runs of ~16 keys per digit instead of scattered words)
    __shared__ int wcnt[SORT_WARPS][RADIX];
    __shared__ int lstart[RADIX], gstart[RADIX];
    __shared__ int skey[SORT_TILE], sval[SORT_TILE];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < SORT_WARPS * RADIX; i += blockDim.x) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int tbase = blockIdx.x * SORT_TILE;
    const int base = tbase + warp * 32 * SORT_ITEMS;
    const unsigned lt = (1u << lane) - 1u;
    constexpr int dmask = (1 << DB) - 1;
    int key[SORT_ITEMS], val[SORT_ITEMS], rank[SORT_ITEMS];
    // all of the warp's loads in flight before the ranking (the ranking's
    // ballots / shuffles would otherwise wait on each load in turn)
#pragma unroll
    for (int it = 0; it < SORT_ITEMS; ++it) {
        const int idx = base + it * 32 + lane;
        key[it] = idx < M ? __ldcs(keys_in + idx) : 0;
        val[it] = idx < M ? (vals_in ? __ldcs(vals_in + idx) : idx) : 0;
    }
#pragma unroll
    for (int it = 0; it < SORT_ITEMS; ++it) {
        int idx = base + it * 32 + lane;
        bool valid = idx < M;
        const int d = (key[it] >> shift) & dmask;
        unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int b = 0; b < DB; ++b) {
            const unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1);
            peers &= ((d >> b) & 1) ? bb : ~bb;
        }
        // the digit group's leader bumps the warp's counter (native shared
        // integer atomic; a warp's atomics land in program order, so ranks
        // stay stable) and broadcasts the old value -- no read / write
        // round trip through shared memory between consecutive items
        const int leader = __ffs(peers) - 1;
        int c = 0;
        if (valid && lane == leader) c = atomicAdd(&wcnt[warp][d], __popc(peers));
        c = __shfl_sync(0xffffffffu, c, valid ? leader : lane);
        rank[it] = valid ? c + __popc(peers & lt) : -1;
    }
    __syncthreads();
    // digit d (thread d): per-warp exclusive offsets inside the digit, the
    // digit's tile total, its global start (scanned upsweep histogram)
    int tot = 0;
    for (int d = threadIdx.x; d < RADIX; d += blockDim.x) {
#pragma unroll
        for (int w = 0; w < SORT_WARPS; ++w) {
            const int cnt = wcnt[w][d];
            wcnt[w][d] = tot;
            tot += cnt;
        }
        gstart[d] = offs[(int64_t)d * ntiles + blockIdx.x];
    }
    int tile_tot;
    static_assert(RADIX == SORT_BLOCK, "one digit per thread");
    const int ex = block_excl_scan(tot, &tile_tot);
    lstart[threadIdx.x] = ex;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < SORT_ITEMS; ++it) {
        if (rank[it] >= 0) {
            const int d = (key[it] >> shift) & dmask;
            const int lp = lstart[d] + wcnt[warp][d] + rank[it];
            skey[lp] = key[it];
            sval[lp] = val[it];
        }
    }
    __syncthreads();
    const int n = min(SORT_TILE, M - tbase);
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int k = skey[t];
        const int d = (k >> shift) & dmask;
        const int pos = gstart[d] + (t - lstart[d]);
        keys_out[pos] = k;
        vals_out[pos] = sval[t];
    }
}

// ---------------------------------------------------------------- K4
__global__ void k_nsub(const int32_t *__restrict__ counts, int nbins, int msub,
                       int32_t *__restrict__ nsub) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nbins) nsub[b] = (counts[b] + msub - 1) / msub;   // binsort.py:183
}

// One thread per subproblem: binary-search its bin in the scanned
// per-bin subproblem counts, then slice (binsort.py:203-211).
__global__ void k_fill_subs(int S, const int32_t *__restrict__ nsub_off, int nbins,
                            const int32_t *__restrict__ starts, int msub,
                            int32_t *__restrict__ sub_bin, int32_t *__restrict__ sub_start,
                            int32_t *__restrict__ sub_stop) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    int lo = 0, hi = nbins - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (nsub_off[mid] <= s) lo = mid;
        else hi = mid - 1;
    }
    int b = lo;
    int r = s - nsub_off[b];
    int st = starts[b] + r * msub;
    int en = min(st + msub, starts[b + 1]);
    sub_bin[s] = b;
    sub_start[s] = st;
    sub_stop[s] = en;
}

__global__ void k_export_subs(int S, Geom g, const int32_t *__restrict__ sub_bin,
                              int32_t *__restrict__ offsets, int32_t *__restrict__ padded) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    int corner[3];
    nk_bin_corner(sub_bin[s], g, corner);
    for (int a = 0; a < g.dim; ++a) {
        int actual = min(g.m[a], g.n[a] - corner[a]);     // binsort.py:200
        if (offsets) offsets[s * g.dim + a] = corner[a] - g.halo;   // :207
        if (padded) padded[s * g.dim + a] = actual + 2 * g.halo;    // :208
    }
}

// ---------------------------------------------------------------- K4m
// Subproblem schedule of the tiled f64 kernels: Morton (Z-order) key of the
// bin, so the CTAs in flight cover a compact block of bins and the halo
// reductions (spread) / halo re-reads (interp) of neighbouring bins hit L2
// (the bin-major order walks a whole 512^2 x halo slab between z-neighbours).
__device__ __forceinline__ unsigned nk_spread_bits3(unsigned v) {   // 10 bits -> every 3rd
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__global__ void k_sched_keys(int S, const int32_t *__restrict__ sub_bin, Geom g,
                             int32_t *__restrict__ keys) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const int b = sub_bin[s];
    const int bx = b % g.nb[0], r = b / g.nb[0];
    const int by = r % g.nb[1], bz = r / g.nb[1];
    keys[s] = (int32_t)(nk_spread_bits3(bx) | (nk_spread_bits3(by) << 1) |
                        (nk_spread_bits3(bz) << 2));
}

// ---------------------------------------------------------------- K4k
// Deterministic type-1 merge order: key = rank of the subproblem inside its
// bin x colours + colour of its bin, colour = per-axis class of bins whose
// padded extents (m + 2 halo) cannot overlap, periodic seam included
// (classes b mod c for the first nb - nb mod c bins, one class each for the
// remainder).  Launched class by class, every fine-grid cell receives at
// most one merge per launch: the summation order is fixed.
__global__ void k_det_keys(int S, const int32_t *__restrict__ sub_bin,
                           const int32_t *__restrict__ nsub_off, Geom g, int3 cc, int3 ncol,
                           int32_t *__restrict__ keys) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const int b = sub_bin[s];
    int c[3] = {b % g.nb[0], 0, 0};
    const int r = b / g.nb[0];
    c[1] = g.dim == 3 ? r % g.nb[1] : r;
    c[2] = g.dim == 3 ? r / g.nb[1] : 0;
    const int cs[3] = {cc.x, cc.y, cc.z};
    int col[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int rem = g.nb[a] % cs[a], reg = g.nb[a] - rem;
        col[a] = c[a] < reg ? c[a] % cs[a] : cs[a] + (c[a] - reg);
    }
    const int color = col[0] + ncol.x * (col[1] + ncol.y * col[2]);
    const int rank = s - nsub_off[b];
    keys[s] = rank * (ncol.x * ncol.y * ncol.z) + color;
}

// ---------------------------------------------------------------- K5
// Visit-order local coordinates u = v - bin corner, in plan precision
// (a float keeps ~4e-6 cell resolution inside a 32-cell bin where a float
// global v would lose 1e-4 cells at n = 2048).  K1 wrote each point's
// coordinates as one aligned record in input order; this gathers the
// records through the visit permutation (one sector per point instead of
// one per coordinate) and writes them as SoA rows.
// FOLD_PPT points per thread, all permutation and record loads issued
// before the first store (memory-level parallelism for the random reads).
template <typename T, int D>
__device__ __forceinline__ void load_rec(const T *__restrict__ rec, int64_t i, T *u) {
    if constexpr (D == 3 && sizeof(T) == 8) {
        const double2 a = __ldg(reinterpret_cast<const double2 *>(rec) + 2 * i);
        u[0] = a.x;
        u[1] = a.y;
        u[2] = __ldg(rec + 4 * i + 2);
    } else if constexpr (D == 3) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(rec) + i);
        u[0] = a.x;
        u[1] = a.y;
        u[2] = a.z;
    } else if constexpr (sizeof(T) == 8) {
        const double2 a = __ldg(reinterpret_cast<const double2 *>(rec) + i);
        u[0] = a.x;
        u[1] = a.y;
    } else {
        const float2 a = __ldg(reinterpret_cast<const float2 *>(rec) + i);
        u[0] = a.x;
        u[1] = a.y;
    }
}

template <typename T, int D>
__global__ void __launch_bounds__(256)
k_gather_points(int M, const int32_t *__restrict__ perm, const T *__restrict__ rec,
                T *__restrict__ pts, int64_t pitch) {
    const int j0 = blockIdx.x * (256 * FOLD_PPT) + threadIdx.x;
    int src[FOLD_PPT];
#pragma unroll
    for (int k = 0; k < FOLD_PPT; ++k) {
        const int j = j0 + k * 256;
        src[k] = j < M ? (perm ? __ldcs(perm + j) : j) : -1;
    }
    T u[FOLD_PPT][D];
#pragma unroll
    for (int k = 0; k < FOLD_PPT; ++k)
        if (src[k] >= 0) load_rec<T, D>(rec, src[k], u[k]);
#pragma unroll
    for (int k = 0; k < FOLD_PPT; ++k) {
        const int j = j0 + k * 256;
        if (src[k] < 0) continue;
#pragma unroll
        for (int a = 0; a < D; ++a) pts[a * pitch + j] = u[k][a];
    }
}

// ---------------------------------------------------------------- K4b
// Visit-order refinement for the staged interpolation (type 2, SM): inside
// each subproblem, deal points round-robin over the shared-memory bank
// residue of their footprint origin, so that the G lanes of one shared
// memory wavefront (16 for 8-byte, 8 for 16-byte complex) gather from
// distinct banks for every footprint cell.  Ranks inside a residue bucket
// follow the sorted order, so the permutation is deterministic.  Only the
// visit order changes; the exported bin-stable layout is untouched.
template <typename T>
__global__ void __launch_bounds__(256)
k_refine_interleave(const int32_t *__restrict__ sub_bin, const int32_t *__restrict__ sub_start,
                    const int32_t *__restrict__ sub_stop, const int32_t *__restrict__ perm_in,
                    const T *__restrict__ pts_in, int64_t pitch, Geom g, int G,
                    int32_t *__restrict__ scratch, int32_t *__restrict__ perm_out,
                    T *__restrict__ pts_out) {
    __shared__ int cnt[16];
    __shared__ int wcnt[8][16];
    extern __shared__ int round_start[];   // max bucket size + 1
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x;
    int corner[3];
    nk_bin_corner(sub_bin[s], g, corner);
    const int h = g.halo;
    const int p1 = min(g.m[0], g.n[0] - corner[0]) + 2 * h;
    const int p2 = min(g.m[1], g.n[1] - corner[1]) + 2 * h;
    const int j0 = sub_start[s], j1 = sub_stop[s];
    if (threadIdx.x < 16) cnt[threadIdx.x] = 0;
    const unsigned lt = (1u << lane) - 1u;
    const T half = (T)(0.5 * g.w);
    for (int base = j0; base < j1; base += blockDim.x) {
        const int j = base + threadIdx.x;
        const bool valid = j < j1;
        int r = 16;
        if (valid) {
            int t1 = (int)nk_ceil<T>(pts_in[j] - half) + h;
            int t2 = (int)nk_ceil<T>(pts_in[pitch + j] - half) + h;
            int t3 = g.dim == 3 ? (int)nk_ceil<T>(pts_in[2 * pitch + j] - half) + h : 0;
            r = ((t3 * p2 + t2) * p1 + t1) & (G - 1);
        }
        if (threadIdx.x < 128) (&wcnt[0][0])[threadIdx.x] = 0;
        __syncthreads();
        unsigned peers = __match_any_sync(0xffffffffu, r);
        if (valid && lane == __ffs(peers) - 1) wcnt[warp][r] = __popc(peers);
        __syncthreads();
        if (threadIdx.x < 16) {
            int run = cnt[threadIdx.x];
            for (int w = 0; w < 8; ++w) {
                int c = wcnt[w][threadIdx.x];
                wcnt[w][threadIdx.x] = run;
                run += c;
            }
            cnt[threadIdx.x] = run;
        }
        __syncthreads();
        if (valid) scratch[j] = ((wcnt[warp][r] + __popc(peers & lt)) << 4) | r;
        __syncthreads();
    }
    // round k holds the k-th point of every bucket larger than k
    int maxsz = 0;
    for (int r = 0; r < G; ++r) maxsz = max(maxsz, cnt[r]);
    int carry = 0;
    for (int k0 = 0; k0 < maxsz; k0 += blockDim.x) {
        const int k = k0 + threadIdx.x;
        int nk = 0;
        if (k < maxsz)
            for (int r = 0; r < G; ++r) nk += cnt[r] > k;
        int tot;
        int ex = block_excl_scan(nk, &tot);
        if (k < maxsz) round_start[k] = carry + ex;
        carry += tot;
    }
    __syncthreads();
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
        const int v = scratch[j];
        const int rank = v >> 4, r = v & 15;
        int pos = round_start[rank];
        for (int q = 0; q < r; ++q) pos += cnt[q] > rank;
        const int d = j0 + pos;
        perm_out[d] = perm_in[j];
        for (int a = 0; a < g.dim; ++a) pts_out[a * pitch + d] = pts_in[a * pitch + j];
    }
}

// ---------------------------------------------------------------- K4c/K4d
// Visit order (bin, footprint start): start offset of every point in its
// bin's padded frame, from the visit-order local coordinates (the same
// T-precision ceil the spread / interp kernels evaluate).  Type 1: points
// sharing a footprint are adjacent (register run accumulation).  Type 2
// (single precision): a warp's 32 gathers of one padded-bin row hit adjacent
// words (one shared-memory wavefront).
template <typename T>
__global__ void __launch_bounds__(256)
k_start_keys(int M, const int32_t *__restrict__ bin_keys, const T *__restrict__ pts,
             int64_t pitch, Geom g, int32_t *__restrict__ skeys) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    int corner[3];
    nk_bin_corner(bin_keys[j], g, corner);
    const int h = g.halo;
    const int p1 = min(g.m[0], g.n[0] - corner[0]) + 2 * h;
    const int p2 = min(g.m[1], g.n[1] - corner[1]) + 2 * h;
    const T half = (T)(0.5 * g.w);
    const int t1 = (int)nk_ceil<T>(pts[j] - half) + h;
    const int t2 = (int)nk_ceil<T>(pts[pitch + j] - half) + h;
    const int t3 = g.dim == 3 ? (int)nk_ceil<T>(pts[2 * pitch + j] - half) + h : 0;
    skeys[j] = nk_start_code(t1, t2, t3, p1, p2, g);
}

__global__ void k_gather_i32(int M, const int32_t *__restrict__ idx,
                             const int32_t *__restrict__ src, int32_t *__restrict__ dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < M) dst[i] = src[idx[i]];
}

template <typename T>
__global__ void k_reorder_points(int M, int dim, const int32_t *__restrict__ q,
                                 const int32_t *__restrict__ perm_in, const T *__restrict__ pts_in,
                                 int64_t pitch, int32_t *__restrict__ perm_out,
                                 T *__restrict__ pts_out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int src = q[i];
    perm_out[i] = perm_in[src];
    for (int a = 0; a < dim; ++a) pts_out[a * pitch + i] = pts_in[a * pitch + src];
}

template <typename T>
int grow(T **ptr, int64_t *cap, int64_t need) {
    if (need <= *cap && *ptr) return NK_OK;
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    int64_t n = std::max<int64_t>(need, 1);
    NK_CUDA(cudaMalloc((void **)ptr, sizeof(T) * n));
    *cap = n;
    return NK_OK;
}

inline unsigned blocks_for(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

int nk_scan_exclusive(nk_plan *p, const int32_t *in, int32_t *out, int64_t n) {
    if (n <= 0) {
        NK_CUDA(cudaMemsetAsync(out, 0, sizeof(int32_t), p->stream));
        return NK_OK;
    }
    int64_t np = (n + SCAN_CHUNK - 1) / SCAN_CHUNK;
    int rc = grow(&p->d_scan_tmp, &p->cap_scan_tmp, np);
    if (rc) return rc;
    k_scan_reduce<<<(unsigned)np, SCAN_BLOCK, 0, p->stream>>>(in, n, p->d_scan_tmp);
    k_scan_partials<<<1, 1024, 0, p->stream>>>(p->d_scan_tmp, (int)np);
    k_scan_down<<<(unsigned)np, SCAN_BLOCK, 0, p->stream>>>(in, n, p->d_scan_tmp, out);
    NK_LAUNCH_CHECK();
    return NK_OK;
}

static int ensure_point_buffers(nk_plan *p, int64_t M) {
    if (M <= p->cap_M && p->d_keys) return NK_OK;
    void **bufs[] = {(void **)&p->d_keys_in, (void **)&p->d_keys, (void **)&p->d_perm,
                     (void **)&p->d_alt_keys, (void **)&p->d_alt_vals, &p->d_pts,
                     (void **)&p->d_vperm_buf, &p->d_pts_alt, (void **)&p->d_sort_scr,
                     &p->d_rec};
    for (void **b : bufs) {
        if (*b) cudaFree(*b);
        *b = nullptr;
    }
    // pitch: a multiple of 16 elements plus 16 of slack, so 16-byte chunked
    // copies of any [j0, j1) slice (the staged interpolation) stay in bounds
    int64_t n = (std::max<int64_t>(M, 1) + 15) / 16 * 16 + 16;
    NK_CUDA(cudaMalloc((void **)&p->d_keys_in, 4 * n));
    NK_CUDA(cudaMalloc((void **)&p->d_keys, 4 * n));
    NK_CUDA(cudaMalloc((void **)&p->d_perm, 4 * n));
    NK_CUDA(cudaMalloc((void **)&p->d_alt_keys, 4 * n));
    NK_CUDA(cudaMalloc((void **)&p->d_alt_vals, 4 * n));
    NK_CUDA(cudaMalloc(&p->d_pts, (size_t)p->csize / 2 * p->dim * n));
    NK_CUDA(cudaMalloc(&p->d_rec, (size_t)p->csize / 2 * (p->dim == 3 ? 4 : 2) * n));
    if (p->method == NK_SM)
        NK_CUDA(cudaMalloc((void **)&p->d_sort_scr, 4 * 4 * n));
    if (p->method == NK_SM) {
        NK_CUDA(cudaMalloc((void **)&p->d_vperm_buf, 4 * n));
        NK_CUDA(cudaMalloc(&p->d_pts_alt, (size_t)p->csize / 2 * p->dim * n));
    }
    p->cap_M = n;
    return NK_OK;
}

template <typename TC>
static int fold_keys(nk_plan *p, const void *x, const void *y, const void *z, int64_t stride,
                     int32_t *ckeys, int sb) {
    int M = (int)p->M;
    if (p->prec == NK_DOUBLE)
        k_fold_keys<TC, double><<<blocks_for(M, 256 * FOLD_PPT), 256, 0, p->stream>>>(
            M, (const TC *)x, (const TC *)y, (const TC *)z, stride, p->geom, p->d_keys_in,
            p->method == NK_GM ? p->d_counts : nullptr, p->d_bad, ckeys, sb, (double *)p->d_rec);
    else
        k_fold_keys<TC, float><<<blocks_for(M, 256 * FOLD_PPT), 256, 0, p->stream>>>(
            M, (const TC *)x, (const TC *)y, (const TC *)z, stride, p->geom, p->d_keys_in,
            p->method == NK_GM ? p->d_counts : nullptr, p->d_bad, ckeys, sb, (float *)p->d_rec);
    NK_LAUNCH_CHECK();
    return NK_OK;
}

template <typename T>
static int gather(nk_plan *p, const int32_t *perm) {
    int M = (int)p->M;
    if (p->dim == 3)
        k_gather_points<T, 3><<<blocks_for(M, 256 * FOLD_PPT), 256, 0, p->stream>>>(
            M, perm, (const T *)p->d_rec, (T *)p->d_pts, p->cap_M);
    else
        k_gather_points<T, 2><<<blocks_for(M, 256 * FOLD_PPT), 256, 0, p->stream>>>(
            M, perm, (const T *)p->d_rec, (T *)p->d_pts, p->cap_M);
    NK_LAUNCH_CHECK();
    return NK_OK;
}

// Stable LSD radix sort of (key, value) pairs on the low `bits` bits of
// the keys; vin == nullptr means values = positions.  The last pass lands
// in (out_k, out_v); (tmp_k, tmp_v) is the ping-pong scratch.  Inputs are
// read by the first pass only.
static int radix_sort_pairs(nk_plan *p, const int32_t *kin, const int32_t *vin, int64_t M,
                            int bits, int32_t *out_k, int32_t *out_v, int32_t *tmp_k,
                            int32_t *tmp_v) {
    cudaStream_t st = p->stream;
    const int passes = std::max(1, (bits + RADIX_BITS - 1) / RADIX_BITS);
    // the bits spread evenly over the passes (C4's 28-bit key: 4 x 7 rather
    // than 8 + 8 + 8 + 4): fewer ranking ballots per pass, longer digit runs
    const int dbits = std::min(RADIX_BITS, std::max(4, (bits + passes - 1) / passes));
    const int ntiles = (int)((M + SORT_TILE - 1) / SORT_TILE);
    int rc = grow(&p->d_tile_hist, &p->cap_tile_hist, (int64_t)RADIX * ntiles + 1);
    if (rc) return rc;
    int32_t *A[2] = {out_k, out_v}, *B[2] = {tmp_k, tmp_v};
    for (int ps = 0; ps < passes; ++ps) {
        const bool toA = ((passes - 1 - ps) % 2) == 0;   // the last pass lands in A
        int32_t **dst = toA ? A : B;
        const int shift = ps * dbits;
        k_radix_hist<<<ntiles, SORT_BLOCK, 0, st>>>(kin, (int)M, shift, (1 << dbits) - 1, ntiles,
                                                    p->d_tile_hist);
        NK_LAUNCH_CHECK();
        rc = nk_scan_exclusive(p, p->d_tile_hist, p->d_tile_hist, (int64_t)RADIX * ntiles);
        if (rc) return rc;
        auto kern = dbits >= 8 ? k_radix_scatter<8>
                  : dbits == 7 ? k_radix_scatter<7>
                  : dbits == 6 ? k_radix_scatter<6>
                  : dbits == 5 ? k_radix_scatter<5>
                  : k_radix_scatter<4>;
        kern<<<ntiles, SORT_BLOCK, 0, st>>>(kin, vin, (int)M, shift, ntiles, p->d_tile_hist,
                                            dst[0], dst[1]);
        NK_LAUNCH_CHECK();
        kin = dst[0];
        vin = dst[1];
    }
    return NK_OK;
}

static int bits_for(int64_t n) {
    int b = 1;
    while ((1ll << b) < n) ++b;
    return b;
}

// SM visit order: stable by (bin, footprint start).  Two stable LSD sorts:
// by start, then by bin key.  The exported bin-stable layout (d_perm) stays.
static int order_by_start(nk_plan *p) {
    const int64_t M = p->M;
    cudaStream_t st = p->stream;
    int32_t *scr = p->d_sort_scr;
    // quarters of the scratch at cap_M offsets (a multiple of 16 elements):
    // every buffer stays 16-byte aligned for the radix passes' int4 loads,
    // whatever the parity of M
    const int64_t q = p->cap_M;
    int32_t *k0 = scr, *v0 = scr + q, *k1 = scr + 2 * q, *v1 = scr + 3 * q;
    const unsigned nb = blocks_for(M, 256);
    if (p->prec == NK_DOUBLE)
        k_start_keys<double><<<nb, 256, 0, st>>>((int)M, p->d_keys, (const double *)p->d_pts,
                                                 p->cap_M, p->geom, k0);
    else
        k_start_keys<float><<<nb, 256, 0, st>>>((int)M, p->d_keys, (const float *)p->d_pts,
                                                p->cap_M, p->geom, k0);
    int rc = radix_sort_pairs(p, k0, nullptr, M, bits_for(p->start_space), p->d_alt_keys,
                              p->d_alt_vals, k1, v1);
    if (!rc) {
        k_gather_i32<<<nb, 256, 0, st>>>((int)M, p->d_alt_vals, p->d_keys, k0);
        rc = radix_sort_pairs(p, k0, p->d_alt_vals, M, bits_for(p->nbins), p->d_alt_keys, v0,
                              k1, v1);
    }
    if (!rc) {
        if (p->prec == NK_DOUBLE)
            k_reorder_points<double><<<nb, 256, 0, st>>>(
                (int)M, p->dim, v0, p->d_perm, (const double *)p->d_pts, p->cap_M,
                p->d_vperm_buf, (double *)p->d_pts_alt);
        else
            k_reorder_points<float><<<nb, 256, 0, st>>>(
                (int)M, p->dim, v0, p->d_perm, (const float *)p->d_pts, p->cap_M,
                p->d_vperm_buf, (float *)p->d_pts_alt);
        std::swap(p->d_pts, p->d_pts_alt);
        p->d_vperm = p->d_vperm_buf;
    }
    return rc;
}

int nk_sort_points(nk_plan *p, int coord_prec, const void *x, const void *y, const void *z,
                   int64_t stride) {
    int rc = ensure_point_buffers(p, p->M);
    if (rc) return rc;
    const int64_t M = p->M;
    const int nbins = (int)p->nbins;
    cudaStream_t st = p->stream;
    const bool sort = p->method != NK_GM && M > 0;
    // SM plans visit points in (bin, footprint start) order: one LSD radix
    // sort of the composite key bin << sb | start (K1 computes both).  The
    // exported bin-stable perm is then derived on demand
    // (nk_compute_bin_perm).
    const int sb = bits_for(p->start_space);
    const bool composite = sort && p->method == NK_SM && sb + bits_for(nbins) <= 32;
    int32_t *ck = composite ? p->d_sort_scr : nullptr;
    NK_CUDA(cudaMemsetAsync(p->d_counts, 0, sizeof(int32_t) * nbins, st));
    NK_CUDA(cudaMemsetAsync(p->d_bad, 0xff, sizeof(unsigned long long), st));
    NK_CUDA(cudaMemsetAsync(p->d_bad + 1, 0, 2 * sizeof(unsigned long long), st));
    if (M > 0) {
        rc = coord_prec == NK_DOUBLE ? fold_keys<double>(p, x, y, z, stride, ck, sb)
                                     : fold_keys<float>(p, x, y, z, stride, ck, sb);
        if (rc) return rc;
    }
    // The non-finite check is read back together with the subproblem count
    // (and the bin-density sum of the type-2 visit-order choice) in setpts'
    // single host synchronisation below: a non-finite point folds to key 0 /
    // coordinate 0, so the sort in between is harmless, and have_points stays
    // false on the error return.
    const int32_t *perm = nullptr;
    p->sorted = false;
    p->perm_valid = false;
    if (sort) {
        if (composite) {
            rc = radix_sort_pairs(p, ck, nullptr, M, sb + bits_for(nbins), p->d_keys,
                                  p->d_vperm_buf, p->d_alt_keys, p->d_alt_vals);
            perm = p->d_vperm_buf;
        } else {
            rc = radix_sort_pairs(p, p->d_keys_in, nullptr, M, bits_for(p->nbins), p->d_keys,
                                  p->d_perm, p->d_alt_keys, p->d_alt_vals);
            perm = p->d_perm;
            p->perm_valid = true;
        }
        if (rc) return rc;
        p->sorted = true;
        k_bin_starts<<<blocks_for(nbins + 1, 256), 256, 0, st>>>((int)M, nbins, p->d_keys,
                                                                 composite ? sb : 0,
                                                                 p->d_starts);
        k_counts_from_starts<<<blocks_for(nbins, 256), 256, 0, st>>>(nbins, p->d_starts,
                                                                     p->d_counts);
        NK_LAUNCH_CHECK();
    } else {
        // starts = exclusive cumsum of counts, length nbins + 1 (binsort.py:150-151)
        rc = nk_scan_exclusive(p, p->d_counts, p->d_starts, nbins);
        if (rc) return rc;
    }
    if (!sort && M > 0) {
        NK_CUDA(cudaMemcpyAsync(p->d_keys, p->d_keys_in, 4 * M, cudaMemcpyDeviceToDevice, st));
    }
    if (M > 0) {
        rc = p->prec == NK_DOUBLE ? gather<double>(p, perm) : gather<float>(p, perm);
        if (rc) return rc;
    }

    // subproblems (binsort.py:166-219), needed by the SM spread and the
    // staged interpolation
    p->S = 0;
    // type-2 SM plans with a composite key and the per-thread gather choose
    // their visit order from the point-weighted bin density (below)
    const bool xwin = nk_interp_xwin(p->type, p->dim, p->prec, p->w, p->method,
                                     p->max_sub_smem) ||
                      p->geom.tiled;
    const bool need_sq = p->method == NK_SM && p->type == 2 && composite && !xwin && M > 0;
    if (p->method == NK_SM && M > 0) {
        k_nsub<<<blocks_for(nbins, 256), 256, 0, st>>>(p->d_counts, nbins, p->msub,
                                                       p->d_nsub_off);
        NK_LAUNCH_CHECK();
        rc = nk_scan_exclusive(p, p->d_nsub_off, p->d_nsub_off, nbins);
        if (rc) return rc;
        NK_CUDA(cudaMemcpyAsync(p->d_bad + 2, p->d_nsub_off + nbins, 4,
                                cudaMemcpyDeviceToDevice, st));
    }
    if (need_sq) {
        k_sum_sq<<<std::min(blocks_for(nbins, 256), 1184u), 256, 0, st>>>(nbins, p->d_counts,
                                                                         p->d_bad + 1);
        NK_LAUNCH_CHECK();
    }
    NK_CUDA(cudaMemcpyAsync(p->h_flags, p->d_bad, 3 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
    NK_CUDA(cudaStreamSynchronize(st));
    const unsigned long long bad = p->h_flags[0];
    if (bad != ~0ull) {
        nk_set_error_index((int64_t)bad);
        nk_set_error("non-finite coordinate at point index " + std::to_string(bad));
        return NK_ERR_NONFINITE;
    }
    if (p->method == NK_SM && M > 0) {
        const int32_t S = (int32_t)p->h_flags[2];
        p->S = S;
        if (S > 0) {
            if (S > p->cap_S || !p->d_sub_bin) {
                cudaFree(p->d_sub_bin);
                cudaFree(p->d_sub_start);
                cudaFree(p->d_sub_stop);
                NK_CUDA(cudaMalloc((void **)&p->d_sub_bin, 4 * (size_t)S));
                NK_CUDA(cudaMalloc((void **)&p->d_sub_start, 4 * (size_t)S));
                NK_CUDA(cudaMalloc((void **)&p->d_sub_stop, 4 * (size_t)S));
                p->cap_S = S;
            }
            k_fill_subs<<<blocks_for(S, 256), 256, 0, st>>>(S, p->d_nsub_off, nbins,
                                                            p->d_starts, p->msub, p->d_sub_bin,
                                                            p->d_sub_start, p->d_sub_stop);
            NK_LAUNCH_CHECK();
        }
    }
    p->d_vperm = composite ? p->d_vperm_buf : p->d_perm;
    // visit-order refinement inside bins (the exported bin-stable layout is
    // untouched).  Start order puts points that share footprint words in the
    // same warp (broadcast loads, register runs in the spread); at low local
    // density there is little to share and the staged interpolation is
    // better served by the bank-residue interleave (K4b: every wavefront
    // gathers from distinct banks).  Measured (type 2): start wins at C2
    // (2.4 points per cell: 166 vs 182 us) and for clustered 3D points (0.90
    // vs 1.35 ms); the interleave wins for uniform 3D f32 at 0.6 points per
    // cell (0.90 vs 1.17 ms) and f64 (15.3 vs 21.0 ms).  The switch is the
    // point-weighted bin density sum_b count_b^2 / (M * bin cells).
    if (p->method == NK_SM && p->S > 0) {
        if (!composite && p->type == 1) {
            rc = order_by_start(p);   // composite key would exceed 32 bits
            if (rc) return rc;
        } else if (p->type == 2) {
            // K7x / K7t group neighbours in footprint-start order
            bool interleave = !composite && p->prec == NK_DOUBLE && !xwin;
            if (xwin) {
                // K7x groups neighbours in footprint-start order
                if (!composite) {
                    rc = order_by_start(p);
                    if (rc) return rc;
                }
            } else if (composite) {
                const unsigned long long sq = p->h_flags[1];   // need_sq: read back above
                double cells = 1;
                for (int i = 0; i < p->dim; ++i) cells *= p->bin_dims[i];
                const double rho = (double)sq / ((double)M * cells);
                interleave = rho < 1.2;
            } else if (p->prec == NK_SINGLE) {
                rc = order_by_start(p);   // composite key would exceed 32 bits
                if (rc) return rc;
            }
            if (interleave && 4 * ((int64_t)p->msub + 1) + 1024 > 227 * 1024)
                interleave = false;   // bucket table would not fit in shared memory
            if (interleave) {
                // in: current visit order; out: scratch-backed visit order
                int32_t *vout = composite ? p->d_sort_scr : p->d_vperm_buf;
                int32_t *scr = composite ? p->d_sort_scr + p->cap_M : p->d_alt_keys;
                // round_start[] holds one int per point of the largest
                // subproblem: past the 48 KB default the kernel opts in
                size_t smem = 4 * ((size_t)p->msub + 1);
                if (smem > 48 * 1024) {
                    if (p->prec == NK_DOUBLE)
                        NK_CUDA(cudaFuncSetAttribute(k_refine_interleave<double>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem));
                    else
                        NK_CUDA(cudaFuncSetAttribute(k_refine_interleave<float>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem));
                }
                if (p->prec == NK_DOUBLE)
                    k_refine_interleave<double><<<(unsigned)p->S, 256, smem, st>>>(
                        p->d_sub_bin, p->d_sub_start, p->d_sub_stop, p->d_vperm,
                        (const double *)p->d_pts, p->cap_M, p->geom, 8, scr, vout,
                        (double *)p->d_pts_alt);
                else
                    k_refine_interleave<float><<<(unsigned)p->S, 256, smem, st>>>(
                        p->d_sub_bin, p->d_sub_start, p->d_sub_stop, p->d_vperm,
                        (const float *)p->d_pts, p->cap_M, p->geom, 16, scr, vout,
                        (float *)p->d_pts_alt);
                NK_LAUNCH_CHECK();
                std::swap(p->d_pts, p->d_pts_alt);
                p->d_vperm = vout;
            }
        }
    }
    free(p->h_det_off);
    p->h_det_off = nullptr;
    p->n_det = 0;
    if (p->deterministic && p->type == 1 && p->method == NK_SM && p->S > 0) {
        // colour classes per axis: ceil((m + 2 halo) / m) residues (+ the
        // remainder bins), then (rank, colour) keys sorted stably
        int cs[3] = {1, 1, 1}, nc[3] = {1, 1, 1};
        for (int a = 0; a < p->dim; ++a) {
            const int m = p->bin_dims[a];
            cs[a] = (int)std::min<int64_t>((m + 2 * p->halo + m - 1) / m, p->nb[a]);
            nc[a] = cs[a] + (int)(p->nb[a] % cs[a]);
        }
        if (p->S > p->cap_sched || !p->d_sub_sched) {
            cudaFree(p->d_sub_sched);
            p->d_sub_sched = nullptr;
            NK_CUDA(cudaMalloc((void **)&p->d_sub_sched, 4 * (size_t)p->S));
            p->cap_sched = p->S;
        }
        const int64_t q = p->cap_M;   // (bin, start) scratch, free once the visit order is set
        int32_t *scr = p->d_sort_scr, *skeys = scr + q;
        k_det_keys<<<blocks_for(p->S, 256), 256, 0, st>>>((int)p->S, p->d_sub_bin,
                                                          p->d_nsub_off, p->geom,
                                                          make_int3(cs[0], cs[1], cs[2]),
                                                          make_int3(nc[0], nc[1], nc[2]), scr);
        NK_LAUNCH_CHECK();
        int maxrank = 1;
        {
            std::vector<int32_t> off(nbins + 1);
            NK_CUDA(cudaMemcpyAsync(off.data(), p->d_nsub_off, 4 * (size_t)(nbins + 1),
                                    cudaMemcpyDeviceToHost, st));
            NK_CUDA(cudaStreamSynchronize(st));
            for (int b = 0; b < nbins; ++b) maxrank = std::max(maxrank, off[b + 1] - off[b]);
        }
        const int64_t nkeys = (int64_t)maxrank * nc[0] * nc[1] * nc[2];
        rc = radix_sort_pairs(p, scr, nullptr, p->S, bits_for(nkeys), skeys, p->d_sub_sched,
                              scr + 2 * q, scr + 3 * q);
        if (rc) return rc;
        std::vector<int32_t> hk((size_t)p->S);
        NK_CUDA(cudaMemcpyAsync(hk.data(), skeys, 4 * (size_t)p->S, cudaMemcpyDeviceToHost, st));
        NK_CUDA(cudaStreamSynchronize(st));
        std::vector<int> offs;
        for (int64_t i = 0; i < p->S; ++i)
            if (i == 0 || hk[i] != hk[i - 1]) offs.push_back((int)i);
        offs.push_back((int)p->S);
        p->n_det = (int)offs.size() - 1;
        p->h_det_off = (int *)malloc(sizeof(int) * offs.size());
        memcpy(p->h_det_off, offs.data(), sizeof(int) * offs.size());
    } else if (p->geom.tiled && p->S > 0 && p->dim == 3 && p->nb[0] <= 1024 &&
               p->nb[1] <= 1024 && p->nb[2] <= 1024 && !getenv("NK_NO_SCHED")) {
        // Morton schedule of the subproblems for the tiled f64 kernels (bins
        // per axis <= 1024; the scratch is free once the visit order is set)
        if (p->S > p->cap_sched || !p->d_sub_sched) {
            cudaFree(p->d_sub_sched);
            p->d_sub_sched = nullptr;
            NK_CUDA(cudaMalloc((void **)&p->d_sub_sched, 4 * (size_t)p->S));
            p->cap_sched = p->S;
        }
        const int64_t q = p->cap_M;
        int32_t *scr = p->d_sort_scr;
        k_sched_keys<<<blocks_for(p->S, 256), 256, 0, st>>>((int)p->S, p->d_sub_bin, p->geom, scr);
        NK_LAUNCH_CHECK();
        rc = radix_sort_pairs(p, scr, nullptr, p->S, 30, scr + q, p->d_sub_sched, scr + 2 * q,
                              scr + 3 * q);
        if (rc) return rc;
    } else if (p->d_sub_sched) {
        cudaFree(p->d_sub_sched);
        p->d_sub_sched = nullptr;
        p->cap_sched = 0;
    }
    NK_CUDA(cudaStreamSynchronize(st));
    return NK_OK;
}

// The reference's bin-stable permutation (binsort.py:153, stable argsort of
// the bin keys) for plans whose visit order is (bin, start): one radix sort
// of the input-order bin keys, run only when the layout is exported.
int nk_compute_bin_perm(nk_plan *p) {
    if (p->perm_valid || p->M == 0) return NK_OK;
    int rc = radix_sort_pairs(p, p->d_keys_in, nullptr, p->M, bits_for(p->nbins), p->d_keys,
                              p->d_perm, p->d_alt_keys, p->d_alt_vals);
    if (rc) return rc;
    p->perm_valid = true;
    return NK_OK;
}

int nk_export_subproblems(const nk_plan *p, int32_t *bin_ids, int32_t *starts, int32_t *stops,
                          int32_t *offsets, int32_t *padded) {
    if (p->S == 0) return NK_OK;
    cudaStream_t st = p->stream;
    size_t b = 4 * (size_t)p->S;
    if (bin_ids) NK_CUDA(cudaMemcpyAsync(bin_ids, p->d_sub_bin, b, cudaMemcpyDeviceToDevice, st));
    if (starts) NK_CUDA(cudaMemcpyAsync(starts, p->d_sub_start, b, cudaMemcpyDeviceToDevice, st));
    if (stops) NK_CUDA(cudaMemcpyAsync(stops, p->d_sub_stop, b, cudaMemcpyDeviceToDevice, st));
    if (offsets || padded) {
        k_export_subs<<<blocks_for(p->S, 256), 256, 0, st>>>((int)p->S, p->geom, p->d_sub_bin,
                                                             offsets, padded);
        NK_LAUNCH_CHECK();
    }
    return NK_OK;
}
