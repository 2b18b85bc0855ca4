// Internal declarations shared by the libnufft_b200 translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <string>

#include "../../include/nufft_b200.h"

#define NK_PI 3.141592653589793
#define NK_TWO_PI (2.0 * NK_PI)

// ---------------------------------------------------------------- errors
void nk_set_error(const std::string &msg);
void nk_set_error_index(int64_t idx);

#define NK_CUDA(expr)                                                                 \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess) {                                                      \
            nk_set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + \
                         __FILE__ + ":" + std::to_string(__LINE__));                  \
            return _e == cudaErrorMemoryAllocation ? NK_ERR_MEMORY : NK_ERR_CUDA;     \
        }                                                                             \
    } while (0)

#define NK_LAUNCH_CHECK() NK_CUDA(cudaGetLastError())

// -------------------------------------------------------------- geometry
// Per-plan geometry passed by value to kernels.  Axis 0 is the reference's
// axis 1 (fastest).
struct Geom {
    int dim;
    int n[3];       // fine sizes
    int N[3];       // mode counts
    int m[3];       // bin dims
    int nb[3];      // bins per axis
    unsigned mdiv[3];  // ceil(2^32 / m): cell / m = umulhi(cell, mdiv) (exact: n m <= 2^32), 0 = divide
    int halo;       // ceil(w/2)
    int w;
    // footprint-start visit code (setpts K4d): 0 = lexicographic
    // (t3 p2 + t2) p1 + t1; else tiles of 2^tile_lg starts per axis, tile
    // major (the tiled f64 spread, nk_spread.cu K6t, groups a tile's points)
    int tile_lg;
    int tiled;
    double scale[3];  // n_i / (2 pi), binsort.py:99
    float betaf, betaf_log2e;
    double beta;
    // per-vector strides of a batched execute (vector = blockIdx.y)
    int64_t ntot;   // fine cells
    int64_t Ntot;   // modes
    int64_t M;      // points
};

template <typename T> struct cplx;
template <> struct cplx<float> { typedef float2 t; };
template <> struct cplx<double> { typedef double2 t; };

// -------------------------------------------------------------- plan
struct nk_plan {
    int type, dim, prec, method;
    int ntrans;     // vectors per execute (cufinufft ntransf), >= 1
    int64_t N[3], n[3];
    double eps;
    int w;
    double beta;
    double alpha[3];
    int eps_clamped;
    int bin_dims[3];
    int64_t nb[3];
    int64_t nbins;
    int msub;
    int halo;
    int device;
    cudaStream_t stream;
    int timing;
    Geom geom;

    int64_t n_tot, N_tot;
    size_t csize;   // bytes per complex element
    void *d_fine;   // fine grid (n_tot complex)
    void *d_corr;   // per-axis correction factors incl. (2/w) and (-1)^k (plan precision)
    cufftHandle fft;
    bool fft_ok;
    // 2D single precision with power-of-two n_1: K9 (type 2) / K8 (type 1)
    // fused with the row FFTs (nk_deconv.cu) + a cuFFT column-only plan
    bool fused_rows;
    cufftHandle fft_col;
    bool fft_col_ok;
    void *d_twiddle;        // n_1 complex exp(+2 pi i k / n_1)
    int *d_work;            // n_trans work counters of the staged interpolation
    void *d_cvis;           // strengths gathered into visit order (tiled f64 spread)
    // TMA descriptor of d_fine as doubles (2 n1, n2, n3, n_trans) with the
    // full padded bin as its box (tiled f64 interpolation, K7t)
    CUtensorMap tmap_fine;
    bool tmap_ok;
    int64_t cap_cvis;

    // points
    int64_t M;
    bool have_points;
    int64_t cap_M;
    int32_t *d_keys_in;     // bin key per input point
    int32_t *d_keys;        // bin key in visit order (sorted, or input order for GM)
    int32_t *d_perm;        // sorted position -> input index (bin-stable; exported layout)
    int32_t *d_vperm;       // visit position -> input index, matches d_pts order
                            // (== d_perm unless refined for bank-conflict-free gathers)
    int32_t *d_vperm_buf;   // storage behind a refined d_vperm
    void *d_pts_alt;        // scratch for reordering d_pts
    int32_t *d_counts;      // nbins
    int32_t *d_starts;      // nbins + 1
    void *d_pts;            // dim arrays of cap_M local coords (plan precision)
    void *d_rec;            // per input point (u1, u2[, u3, 0]) records (K1 -> K5)
    int32_t *d_alt_keys, *d_alt_vals;  // radix scratch
    int32_t *d_sort_scr;    // 4 cap_M int32: (bin, start) ordering scratch (type-1 SM)
    int32_t *d_tile_hist;
    int64_t cap_tile_hist;
    int32_t *d_scan_tmp;
    int64_t cap_scan_tmp;
    unsigned long long *d_bad;    // [0] first non-finite index, [1] sum count^2, [2] S
    unsigned long long *h_flags;  // pinned copy of d_bad[0..2]: setpts' one host sync
    bool sorted;
    bool perm_valid;        // d_perm holds the bin-stable layout (else derived on demand)

    // subproblems
    int64_t S, cap_S;
    int32_t *d_nsub_off;    // nbins + 1
    int32_t *d_sub_bin, *d_sub_start, *d_sub_stop;
    int32_t *d_sub_sched;   // tiled f64 kernels: CTA -> subproblem in Morton order of bins
    int64_t cap_sched;
    // deterministic type-1 merge: subproblems sorted by (rank in bin, colour
    // class of non-overlapping bins); launch g covers sched[off[g], off[g+1])
    int deterministic;
    int *h_det_off;
    int n_det;
    int max_sub_smem;       // bytes of dynamic smem for the SM kernels
    int64_t max_pad_cells;  // prod(m_i + 2 halo)
    int64_t start_space;    // footprint-start codes per bin (nk_start_code range)

    // staging for host pointers
    void *d_in_stage, *d_out_stage;
    size_t cap_in_stage, cap_out_stage;

    // timing
    cudaEvent_t ev[4];
    bool ev_ok;
    int last_launches;

    // CUDA graph of execute() for a fixed (in, out) pair: captured on a
    // private stream, replayed into the caller's stream (cudaGraphLaunch)
    bool use_graph;
    cudaStream_t cap_stream;
    cudaGraphExec_t gexec;
    const void *g_in;
    void *g_out;
    int g_launches;
};

// Warps per CTA of the plane-owned 3D SM spread (nk_spread.cu): warp w owns
// padded-bin planes z == w (mod NW), ceil(w / NW) planes per footprint.
// With the tuned small bins, 2 measured fastest for w <= 8 (C3a 1.24 ms
// vs 1.37 with 4, 2.10 with 8, 1.61 with 1); above, NW = w: every warp owns
// exactly one plane of every footprint.
constexpr int nk_sm3_warps(int w) { return w <= 8 ? 2 : w; }
// Tiled f64 3D spread (K6t, nk_spread.cu): 3D double type 1 SM plans with
// 9 <= w <= 16.  A CTA of 16 warps holds a 16 x 16 x 16 register window
// (warp = plane, lane = 16 x-cells x 8 rows); all points whose footprint
// starts fall in one tile of 2^L x 2^L x 2^L start values share it, with
// 2^L the largest power of two such that w + 2^L - 1 <= 16.
constexpr int kTileWin = 16;
#ifndef NK_TILE_NB
#define NK_TILE_NB 32
#endif
constexpr int kTileBatch = NK_TILE_NB;   // points per staged batch (two buffers)
constexpr int kTileMsub = 1024;          // max subproblem of the tiled interp (chunk table)
constexpr int nk_tile_lg(int w) { return w + 7 <= kTileWin ? 3 : (w + 3 <= kTileWin ? 2 : (w + 1 <= kTileWin ? 1 : 0)); }
inline bool nk_spread_tiled(int type, int dim, int prec, int w, int method) {
    return type == 1 && dim == 3 && prec == NK_DOUBLE && w >= 9 && w <= 16 && method == NK_SM &&
           !getenv("NK_SPREAD_NO_TILE");
}
// Tiled f64 3D interpolation (K7t, nk_interp.cu): the adjoint of K6t on the
// same tile groups (type 2, same plans).
inline bool nk_interp_tiled(int type, int dim, int prec, int w, int method, int msub = 0) {
    return type == 2 && dim == 3 && prec == NK_DOUBLE && w >= 9 && w <= 16 && method == NK_SM &&
           msub <= kTileMsub && !getenv("NK_INTERP_NO_TILE");
}
inline bool nk_tiled(int type, int dim, int prec, int w, int method, int msub) {
    return nk_spread_tiled(type, dim, prec, w, method) ||
           nk_interp_tiled(type, dim, prec, w, method, msub);
}
// Points staged per batch by the plane-owned 3D SM spread (nk_spread.cu):
// 64 keeps the staging small enough for more resident CTAs (C3a spread
// 1.24 -> 1.08 ms vs 128).
inline int nk_sm3_batch(int prec) { return 64; }
// Dynamic shared memory (bytes) of the SM spread / staged interp for a plan
// shape: padded bin (+ point staging for the 3D spread).
inline int64_t nk_sm_smem_bytes(int type, int dim, int prec, int w, const int *bin_dims,
                                int halo, int msub) {
    int64_t cells = 1;
    for (int i = 0; i < dim; ++i) cells *= bin_dims[i] + 2 * halo;
    int64_t rs = prec == NK_DOUBLE ? 8 : 4;
    int64_t b = (cells * 2 * rs + 15) / 16 * 16;
    // staging per point: int4 start, k1 row (double: zero-padded to 32),
    // k2 row, c * k3 row (complex)
    if (nk_spread_tiled(type, dim, prec, w, NK_SM))
        // per point: int4 info, k1 / k2 window rows, c k3 window row (complex)
        b += 2 * ((int64_t)kTileBatch * (16 + 2 * kTileWin * rs + 2 * kTileWin * rs) +
                  2 * kTileWin * 4 * rs) +
             3 * (3 * (kTileBatch + 2) * rs + kTileBatch * 2 * rs) + 32;   // + TMA ring
    else if (nk_interp_tiled(type, dim, prec, w, NK_SM, msub))
        // per warp (16): kernel rows [3][16][8] doubles; chunk starts
        b += 16 * 3 * kTileWin * 8 * rs + 4 * (int64_t)(kTileMsub + 4) + 16;
    else if (type == 1 && dim == 3)
        b += (int64_t)nk_sm3_batch(prec) *
             (((prec == NK_DOUBLE && w <= 16) ? 32 : w) * rs + 3 * w * rs + 16);
    if (type == 1 && dim == 2) b += 128 + (32 * w * rs + 15) / 16 * 16 + 32 * w * 2 * rs;
    return b;
}

// Does the type-2 plan use the x-window group interpolation (K7x,
// nk_interp.cu: 3D, wide double footprints, padded bin + per-warp staging
// within the 227 KB opt-in shared memory)?  Its setpts keeps the
// footprint-start visit order.
#ifndef NK_XWIN_NB
#define NK_XWIN_NB 10  // points staged per warp batch (K7x; 8: 12.5, 10: 11.9 ms at C5)
#endif
#ifndef NK_XWIN_G
#define NK_XWIN_G 4    // max points per K7x group (2 / 3 / 6 / 8: 12.7 / 12.1 / 12.9 / 14.5 ms)
#endif
#ifndef NK_XWIN_WARPS
#define NK_XWIN_WARPS 16  // K7x warps per CTA (one CTA per SM)
#endif
inline int64_t nk_xwin_smem_bytes(int w) { return NK_XWIN_WARPS * NK_XWIN_NB * (16 + 3 * w * 8); }
inline bool nk_interp_xwin(int type, int dim, int prec, int w, int method, int64_t max_sub_smem) {
    return type == 2 && dim == 3 && prec == NK_DOUBLE && w > 8 && method == NK_SM &&
           max_sub_smem + nk_xwin_smem_bytes(w) + 1024 <= 227 * 1024 &&
           !getenv("NK_INTERP_NO_XWIN");
}

// -------------------------------------------------------------- launchers
int nk_scan_exclusive(nk_plan *p, const int32_t *in, int32_t *out, int64_t n);
int nk_sort_points(nk_plan *p, int coord_prec, const void *x, const void *y,
                   const void *z, int64_t stride);
int nk_launch_spread(nk_plan *p, const void *c, void *fine, int *launches);
int nk_launch_interp(nk_plan *p, const void *fine, void *out, int *launches);
int nk_launch_deconv1(nk_plan *p, const void *spec, void *modes);
int nk_launch_deconv2(nk_plan *p, const void *modes, void *spec);
int nk_launch_pad_rowfft(nk_plan *p, const void *modes, void *spec);
int nk_launch_rowfft_deconv(nk_plan *p, const void *spec, void *modes);
int nk_compute_bin_perm(nk_plan *p);
int nk_export_subproblems(const nk_plan *p, int32_t *bin_ids, int32_t *starts,
                          int32_t *stops, int32_t *offsets, int32_t *padded);

// plan-time host math (nk_host.cpp)
void nk_kernel_fourier_host(double beta, const double *xi, int64_t n, double *out);
