/*
 * nufft_b200.h -- C-ABI of libnufft_b200.so, the B200 (sm_100a) NUFFT hot path.
 *
 * The reference (nufftkit, /root/reference/pkg/src/nufftkit) is a Python
 * package with no FFI of its own; these entry points are what a binding of
 * its plan / stage API would call.  Each function cites the reference
 * interface it replaces.  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *  - Return 0 (NK_OK) on success, a nonzero NK_ERR_* code otherwise; the
 *    message is in nk_last_error() (thread-local).  NK_ERR_VALUE and
 *    NK_ERR_NONFINITE map to Python ValueError (kernel.py:77,92-93,168,196;
 *    binsort.py:144,175; spread.py:138,156,172,175).
 *  - Complex arrays are interleaved (re, im) in the plan precision
 *    (complex64 for NK_SINGLE, complex128 for NK_DOUBLE).
 *  - Uniform (mode) arrays are (N_d, ..., N_1), k_1 fastest, each axis
 *    -floor(N/2) .. ceil(N/2)-1 (kernel.py:176-178).
 *    Fine grids are (n_d, ..., n_1), n_1 fastest (spread.py:132).
 *  - Pointers passed to nk_setpts / nk_execute may be device or host memory
 *    (detected with cudaPointerGetAttributes).  With device pointers the
 *    work is enqueued on the plan stream and the call returns without
 *    synchronising (like cuFINUFFT); with any host pointer the call copies
 *    through device staging buffers and synchronises before returning.
 *    Stage-level functions (nk_spread ... nk_deconv_type2) take device
 *    pointers only.
 */
#ifndef NUFFT_B200_H
#define NUFFT_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define NK_API __attribute__((visibility("default")))
#else
#define NK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define NK_OK 0
#define NK_ERR_VALUE 1     /* invalid argument -> ValueError */
#define NK_ERR_NONFINITE 2 /* non-finite coordinate at nk_error_index() -> ValueError */
#define NK_ERR_STATE 3     /* e.g. execute before setpts -> ValueError */
#define NK_ERR_MEMORY 4    /* device allocation failed -> MemoryError */
#define NK_ERR_CUDA 5      /* CUDA / cuFFT runtime error -> RuntimeError */

#define NK_SINGLE 0
#define NK_DOUBLE 1

/* Spreading method tags (spread.py:3-8). */
#define NK_METHOD_DEFAULT (-1)
#define NK_GM 0
#define NK_GMSORT 1
#define NK_SM 2

typedef struct nk_plan nk_plan;

typedef struct {
    int method;          /* NK_METHOD_DEFAULT: SM for both types.  Type 1 follows
                            SPEC.md:170; for type 2 SPEC.md:170 says GM-sort, this
                            library deviates and picks the shared-memory staged
                            gather ("sm", measured faster on B200) */
    int bin_dims[3];     /* 0 = default.  GM-sort plans: the reference's (32,32) /
                            (16,16,2) (binsort.py:34-35).  SM plans: B200-tuned shapes
                            -- type 1: 2D (16,8), 3D f32 (4,4,4), 3D f64 (11,7,7);
                            type 2: 2D (32,32), 3D f32 (16,16,4), 3D f64 (11,7,7);
                            halved along axes 1/2 while the padded bin exceeds
                            shared memory */
    int max_subproblem;  /* 0 = default.  The reference default is 1024
                            (binsort.py:38); SM plans use 128 for 2D type 1, 1024
                            for 3D type 1 and 3D double type 2, 4096 for other
                            type 2 */
    int64_t fine[3];     /* 0 = sizing rule n_i = next_smooth(max(2N_i, 2w)) */
    int device;          /* -1 = current device.  Every call on the plan runs on this
                            device and restores the caller's current device */
    void *stream;        /* cudaStream_t, NULL = default stream */
    int timing;          /* nonzero: record per-stage CUDA events (nk_stage_times) */
    int n_trans;         /* vectors per execute (cufinufft ntransf); 0 or 1 = one.  The
                            reference has no batching; the paper reuses
                            one setpts across many transforms */
    int deterministic;   /* nonzero: repeated type-1 executes are bit-identical
                            (SPEC.md:163).  SM plans merge their padded bins in
                            colour classes of non-overlapping bins, one launch per
                            class, so every fine-grid cell is summed in a fixed
                            order.  Type 2 is always deterministic; GM / GM-sort
                            type 1 (per-point atomics) is not */
} nk_opts;

typedef struct {
    int type, dim, precision, method;
    int64_t modes[3], fine[3];
    double epsilon; /* effective epsilon after the single-precision floor */
    int w;
    double beta;
    double alpha[3];
    int eps_clamped; /* 1 if a single-precision epsilon < 1e-6 was clamped */
    int bin_dims[3];
    int64_t bins_per_axis[3];
    int64_t nbins;
    int max_subproblem;
    int halo;
    int64_t num_points;
    int64_t num_subproblems;
    int n_trans;
} nk_plan_info;

/* ---- plan-time host math (kernel.py) --------------------------------- */

/* kernel.py:83-103 tolerance_to_width: (eps_eff, w, beta); *clamped set when
 * a single-precision eps < 1e-6 was raised to 1e-6. */
NK_API int nk_tolerance_to_width(double eps, int precision, double *eps_eff, int *w,
                          double *beta, int *clamped);

/* SPEC.md:122-130 next_smooth: smallest 2^q 3^p 5^r >= n (n >= 1), or -1. */
NK_API int64_t nk_next_smooth(int64_t n);

/* kernel.py:149-173 kernel_fourier: phi_hat(xi) by 100-node Gauss-Legendre
 * after z = sin(theta).  Host arrays. */
NK_API int nk_kernel_fourier(double beta, const double *xi, int64_t n, double *out);

/* kernel.py:181-205 build_correction_factors: writes the (N_d, ..., N_1)
 * table (2/w)^d / prod_i phi_hat(alpha_i k_i) over centered k_i into host
 * memory `out` (float for NK_SINGLE, double for NK_DOUBLE).  modes / alpha
 * are axis 1 first.  NK_ERR_VALUE when phi_hat underflows (kernel.py:195-199). */
NK_API int nk_correction_factors(double beta, int w, int dim, const int64_t *modes,
                                 const double *alpha, int precision, void *out);

/* ---- plan lifecycle -------- */

NK_API void nk_default_opts(nk_opts *opts);

/* make_plan(type, N, epsilon, method, precision). */
NK_API int nk_plan_create(int type, int dim, const int64_t *modes, double eps, int precision,
                   const nk_opts *opts, nk_plan **plan);

NK_API int nk_plan_get_info(const nk_plan *plan, nk_plan_info *info);

/* Re-target the plan's stream (cudaStream_t). */
NK_API int nk_set_stream(nk_plan *plan, void *stream);

/* set_points(plan, coords): coordinate i of axis a is
 * read at coord_a[i * stride] (stride 1 = SoA x/y/z as in the paper's
 * set_pts(X, Y, Z); stride d = the reference's (M, d) array).  coord_prec
 * is NK_SINGLE or NK_DOUBLE (coordinates are widened to FP64 for the fold,
 * binsort.py:123).  Non-finite coordinates -> NK_ERR_NONFINITE naming the
 * first offending index.  M = 0 is legal.  Unlike nk_execute, setpts always
 * waits for the plan stream before returning: the subproblem count sizes
 * host-side launches, so it reads that count back together with the
 * non-finite check (one synchronisation; the deterministic option adds its
 * colour-class readback). */
NK_API int nk_setpts(nk_plan *plan, int64_t M, int coord_prec, const void *x, const void *y,
              const void *z, int64_t stride);

/* execute(plan, input, output): type 1 reads M strengths
 * and writes prod(N) modes; type 2 the reverse.  Input is not modified.
 * With n_trans = K > 1 the input and output hold K vectors back to back
 * (type 1: K x M strengths -> K x prod(N) modes). */
NK_API int nk_execute(nk_plan *plan, const void *in, void *out);

/* destroy. */
NK_API int nk_destroy(nk_plan *plan);

NK_API const char *nk_last_error(void);
NK_API int64_t nk_error_index(void);

/* ---- stage level (device pointers; parity hooks) --------------------- */

/* bin_sort (binsort.py:134-163) results of the last setpts, as int32:
 * point_bins (M, input order), counts (nbins), starts (nbins+1), perm (M).
 * Any pointer may be NULL.  Requires a GM-sort or SM plan. */
NK_API int nk_get_layout(const nk_plan *plan, int32_t *point_bins, int32_t *counts,
                  int32_t *starts, int32_t *perm);

/* build_subproblems (binsort.py:166-219) results: bin_ids, slice_starts,
 * slice_stops (S), offsets and padded_dims (S, d) row-major.  SM plans. */
NK_API int nk_get_subproblems(const nk_plan *plan, int32_t *bin_ids, int32_t *slice_starts,
                       int32_t *slice_stops, int32_t *offsets, int32_t *padded_dims);

/* spread_gm / spread_gm_sort / spread_sm (spread.py:142-182): zero `fine`
 * then spread the M strengths with the plan method.  Stage functions act on
 * all n_trans vectors (buffers hold n_trans back-to-back arrays). */
NK_API int nk_spread(nk_plan *plan, const void *strengths, void *fine);

/* interpolate: out[j] = gather at point j. */
NK_API int nk_interp(nk_plan *plan, const void *fine, void *out);

/* fft_fine: in place, direction -1 forward (e^{-}),
 * +1 inverse unnormalised (e^{+}). cuFFT. */
NK_API int nk_fft(nk_plan *plan, void *fine, int direction);

/* deconvolve_type1 (with the (-1)^{sum k} phase). */
NK_API int nk_deconv_type1(nk_plan *plan, const void *fine_spectrum, void *modes);

/* fft_fine(forward) followed by deconvolve_type1, in place on `fine`: the
 * type-1 back half of execute() (2D single precision with n_1 = 2^L: cuFFT
 * column pass + the fused row-FFT / mode-selection kernel).  Used by the
 * sharded type-1 path after the fine-grid reduce. */
NK_API int nk_fft_deconv_type1(nk_plan *plan, void *fine, void *modes);

/* deconvolve_type2 (with the phase): writes every fine cell. */
NK_API int nk_deconv_type2(nk_plan *plan, const void *modes, void *fine_spectrum);

/* Device milliseconds of the stages of the last nk_execute when the plan was
 * created with opts.timing: ms[0] spread|interp, ms[1] fft, ms[2]
 * deconv|pad, ms[3] total.  Synchronises on the plan's last event. */
NK_API int nk_stage_times(nk_plan *plan, float *ms, int n);

/* Turn per-stage CUDA-event timing on/off (events are created on first
 * use).  While timing is on, execute() launches directly instead of
 * replaying its CUDA graph, so the events bracket each stage. */
NK_API int nk_set_timing(nk_plan *plan, int on);

/* Number of this library's kernels launched by the last nk_execute. */
NK_API int nk_last_launch_count(const nk_plan *plan);

#ifdef __cplusplus
}
#endif

#endif /* NUFFT_B200_H */
