/*
 * nufft_oracle.c -- CPU restatement of the reference `nufftkit` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_2102_08463_b200/csrc) and the CPU baseline timed by
 * bench.py's `cpu_baseline` leg / `--impl reference` arm.  Nothing in the
 * product imports, links or executes it.
 *
 * Every function restates one reference function (file:line relative to
 * /root/reference/pkg/src/nufftkit/):
 *
 *   or_remainder          numpy npy_remainder used by binsort.py:100
 *   or_grid_coords        binsort.py:91-100   grid_coords
 *   or_bin_keys           binsort.py:103-131  _bins_from_cells / bin_index
 *   or_bin_sort           binsort.py:134-163  bin_sort (bincount, cumsum,
 *                                             stable argsort == counting sort)
 *   or_build_subproblems  binsort.py:166-219  build_subproblems
 *   or_spread_gm          _kernels.py:36-79 (spread_2d/3d) via
 *                         spread.py:67-90 (_spread_chunked, ordered merge)
 *   or_spread_sm          _kernels.py:82-147 (spread_local_*, merge_wrap_*)
 *                         via spread.py:93-111 (_spread_blocked)
 *   or_interp             _kernels.py:150-198 (interp_2d/3d); the missing
 *                         interpolate wrapper is restated from SPEC.md:358-366
 *   or_deconv_type1/2     SPEC.md:408-425 plus the (-1)^{sum k} phase forced by
 *                         the reference's -pi-origin grid frame (binsort.py:10-12)
 *   or_direct_type1/2     SPEC.md:473-490 (direct sums of Eqs. (1),(3)),
 *                         compensated (Neumaier) summation per SPEC.md:506
 *
 * Arithmetic mirrors the Numba loops: kernel rows in FP64 (_kernels.py:20-33),
 * strength*row promoted to complex128, accumulation stored back in the array
 * dtype (complex64 for single, complex128 for double).
 *
 * Complex arrays are interleaved (re, im) like numpy complex64/complex128.
 * Arrays with "prec" take float (prec=0) or double (prec=1) storage.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.141592653589793
#define OR_TWO_PI (2.0 * OR_PI)

/* numpy float remainder (npy_divmod): fmod, then shift into the sign of b;
 * an exact zero becomes +0.0.  Used by grid_coords (binsort.py:100). */
double or_remainder(double a, double b) {
    double mod = fmod(a, b);
    if (b == 0.0) return mod;
    if (mod != 0.0) {
        if ((b < 0) != (mod < 0)) mod += b;
    } else {
        mod = copysign(0.0, b);
    }
    return mod;
}

/* binsort.py:98-100: v_i = remainder(x_i + pi, 2 pi) * (n_i / 2 pi). */
static inline double fold_coord(double x, int64_t n) {
    double scale = (double)n / OR_TWO_PI;
    return or_remainder(x + OR_PI, OR_TWO_PI) * scale;
}

/* pts: (M, d) float64 row-major.  out: (M, d) float64. */
void or_grid_coords(int64_t M, int d, const double *pts, const int64_t *fine,
                    double *out) {
    for (int64_t j = 0; j < M; ++j)
        for (int i = 0; i < d; ++i)
            out[j * d + i] = fold_coord(pts[j * d + i], fine[i]);
}

static inline int64_t nbins_axis(int64_t n, int64_t m) { return (n + m - 1) / m; }

/* binsort.py:114-131 (bin_index) with _bins_from_cells (103-111). */
void or_bin_keys(int64_t M, int d, const double *pts, const int64_t *fine,
                 const int64_t *bin_dims, int64_t *keys) {
    int64_t nb[3];
    for (int i = 0; i < d; ++i) nb[i] = nbins_axis(fine[i], bin_dims[i]);
    for (int64_t j = 0; j < M; ++j) {
        int64_t key = 0, stride = 1;
        for (int i = 0; i < d; ++i) {
            double v = fold_coord(pts[j * d + i], fine[i]);
            double fl = floor(v);
            int64_t cell;
            /* np.floor(v).astype(int64) then clamp [0, n-1]; NaN maps to
             * INT64_MIN under numpy's cast and is clamped to 0. */
            if (fl != fl) cell = INT64_MIN;
            else if (fl >= 9.2e18) cell = INT64_MAX;
            else if (fl <= -9.2e18) cell = INT64_MIN;
            else cell = (int64_t)fl;
            if (cell > fine[i] - 1) cell = fine[i] - 1;
            if (cell < 0) cell = 0;
            key += stride * (cell / bin_dims[i]);
            stride *= nb[i];
        }
        keys[j] = key;
    }
}

/* binsort.py:134-163.  counts (nbins), starts (nbins+1), perm (M). */
void or_bin_sort(int64_t M, int d, const double *pts, const int64_t *fine,
                 const int64_t *bin_dims, int64_t *keys, int64_t *counts,
                 int64_t *starts, int64_t *perm) {
    int64_t nbins = 1;
    for (int i = 0; i < d; ++i) nbins *= nbins_axis(fine[i], bin_dims[i]);
    or_bin_keys(M, d, pts, fine, bin_dims, keys);
    memset(counts, 0, sizeof(int64_t) * nbins);
    for (int64_t j = 0; j < M; ++j) counts[keys[j]]++;
    starts[0] = 0;
    for (int64_t b = 0; b < nbins; ++b) starts[b + 1] = starts[b] + counts[b];
    /* stable counting-sort scatter == np.argsort(kind="stable") */
    int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (nbins ? nbins : 1));
    memcpy(next, starts, sizeof(int64_t) * nbins);
    for (int64_t j = 0; j < M; ++j) perm[next[keys[j]]++] = j;
    free(next);
}

/* binsort.py:166-219.  Returns S; when out arrays are NULL only counts.
 * offsets/padded: (S, d) row-major. */
int64_t or_build_subproblems(int d, const int64_t *fine, const int64_t *bin_dims,
                             int64_t nbins, const int64_t *counts,
                             const int64_t *starts, int64_t max_size, int64_t halo,
                             int64_t *bin_ids, int64_t *slice_starts,
                             int64_t *slice_stops, int64_t *offsets,
                             int64_t *padded) {
    int64_t nb[3];
    for (int i = 0; i < d; ++i) nb[i] = nbins_axis(fine[i], bin_dims[i]);
    int64_t pos = 0;
    for (int64_t b = 0; b < nbins; ++b) {
        if (counts[b] == 0) continue;
        int64_t reps = (counts[b] + max_size - 1) / max_size;
        if (bin_ids) {
            int64_t rem = b, corner[3], actual[3];
            for (int i = 0; i < d; ++i) {
                corner[i] = (rem % nb[i]) * bin_dims[i];
                rem /= nb[i];
                actual[i] = bin_dims[i] < fine[i] - corner[i] ? bin_dims[i]
                                                               : fine[i] - corner[i];
            }
            int64_t lo = starts[b], hi = starts[b + 1];
            for (int64_t r = 0; r < reps; ++r) {
                int64_t p = pos + r;
                bin_ids[p] = b;
                slice_starts[p] = lo + r * max_size;
                slice_stops[p] = lo + (r + 1) * max_size < hi ? lo + (r + 1) * max_size : hi;
                for (int i = 0; i < d; ++i) {
                    offsets[p * d + i] = corner[i] - halo;
                    padded[p * d + i] = actual[i] + 2 * halo;
                }
            }
        }
        pos += reps;
    }
    return pos;
}

/* _kernels.py:20-26 */
static inline double es_value(double beta, double z) {
    double t = 1.0 - z * z;
    if (t < 0.0) return 0.0;
    return exp(beta * (sqrt(t) - 1.0));
}

/* _kernels.py:29-33 */
static inline void kernel_row(double v, int w, double beta, int64_t start, double *row) {
    double inv = 2.0 / w;
    for (int r = 0; r < w; ++r) row[r] = es_value(beta, ((double)(start + r) - v) * inv);
}

static inline int64_t pymod(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

/* Accumulate (re, im) into a complex cell of the given precision the way
 * numba does for `out[...] += t2 * row1[a]`: complex128 add, then store in
 * the array dtype. */
static inline void cadd(void *arr, int prec, int64_t idx, double re, double im) {
    if (prec) {
        double *p = (double *)arr + 2 * idx;
        p[0] = p[0] + re;
        p[1] = p[1] + im;
    } else {
        float *p = (float *)arr + 2 * idx;
        p[0] = (float)((double)p[0] + re);
        p[1] = (float)((double)p[1] + im);
    }
}

static inline void cget(const void *arr, int prec, int64_t idx, double *re, double *im) {
    if (prec) {
        const double *p = (const double *)arr + 2 * idx;
        *re = p[0];
        *im = p[1];
    } else {
        const float *p = (const float *)arr + 2 * idx;
        *re = p[0];
        *im = p[1];
    }
}

/* One point into a global grid with wrap (_kernels.py:36-79) or into a local
 * padded buffer without wrap (_kernels.py:82-124) when `offs` is non-NULL.
 * dims: (n1, n2, n3) of the target, axis 1 fastest. */
static void spread_one(int d, const double *v, double cre, double cim, int w,
                       double beta, void *out, int prec, const int64_t *dims,
                       const int64_t *offs) {
    double rows[3][16];
    int64_t st[3];
    double half = 0.5 * w;
    for (int i = 0; i < d; ++i) {
        st[i] = (int64_t)ceil(v[i] - half);
        kernel_row(v[i], w, beta, st[i], rows[i]);
    }
    if (d == 2) {
        for (int b = 0; b < w; ++b) {
            int64_t l2 = offs ? st[1] - offs[1] + b : pymod(st[1] + b, dims[1]);
            double t2r = cre * rows[1][b], t2i = cim * rows[1][b];
            for (int a = 0; a < w; ++a) {
                int64_t l1 = offs ? st[0] - offs[0] + a : pymod(st[0] + a, dims[0]);
                cadd(out, prec, l2 * dims[0] + l1, t2r * rows[0][a], t2i * rows[0][a]);
            }
        }
    } else {
        for (int e = 0; e < w; ++e) {
            int64_t l3 = offs ? st[2] - offs[2] + e : pymod(st[2] + e, dims[2]);
            double t3r = cre * rows[2][e], t3i = cim * rows[2][e];
            for (int b = 0; b < w; ++b) {
                int64_t l2 = offs ? st[1] - offs[1] + b : pymod(st[1] + b, dims[1]);
                double t2r = t3r * rows[1][b], t2i = t3i * rows[1][b];
                for (int a = 0; a < w; ++a) {
                    int64_t l1 = offs ? st[0] - offs[0] + a : pymod(st[0] + a, dims[0]);
                    cadd(out, prec, (l3 * dims[1] + l2) * dims[0] + l1,
                         t2r * rows[0][a], t2i * rows[0][a]);
                }
            }
        }
    }
}

/* Fold a sample of points to grid coords, optionally through a permutation. */
static inline void point_v(int d, const double *pts, const int64_t *fine,
                           int64_t j, double *v) {
    for (int i = 0; i < d; ++i) v[i] = fold_coord(pts[j * d + i], fine[i]);
}

static int64_t grid_cells(int d, const int64_t *fine) {
    int64_t n = 1;
    for (int i = 0; i < d; ++i) n *= fine[i];
    return n;
}

/* GM / GM-sort (spread.py:142-163 via _spread_chunked spread.py:67-90):
 * visit points in `order` (NULL = input order); `nworkers` contiguous chunks
 * each into a private grid, merged in worker order.  out must be zeroed. */
void or_spread_gm(int64_t M, int d, const double *pts, const int64_t *perm,
                  const void *c, const int64_t *fine, int w, double beta, int prec,
                  int nworkers, void *out) {
    int64_t ncell = grid_cells(d, fine);
    size_t cbytes = (size_t)(prec ? 16 : 8);
    if (nworkers < 1) nworkers = 1;
    if (nworkers > M) nworkers = M > 0 ? (int)M : 1;
    if (nworkers == 1) {
        for (int64_t j = 0; j < M; ++j) {
            int64_t src = perm ? perm[j] : j;
            double v[3], cr, ci;
            point_v(d, pts, fine, src, v);
            cget(c, prec, src, &cr, &ci);
            spread_one(d, v, cr, ci, w, beta, out, prec, fine, NULL);
        }
        return;
    }
    void **parts = (void **)calloc(nworkers, sizeof(void *));
    for (int t = 0; t < nworkers; ++t) parts[t] = calloc(ncell, cbytes);
#pragma omp parallel for schedule(static, 1) num_threads(nworkers)
    for (int t = 0; t < nworkers; ++t) {
        /* _parallel.py:32-42 chunk_bounds */
        int64_t step = M / nworkers, extra = M % nworkers;
        int64_t lo = t * step + (t < extra ? t : extra);
        int64_t hi = lo + step + (t < extra ? 1 : 0);
        for (int64_t j = lo; j < hi; ++j) {
            int64_t src = perm ? perm[j] : j;
            double v[3], cr, ci;
            point_v(d, pts, fine, src, v);
            cget(c, prec, src, &cr, &ci);
            spread_one(d, v, cr, ci, w, beta, parts[t], prec, fine, NULL);
        }
    }
    for (int t = 0; t < nworkers; ++t) {
        if (prec) {
            double *o = (double *)out, *p = (double *)parts[t];
            for (int64_t k = 0; k < 2 * ncell; ++k) o[k] += p[k];
        } else {
            float *o = (float *)out, *p = (float *)parts[t];
            for (int64_t k = 0; k < 2 * ncell; ++k) o[k] += p[k];
        }
        free(parts[t]);
    }
    free(parts);
}

/* merge_wrap_2d/3d (_kernels.py:127-147). buf dims pd (p1,p2,p3). */
static void merge_wrap(int d, const void *buf, const int64_t *pd, const int64_t *offs,
                       void *out, int prec, const int64_t *fine) {
    int64_t p3 = d == 3 ? pd[2] : 1;
    for (int64_t s3 = 0; s3 < p3; ++s3) {
        int64_t l3 = d == 3 ? pymod(offs[2] + s3, fine[2]) : 0;
        for (int64_t s2 = 0; s2 < pd[1]; ++s2) {
            int64_t l2 = pymod(offs[1] + s2, fine[1]);
            for (int64_t s1 = 0; s1 < pd[0]; ++s1) {
                int64_t l1 = pymod(offs[0] + s1, fine[0]);
                int64_t src = (s3 * pd[1] + s2) * pd[0] + s1;
                int64_t dst = (l3 * fine[1] + l2) * fine[0] + l1;
                if (prec) {
                    const double *b = (const double *)buf + 2 * src;
                    double *o = (double *)out + 2 * dst;
                    o[0] += b[0];
                    o[1] += b[1];
                } else {
                    const float *b = (const float *)buf + 2 * src;
                    float *o = (float *)out + 2 * dst;
                    o[0] += b[0];
                    o[1] += b[1];
                }
            }
        }
    }
}

/* SM (spread.py:166-182 via _spread_blocked spread.py:93-111): per
 * subproblem padded buffers, merged in subproblem order. out must be zeroed. */
void or_spread_sm(int64_t M, int d, const double *pts, const int64_t *perm,
                  const void *c, const int64_t *fine, int w, double beta, int prec,
                  int64_t S, const int64_t *slice_starts, const int64_t *slice_stops,
                  const int64_t *offsets, const int64_t *padded, int nworkers,
                  void *out) {
    size_t cbytes = (size_t)(prec ? 16 : 8);
    (void)M;
    if (nworkers < 1) nworkers = 1;
#pragma omp parallel for ordered schedule(dynamic, 1) num_threads(nworkers)
    for (int64_t s = 0; s < S; ++s) {
        const int64_t *pd = padded + s * d, *of = offsets + s * d;
        int64_t nb = 1;
        for (int i = 0; i < d; ++i) nb *= pd[i];
        void *buf = calloc(nb, cbytes);
        for (int64_t j = slice_starts[s]; j < slice_stops[s]; ++j) {
            int64_t src = perm[j];
            double v[3], cr, ci;
            point_v(d, pts, fine, src, v);
            cget(c, prec, src, &cr, &ci);
            spread_one(d, v, cr, ci, w, beta, buf, prec, pd, of);
        }
#pragma omp ordered
        merge_wrap(d, buf, pd, of, out, prec, fine);
        free(buf);
    }
}

/* interp_2d/3d (_kernels.py:150-198); output slot = original index
 * (SPEC.md:361).  Visit order `perm` (NULL = input order). */
void or_interp(int64_t M, int d, const double *pts, const int64_t *perm,
               const void *grid, const int64_t *fine, int w, double beta, int prec,
               int nworkers, void *out) {
    if (nworkers < 1) nworkers = 1;
#pragma omp parallel for schedule(static) num_threads(nworkers)
    for (int64_t j = 0; j < M; ++j) {
        int64_t src = perm ? perm[j] : j;
        double v[3], rows[3][16];
        int64_t st[3];
        double half = 0.5 * w;
        point_v(d, pts, fine, src, v);
        for (int i = 0; i < d; ++i) {
            st[i] = (int64_t)ceil(v[i] - half);
            kernel_row(v[i], w, beta, st[i], rows[i]);
        }
        double accr = 0.0, acci = 0.0;
        if (d == 2) {
            for (int b = 0; b < w; ++b) {
                int64_t l2 = pymod(st[1] + b, fine[1]);
                double ir = 0.0, ii = 0.0;
                for (int a = 0; a < w; ++a) {
                    int64_t l1 = pymod(st[0] + a, fine[0]);
                    double gr, gi;
                    cget(grid, prec, l2 * fine[0] + l1, &gr, &gi);
                    ir += gr * rows[0][a];
                    ii += gi * rows[0][a];
                }
                accr += ir * rows[1][b];
                acci += ii * rows[1][b];
            }
        } else {
            for (int e = 0; e < w; ++e) {
                int64_t l3 = pymod(st[2] + e, fine[2]);
                double mr = 0.0, mi = 0.0;
                for (int b = 0; b < w; ++b) {
                    int64_t l2 = pymod(st[1] + b, fine[1]);
                    double ir = 0.0, ii = 0.0;
                    for (int a = 0; a < w; ++a) {
                        int64_t l1 = pymod(st[0] + a, fine[0]);
                        double gr, gi;
                        cget(grid, prec, (l3 * fine[1] + l2) * fine[0] + l1, &gr, &gi);
                        ir += gr * rows[0][a];
                        ii += gi * rows[0][a];
                    }
                    mr += ir * rows[1][b];
                    mi += ii * rows[1][b];
                }
                accr += mr * rows[2][e];
                acci += mi * rows[2][e];
            }
        }
        if (prec) {
            ((double *)out)[2 * src] = accr;
            ((double *)out)[2 * src + 1] = acci;
        } else {
            ((float *)out)[2 * src] = (float)accr;
            ((float *)out)[2 * src + 1] = (float)acci;
        }
    }
}

/* Type-1 deconvolution (SPEC.md:408-416 + phase): modes (N_d..N_1), k_1
 * fastest, centered (kernel.py:176-178).  corr: per-axis real factors
 * phi_hat^-1 * (2/w) (double), length N_i each, concatenated. */
void or_deconv_type1(int d, const int64_t *N, const int64_t *fine, const double *corr,
                     const void *spec, int prec, void *modes) {
    int64_t N3 = d == 3 ? N[2] : 1;
    const double *c1 = corr, *c2 = corr + N[0], *c3 = corr + N[0] + N[1];
    for (int64_t i3 = 0; i3 < N3; ++i3) {
        int64_t k3 = i3 - N3 / 2;
        int64_t l3 = d == 3 ? pymod(k3, fine[2]) : 0;
        double f3 = d == 3 ? c3[i3] * ((k3 & 1) ? -1.0 : 1.0) : 1.0;
        for (int64_t i2 = 0; i2 < N[1]; ++i2) {
            int64_t k2 = i2 - N[1] / 2;
            int64_t l2 = pymod(k2, fine[1]);
            double f2 = f3 * c2[i2] * ((k2 & 1) ? -1.0 : 1.0);
            for (int64_t i1 = 0; i1 < N[0]; ++i1) {
                int64_t k1 = i1 - N[0] / 2;
                int64_t l1 = pymod(k1, fine[0]);
                double f = f2 * c1[i1] * ((k1 & 1) ? -1.0 : 1.0);
                double re, im;
                cget(spec, prec, (l3 * fine[1] + l2) * fine[0] + l1, &re, &im);
                int64_t o = (i3 * N[1] + i2) * N[0] + i1;
                if (prec) {
                    ((double *)modes)[2 * o] = re * f;
                    ((double *)modes)[2 * o + 1] = im * f;
                } else {
                    ((float *)modes)[2 * o] = (float)(re * f);
                    ((float *)modes)[2 * o + 1] = (float)(im * f);
                }
            }
        }
    }
}

/* Type-2 amplify + zero-pad (SPEC.md:418-425 + phase).  spec is zeroed here. */
void or_deconv_type2(int d, const int64_t *N, const int64_t *fine, const double *corr,
                     const void *modes, int prec, void *spec) {
    int64_t ncell = grid_cells(d, fine);
    memset(spec, 0, (size_t)ncell * (prec ? 16 : 8));
    int64_t N3 = d == 3 ? N[2] : 1;
    const double *c1 = corr, *c2 = corr + N[0], *c3 = corr + N[0] + N[1];
    for (int64_t i3 = 0; i3 < N3; ++i3) {
        int64_t k3 = i3 - N3 / 2;
        int64_t l3 = d == 3 ? pymod(k3, fine[2]) : 0;
        double f3 = d == 3 ? c3[i3] * ((k3 & 1) ? -1.0 : 1.0) : 1.0;
        for (int64_t i2 = 0; i2 < N[1]; ++i2) {
            int64_t k2 = i2 - N[1] / 2;
            int64_t l2 = pymod(k2, fine[1]);
            double f2 = f3 * c2[i2] * ((k2 & 1) ? -1.0 : 1.0);
            for (int64_t i1 = 0; i1 < N[0]; ++i1) {
                int64_t k1 = i1 - N[0] / 2;
                int64_t l1 = pymod(k1, fine[0]);
                double f = f2 * c1[i1] * ((k1 & 1) ? -1.0 : 1.0);
                double re, im;
                int64_t o = (i3 * N[1] + i2) * N[0] + i1;
                cget(modes, prec, o, &re, &im);
                int64_t dst = (l3 * fine[1] + l2) * fine[0] + l1;
                if (prec) {
                    ((double *)spec)[2 * dst] = re * f;
                    ((double *)spec)[2 * dst + 1] = im * f;
                } else {
                    ((float *)spec)[2 * dst] = (float)(re * f);
                    ((float *)spec)[2 * dst + 1] = (float)(im * f);
                }
            }
        }
    }
}

/* Neumaier compensated accumulator. */
typedef struct { double s, c; } nsum;
static inline void nadd(nsum *a, double x) {
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else a->c += (x - t) + a->s;
    a->s = t;
}

/* direct_type1: f_k = sum_j c_j exp(-i k.x_j). pts (M,d)
 * double, c complex128, modes complex128 in the library layout. */
void or_direct_type1(int64_t M, int d, const double *pts, const double *c,
                     const int64_t *N, int nthreads, double *modes) {
    int64_t N3 = d == 3 ? N[2] : 1;
    int64_t tot = N[0] * N[1] * N3;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
    for (int64_t o = 0; o < tot; ++o) {
        int64_t i1 = o % N[0], i2 = (o / N[0]) % N[1], i3 = o / (N[0] * N[1]);
        double k1 = (double)(i1 - N[0] / 2), k2 = (double)(i2 - N[1] / 2);
        double k3 = d == 3 ? (double)(i3 - N3 / 2) : 0.0;
        nsum re = {0, 0}, im = {0, 0};
        for (int64_t j = 0; j < M; ++j) {
            double ph = k1 * pts[j * d] + k2 * pts[j * d + 1];
            if (d == 3) ph += k3 * pts[j * d + 2];
            double s = sin(ph), co = cos(ph);
            double cr = c[2 * j], ci = c[2 * j + 1];
            /* (cr + i ci)(co - i s) */
            nadd(&re, cr * co + ci * s);
            nadd(&im, ci * co - cr * s);
        }
        modes[2 * o] = re.s + re.c;
        modes[2 * o + 1] = im.s + im.c;
    }
}

/* direct_type1 at selected modes only (SPEC.md:473-481 restricted to the
 * integer wave vectors kv (nk, d)): spot checks at geometries whose full
 * direct sum is out of reach (BASELINE C3-C5). */
void or_direct_type1_at(int64_t M, int d, const double *pts, const double *c, int64_t nk,
                        const int64_t *kv, int nthreads, double *out) {
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int64_t o = 0; o < nk; ++o) {
        double k1 = (double)kv[o * d], k2 = (double)kv[o * d + 1];
        double k3 = d == 3 ? (double)kv[o * d + 2] : 0.0;
        nsum re = {0, 0}, im = {0, 0};
        for (int64_t j = 0; j < M; ++j) {
            double ph = k1 * pts[j * d] + k2 * pts[j * d + 1];
            if (d == 3) ph += k3 * pts[j * d + 2];
            double s = sin(ph), co = cos(ph);
            double cr = c[2 * j], ci = c[2 * j + 1];
            nadd(&re, cr * co + ci * s);
            nadd(&im, ci * co - cr * s);
        }
        out[2 * o] = re.s + re.c;
        out[2 * o + 1] = im.s + im.c;
    }
}

/* direct_type2: c_j = sum_k f_k exp(+i k.x_j). */
void or_direct_type2(int64_t M, int d, const double *pts, const double *modes,
                     const int64_t *N, int nthreads, double *c) {
    int64_t N3 = d == 3 ? N[2] : 1;
    int64_t tot = N[0] * N[1] * N3;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
    for (int64_t j = 0; j < M; ++j) {
        nsum re = {0, 0}, im = {0, 0};
        for (int64_t o = 0; o < tot; ++o) {
            int64_t i1 = o % N[0], i2 = (o / N[0]) % N[1], i3 = o / (N[0] * N[1]);
            double ph = (double)(i1 - N[0] / 2) * pts[j * d] +
                        (double)(i2 - N[1] / 2) * pts[j * d + 1];
            if (d == 3) ph += (double)(i3 - N3 / 2) * pts[j * d + 2];
            double s = sin(ph), co = cos(ph);
            double fr = modes[2 * o], fi = modes[2 * o + 1];
            nadd(&re, fr * co - fi * s);
            nadd(&im, fr * s + fi * co);
        }
        c[2 * j] = re.s + re.c;
        c[2 * j + 1] = im.s + im.c;
    }
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
