// C-ABI entry points of libnufft_b200.so (include/nufft_b200.h): plan
// lifecycle, stage-level parity hooks and cuFFT glue.
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "nk_internal.cuh"

namespace {
thread_local std::string g_err;
thread_local int64_t g_err_idx = -1;

const char *cufft_msg(cufftResult r) {
    switch (r) {
    case CUFFT_SUCCESS: return "success";
    case CUFFT_ALLOC_FAILED: return "allocation failed";
    case CUFFT_INVALID_VALUE: return "invalid value";
    case CUFFT_EXEC_FAILED: return "exec failed";
    case CUFFT_SETUP_FAILED: return "setup failed";
    case CUFFT_INVALID_SIZE: return "invalid size";
    default: return "cuFFT error";
    }
}

#define NK_CUFFT(expr)                                                            \
    do {                                                                          \
        cufftResult _r = (expr);                                                  \
        if (_r != CUFFT_SUCCESS) {                                                \
            nk_set_error(std::string("cuFFT: ") + cufft_msg(_r) + " (" +          \
                         std::to_string((int)_r) + ") at " + __FILE__ + ":" +     \
                         std::to_string(__LINE__));                               \
            return _r == CUFFT_ALLOC_FAILED ? NK_ERR_MEMORY : NK_ERR_CUDA;        \
        }                                                                         \
    } while (0)

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int stage_buffer(void **buf, size_t *cap, size_t need) {
    if (need <= *cap && *buf) return NK_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    NK_CUDA(cudaMalloc(buf, std::max<size_t>(need, 16)));
    *cap = std::max<size_t>(need, 16);
    return NK_OK;
}

void free_plan(nk_plan *p) {
    if (!p) return;
    void *bufs[] = {p->d_fine, p->d_corr, p->d_keys_in, p->d_keys, p->d_perm, p->d_counts,
                    p->d_starts, p->d_pts, p->d_alt_keys, p->d_alt_vals, p->d_tile_hist,
                    p->d_scan_tmp, p->d_bad, p->d_nsub_off, p->d_sub_bin, p->d_sub_start,
                    p->d_sub_stop, p->d_in_stage, p->d_out_stage, p->d_vperm_buf,
                    p->d_pts_alt, p->d_sort_scr, p->d_work, p->d_cvis, p->d_rec, p->d_sub_sched};
    for (void *b : bufs)
        if (b) cudaFree(b);
    free(p->h_det_off);
    if (p->h_flags) cudaFreeHost(p->h_flags);
    if (p->fft_ok) cufftDestroy(p->fft);
    if (p->fft_col_ok) cufftDestroy(p->fft_col);
    if (p->d_twiddle) cudaFree(p->d_twiddle);
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    if (p->ev_ok)
        for (auto &e : p->ev) cudaEventDestroy(e);
    delete p;
}

// Every entry point that touches the device runs on the plan's device and
// restores the caller's current device on return (a single process may
// drive plans on several GPUs, PAPER.md:1617-1618 gpu_device_id).
struct DevGuard {
    int prev = -1;
    bool switched = false;
    explicit DevGuard(int dev) {
        if (dev < 0 || cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        if (prev != dev) switched = cudaSetDevice(dev) == cudaSuccess;
        if (!switched) cudaGetLastError();
    }
    ~DevGuard() {
        if (switched) cudaSetDevice(prev);
    }
};
#define NK_DEVICE_GUARD(p) DevGuard _nk_dev_guard((p)->device)

int check_plan(const nk_plan *p) {
    if (!p) {
        nk_set_error("null plan");
        return NK_ERR_VALUE;
    }
    return NK_OK;
}

int do_fft(nk_plan *p, void *fine, int direction) {
    int dir = direction < 0 ? CUFFT_FORWARD : CUFFT_INVERSE;
    if (p->prec == NK_DOUBLE)
        NK_CUFFT(cufftExecZ2Z(p->fft, (cufftDoubleComplex *)fine, (cufftDoubleComplex *)fine, dir));
    else
        NK_CUFFT(cufftExecC2C(p->fft, (cufftComplex *)fine, (cufftComplex *)fine, dir));
    return NK_OK;
}

}  // namespace

void nk_set_error(const std::string &msg) { g_err = msg; }
void nk_set_error_index(int64_t idx) { g_err_idx = idx; }

extern "C" const char *nk_last_error(void) { return g_err.c_str(); }
extern "C" int64_t nk_error_index(void) { return g_err_idx; }

extern "C" void nk_default_opts(nk_opts *o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->method = NK_METHOD_DEFAULT;
    o->device = -1;
    o->n_trans = 1;
}

extern "C" int nk_plan_create(int type, int dim, const int64_t *modes, double eps, int precision,
                              const nk_opts *opts_in, nk_plan **out) {
    if (!out || !modes) {
        nk_set_error("null argument");
        return NK_ERR_VALUE;
    }
    *out = nullptr;
    nk_opts opts;
    if (opts_in) opts = *opts_in;
    else nk_default_opts(&opts);
    if (type != 1 && type != 2) {
        nk_set_error("transform type must be 1 or 2, got " + std::to_string(type));
        return NK_ERR_VALUE;
    }
    if (dim != 2 && dim != 3) {   // reject dim 1 or > 3
        nk_set_error("dimension must be 2 or 3, got " + std::to_string(dim));
        return NK_ERR_VALUE;
    }
    for (int i = 0; i < dim; ++i)
        if (modes[i] < 1 || modes[i] > (1 << 24)) {
            nk_set_error("mode counts must be >= 1, got " + std::to_string(modes[i]));
            return NK_ERR_VALUE;
        }
    double eps_eff, beta;
    int w, clamped;
    int rc = nk_tolerance_to_width(eps, precision, &eps_eff, &w, &beta, &clamped);
    if (rc) return rc;
    if (opts.method < NK_METHOD_DEFAULT || opts.method > NK_SM) {
        nk_set_error("method must be gm, gmsort or sm");
        return NK_ERR_VALUE;
    }

    if (opts.n_trans < 0 || opts.n_trans > (1 << 20)) {
        nk_set_error("n_trans must be >= 1, got " + std::to_string(opts.n_trans));
        return NK_ERR_VALUE;
    }
    nk_plan *p = new nk_plan();
    memset((void *)p, 0, sizeof(*p));
    p->ntrans = opts.n_trans > 0 ? opts.n_trans : 1;
    p->deterministic = opts.deterministic ? 1 : 0;
    p->type = type;
    p->dim = dim;
    p->prec = precision;
    p->eps = eps_eff;
    p->w = w;
    p->beta = beta;
    p->eps_clamped = clamped;
    p->halo = (w + 1) / 2;   // kernel.py:72
    p->csize = precision == NK_DOUBLE ? 16 : 8;
    p->stream = (cudaStream_t)opts.stream;
    p->timing = opts.timing;
    p->n_tot = 1;
    p->N_tot = 1;
    for (int i = 0; i < 3; ++i) {
        p->N[i] = i < dim ? modes[i] : 1;
        int64_t n = i < dim ? opts.fine[i] : 1;
        if (i < dim && n <= 0) n = nk_next_smooth(std::max<int64_t>(2 * p->N[i], 2 * w));
        p->n[i] = n;
        if (i < dim && (n < w || n < p->N[i] || n > (1 << 30))) {
            nk_set_error("fine grid size " + std::to_string(n) + " too small for axis " +
                         std::to_string(i + 1));
            delete p;
            return NK_ERR_VALUE;
        }
        p->alpha[i] = i < dim ? w * NK_PI / (double)n : 0.0;   // kernel.py:115
        p->n_tot *= p->n[i];
        p->N_tot *= p->N[i];
    }
    // bins (binsort.py:34-35,143-145)
    const int def2[3] = {32, 32, 1}, def3[3] = {16, 16, 2};
    p->nbins = 1;
    for (int i = 0; i < 3; ++i) {
        int m = i < dim ? opts.bin_dims[i] : 1;
        if (i < dim && m == 0) m = dim == 2 ? def2[i] : def3[i];
        if (m < 1) {
            nk_set_error("invalid bin dims");
            delete p;
            return NK_ERR_VALUE;
        }
        p->bin_dims[i] = m;
        p->nb[i] = (p->n[i] + m - 1) / m;
        p->nbins *= p->nb[i];
    }
    if (p->nbins >= (1ll << 30)) {
        nk_set_error("too many bins");
        delete p;
        return NK_ERR_VALUE;
    }
    // M_sub: the reference default is 1024 (binsort.py:38).  A plan that is
    // not given one picks the B200-tuned size for its kernel: 128 for the
    // one-warp 2D spread (more warps in flight), 4096 for the staged
    // interpolation (one padded-bin load per bin).  Stage-level
    // build_subproblems keeps the reference default.
    // (the tiled f64 3D interpolation, K7t, takes subproblems of <= 1024)
    p->msub = opts.max_subproblem
                  ? opts.max_subproblem
                  : (type == 2 ? (dim == 3 && precision == NK_DOUBLE ? kTileMsub : 4096)
                               : (dim == 2 ? 128 : 1024));
    if (p->msub < 1) {
        nk_set_error("max subproblem size must be >= 1, got " + std::to_string(p->msub));
        delete p;
        return NK_ERR_VALUE;
    }

    // device: the plan lives on opts.device (or the current one); the
    // caller's current device is restored on return
    if (opts.device >= 0) {
        int ndev = 0;
        cudaGetDeviceCount(&ndev);
        cudaGetLastError();
        if (opts.device >= ndev) {
            nk_set_error("invalid CUDA device " + std::to_string(opts.device));
            delete p;
            return NK_ERR_VALUE;
        }
        p->device = opts.device;
    } else {
        cudaGetDevice(&p->device);
    }
    DevGuard dev_guard(p->device);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);

    // method (SPEC.md:170 defaults: SM for type 1; type 2 defaults to the
    // shared-memory staged gather, measured faster than GM-sort on B200) and
    // the shared-memory budget of the SM kernels.  Default bin dims are the
    // reference's; if the padded bin does not fit in shared memory they are
    // halved along the larger of axes 1/2 until it does.
    int method = opts.method;
    const bool user_bins = opts.bin_dims[0] || opts.bin_dims[1] || opts.bin_dims[2];
    if (method == NK_METHOD_DEFAULT) method = NK_SM;
    // B200-tuned bin shapes for the SM kernels when the caller gave none
    // (measured sweeps): smaller padded bins keep more CTAs
    // (or the 2D one-warp subproblems) resident per SM.  GM / GM-sort and the
    // stage-level bin_sort keep the reference defaults (binsort.py:34-35).
    if (method == NK_SM && !user_bins) {
        static const int t1_2d[3] = {16, 8, 1}, t1_3s[3] = {4, 4, 4}, t1_3d[3] = {11, 7, 7},
                         t2_2d[3] = {32, 32, 1}, t2_3s[3] = {16, 16, 4}, t2_3d[3] = {11, 7, 7};
        const int *tb = type == 1 ? (dim == 2 ? t1_2d : (precision == NK_SINGLE ? t1_3s : t1_3d))
                                  : (dim == 2 ? t2_2d : (precision == NK_SINGLE ? t2_3s : t2_3d));
        p->nbins = 1;
        for (int i = 0; i < 3; ++i) {
            p->bin_dims[i] = i < dim ? tb[i] : 1;
            p->nb[i] = (p->n[i] + p->bin_dims[i] - 1) / p->bin_dims[i];
            p->nbins *= p->nb[i];
        }
        if (p->nbins >= (1ll << 30)) {
            nk_set_error("too many bins");
            delete p;
            return NK_ERR_VALUE;
        }
    }
    int64_t need = nk_sm_smem_bytes(type, dim, precision, w, p->bin_dims, p->halo, p->msub);
    if (method == NK_SM && need > smem_optin) {
        if (user_bins) {
            if (opts.method == NK_SM) {
                nk_set_error("padded bin needs " + std::to_string(need) +
                             " bytes of shared memory, more than the per-block " +
                             std::to_string(smem_optin) + "; use smaller bin dims or gmsort");
                delete p;
                return NK_ERR_VALUE;
            }
            method = NK_GMSORT;
        } else {
            while (need > smem_optin && (p->bin_dims[0] > 1 || p->bin_dims[1] > 1)) {
                int ax = p->bin_dims[0] >= p->bin_dims[1] ? 0 : 1;
                p->bin_dims[ax] = (p->bin_dims[ax] + 1) / 2;
                need = nk_sm_smem_bytes(type, dim, precision, w, p->bin_dims, p->halo, p->msub);
            }
            if (need > smem_optin) method = NK_GMSORT;
            p->nbins = 1;
            for (int i = 0; i < 3; ++i) {
                p->nb[i] = (p->n[i] + p->bin_dims[i] - 1) / p->bin_dims[i];
                p->nbins *= p->nb[i];
            }
        }
    }
    p->max_sub_smem = (int)std::min<int64_t>(need, INT32_MAX);
    p->max_pad_cells = 1;
    for (int i = 0; i < dim; ++i) p->max_pad_cells *= p->bin_dims[i] + 2 * p->halo;
    p->method = method;
    // footprint-start code space (setpts K4d): lexicographic in the padded
    // bin, or tile-major for the tiled f64 spread
    const bool tiled = nk_tiled(type, dim, precision, w, method, p->msub);
    const int tlg = tiled ? nk_tile_lg(w) : 0;
    p->start_space = p->max_pad_cells;
    if (tiled) {
        p->start_space = (int64_t)1 << (3 * tlg);
        for (int i = 0; i < dim; ++i)
            p->start_space *= (p->bin_dims[i] + 1 + (1 << tlg) - 1) >> tlg;
    }

    // geometry for kernels
    Geom &g = p->geom;
    g.dim = dim;
    for (int i = 0; i < 3; ++i) {
        g.n[i] = (int)p->n[i];
        g.N[i] = (int)p->N[i];
        g.m[i] = p->bin_dims[i];
        g.nb[i] = (int)p->nb[i];
        // multiply-high division of a cell index by the bin width (K1): exact
        // when cell * m < 2^32 for every cell < n (floor(c ceil(2^32/m) / 2^32)
        // = floor(c / m) while c m <= 2^32)
        g.mdiv[i] = g.m[i] > 1 && (uint64_t)p->n[i] * (uint64_t)g.m[i] <= (1ull << 32)
                        ? (unsigned)(((1ull << 32) + g.m[i] - 1) / g.m[i])
                        : 0u;
        g.scale[i] = (double)p->n[i] / NK_TWO_PI;   // binsort.py:99
    }
    g.halo = p->halo;
    g.w = w;
    g.tiled = tiled ? 1 : 0;
    g.tile_lg = tlg;
    g.beta = beta;
    g.betaf = (float)beta;
    g.betaf_log2e = (float)(beta * 1.4426950408889634);
    g.ntot = p->n_tot;
    g.Ntot = p->N_tot;
    g.M = 0;

    // correction factors, per axis, with (2/w) and the (-1)^k phase folded in
    std::vector<double> corr;
    const double floor_v = (precision == NK_DOUBLE ? DBL_MIN : FLT_MIN) * 100;  // kernel.py:190
    for (int i = 0; i < dim; ++i) {
        int64_t Ni = p->N[i];
        std::vector<double> xi(Ni), ft(Ni);
        for (int64_t k = 0; k < Ni; ++k) xi[k] = p->alpha[i] * (double)(k - Ni / 2);
        nk_kernel_fourier_host(beta, xi.data(), Ni, ft.data());
        for (int64_t k = 0; k < Ni; ++k) {
            if (!(ft[k] > floor_v)) {   // kernel.py:195-199
                nk_set_error("kernel Fourier transform underflowed on axis " +
                             std::to_string(i + 1) + "; correction factors would overflow");
                delete p;
                return NK_ERR_VALUE;
            }
            int64_t kk = k - Ni / 2;
            corr.push_back((2.0 / w) / ft[k] * ((kk & 1) ? -1.0 : 1.0));
        }
    }

    auto fail = [&](int code) {
        free_plan(p);
        return code;
    };
    cudaError_t e;
#define NK_ALLOC(ptr, bytes)                                                        \
    e = cudaMalloc((void **)&(ptr), std::max<size_t>((bytes), 16));                 \
    if (e != cudaSuccess) {                                                         \
        cudaGetLastError();                                                         \
        nk_set_error(std::string("device allocation failed: ") + cudaGetErrorString(e)); \
        return fail(NK_ERR_MEMORY);                                                 \
    }
    NK_ALLOC(p->d_fine, p->n_tot * p->csize * p->ntrans);
    // TMA tensor map of the fine grid for the tiled interpolation: one
    // cp.async.bulk.tensor box per (non-wrapping) padded bin
    if (type == 2 && method == NK_SM) {
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        if (!encode) {
            cudaDriverEntryPointQueryResult q;
            void *fn = nullptr;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                    cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
            cudaGetLastError();
        }
        // the grid as reals (2 n1, n2, n3, n_trans); 2D grids have n3 = 1
        const int h2 = 2 * p->halo;
        const cuuint64_t rs = precision == NK_DOUBLE ? 8 : 4;
        const cuuint64_t dims[4] = {(cuuint64_t)(2 * p->n[0]), (cuuint64_t)p->n[1],
                                    (cuuint64_t)p->n[2], (cuuint64_t)p->ntrans};
        const cuuint64_t strides[3] = {(cuuint64_t)(2 * rs * p->n[0]),
                                       (cuuint64_t)(2 * rs * p->n[0] * p->n[1]),
                                       (cuuint64_t)(2 * rs * p->n_tot)};
        const cuuint32_t box[4] = {(cuuint32_t)(2 * (p->bin_dims[0] + h2)),
                                   (cuuint32_t)(p->bin_dims[1] + h2),
                                   (cuuint32_t)(dim == 3 ? p->bin_dims[2] + h2 : 1), 1};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        p->tmap_ok = encode && box[0] <= 256 && box[1] <= 256 && box[2] <= 256 &&
                     (box[0] * rs) % 16 == 0 && strides[0] % 16 == 0 &&
                     encode(&p->tmap_fine,
                            precision == NK_DOUBLE ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                                   : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                            4, p->d_fine, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    NK_ALLOC(p->d_corr, corr.size() * p->csize / 2);
    NK_ALLOC(p->d_counts, 4 * p->nbins);
    NK_ALLOC(p->d_starts, 4 * (p->nbins + 1));
    NK_ALLOC(p->d_nsub_off, 4 * (p->nbins + 1));
    NK_ALLOC(p->d_bad, 4 * sizeof(unsigned long long));
    e = cudaMallocHost((void **)&p->h_flags, 4 * sizeof(unsigned long long));
    if (e != cudaSuccess) {
        cudaGetLastError();
        p->h_flags = nullptr;
        nk_set_error(std::string("pinned host allocation failed: ") + cudaGetErrorString(e));
        return fail(NK_ERR_MEMORY);
    }
    NK_ALLOC(p->d_work, sizeof(int) * p->ntrans);
#undef NK_ALLOC
    if (precision == NK_DOUBLE) {
        e = cudaMemcpy(p->d_corr, corr.data(), 8 * corr.size(), cudaMemcpyHostToDevice);
    } else {
        std::vector<float> cf(corr.begin(), corr.end());
        e = cudaMemcpy(p->d_corr, cf.data(), 4 * cf.size(), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        nk_set_error(std::string("cudaMemcpy: ") + cudaGetErrorString(e));
        return fail(NK_ERR_CUDA);
    }

    // cuFFT plan on the fine grid, slowest axis first
    int nn[3];
    for (int i = 0; i < dim; ++i) nn[i] = (int)p->n[dim - 1 - i];
    cufftResult fr = cufftPlanMany(&p->fft, dim, nn, nn, 1, (int)p->n_tot, nn, 1,
                                   (int)p->n_tot, precision == NK_DOUBLE ? CUFFT_Z2Z : CUFFT_C2C,
                                   p->ntrans);
    if (fr != CUFFT_SUCCESS) {
        nk_set_error(std::string("cufftPlanMany failed: ") + cufft_msg(fr));
        return fail(fr == CUFFT_ALLOC_FAILED ? NK_ERR_MEMORY : NK_ERR_CUDA);
    }
    p->fft_ok = true;
    cufftSetStream(p->fft, p->stream);
    // 2D, single precision, one vector, n_1 = 2^L in [256, 4096]: the pad
    // (type 2) or the deconvolution (type 1) is fused with the x-row FFTs;
    // cuFFT only runs the y axis
    {
        const int64_t n1 = p->n[0];
        const char *fe = getenv("NK_FUSED_ROWS");
        // 2D only: in 3D the strided rank-2 (z, y) cuFFT plan took 390 us
        // against 144 us for the whole 3D transform at 256^3
        if (dim == 2 && precision == NK_SINGLE && p->ntrans == 1 && (n1 & (n1 - 1)) == 0 &&
            n1 >= 256 && n1 <= 4096 && !(fe && fe[0] == '0')) {
            // the y axis of every x column: a strided batch of 1D transforms
            int nc[2] = {(int)p->n[dim - 1], (int)p->n[1]};
            fr = cufftPlanMany(&p->fft_col, dim - 1, nc, nc, (int)n1, 1, nc, (int)n1, 1,
                               CUFFT_C2C, (int)n1);
            if (fr == CUFFT_SUCCESS) {
                p->fft_col_ok = true;
                cufftSetStream(p->fft_col, p->stream);
                std::vector<float> twh((size_t)(2 * n1));
                for (int64_t k = 0; k < n1; ++k) {
                    const double ang = NK_TWO_PI * (double)k / (double)n1;
                    twh[2 * k] = (float)cos(ang);
                    twh[2 * k + 1] = (float)sin(ang);
                }
                e = cudaMalloc(&p->d_twiddle, sizeof(float) * 2 * n1);
                if (e == cudaSuccess)
                    e = cudaMemcpy(p->d_twiddle, twh.data(), sizeof(float) * 2 * n1,
                                   cudaMemcpyHostToDevice);
                p->fused_rows = e == cudaSuccess;
                if (e != cudaSuccess) cudaGetLastError();
            }
        }
    }
    if (p->timing) {
        for (auto &ev : p->ev) cudaEventCreate(&ev);
        p->ev_ok = true;
    }
    {
        const char *ng = getenv("NK_NO_GRAPH");
        p->use_graph = !(ng && ng[0] == '1');
        if (p->use_graph &&
            cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            p->use_graph = false;
            p->cap_stream = nullptr;
        }
    }
    *out = p;
    return NK_OK;
}

extern "C" int nk_plan_get_info(const nk_plan *p, nk_plan_info *info) {
    int rc = check_plan(p);
    if (rc) return rc;
    memset(info, 0, sizeof(*info));
    info->type = p->type;
    info->dim = p->dim;
    info->precision = p->prec;
    info->method = p->method;
    for (int i = 0; i < 3; ++i) {
        info->modes[i] = p->N[i];
        info->fine[i] = p->n[i];
        info->alpha[i] = p->alpha[i];
        info->bin_dims[i] = p->bin_dims[i];
        info->bins_per_axis[i] = p->nb[i];
    }
    info->epsilon = p->eps;
    info->w = p->w;
    info->beta = p->beta;
    info->eps_clamped = p->eps_clamped;
    info->nbins = p->nbins;
    info->max_subproblem = p->msub;
    info->halo = p->halo;
    info->num_points = p->have_points ? p->M : 0;
    info->num_subproblems = p->S;
    info->n_trans = p->ntrans;
    return NK_OK;
}

extern "C" int nk_set_stream(nk_plan *p, void *stream) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    p->stream = (cudaStream_t)stream;
    NK_CUFFT(cufftSetStream(p->fft, p->stream));
    if (p->fft_col_ok) NK_CUFFT(cufftSetStream(p->fft_col, p->stream));
    return NK_OK;
}

extern "C" int nk_setpts(nk_plan *p, int64_t M, int coord_prec, const void *x, const void *y,
                         const void *z, int64_t stride) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    if (M < 0 || M >= INT32_MAX) {
        nk_set_error("number of points must be in [0, 2^31-1), got " + std::to_string(M));
        return NK_ERR_VALUE;
    }
    if (coord_prec != NK_SINGLE && coord_prec != NK_DOUBLE) {
        nk_set_error("coordinate precision must be single or double");
        return NK_ERR_VALUE;
    }
    if (stride < 1) stride = 1;
    const void *ax[3] = {x, y, z};
    for (int i = 0; i < p->dim; ++i)
        if (M > 0 && !ax[i]) {
            nk_set_error("missing coordinate array for axis " + std::to_string(i + 1));
            return NK_ERR_VALUE;
        }
    p->have_points = false;
    p->M = M;
    p->geom.M = M;
    if (p->gexec) {   // kernel parameters (M, S, buffers) change with the points
        cudaGraphExecDestroy(p->gexec);
        p->gexec = nullptr;
    }
    // host coordinates: copy each axis (strided) into a device SoA buffer
    void *dev_axes[3] = {nullptr, nullptr, nullptr};
    const void *use[3] = {x, y, z};
    int64_t use_stride = stride;
    bool host = false;
    for (int i = 0; i < p->dim; ++i)
        if (M > 0 && !is_device_ptr(ax[i])) host = true;
    if (host) {
        size_t es = coord_prec == NK_DOUBLE ? 8 : 4;
        for (int i = 0; i < p->dim; ++i) {
            NK_CUDA(cudaMalloc(&dev_axes[i], es * M));
            NK_CUDA(cudaMemcpy2DAsync(dev_axes[i], es, ax[i], es * stride, es, M,
                                      cudaMemcpyHostToDevice, p->stream));
            use[i] = dev_axes[i];
        }
        use_stride = 1;
    }
    rc = nk_sort_points(p, coord_prec, use[0], use[1], use[2], use_stride);
    for (void *d : dev_axes)
        if (d) cudaFree(d);
    if (rc) return rc;
    p->have_points = true;
    return NK_OK;
}

static int execute_device(nk_plan *p, const void *in, void *out) {
    int launches = 0;
    int rc;
    if (p->timing) NK_CUDA(cudaEventRecord(p->ev[0], p->stream));
    if (p->type == 1) {
        rc = nk_launch_spread(p, in, p->d_fine, &launches);
        if (rc) return rc;
        if (p->timing) NK_CUDA(cudaEventRecord(p->ev[1], p->stream));
        if (p->fused_rows) {
            NK_CUFFT(cufftExecC2C(p->fft_col, (cufftComplex *)p->d_fine,
                                  (cufftComplex *)p->d_fine, CUFFT_FORWARD));
            if (p->timing) NK_CUDA(cudaEventRecord(p->ev[2], p->stream));
            rc = nk_launch_rowfft_deconv(p, p->d_fine, out);
            if (rc) return rc;
            launches += 1;
        } else {
            rc = do_fft(p, p->d_fine, -1);
            if (rc) return rc;
            if (p->timing) NK_CUDA(cudaEventRecord(p->ev[2], p->stream));
            rc = nk_launch_deconv1(p, p->d_fine, out);
            if (rc) return rc;
            launches += p->N_tot > 0;
        }
    } else {
        if (p->fused_rows) {
            rc = nk_launch_pad_rowfft(p, in, p->d_fine);
            if (rc) return rc;
            launches += 1;
            if (p->timing) NK_CUDA(cudaEventRecord(p->ev[1], p->stream));
            NK_CUFFT(cufftExecC2C(p->fft_col, (cufftComplex *)p->d_fine,
                                  (cufftComplex *)p->d_fine, CUFFT_INVERSE));
        } else {
            rc = nk_launch_deconv2(p, in, p->d_fine);
            if (rc) return rc;
            launches += 1;
            if (p->timing) NK_CUDA(cudaEventRecord(p->ev[1], p->stream));
            rc = do_fft(p, p->d_fine, +1);
            if (rc) return rc;
        }
        if (p->timing) NK_CUDA(cudaEventRecord(p->ev[2], p->stream));
        rc = nk_launch_interp(p, p->d_fine, out, &launches);
        if (rc) return rc;
    }
    if (p->timing) NK_CUDA(cudaEventRecord(p->ev[3], p->stream));
    p->last_launches = launches;
    return NK_OK;
}

// Capture execute_device() once per (in, out) pair on the plan's private
// capture stream and replay it into the caller's stream: one cudaGraphLaunch
// instead of ~4 kernel/cuFFT launches per execute.
static int execute_graph(nk_plan *p, const void *in, void *out) {
    if (p->g_in != in || p->g_out != out) {
        // a new (in, out) pair: launch directly; capture only when the same
        // pair comes back (repeated executes on fixed buffers)
        if (p->gexec) {
            cudaGraphExecDestroy(p->gexec);
            p->gexec = nullptr;
        }
        p->g_in = in;
        p->g_out = out;
        return execute_device(p, in, out);
    }
    if (!p->gexec) {
        cudaStream_t user = p->stream;
        p->stream = p->cap_stream;
        NK_CUFFT(cufftSetStream(p->fft, p->cap_stream));
        if (p->fft_col_ok) NK_CUFFT(cufftSetStream(p->fft_col, p->cap_stream));
        NK_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
        int rc = execute_device(p, in, out);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(p->cap_stream, &graph);
        p->stream = user;
        cufftSetStream(p->fft, user);
        if (p->fft_col_ok) cufftSetStream(p->fft_col, user);
        if (rc || e != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            // fall back to direct launches for this plan
            p->use_graph = false;
            return execute_device(p, in, out);
        }
        e = cudaGraphInstantiate(&p->gexec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p->gexec = nullptr;
            p->use_graph = false;
            return execute_device(p, in, out);
        }
        p->g_in = in;
        p->g_out = out;
        p->g_launches = p->last_launches;
    }
    NK_CUDA(cudaGraphLaunch(p->gexec, p->stream));
    p->last_launches = p->g_launches;
    return NK_OK;
}

extern "C" int nk_execute(nk_plan *p, const void *in, void *out) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    if (!p->have_points) {
        nk_set_error("execute called before set_points");
        return NK_ERR_STATE;
    }
    const size_t in_bytes = (p->type == 1 ? p->M : p->N_tot) * p->csize * p->ntrans;
    const size_t out_bytes = (p->type == 1 ? p->N_tot : p->M) * p->csize * p->ntrans;
    if ((in_bytes && !in) || (out_bytes && !out)) {
        nk_set_error("null input or output buffer");
        return NK_ERR_VALUE;
    }
    const bool in_host = in_bytes && !is_device_ptr(in);
    const bool out_host = out_bytes && !is_device_ptr(out);
    const void *din = in;
    void *dout = out;
    if (in_host) {
        rc = stage_buffer(&p->d_in_stage, &p->cap_in_stage, in_bytes);
        if (rc) return rc;
        NK_CUDA(cudaMemcpyAsync(p->d_in_stage, in, in_bytes, cudaMemcpyHostToDevice, p->stream));
        din = p->d_in_stage;
    }
    if (out_host) {
        rc = stage_buffer(&p->d_out_stage, &p->cap_out_stage, out_bytes);
        if (rc) return rc;
        dout = p->d_out_stage;
    }
    rc = (p->use_graph && !p->timing) ? execute_graph(p, din, dout)
                                      : execute_device(p, din, dout);
    if (rc) return rc;
    if (out_host)
        NK_CUDA(cudaMemcpyAsync(out, dout, out_bytes, cudaMemcpyDeviceToHost, p->stream));
    if (in_host || out_host) NK_CUDA(cudaStreamSynchronize(p->stream));
    return NK_OK;
}

extern "C" int nk_destroy(nk_plan *p) {
    if (!p) return NK_OK;
    NK_DEVICE_GUARD(p);
    if (p->stream) cudaStreamSynchronize(p->stream);
    free_plan(p);
    return NK_OK;
}

// ------------------------------------------------------------ stage level

extern "C" int nk_get_layout(const nk_plan *p, int32_t *point_bins, int32_t *counts,
                             int32_t *starts, int32_t *perm) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    if (!p->have_points) {
        nk_set_error("no points set");
        return NK_ERR_STATE;
    }
    if (!p->sorted && (perm || counts || starts) && p->M > 0) {
        nk_set_error("bin layout requires a gmsort or sm plan");
        return NK_ERR_STATE;
    }
    cudaStream_t st = p->stream;
    if (perm && p->M && !p->perm_valid) {
        // the plan visits points in (bin, start) order; derive the
        // reference's bin-stable permutation now (a cached parity export)
        rc = nk_compute_bin_perm(const_cast<nk_plan *>(p));
        if (rc) return rc;
    }
    if (point_bins && p->M)
        NK_CUDA(cudaMemcpyAsync(point_bins, p->d_keys_in, 4 * p->M, cudaMemcpyDefault, st));
    if (counts) NK_CUDA(cudaMemcpyAsync(counts, p->d_counts, 4 * p->nbins, cudaMemcpyDefault, st));
    if (starts)
        NK_CUDA(cudaMemcpyAsync(starts, p->d_starts, 4 * (p->nbins + 1), cudaMemcpyDefault, st));
    if (perm && p->M) NK_CUDA(cudaMemcpyAsync(perm, p->d_perm, 4 * p->M, cudaMemcpyDefault, st));
    NK_CUDA(cudaStreamSynchronize(st));
    return NK_OK;
}

extern "C" int nk_get_subproblems(const nk_plan *p, int32_t *bin_ids, int32_t *slice_starts,
                                  int32_t *slice_stops, int32_t *offsets, int32_t *padded) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    if (p->method != NK_SM) {
        nk_set_error("subproblems exist only for sm plans");
        return NK_ERR_STATE;
    }
    if (p->S == 0) return NK_OK;
    size_t b = 4 * (size_t)p->S, bd = b * p->dim;
    int32_t *tmp = nullptr;
    NK_CUDA(cudaMalloc((void **)&tmp, 3 * b + 2 * bd));
    int32_t *tb = tmp, *ts = tmp + p->S, *te = tmp + 2 * p->S, *to = tmp + 3 * p->S,
            *tp = to + p->S * p->dim;
    rc = nk_export_subproblems(p, tb, ts, te, to, tp);
    if (!rc) {
        cudaStream_t st = p->stream;
        if (bin_ids) cudaMemcpyAsync(bin_ids, tb, b, cudaMemcpyDefault, st);
        if (slice_starts) cudaMemcpyAsync(slice_starts, ts, b, cudaMemcpyDefault, st);
        if (slice_stops) cudaMemcpyAsync(slice_stops, te, b, cudaMemcpyDefault, st);
        if (offsets) cudaMemcpyAsync(offsets, to, bd, cudaMemcpyDefault, st);
        if (padded) cudaMemcpyAsync(padded, tp, bd, cudaMemcpyDefault, st);
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            nk_set_error(std::string("CUDA error: ") + cudaGetErrorString(e));
            rc = NK_ERR_CUDA;
        }
    }
    cudaFree(tmp);
    return rc;
}

extern "C" int nk_spread(nk_plan *p, const void *strengths, void *fine) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    if (!p->have_points) {
        nk_set_error("spread called before set_points");
        return NK_ERR_STATE;
    }
    int launches = 0;
    return nk_launch_spread(p, strengths, fine, &launches);
}

extern "C" int nk_interp(nk_plan *p, const void *fine, void *out) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    if (!p->have_points) {
        nk_set_error("interp called before set_points");
        return NK_ERR_STATE;
    }
    int launches = 0;
    return nk_launch_interp(p, fine, out, &launches);
}

extern "C" int nk_fft(nk_plan *p, void *fine, int direction) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    return do_fft(p, fine, direction);
}

extern "C" int nk_deconv_type1(nk_plan *p, const void *spec, void *modes) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    return nk_launch_deconv1(p, spec, modes);
}

extern "C" int nk_fft_deconv_type1(nk_plan *p, void *fine, void *modes) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    if (p->fused_rows) {
        NK_CUFFT(cufftExecC2C(p->fft_col, (cufftComplex *)fine, (cufftComplex *)fine,
                              CUFFT_FORWARD));
        return nk_launch_rowfft_deconv(p, fine, modes);
    }
    rc = do_fft(p, fine, -1);
    if (rc) return rc;
    return nk_launch_deconv1(p, fine, modes);
}

extern "C" int nk_deconv_type2(nk_plan *p, const void *modes, void *spec) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    return nk_launch_deconv2(p, modes, spec);
}

extern "C" int nk_stage_times(nk_plan *p, float *ms, int n) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    if (!p->timing || !p->ev_ok) {
        nk_set_error("plan was not created with timing enabled");
        return NK_ERR_STATE;
    }
    NK_CUDA(cudaEventSynchronize(p->ev[3]));
    float t[4] = {0, 0, 0, 0};
    if (p->type == 1) {
        cudaEventElapsedTime(&t[0], p->ev[0], p->ev[1]);   // spread
        cudaEventElapsedTime(&t[1], p->ev[1], p->ev[2]);   // fft
        cudaEventElapsedTime(&t[2], p->ev[2], p->ev[3]);   // deconv
    } else {
        cudaEventElapsedTime(&t[0], p->ev[2], p->ev[3]);   // interp
        cudaEventElapsedTime(&t[1], p->ev[1], p->ev[2]);   // fft
        cudaEventElapsedTime(&t[2], p->ev[0], p->ev[1]);   // pad
    }
    cudaEventElapsedTime(&t[3], p->ev[0], p->ev[3]);
    for (int i = 0; i < n && i < 4; ++i) ms[i] = t[i];
    return NK_OK;
}

extern "C" int nk_set_timing(nk_plan *p, int on) {
    int rc = check_plan(p);
    if (rc) return rc;
    NK_DEVICE_GUARD(p);
    if (on && !p->ev_ok) {
        for (auto &ev : p->ev) NK_CUDA(cudaEventCreate(&ev));
        p->ev_ok = true;
    }
    p->timing = on ? 1 : 0;
    return NK_OK;
}

extern "C" int nk_last_launch_count(const nk_plan *p) { return p ? p->last_launches : 0; }
