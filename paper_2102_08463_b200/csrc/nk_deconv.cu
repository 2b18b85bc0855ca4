// K8 / K9: kernel-Fourier deconvolution with mode selection (type 1) and
// its adjoint amplify + zero-pad (type 2).
//
// SPEC.md:408-425 plus the (-1)^{sum k} phase forced by the reference's
// -pi-origin grid frame (binsort.py:10-12).  The correction
// factor p_k = (2/w)^d / prod_i phi_hat(alpha_i k_i) (kernel.py:181-205) is
// applied as a product of per-axis factors corr_i[k_i] = (2/w)(-1)^{k_i} /
// phi_hat(alpha_i k_i), so no N_tot-sized table is read per execute.
#include "nk_device.cuh"

namespace {

// type 1: modes (N_d..N_1) <- p_k (-1)^{sum k} bhat[k mod n].  One CTA per
// mode row (k_2, k_3): the row's factor and fine-row pointer are computed
// once; threads stream k_1 (coalesced reads of the two wrapped segments).
template <typename T>
__global__ void __launch_bounds__(256)
k_deconv1(Geom g, const T *__restrict__ corr, const typename cplx<T>::t *__restrict__ spec,
          typename cplx<T>::t *__restrict__ modes) {
    typedef typename cplx<T>::t C;
    const int N1 = g.N[0], N2 = g.N[1];
    const int row = blockIdx.x;            // i2 + N2 * i3
    spec += blockIdx.y * g.ntot;           // batched execute: vector blockIdx.y
    modes += blockIdx.y * g.Ntot;
    const int i2 = row % N2, i3 = row / N2;
    const int l2 = nk_wrap(i2 - N2 / 2, g.n[1]);
    T frow = corr[N1 + i2];
    int64_t fine_row = (int64_t)g.n[0] * l2;
    if (g.dim == 3) {
        frow *= corr[N1 + N2 + i3];
        fine_row += (int64_t)g.n[0] * g.n[1] * nk_wrap(i3 - g.N[2] / 2, g.n[2]);
    }
    const C *src = spec + fine_row;
    C *dst = modes + (int64_t)row * N1;
    for (int i1 = threadIdx.x; i1 < N1; i1 += blockDim.x) {
        C v = src[nk_wrap(i1 - N1 / 2, g.n[0])];
        const T f = frow * corr[i1];
        v.x *= f;
        v.y *= f;
        dst[i1] = v;
    }
}

// Mode index along one axis for fine index l, or -1 outside the band.
__device__ __forceinline__ int mode_of(int l, int N, int n) {
    const int kneg = N / 2;          // number of negative frequencies
    const int kpos = N - kneg;       // 0 .. kpos-1 non-negative
    if (l < kpos) return l + kneg;
    if (l >= n - kneg) return l - n + kneg;
    return -1;
}

// type 2: every fine cell written once: p_k (-1)^{sum k} f_k inside the
// band, zero elsewhere (fused zero-fill + scatter).  One CTA per fine row
// (l_2, l_3); rows outside the band are pure zero streams.
template <typename T>
__global__ void __launch_bounds__(256)
k_deconv2(Geom g, const T *__restrict__ corr, const typename cplx<T>::t *__restrict__ modes,
          typename cplx<T>::t *__restrict__ spec) {
    typedef typename cplx<T>::t C;
    const int n1 = g.n[0], n2 = g.n[1];
    const int N1 = g.N[0], N2 = g.N[1];
    const int row = blockIdx.x;            // l2 + n2 * l3
    modes += blockIdx.y * g.Ntot;          // batched execute: vector blockIdx.y
    spec += blockIdx.y * g.ntot;
    const int l2 = row % n2, l3 = row / n2;
    const int i2 = mode_of(l2, N2, n2);
    const int i3 = g.dim == 3 ? mode_of(l3, g.N[2], g.n[2]) : 0;
    C *dst = spec + (int64_t)row * n1;
    C zero;
    zero.x = 0;
    zero.y = 0;
    if (i2 < 0 || i3 < 0) {
        for (int l1 = threadIdx.x; l1 < n1; l1 += blockDim.x) dst[l1] = zero;
        return;
    }
    T frow = corr[N1 + i2];
    if (g.dim == 3) frow *= corr[N1 + N2 + i3];
    const C *src = modes + ((int64_t)i3 * N2 + i2) * N1;
    for (int l1 = threadIdx.x; l1 < n1; l1 += blockDim.x) {
        const int i1 = mode_of(l1, N1, n1);
        C v = zero;
        if (i1 >= 0) {
            v = src[i1];
            const T f = frow * corr[i1];
            v.x *= f;
            v.y *= f;
        }
        dst[l1] = v;
    }
}

// K9 + row FFTs fused (type 2, 2D/3D, single precision, n_1 = 2^L <= 4096).
// One CTA per fine row l_2: rows outside the mode band are written as
// zeros; band rows load their N_1 corrected modes into shared memory and run
// an in-place Stockham radix-8 (radix-4 / -2 last stage) inverse FFT (e^{+},
// unnormalised like cuFFT; twiddle table from FP64 on the host), then write
// the row once.  The separate pad kernel's full-grid write and the FFT's
// first full-grid pass disappear; a cuFFT column-only plan finishes the 2D
// transform.
__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// y = DFT_R(v) with kernel e^{+2 pi i k r / R} (inverse direction)
__device__ __forceinline__ void dft2(float2 &a, float2 &b) {
    const float2 t = a;
    a = make_float2(t.x + b.x, t.y + b.y);
    b = make_float2(t.x - b.x, t.y - b.y);
}
__device__ __forceinline__ void dft4(float2 &v0, float2 &v1, float2 &v2, float2 &v3) {
    const float2 a = make_float2(v0.x + v2.x, v0.y + v2.y), b = make_float2(v0.x - v2.x, v0.y - v2.y);
    const float2 c = make_float2(v1.x + v3.x, v1.y + v3.y), d = make_float2(v1.x - v3.x, v1.y - v3.y);
    // i * d = (-d.y, d.x)
    v0 = make_float2(a.x + c.x, a.y + c.y);
    v2 = make_float2(a.x - c.x, a.y - c.y);
    v1 = make_float2(b.x - d.y, b.y + d.x);
    v3 = make_float2(b.x + d.y, b.y - d.x);
}
__device__ __forceinline__ void dft8(float2 *v) {
    dft4(v[0], v[2], v[4], v[6]);
    dft4(v[1], v[3], v[5], v[7]);
    const float c = 0.70710678118654752f;
    // odd terms times w8^k, w8 = e^{i pi / 4}
    const float2 o1 = make_float2(c * (v[3].x - v[3].y), c * (v[3].x + v[3].y));
    const float2 o2 = make_float2(-v[5].y, v[5].x);
    const float2 o3 = make_float2(-c * (v[7].x + v[7].y), c * (v[7].x - v[7].y));
    const float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], o0 = v[1];
    v[0] = make_float2(e0.x + o0.x, e0.y + o0.y);
    v[4] = make_float2(e0.x - o0.x, e0.y - o0.y);
    v[1] = make_float2(e1.x + o1.x, e1.y + o1.y);
    v[5] = make_float2(e1.x - o1.x, e1.y - o1.y);
    v[2] = make_float2(e2.x + o2.x, e2.y + o2.y);
    v[6] = make_float2(e2.x - o2.x, e2.y - o2.y);
    v[3] = make_float2(e3.x + o3.x, e3.y + o3.y);
    v[7] = make_float2(e3.x - o3.x, e3.y - o3.y);
}

// One Stockham stage of a length-N (power of two) inverse FFT in shared
// memory (pad cell every 16 entries), radix R = 8 / 4 / 2 chosen at compile
// time; recursion unrolls the whole transform for a fixed N.
__device__ __forceinline__ int rpad(int i) { return i + (i >> 4); }

template <int N, int NS>
__device__ __forceinline__ void rowfft_stages(float2 *xs, const float2 *__restrict__ tw) {
    if constexpr (NS < N) {
        constexpr int LEFT = N / NS;
        constexpr int R = LEFT >= 8 ? 8 : (LEFT >= 4 ? 4 : 2);
        constexpr int NB = N / R;
        constexpr int NBT = (NB + 255) / 256;
        constexpr int TSTEP = N / (NS * R);
        float2 v[NBT][R];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NBT; ++q) {
            const int j = threadIdx.x + q * 256;
            if (NB % 256 == 0 || j < NB) {
                const int k = j & (NS - 1);
                // one table twiddle per butterfly, powers by recurrence
                const float2 w1 = NS > 1 ? __ldg(tw + k * TSTEP) : make_float2(1.f, 0.f);
                float2 w = w1;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float2 x = xs[rpad(j + r * NB)];
                    if (r && NS > 1) {
                        x = cmulf(x, w);
                        w = cmulf(w, w1);
                    }
                    v[q][r] = x;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NBT; ++q) {
            const int j = threadIdx.x + q * 256;
            if (NB % 256 == 0 || j < NB) {
                if constexpr (R == 8) dft8(v[q]);
                else if constexpr (R == 4) dft4(v[q][0], v[q][1], v[q][2], v[q][3]);
                else dft2(v[q][0], v[q][1]);
                const int k = j & (NS - 1);
                const int base = (j - k) * R + k;
#pragma unroll
                for (int r = 0; r < R; ++r) xs[rpad(base + r * NS)] = v[q][r];
            }
        }
        rowfft_stages<N, NS * R>(xs, tw);
    }
}

template <int N>
__global__ void __launch_bounds__(256)
k_pad_rowfft(Geom g, const float *__restrict__ corr, const float2 *__restrict__ modes,
             const float2 *__restrict__ tw, float2 *__restrict__ spec) {
    extern __shared__ __align__(16) float2 xs[];
    const int n2 = g.n[1];
    const int N1 = g.N[0], N2 = g.N[1];
    const int row = blockIdx.x;            // l2 + n2 * l3
    const int l2 = row % n2, l3 = row / n2;
    const int i2 = mode_of(l2, N2, n2);
    const int i3 = g.dim == 3 ? mode_of(l3, g.N[2], g.n[2]) : 0;
    float2 *dst = spec + (int64_t)row * N;
    if (i2 < 0 || i3 < 0) {
        float4 *d4 = reinterpret_cast<float4 *>(dst);
#pragma unroll
        for (int l = threadIdx.x; l < N / 2; l += 256) d4[l] = make_float4(0, 0, 0, 0);
        return;
    }
    float frow = corr[N1 + i2];
    if (g.dim == 3) frow *= corr[N1 + N2 + i3];
    const float2 *src = modes + ((int64_t)i3 * N2 + i2) * N1;
    const int kneg = N1 / 2, kpos = N1 - kneg;
#pragma unroll
    for (int l1 = threadIdx.x; l1 < N; l1 += 256) {
        const int i1 = l1 < kpos ? l1 + kneg : (l1 >= N - kneg ? l1 - N + kneg : -1);
        float2 v = make_float2(0.f, 0.f);
        if (i1 >= 0) {
            v = src[i1];
            const float f = frow * corr[i1];
            v.x *= f;
            v.y *= f;
        }
        xs[rpad(l1)] = v;
    }
    rowfft_stages<N, 1>(xs, tw);
    __syncthreads();
#pragma unroll
    for (int l = threadIdx.x; l < N; l += 256) dst[l] = xs[rpad(l)];
}

// K8 fused with the row FFTs (type 1, 2D/3D, single precision, n_1 = 2^L):
// after cuFFT's column pass, CTA i_2 loads fine row (i_2 - N_2/2) mod n_2,
// runs the forward row FFT in shared memory (forward = conj(inverse(conj))),
// and writes only the N_1 band modes with the correction factor and phase.
// The FFT's second full-grid pass and the deconvolution's read disappear.
template <int N>
__global__ void __launch_bounds__(256)
k_rowfft_deconv(Geom g, const float *__restrict__ corr, const float2 *__restrict__ spec,
                const float2 *__restrict__ tw, float2 *__restrict__ modes) {
    extern __shared__ __align__(16) float2 xs[];
    const int N1 = g.N[0], N2 = g.N[1];
    const int row = blockIdx.x;            // i2 + N2 * i3
    const int i2 = row % N2, i3 = row / N2;
    const int l2 = nk_wrap(i2 - N2 / 2, g.n[1]);
    const int l3 = g.dim == 3 ? nk_wrap(i3 - g.N[2] / 2, g.n[2]) : 0;
    const float2 *src = spec + ((int64_t)l3 * g.n[1] + l2) * N;
#pragma unroll
    for (int l = threadIdx.x; l < N; l += 256) {
        const float2 v = src[l];
        xs[rpad(l)] = make_float2(v.x, -v.y);
    }
    rowfft_stages<N, 1>(xs, tw);
    __syncthreads();
    float frow = corr[N1 + i2];
    if (g.dim == 3) frow *= corr[N1 + N2 + i3];
    float2 *dst = modes + (int64_t)row * N1;
    for (int i1 = threadIdx.x; i1 < N1; i1 += 256) {
        const float2 v = xs[rpad(nk_wrap(i1 - N1 / 2, N))];
        const float f = frow * corr[i1];
        dst[i1] = make_float2(v.x * f, -v.y * f);
    }
}

}  // namespace

int nk_launch_deconv1(nk_plan *p, const void *spec, void *modes) {
    if (p->N_tot == 0) return NK_OK;
    const dim3 grid((unsigned)(p->N[1] * p->N[2]), p->ntrans);
    if (p->prec == NK_DOUBLE)
        k_deconv1<double><<<grid, 256, 0, p->stream>>>(p->geom, (const double *)p->d_corr,
                                                       (const double2 *)spec, (double2 *)modes);
    else
        k_deconv1<float><<<grid, 256, 0, p->stream>>>(p->geom, (const float *)p->d_corr,
                                                      (const float2 *)spec, (float2 *)modes);
    NK_LAUNCH_CHECK();
    return NK_OK;
}

int nk_launch_deconv2(nk_plan *p, const void *modes, void *spec) {
    const dim3 grid((unsigned)(p->n[1] * p->n[2]), p->ntrans);
    if (p->prec == NK_DOUBLE)
        k_deconv2<double><<<grid, 256, 0, p->stream>>>(p->geom, (const double *)p->d_corr,
                                                       (const double2 *)modes, (double2 *)spec);
    else
        k_deconv2<float><<<grid, 256, 0, p->stream>>>(p->geom, (const float *)p->d_corr,
                                                      (const float2 *)modes, (float2 *)spec);
    NK_LAUNCH_CHECK();
    return NK_OK;
}

int nk_launch_pad_rowfft(nk_plan *p, const void *modes, void *spec) {
    const size_t smem = sizeof(float2) * (size_t)(p->n[0] + p->n[0] / 16);
    const unsigned rows = (unsigned)(p->n[1] * p->n[2]);
    const float *corr = (const float *)p->d_corr;
    const float2 *tw = (const float2 *)p->d_twiddle;
    switch (p->n[0]) {
#define NK_RF(N)                                                                          \
    case N:                                                                               \
        k_pad_rowfft<N><<<rows, 256, smem, p->stream>>>(p->geom, corr, (const float2 *)modes, \
                                                         tw, (float2 *)spec);             \
        break;
        NK_RF(256) NK_RF(512) NK_RF(1024) NK_RF(2048) NK_RF(4096)
#undef NK_RF
    default:
        nk_set_error("fused row FFT: unsupported n_1");
        return NK_ERR_VALUE;
    }
    NK_LAUNCH_CHECK();
    return NK_OK;
}

int nk_launch_rowfft_deconv(nk_plan *p, const void *spec, void *modes) {
    const size_t smem = sizeof(float2) * (size_t)(p->n[0] + p->n[0] / 16);
    const unsigned rows = (unsigned)(p->N[1] * p->N[2]);
    const float *corr = (const float *)p->d_corr;
    const float2 *tw = (const float2 *)p->d_twiddle;
    switch (p->n[0]) {
#define NK_RF(N)                                                                          \
    case N:                                                                               \
        k_rowfft_deconv<N><<<rows, 256, smem, p->stream>>>(p->geom, corr,                 \
                                                            (const float2 *)spec, tw,     \
                                                            (float2 *)modes);             \
        break;
        NK_RF(256) NK_RF(512) NK_RF(1024) NK_RF(2048) NK_RF(4096)
#undef NK_RF
    default:
        nk_set_error("fused row FFT: unsupported n_1");
        return NK_ERR_VALUE;
    }
    NK_LAUNCH_CHECK();
    return NK_OK;
}
