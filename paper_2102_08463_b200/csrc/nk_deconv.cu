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
