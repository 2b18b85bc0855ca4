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

// type 1: modes (N_d..N_1) <- p_k (-1)^{sum k} bhat[k mod n]
template <typename T>
__global__ void __launch_bounds__(256)
k_deconv1(int64_t Ntot, Geom g, const T *__restrict__ corr,
          const typename cplx<T>::t *__restrict__ spec, typename cplx<T>::t *__restrict__ modes) {
    typedef typename cplx<T>::t C;
    int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= Ntot) return;
    const int N1 = g.N[0], N2 = g.N[1];
    const int i1 = (int)(o % N1);
    const int64_t r = o / N1;
    const int i2 = (int)(r % N2);
    const int i3 = (int)(r / N2);
    int l1 = nk_wrap(i1 - N1 / 2, g.n[0]);
    int l2 = nk_wrap(i2 - N2 / 2, g.n[1]);
    T f = corr[i1] * corr[N1 + i2];
    int64_t l = l1 + (int64_t)g.n[0] * l2;
    if (g.dim == 3) {
        int l3 = nk_wrap(i3 - g.N[2] / 2, g.n[2]);
        f *= corr[N1 + N2 + i3];
        l += (int64_t)g.n[0] * g.n[1] * l3;
    }
    C v = spec[l];
    v.x *= f;
    v.y *= f;
    modes[o] = v;
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
// band, zero elsewhere (fused zero-fill + scatter).
template <typename T>
__global__ void __launch_bounds__(256)
k_deconv2(int64_t ntot, Geom g, const T *__restrict__ corr,
          const typename cplx<T>::t *__restrict__ modes, typename cplx<T>::t *__restrict__ spec) {
    typedef typename cplx<T>::t C;
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ntot) return;
    const int n1 = g.n[0], n2 = g.n[1];
    const int l1 = (int)(q % n1);
    const int64_t r = q / n1;
    const int l2 = (int)(r % n2);
    const int l3 = (int)(r / n2);
    C v;
    v.x = 0;
    v.y = 0;
    const int N1 = g.N[0], N2 = g.N[1];
    int i1 = mode_of(l1, N1, n1), i2 = mode_of(l2, N2, n2);
    int i3 = g.dim == 3 ? mode_of(l3, g.N[2], g.n[2]) : 0;
    if (i1 >= 0 && i2 >= 0 && i3 >= 0) {
        T f = corr[i1] * corr[N1 + i2];
        int64_t o = i1 + (int64_t)N1 * i2;
        if (g.dim == 3) {
            f *= corr[N1 + N2 + i3];
            o += (int64_t)N1 * N2 * i3;
        }
        v = modes[o];
        v.x *= f;
        v.y *= f;
    }
    spec[q] = v;
}

}  // namespace

int nk_launch_deconv1(nk_plan *p, const void *spec, void *modes) {
    if (p->N_tot == 0) return NK_OK;
    unsigned nb = (unsigned)((p->N_tot + 255) / 256);
    if (p->prec == NK_DOUBLE)
        k_deconv1<double><<<nb, 256, 0, p->stream>>>(p->N_tot, p->geom, (const double *)p->d_corr,
                                                     (const double2 *)spec, (double2 *)modes);
    else
        k_deconv1<float><<<nb, 256, 0, p->stream>>>(p->N_tot, p->geom, (const float *)p->d_corr,
                                                    (const float2 *)spec, (float2 *)modes);
    NK_LAUNCH_CHECK();
    return NK_OK;
}

int nk_launch_deconv2(nk_plan *p, const void *modes, void *spec) {
    unsigned nb = (unsigned)((p->n_tot + 255) / 256);
    if (p->prec == NK_DOUBLE)
        k_deconv2<double><<<nb, 256, 0, p->stream>>>(p->n_tot, p->geom, (const double *)p->d_corr,
                                                     (const double2 *)modes, (double2 *)spec);
    else
        k_deconv2<float><<<nb, 256, 0, p->stream>>>(p->n_tot, p->geom, (const float *)p->d_corr,
                                                    (const float2 *)modes, (float2 *)spec);
    NK_LAUNCH_CHECK();
    return NK_OK;
}
