// Plan-time host math: tolerance -> (w, beta), 5-smooth sizing, and the ES
// kernel Fourier transform used for the correction factors.
//
// Reference: kernel.py:83-103 (tolerance_to_width), kernel.py:138-173
// (Gauss-Legendre kernel_fourier), SPEC.md:122-140 (next_smooth, sizing).
#include <math.h>
#include <stdint.h>

#include <mutex>
#include <vector>

#include "nk_internal.cuh"

namespace {

constexpr int kQuadNodes = 100;      // kernel.py:36
constexpr int kMinWidth = 2;         // kernel.py:27
constexpr int kMaxWidth = 16;        // kernel.py:28
constexpr double kSingleFloor = 1e-6;  // kernel.py:31

struct GaussLegendre {
    double theta[kQuadNodes];
    double wq[kQuadNodes];
    GaussLegendre() {
        // Roots of P_n by Newton iteration (numpy.polynomial.legendre.leggauss
        // gives the same rule to ~1e-16), mapped to [-pi/2, pi/2]
        // (kernel.py:138-143).
        const int n = kQuadNodes;
        for (int i = 0; i < n; ++i) {
            double x = cos(NK_PI * (i + 0.75) / (n + 0.5));
            double dp = 0.0;
            for (int it = 0; it < 100; ++it) {
                double p0 = 1.0, p1 = x;
                for (int k = 2; k <= n; ++k) {
                    double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
                    p0 = p1;
                    p1 = p2;
                }
                dp = n * (x * p1 - p0) / (x * x - 1.0);
                double dx = p1 / dp;
                x -= dx;
                if (fabs(dx) < 1e-17) break;
            }
            double p0 = 1.0, p1 = x;
            for (int k = 2; k <= n; ++k) {
                double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (x * p1 - p0) / (x * x - 1.0);
            // ascending order like leggauss
            theta[n - 1 - i] = x * (NK_PI / 2);
            wq[n - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp) * (NK_PI / 2);
        }
    }
};

const GaussLegendre &rule() {
    static GaussLegendre gl;
    return gl;
}

}  // namespace

void nk_kernel_fourier_host(double beta, const double *xi, int64_t n, double *out) {
    const GaussLegendre &g = rule();
    double env[kQuadNodes], s[kQuadNodes];
    for (int q = 0; q < kQuadNodes; ++q) {
        double c = cos(g.theta[q]);
        env[q] = g.wq[q] * c * exp(beta * (c - 1.0));   // kernel.py:163
        s[q] = sin(g.theta[q]);
    }
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int q = 0; q < kQuadNodes; ++q) acc += cos(xi[i] * s[q]) * env[q];  // kernel.py:164
        out[i] = acc;
    }
}

extern "C" int nk_tolerance_to_width(double eps, int precision, double *eps_eff, int *w,
                                     double *beta, int *clamped) {
    if (precision != NK_SINGLE && precision != NK_DOUBLE) {
        nk_set_error("precision must be 'single' or 'double'");
        return NK_ERR_VALUE;
    }
    if (!isfinite(eps) || !(eps > 0.0 && eps < 1.0)) {
        nk_set_error("tolerance must lie in (0, 1), got " + std::to_string(eps));
        return NK_ERR_VALUE;
    }
    int cl = 0;
    if (precision == NK_SINGLE && eps < kSingleFloor) {   // kernel.py:94-100
        eps = kSingleFloor;
        cl = 1;
    }
    int ww = (int)ceil(log10(1.0 / eps)) + 1;             // kernel.py:101
    if (ww < kMinWidth) ww = kMinWidth;
    if (ww > kMaxWidth) ww = kMaxWidth;
    if (eps_eff) *eps_eff = eps;
    if (w) *w = ww;
    if (beta) *beta = 2.30 * ww;                          // kernel.py:103
    if (clamped) *clamped = cl;
    return NK_OK;
}

extern "C" int64_t nk_next_smooth(int64_t n) {
    if (n < 1) return -1;
    for (int64_t m = n; m > 0; ++m) {
        int64_t r = m;
        while (r % 2 == 0) r /= 2;
        while (r % 3 == 0) r /= 3;
        while (r % 5 == 0) r /= 5;
        if (r == 1) return m;
    }
    return -1;
}

extern "C" int nk_kernel_fourier(double beta, const double *xi, int64_t n, double *out) {
    if (n < 0 || (n > 0 && (!xi || !out))) {
        nk_set_error("invalid kernel_fourier arguments");
        return NK_ERR_VALUE;
    }
    nk_kernel_fourier_host(beta, xi, n, out);
    double mx = 0.0;
    bool finite = true;
    for (int64_t i = 0; i < n; ++i) {
        if (!isfinite(out[i])) finite = false;
        mx = fmax(mx, fabs(out[i]));
    }
    // kernel.py:165-170 (np.finfo(float64).tiny * 8)
    if (n > 0 && (!finite || mx < 2.2250738585072014e-308 * 8)) {
        nk_set_error("kernel Fourier transform underflowed below the precision floor");
        return NK_ERR_VALUE;
    }
    return NK_OK;
}

// kernel.py:181-205 build_correction_factors: the full (N_d, ..., N_1) table
// p_k = (2/w)^d / prod_i phi_hat(alpha_i k_i), k_i centered (kernel.py:176-178),
// with the reference's product order (axis d outermost, multiplied down to
// axis 1, kernel.py:201-203) and the cast to the plan's real dtype
// (kernel.py:205).  Host output; the CUDA path uses per-axis factors instead.
extern "C" int nk_correction_factors(double beta, int w, int dim, const int64_t *modes,
                                     const double *alpha, int precision, void *out) {
    if (dim < 1 || dim > 3 || !modes || !alpha || !out || w < 1 ||
        (precision != NK_SINGLE && precision != NK_DOUBLE)) {
        nk_set_error("invalid correction-factor arguments");
        return NK_ERR_VALUE;
    }
    // np.finfo(real dtype).tiny * 100 (kernel.py:190)
    const double floor_v = (precision == NK_DOUBLE ? 2.2250738585072014e-308
                                                   : 1.1754943508222875e-38) * 100;
    std::vector<std::vector<double>> ft(dim);
    int64_t total = 1;
    for (int i = 0; i < dim; ++i) {
        const int64_t Ni = modes[i];
        if (Ni < 0) {
            nk_set_error("invalid mode count");
            return NK_ERR_VALUE;
        }
        std::vector<double> xi(Ni);
        for (int64_t k = 0; k < Ni; ++k) xi[k] = alpha[i] * (double)(k - Ni / 2);
        ft[i].resize(Ni);
        nk_kernel_fourier_host(beta, xi.data(), Ni, ft[i].data());
        for (int64_t k = 0; k < Ni; ++k)
            if (!(ft[i][k] > floor_v)) {   // kernel.py:195-199
                nk_set_error("kernel Fourier transform underflowed on axis " +
                             std::to_string(i + 1) + "; correction factors would overflow");
                return NK_ERR_VALUE;
            }
        total *= Ni;
    }
    const double c = pow(2.0 / w, (double)dim);
    const int64_t N1 = modes[0], N2 = dim > 1 ? modes[1] : 1, N3 = dim > 2 ? modes[2] : 1;
    int64_t o = 0;
    for (int64_t k3 = 0; k3 < N3; ++k3)
        for (int64_t k2 = 0; k2 < N2; ++k2)
            for (int64_t k1 = 0; k1 < N1; ++k1, ++o) {
                double prod;
                if (dim == 1) prod = ft[0][k1];
                else if (dim == 2) prod = ft[1][k2] * ft[0][k1];
                else prod = (ft[2][k3] * ft[1][k2]) * ft[0][k1];
                const double v = c / prod;
                if (precision == NK_DOUBLE) ((double *)out)[o] = v;
                else ((float *)out)[o] = (float)v;
            }
    (void)total;
    return NK_OK;
}
