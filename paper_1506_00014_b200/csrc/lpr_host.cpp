// Plan-time host code of the product library: sampling geometry and the
// kernel spectra zeta / zeta#. These are per-plan constants (computed once,
// uploaded once); nothing here runs per slice.
//
//   geometry  follows lpr::sampling_plan   (geometry.cpp:51-98)
//   spectra   follow the quadrature path    (kernel.cpp:293-429): for each
//             rho frequency, one power-of-two FFT of end-corrected trapezoid
//             samples of cos(t)^alpha on [-beta, beta] yields the integral
//             P(mu, alpha, beta) at every theta frequency mu = -pi k / beta.
#include <algorithm>
#include <cmath>
#include <complex>
#include <stdexcept>
#include <thread>
#include <vector>

#include "lpradon_gpu.h"
#include "lpr_host.hpp"

namespace lpr::host {

namespace {
constexpr double kPi = 3.14159265358979323846;
using cd = std::complex<double>;

// In-place iterative radix-2 transform, sign -1 (forward), unnormalised.
void fft_pow2(std::vector<cd>& x) {
    const size_t n = x.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(x[i], x[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len / 2;
        std::vector<cd> w(half);
        for (size_t k = 0; k < half; ++k) w[k] = std::polar(1.0, -2.0 * kPi * double(k) / double(len));
        for (size_t s = 0; s < n; s += len)
            for (size_t k = 0; k < half; ++k) {
                const cd u = x[s + k], v = x[s + k + half] * w[k];
                x[s + k] = u + v;
                x[s + k + half] = u - v;
            }
    }
}

bool smooth7(long n) {
    for (long f : {2L, 3L, 5L, 7L})
        while (n % f == 0) n /= f;
    return n == 1;
}
}  // namespace

int minimal_n_rho(int N, int M) {
    const double beta = kPi / M;
    const double sh = std::sin(beta / 2), ch = std::cos(beta / 2);
    const double aR = sh / (1 + sh), ar = (ch - sh) / (1 + sh);
    return int(std::ceil(std::log(ar) / std::log1p(-2.0 * aR / N)));
}

int smooth_n_rho(int N, int M) {
    long n = minimal_n_rho(N, M);
    while (!smooth7(n)) ++n;
    return int(n);
}

lpr_geometry make_geometry(int N, int M, int n_theta, int n_rho) {
    if (N < 16 || N % 2) throw std::invalid_argument("sampling_plan: N must be even and >= 16");
    if (M < 3) throw std::invalid_argument("sampling_plan: M must be >= 3");
    lpr_geometry g{};
    g.N = N;
    g.M = M;
    g.beta = kPi / M;
    const double sh = std::sin(g.beta / 2), ch = std::cos(g.beta / 2);
    g.a_R = sh / (1 + sh);
    g.a_r = (ch - sh) / (1 + sh);
    g.log_ar = std::log(g.a_r);
    if (n_theta <= 0) n_theta = int(std::ceil(1.5 * N));
    if (n_theta < 2 * M) throw std::invalid_argument("sampling_plan: n_theta must be positive");
    g.n_theta = (n_theta + 2 * M - 1) / (2 * M) * (2 * M);
    g.nts = g.n_theta / M;
    g.ds = 1.0 / N;
    g.dtheta_p = kPi / g.n_theta;
    const int nmin = minimal_n_rho(N, M);
    if (n_rho <= 0) n_rho = nmin;
    if (n_rho < nmin) throw std::invalid_argument("sampling_plan: n_rho below the sampling bound (Eq. vrho)");
    g.n_rho = n_rho;
    g.drho = -g.log_ar / n_rho;
    g.refine = int(std::ceil(g.dtheta_p * N / (2.0 * g.a_R) - 1e-12));
    g.dtheta_lp = g.dtheta_p / g.refine;
    return g;
}

void spectrum(const lpr_geometry& g, int kind, double* out) {
    // end-point correction deltas for the first/last seven nodes
    static const double dc[7] = {-23681, 55688, -66109, 57024, -31523, 9976, -1375};
    const long nts = g.nts, rows = 2 * nts, cols = g.n_rho;
    const double beta = g.beta, ell = -g.log_ar;
    auto put = [&](long kt, long v, cd val) {
        const long r = ((kt % rows) + rows) % rows;
        out[2 * (r * cols + v)] = val.real();
        out[2 * (r * cols + v) + 1] = val.imag();
    };
    auto column = [&](long v) {
        const long kr = v < (cols + 1) / 2 ? v : v - cols;  // signed rho frequency
        const double y = 2.0 * kPi * double(kr) / ell;
        if (kind == 1 && kr == 0) {  // alpha = 0: elementary 2 sin(mu beta) / mu
            for (long kt = -nts; kt < nts; ++kt) {
                const double mu = -kPi * double(kt) / beta;
                put(kt, v, kt == 0 ? cd(2 * beta) : cd(2 * std::sin(mu * beta) / mu));
            }
            return;
        }
        const cd alpha = kind == 0 ? cd(-1.0, -y) : cd(0.0, y);
        const double rate = (kPi * double(nts) / beta + std::fabs(y) * std::tan(beta)) * beta / kPi;
        long n = 1;
        while (n < 16 * std::max<long>(32, long(std::ceil(rate)))) n <<= 1;
        const double h = 2.0 * beta / double(n);
        std::vector<cd> s(n);
        for (long j = 0; j < n; ++j) {
            double w = 1.0;
            if (j == 0) w += 2.0 * dc[0] / 120960.0;  // both ends meet at node 0 on the circle
            else if (j < 7) w += dc[j] / 120960.0;
            if (n - j < 7) w += dc[n - j] / 120960.0;
            s[j] = w * std::exp(alpha * std::log(std::cos(-beta + double(j) * h)));
        }
        fft_pow2(s);
        for (long kt = -nts; kt < nts; ++kt) {
            cd val = h * s[((kt % n) + n) % n];
            put(kt, v, (kt & 1) ? -val : val);
        }
    };
    const unsigned nthreads = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nthreads; ++t)
        pool.emplace_back([&, t] {
            for (long v = t; v < cols; v += nthreads) column(v);
        });
    for (auto& th : pool) th.join();
    if (cols % 2 == 0)  // a Hermitian multiplier is real on the rho Nyquist column
        for (long r = 0; r < rows; ++r) out[2 * (r * cols + cols / 2) + 1] = 0.0;
}

}  // namespace lpr::host
