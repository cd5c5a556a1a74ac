// ORACLE — test infrastructure only (see lpo.hpp). Flat C entry points for
// the Python test harness (ctypes). Plans are passed as (N, M, n_theta,
// n_rho) and rebuilt per call; spectra travel as interleaved re/im doubles.
// Every function returns 0 on success and -1 after storing a message that
// lpo_last_error() returns.
#include <cstring>
#include <exception>
#include <string>

#include "lpo.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

inline const lpo::cd* as_cd(const double* p) { return reinterpret_cast<const lpo::cd*>(p); }
inline lpo::cd* as_cd(double* p) { return reinterpret_cast<lpo::cd*>(p); }
}  // namespace

extern "C" {

const char* lpo_last_error() { return g_err.c_str(); }

// ints: N, M, n_theta, nts, n_rho, refine; dbls: beta, aR, ar, log_ar,
// dtheta_p, dtheta_lp, drho, ds
int lpo_plan(int N, int M, int nt, int nr, int* ints, double* dbls) {
    return guard([&] {
        const lpo::Plan p = lpo::make_plan(N, M, nt, nr);
        const int iv[6] = {p.N, p.M, p.n_theta, p.nts, p.n_rho, p.refine};
        const double dv[8] = {p.beta, p.aR, p.ar, p.log_ar, p.dtheta_p, p.dtheta_lp, p.drho, p.ds};
        std::memcpy(ints, iv, sizeof iv);
        std::memcpy(dbls, dv, sizeof dv);
    });
}

int lpo_spectrum(int N, int M, int nt, int nr, int kind, double* out) {
    return guard([&] { lpo::spectrum(lpo::make_plan(N, M, nt, nr), kind, as_cd(out)); });
}

int lpo_fast_radon(int N, int M, int nt, int nr, const double* zeta, const double* img, double* sino, int batch) {
    return guard([&] {
        const lpo::Plan p = lpo::make_plan(N, M, nt, nr);
        for (int b = 0; b < batch; ++b)
            lpo::fast_radon(p, as_cd(zeta), img + long(b) * N * N, sino + long(b) * p.n_theta * N);
    });
}

int lpo_fast_backprojection(int N, int M, int nt, int nr, const double* zeta_bp, const double* sino, double* img,
                            int batch) {
    return guard([&] {
        const lpo::Plan p = lpo::make_plan(N, M, nt, nr);
        for (int b = 0; b < batch; ++b)
            lpo::fast_backprojection(p, as_cd(zeta_bp), sino + long(b) * p.n_theta * N, img + long(b) * N * N);
    });
}

int lpo_radon_transpose(int N, int M, int nt, int nr, const double* zeta, const double* sino, double* img,
                        int batch) {
    return guard([&] {
        const lpo::Plan p = lpo::make_plan(N, M, nt, nr);
        for (int b = 0; b < batch; ++b)
            lpo::radon_transpose(p, as_cd(zeta), sino + long(b) * p.n_theta * N, img + long(b) * N * N);
    });
}

int lpo_radon_sector_coeffs(int N, int M, int nt, int nr, const double* zeta, const double* qf, int m,
                            double* out) {
    return guard([&] { lpo::radon_sector_coeffs(lpo::make_plan(N, M, nt, nr), as_cd(zeta), qf, m, out); });
}

int lpo_lp_convolve(const double* spec, int divide_bspline, double* data, long rows, long cols) {
    return guard([&] { lpo::lp_convolve(as_cd(spec), divide_bspline != 0, data, rows, cols); });
}

int lpo_direct_radon(int N, int M, int nt, int nr, const double* img, double* sino) {
    return guard([&] { lpo::direct_radon(lpo::make_plan(N, M, nt, nr), img, sino); });
}

int lpo_direct_backprojection(int N, int M, int nt, int nr, const double* sino, double* img) {
    return guard([&] { lpo::direct_backprojection(lpo::make_plan(N, M, nt, nr), sino, img); });
}

int lpo_phantom_image(int N, double* img) {
    return guard([&] { lpo::phantom_image(N, img); });
}

int lpo_phantom_sinogram(int N, int M, int nt, int nr, double* sino) {
    return guard([&] { lpo::phantom_sinogram(lpo::make_plan(N, M, nt, nr), sino); });
}

int lpo_prefilter_1d(double* x, long n) {
    return guard([&] { lpo::prefilter_1d(x, n, 1); });
}

int lpo_prefilter_2d(double* img, long rows, long cols) {
    return guard([&] { lpo::prefilter_2d(img, rows, cols); });
}

int lpo_eval_mirror_2d(const double* c, long rows, long cols, const double* tr, const double* tc, double* out,
                       long npts) {
    return guard([&] {
        for (long i = 0; i < npts; ++i) out[i] = lpo::eval_mirror_2d(c, rows, cols, tr[i], tc[i]);
    });
}

int lpo_eval_periodic_2d(const double* c, long rows, long cols, const double* tr, const double* tc, double* out,
                         long npts) {
    return guard([&] {
        for (long i = 0; i < npts; ++i) out[i] = lpo::eval_periodic_2d(c, rows, cols, tr[i], tc[i]);
    });
}

int lpo_fft1d(double* x, long n, int sign) {
    return guard([&] { lpo::fft1d(as_cd(x), n, sign); });
}

int lpo_fft2d(double* x, long rows, long cols, int sign) {
    return guard([&] { lpo::fft2d(as_cd(x), rows, cols, sign); });
}

unsigned long long lpo_fft2d_count() { return lpo::fft2d_count(); }
void lpo_fft2d_count_reset() { lpo::fft2d_count_reset(); }

}  // extern "C"
