// ORACLE bridge — test infrastructure only. Flat C entry points onto the
// reference's own compiled building blocks (geometry.cpp, bspline.cpp,
// kernel.cpp, oracle.cpp under /root/reference/proj/src), so the Python tests
// can pin the oracle restatement (oracle/lpo.cpp) against them and generate
// golden fixtures. Built only into oracle/_ref/liblpr_ref.so.
#include <cstring>
#include <exception>
#include <string>

#include "lpradon/bspline.hpp"
#include "lpradon/geometry.hpp"
#include "lpradon/kernel.hpp"
#include "lpradon/oracle.hpp"

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
lpr::Array2D<double> wrap2d(const double* p, long rows, long cols) {
    lpr::Array2D<double> a(rows, cols);
    std::memcpy(a.data(), p, sizeof(double) * rows * cols);
    return a;
}
}  // namespace

extern "C" {

const char* lpr_ref_last_error() { return g_err.c_str(); }

// ints: N, M, N_theta, N_theta_sector, N_rho, theta_refine, N_s
// dbls: beta, a_R, a_r, log_ar, dtheta_p, dtheta_lp, drho, ds
int lpr_ref_plan(int N, int M, int nt, int* ints, double* dbls) {
    return guard([&] {
        const auto p = nt > 0 ? lpr::sampling_plan(N, M, nt) : lpr::sampling_plan(N, M);
        const int iv[7] = {p.N, p.M, p.N_theta, p.N_theta_sector, p.N_rho, p.theta_refine, p.N_s};
        const double dv[8] = {p.constants.beta, p.constants.a_R, p.constants.a_r, p.log_ar(),
                              p.dtheta_p,       p.dtheta_lp,     p.drho,          p.ds};
        std::memcpy(ints, iv, sizeof iv);
        std::memcpy(dbls, dv, sizeof dv);
    });
}

int lpr_ref_spectrum(int N, int M, int nt, int kind, int closed_form, double* out, long* fallback_bins) {
    return guard([&] {
        const auto p = nt > 0 ? lpr::sampling_plan(N, M, nt) : lpr::sampling_plan(N, M);
        const auto method = closed_form ? lpr::KernelMethod::closed_form : lpr::KernelMethod::quadrature;
        const auto s = kind == 0 ? lpr::zeta_spectrum(p, method) : lpr::zeta_bp_spectrum(p, method);
        std::memcpy(out, s.coeffs.data(), sizeof(double) * 2 * s.coeffs.size());
        if (fallback_bins) *fallback_bins = long(s.fallback_bins);
    });
}

int lpr_ref_p_quadrature(double mu, double are, double aim, double beta, int os, double* out) {
    return guard([&] {
        const auto v = lpr::p_quadrature(mu, {are, aim}, beta, os);
        out[0] = v.real();
        out[1] = v.imag();
    });
}

int lpr_ref_p_closed_form(double mu, double are, double aim, double beta, double* out) {
    return guard([&] {
        const auto v = lpr::p_closed_form(mu, {are, aim}, beta);
        out[0] = v.real();
        out[1] = v.imag();
    });
}

int lpr_ref_prefilter_1d(double* x, long n) {
    return guard([&] { lpr::prefilter_1d(x, std::size_t(n)); });
}

int lpr_ref_prefilter_2d(double* img, long rows, long cols) {
    return guard([&] {
        lpr::GridSpec g{lpr::GridKind::cartesian, {std::size_t(rows), 0.0, 1.0}, {std::size_t(cols), 0.0, 1.0}};
        const auto c = lpr::prefilter_2d(wrap2d(img, rows, cols), g);
        std::memcpy(img, c.values.data(), sizeof(double) * rows * cols);
    });
}

int lpr_ref_interp_cubic_2d(const double* coef, long rows, long cols, const double* tr, const double* tc,
                            double* out, long npts) {
    return guard([&] {
        lpr::SplineCoeffs c;
        c.values = wrap2d(coef, rows, cols);
        for (long i = 0; i < npts; ++i) out[i] = lpr::interp_cubic_2d(c, tr[i], tc[i]);
    });
}

int lpr_ref_eval_periodic_2d(const double* coef, long rows, long cols, const double* tr, const double* tc,
                             double* out, long npts) {
    return guard([&] {
        const auto c = wrap2d(coef, rows, cols);
        for (long i = 0; i < npts; ++i) out[i] = lpr::detail::eval_periodic_2d(c, tr[i], tc[i]);
    });
}

int lpr_ref_eval_zero_1d(const double* coef, long n, const double* t, double* out, long npts) {
    return guard([&] {
        for (long i = 0; i < npts; ++i) out[i] = lpr::detail::eval_zero_1d(coef, std::size_t(n), t[i]);
    });
}

int lpr_ref_line_to_sector(int M, double theta, double s, int* m, double* theta_res, double* s_out) {
    return guard([&] {
        const auto l = lpr::line_to_sector(theta, s, lpr::sector_constants(M), M);
        *m = l.m;
        *theta_res = l.theta_res;
        *s_out = l.s;
    });
}

int lpr_ref_map_T_inv(int M, int m, double px, double py, double* out) {
    return guard([&] {
        const auto v = lpr::map_T_inv(m, {px, py}, lpr::sector_constants(M));
        out[0] = v.x;
        out[1] = v.y;
    });
}

int lpr_ref_map_S(int M, int m, double theta, double s, double* out) {
    return guard([&] {
        const auto v = lpr::map_S(m, theta, s, lpr::sector_constants(M));
        out[0] = v.first;
        out[1] = v.second;
    });
}

int lpr_ref_direct_radon(int N, int M, int nt, const double* img, double* sino) {
    return guard([&] {
        const auto p = nt > 0 ? lpr::sampling_plan(N, M, nt) : lpr::sampling_plan(N, M);
        lpr::Image im{wrap2d(img, N, N), p.cartesian_grid()};
        const auto s = lpr::direct_radon(im, p.polar_grid());
        std::memcpy(sino, s.values.data(), sizeof(double) * s.values.size());
    });
}

int lpr_ref_direct_backprojection(int N, int M, int nt, const double* sino, double* img) {
    return guard([&] {
        const auto p = nt > 0 ? lpr::sampling_plan(N, M, nt) : lpr::sampling_plan(N, M);
        lpr::Sinogram sg{wrap2d(sino, p.N_theta, N), p.polar_grid()};
        const auto im = lpr::direct_backprojection(sg);
        std::memcpy(img, im.pixels.data(), sizeof(double) * N * N);
    });
}

int lpr_ref_phantom_image(int N, double* img) {
    return guard([&] {
        const auto im = lpr::phantom_image(N);
        std::memcpy(img, im.pixels.data(), sizeof(double) * N * N);
    });
}

int lpr_ref_phantom_sinogram(int N, int M, int nt, double* sino) {
    return guard([&] {
        const auto p = nt > 0 ? lpr::sampling_plan(N, M, nt) : lpr::sampling_plan(N, M);
        const auto s = lpr::phantom_sinogram(lpr::shepp_logan_ellipses(), p.polar_grid());
        std::memcpy(sino, s.values.data(), sizeof(double) * s.values.size());
    });
}

}  // extern "C"
