// ORACLE — test infrastructure only. Nothing in the product path may include,
// link or call this code; only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py use it, as the checker.
//
// lpo: an fp64 CPU restatement of arXiv 1506.00014 Algorithms 1-2 (fast
// log-polar Radon transform R and back-projection R#), plus the exact
// discrete transpose of R, composed from restated versions of the
// reference's building blocks:
//   geometry   /root/reference/proj/src/geometry.cpp:51-142
//   B-spline   /root/reference/proj/src/bspline.cpp:33-216
//   spectra    /root/reference/proj/src/kernel.cpp:293-429 (quadrature path)
//   FFT        /root/reference/proj/src/fft.cpp (FFTW replaced by our own)
//   direct     /root/reference/proj/src/oracle.cpp:95-265
// The operator composition follows PAPER.md:433-468 and SPEC.md:250-328;
// every convention the reference leaves open is fixed in DESIGN.md §3 and
// restated at the definition below.
#pragma once

#include <complex>
#include <cstdint>
#include <vector>

namespace lpo {

using cd = std::complex<double>;

// ---------------------------------------------------------------- geometry
// Mirrors GeometryPlan/sampling_plan (geometry.hpp:23-61, geometry.cpp:51-98).
struct Plan {
    int N = 0, M = 0;
    int n_theta = 0;   // polar angles over [0, pi)
    int nts = 0;       // angles per sector on the coarse grid (N_theta_sector)
    int n_rho = 0;     // log-radial count
    int refine = 0;    // fine/coarse theta ratio (theta_refine)
    double beta = 0, aR = 0, ar = 0, log_ar = 0;
    double dtheta_p = 0, dtheta_lp = 0, drho = 0, ds = 0;
};

// n_theta <= 0 -> ceil(3N/2); n_rho <= 0 -> the minimal count of Eq. (vrho).
// An explicit n_rho must be >= the minimal count.
Plan make_plan(int N, int M, int n_theta = 0, int n_rho = 0);
int min_n_rho(int N, int M);

// ---------------------------------------------------------------- FFT
// Unnormalised in-place c2c, sign -1 forward / +1 backward (fft.hpp:9-16).
void fft1d(cd* x, long n, int sign);
void fft2d(cd* x, long rows, long cols, int sign);
std::uint64_t fft2d_count();
void fft2d_count_reset();

// ---------------------------------------------------------------- B-spline
void bspline_weights(double a, double w[4]);     // taps k-1..k+2 for t = k + a
void prefilter_1d(double* x, long n, long stride);  // mirror boundary, in place
void prefilter_2d(double* img, long rows, long cols);  // rows then columns
double eval_mirror_2d(const double* c, long rows, long cols, double tr, double tc);
double eval_periodic_2d(const double* c, long rows, long cols, double tr, double tc);
double eval_periodic_1d(const double* c, long n, double t);
double eval_zero_1d(const double* c, long n, double t);

// ---------------------------------------------------------------- spectra
// kind 0 = zeta (radon), 1 = zeta# (back-projection). Output row-major
// (2*nts) x n_rho, theta rows in FFT order (kernel.hpp:19-26).
void spectrum(const Plan& p, int kind, cd* out);

// ---------------------------------------------------------------- operators
// All rasters row-major fp64. Image N x N (rows = x2), sinogram n_theta x N.
// zeta / zeta_bp are spectra from spectrum() (or the reference's).
void fast_radon(const Plan& p, const cd* zeta, const double* img, double* sino);
void fast_backprojection(const Plan& p, const cd* zeta_bp, const double* sino, double* img);
// Exact transpose of fast_radon under the weighted inner products
// <.,.>_Sigma = 2 dtheta ds sum and <.,.>_X = sum / N^2.
void radon_transpose(const Plan& p, const cd* zeta, const double* sino, double* img);
// lp_convolve: IFFT(FFT(data) * spec / (Bhat?)) real part,
// on a rows x cols doubled grid, normalised by 1/(rows*cols).
void lp_convolve(const cd* spec, bool divide_bspline, double* data, long rows, long cols);

// Stage probes used by the GPU parity tests (same conventions as above).
// Spectral coefficients of one sector, half theta spectrum k in [0, nts]:
// out (nts+1) x n_rho complex, already multiplied by the spectrum and scaled.
void radon_sector_coeffs(const Plan& p, const cd* zeta, const double* qf, int m, double* out);

// ---------------------------------------------------------------- direct
void direct_radon(const Plan& p, const double* img, double* sino);
void direct_backprojection(const Plan& p, const double* sino, double* img);
void phantom_image(int N, double* img);
void phantom_sinogram(const Plan& p, double* sino);

}  // namespace lpo
