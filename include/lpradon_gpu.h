/* lpradon_gpu.h — C ABI of the B200 log-polar Radon transform library
 * (paper_1506_00014_b200/liblpradon_gpu.so).
 *
 * This is the drop-in boundary for the reference's (specified but
 * unimplemented) fast operators. Each entry point replaces one reference
 * interface:
 *
 *   lpr_geometry_make       <- lpr::sampling_plan        (proj/include/lpradon/geometry.hpp:48-61,
 *                                                          proj/src/geometry.cpp:69-98)
 *   lpr_spectrum_quadrature, lpr_gpu_spectrum_quadrature
 *                           <- lpr::zeta_spectrum / zeta_bp_spectrum
 *                                                         (proj/include/lpradon/kernel.hpp:41-47,
 *                                                          proj/src/kernel.cpp:341-439)
 *   lpr_gpu_plan_create     <- RadonPlan construction
 *   lpr_gpu_radon[_host]    <- fast_radon(Image, RadonPlan) -> Sinogram
 *   lpr_gpu_backproject[_host] <- fast_backprojection(Sinogram, RadonPlan) -> Image
 *   lpr_gpu_radon_transpose <- the exact discrete adjoint used by adjoint_gap
 *   lpr_gpu_sensitivity     <- sensitivity_image(plan)
 *   lpr_gpu_em[_host]       <- em_run(g, plan, iters, f0) / em_step
 *
 * No C++ or CUDA types cross the boundary: plain pointers, sizes and an
 * opaque stream handle (a cudaStream_t passed as void*, NULL = default).
 *
 * Layouts (row-major fp32): images batch x N x N (rows index x2, the
 * raster covers [-1/2, 1/2)^2); sinograms batch x n_theta x N (rows theta =
 * i pi / n_theta, columns s = -1/2 + j / N). Device pointers for the lpr_gpu_*
 * calls, host pointers for the *_host calls (copies happen inside).
 *
 * Errors: every function returns an lpr_status; on failure a message is
 * kept per thread for lpr_gpu_last_error(). LPR_ERR_ARG mirrors the
 * reference's std::invalid_argument (types.hpp:72-74), LPR_ERR_CUDA/OOM its
 * runtime_error class. There is no CPU fallback: without a usable sm_100
 * device every compute call fails with LPR_ERR_CUDA.
 */
#ifndef LPRADON_GPU_H
#define LPRADON_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LPR_OK = 0,
    LPR_ERR_ARG = 1,
    LPR_ERR_CUDA = 2,
    LPR_ERR_OOM = 3,
} lpr_status;

/* Mirrors lpr::GeometryPlan (geometry.hpp:23-43). */
typedef struct {
    int N, M, n_theta, nts, n_rho, refine;
    double beta, a_R, a_r, log_ar, dtheta_p, dtheta_lp, drho, ds;
} lpr_geometry;

typedef struct lpr_gpu_plan lpr_gpu_plan;

/* sampling_plan(N, M[, n_theta]) with an optional n_rho override (>= the
 * minimal count of Eq. (vrho); 0 selects the minimal count). n_theta <= 0
 * selects ceil(3N/2); it is rounded up to a multiple of 2M. */
int lpr_geometry_make(int N, int M, int n_theta, int n_rho, lpr_geometry* out);

/* Smallest n_rho >= the sampling bound whose FFT length factors into
 * {2,3,5,7} (the fast plan variant; the default plan uses the bound itself). */
int lpr_smooth_n_rho(int N, int M);

/* Kernel spectrum on the doubled grid, (2 nts) x n_rho complex interleaved
 * re/im fp64, theta rows in FFT order: kind 0 = zeta (Radon), 1 = zeta#
 * (back-projection). Host fp64, trapezoid + eighth-order end corrections. */
int lpr_spectrum_quadrature(const lpr_geometry* geom, int kind, double* out_re_im);
/* The same spectrum computed on `device` (fp64 sample kernels + batched
 * double-precision FFTs; ~100x faster than the host version at N=2048),
 * written to the host array out_re_im. Plans created with NULL spectra use it. */
int lpr_gpu_spectrum_quadrature(int device, const lpr_geometry* geom, int kind, double* out_re_im);

/* On-disk spectrum cache keyed by (kind, N, M, n_theta, n_rho):
 * lpr_spectrum_quadrature, lpr_gpu_spectrum_quadrature and plan creation with
 * NULL spectra read a cached spectrum (full fp64) instead of recomputing it,
 * and store what they compute. dir = NULL disables the cache; until this is
 * called the directory comes from the environment variable
 * LPR_SPECTRUM_CACHE (unset: disabled). The counters report cache reads and
 * writes since the library was loaded. */
int lpr_spectrum_cache_dir(const char* dir);
long long lpr_spectrum_cache_hits(void);
long long lpr_spectrum_cache_stores(void);

/* Device plan: uploads the spectra (folded with 1/Bhat and the FFT
 * normalisation, fp32) and allocates scratch for max_batch slices. Either
 * spectrum may be NULL, in which case it is computed here. */
int lpr_gpu_plan_create(int device, const lpr_geometry* geom, const double* zeta_re_im,
                        const double* zeta_bp_re_im, int max_batch, lpr_gpu_plan** out);
/* Plan flags. LPR_PLAN_TEXTURE_GATHER: the fine-grid gather of R uses
 * hardware bilinear texture filtering (two linear lookups per axis,
 * PAPER.md:332-349) instead of fp32 software taps — a measured ablation only
 * (the texture unit's fixed-point weights cost ~1e-3 relative accuracy);
 * radon_transpose is not defined for such a plan. */
enum { LPR_PLAN_TEXTURE_GATHER = 1 };
int lpr_gpu_plan_create_ex(int device, const lpr_geometry* geom, const double* zeta_re_im,
                           const double* zeta_bp_re_im, int max_batch, unsigned flags, lpr_gpu_plan** out);
void lpr_gpu_plan_destroy(lpr_gpu_plan* plan);

/* Algorithm 1: d_img (batch x N x N) -> d_sino (batch x n_theta x N). */
int lpr_gpu_radon(lpr_gpu_plan* plan, const float* d_img, float* d_sino, int batch, void* stream);
/* Algorithm 2: d_sino -> d_img (sector sum, factor 2; zero outside the unit disc). */
int lpr_gpu_backproject(lpr_gpu_plan* plan, const float* d_sino, float* d_img, int batch, void* stream);
/* Exact transpose of lpr_gpu_radon under <g,h>_Sigma = 2 dtheta ds sum(g h)
 * and <f,u>_X = sum(f u) / N^2, so <R f, g>_Sigma = <f, R^T g>_X. */
int lpr_gpu_radon_transpose(lpr_gpu_plan* plan, const float* d_sino, float* d_img, int batch, void* stream);

/* lp_convolve, the spectral convolution of Alg. 1 step 6 /
 * Alg. 2 step 4 as a standalone operator: for each of `batch` real rasters on
 * the doubled grid (2 nts rows in periodic order x n_rho columns, row-major,
 * device), out = Re IFFT2(FFT2(in) * S [/ (Bhat_theta Bhat_rho)]) with S the
 * host (2 nts) x n_rho complex fp64 spectrum (re/im interleaved, theta rows in
 * FFT order, even in k_theta like zeta and zeta#: kernel.cpp:228) and its
 * theta-Nyquist row treated as zero, as Algorithms 1-2 do. Runs the plan's
 * own theta / rho / theta-inverse kernels; batch may exceed max_batch. */
int lpr_gpu_lp_convolve(lpr_gpu_plan* plan, const double* spectrum_re_im, int divide_bspline, const float* d_in,
                        float* d_out, int batch, void* stream);
int lpr_gpu_lp_convolve_host(lpr_gpu_plan* plan, const double* spectrum_re_im, int divide_bspline, const float* h_in,
                             float* h_out, int batch);

/* Filtered back-projection (the main caller of R#):
 * kind 0 = ramp, 1 = Shepp-Logan, 2 = cosine transfer functions along s
 * (discrete band-limited ramp with end-point correction, 2N zero padding).
 * lpr_gpu_filter: d_in sinograms -> filtered sinograms (no normalisation);
 * lpr_gpu_fbp: c_norm * R#(filter(d_sino)) with c_norm = 1/2. */
int lpr_gpu_filter(lpr_gpu_plan* plan, int kind, const float* d_in, float* d_out, int batch, void* stream);
int lpr_gpu_fbp(lpr_gpu_plan* plan, int kind, const float* d_sino, float* d_img, int batch, void* stream);
int lpr_gpu_fbp_host(lpr_gpu_plan* plan, int kind, const float* h_sino, float* h_img, int batch);

/* EM reconstruction, device resident:
 * f <- f R#(g / max(R f, eps)) / R# chi_C with eps = 1e-6 max(g) per slice
 * (bins under eps give ratio 0), the sensitivity floor-clamped at 1e-6 of its
 * max, estimates kept >= 0 and 0 outside the unit disc.
 * lpr_gpu_sensitivity: R# chi_C (one N x N image) <- sensitivity_image(plan).
 * lpr_gpu_em: `iters` steps <- em_run(g, plan, iters, f0); d_img holds f0 on
 * entry (init != 0: f0 = 1 inside the unit disc) and the estimate on return;
 * h_loglik (host, batch x iters doubles, may be NULL) receives the Poisson
 * log-likelihood sum(g log Rf - Rf) over Rf > eps of every iterate f^1..f^iters.
 * A negative or non-finite g is LPR_ERR_ARG; a non-finite estimate LPR_ERR_CUDA. */
int lpr_gpu_sensitivity(lpr_gpu_plan* plan, float* d_img, void* stream);
int lpr_gpu_sensitivity_host(lpr_gpu_plan* plan, float* h_img);
int lpr_gpu_em(lpr_gpu_plan* plan, const float* d_sino, float* d_img, int batch, int iters, int init,
               double* h_loglik, void* stream);
int lpr_gpu_em_host(lpr_gpu_plan* plan, const float* h_sino, float* h_img, int batch, int iters, int init,
                    double* h_loglik);

/* Same operators on host buffers: pinned staging, H2D, compute, D2H and a
 * stream synchronisation inside the call (the end-to-end path). */
int lpr_gpu_radon_host(lpr_gpu_plan* plan, const float* h_img, float* h_sino, int batch);
int lpr_gpu_backproject_host(lpr_gpu_plan* plan, const float* h_sino, float* h_img, int batch);
int lpr_gpu_radon_transpose_host(lpr_gpu_plan* plan, const float* h_sino, float* h_img, int batch);
/* R then R# of the same slices in one call (the normal operator R# R of
 * iterative reconstruction, the bench step): h_img in, both the sinograms
 * R f (h_sino) and R# R f (h_back) out; R#'s input stays on the device. */
int lpr_gpu_radon_backproject_host(lpr_gpu_plan* plan, const float* h_img, float* h_sino, float* h_back, int batch);

/* Instrumentation: run one chunk of op (0 = R, 1 = R#) on device buffers
 * `reps` times on the plan's stream with CUDA events between the launches;
 * ms[i] is the mean duration of kernel i, names[i] its stage name (static
 * strings; pass arrays of at least 8). batch <= max_batch. */
int lpr_gpu_profile_stages(lpr_gpu_plan* plan, int op, const float* d_in, float* d_out, int batch, int reps,
                           double* ms, int* nstages, const char** names);

/* The same on host input h_in (copied once into the plan's staging buffer
 * before the timed launches; the outputs stay on the device). */
int lpr_gpu_profile_stages_host(lpr_gpu_plan* plan, int op, const float* h_in, int batch, int reps, double* ms,
                                int* nstages, const char** names);

/* Kernel launches issued by this plan since creation (instrumentation). */
long long lpr_gpu_launch_count(const lpr_gpu_plan* plan);
/* Spectral-convolution launches (the reference's 2-D FFT counter analogue:
 * 2 per sector per operator call). */
long long lpr_gpu_fft_count(const lpr_gpu_plan* plan);

const char* lpr_gpu_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* LPRADON_GPU_H */
