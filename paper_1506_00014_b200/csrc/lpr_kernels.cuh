// Device-side plan constants and kernel declarations for the log-polar
// Radon transform R (Alg. 1) and back-projection R# (Alg. 2).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "lpr_fft.cuh"

namespace lpr {

constexpr int kMaxSectors = 16;

// The image B-spline coefficients read by the fine-grid gather: quad taps,
// element [r][c] = Q[r][c..c+3] (one 16-byte load per spline tap row), plus
// the transposed raster for sector 0 (element [c][r] = Q[r..r+3][c]).
using Tap = float4;
constexpr int kApron = 4;     // mirrored border around the image coefficients
constexpr int kFirHalf = 16;  // B-spline prefilter impulse-response half length
constexpr int kOutSlices = 4;  // slices per block of the R output resampling kernel

// Row stride of the theta-inverse window buffer lp: n_rho columns + 3
// periodic copies (rho taps never wrap), rounded up to 8 floats (32-byte rows,
// the texture pitch of k_bp_out's tld4 view). One definition for the plan and
// the kernels specialised on a compile-time N_rho.
__host__ __device__ constexpr int lp_stride(int n_rho) { return (n_rho + 3 + 7) / 8 * 8; }

// Everything a kernel needs about the plan, passed by value.
struct DevGeom {
    int N, M, n_theta, nts, n_rho, refine;
    int nf;      // fine theta rows per sector (refine * nts)
    int Lf;      // doubled fine period (2 * nf)
    int L2;      // doubled coarse period (2 * nts)
    int win;     // rows kept from the coarse theta inverse
    int j0;      // coarse theta index of window row 0 (= -nts/2 - 4)
    int pitch;   // row pitch of the apron image (N + 2 kApron)
    int lps;     // row stride of the theta-inverse window buffer lp: n_rho + 3 periodic columns, rounded up to 4 (16-byte rows)
    float aR, inv_aR, one_m_aR, aR2, log_ar, inv_drho, inv_dtheta_p, out_scale;
    float cosm[kMaxSectors], sinm[kMaxSectors];
    float vcm[kMaxSectors], vrm[kMaxSectors];  // pixel coords of T_m^{-1}(0): (N/2)(1 - (cos, sin)(m beta)(1 - aR)/aR)
    float mask_k;                               // 1 - 2 aR (sector-disc test)
    // tables (device)
    const float* fine_cos;    // nf entries: cos(q dtheta_lp), q = i - nf/2
    const float* fine_sin;
    int fine_b1;              // stride of a thread's rows in the fused fine first pass (0: use the tables)
    float2 fine_rot[16];      // (cos, sin)(j fine_b1 dtheta_lp), j < 16
    const float* coarse_cos;  // nts entries: cos(j dtheta_p), j = jj - nts/2
    const float* erho;        // n_rho entries: exp(log a_r + l drho)
    const float* fir;         // 2 kFirHalf + 1 prefilter taps
    cudaTextureObject_t qtex; // texture-gather ablation: coefficient raster (0 unless enabled)
    cudaTextureObject_t lptex; // tld4 view of lp for k_bp_out (0 unless enabled)
};

// FFT kernel variants: a compile-time register FFT for the hot lengths
// (lpr_fft_ct.cuh) or the generic runtime Stockham / Bluestein.
enum FftVariant : int { kFftGeneric = 0, kFft2048, kFft4096, kFft4374, kFft8192, kFft16384 };
struct FftLaunch {
    int variant;
    int threads;   // block size of the theta kernels (kT * kP)
    int tpt;       // threads per transform (block size of the rho pass)
    int per_block; // transforms (column pairs) per theta block
    size_t smem;   // shared bytes of one transform
    int rho_stream = 0;  // rho pass: 1 = the TMA-streamed two-rows-per-block kernel (k_rho_stream)
};

// host-side launchers (lpr_kernels.cu)
FftLaunch fft_launch_config(const FftDesc& d);
int fft_first_radix(int variant);  // 0 for the generic plan
std::vector<float2> fft_pass_twiddles(int variant);
cudaError_t prepare_fft_kernels(const FftLaunch& fine, const FftLaunch& rho, const FftLaunch& coarse,
                                size_t rho_mult_bytes);
void launch_radon_theta_fwd(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                            const Tap* qf, const Tap* qft, float2* spec, int tex);  // tex: 0 quad taps, 1 hardware bilinear (ablation)
void launch_prefilter_2d(bool quad, int nb, cudaStream_t st, const DevGeom& g, const float* img, void* out,
                         void* out_t);
size_t rho_stream_smem(int variant);  // 0: no streamed rho kernel for this length
std::vector<float4> rho_stream_inv_twiddles(int variant);
std::vector<float4> rho_stream_fwd_twiddles(int variant);
size_t rho_pad_length(int n_rho);  // padded convolution length for a non-smooth n_rho (0: none)
size_t rho_direct_length();       // the compile-time length k_rho_pad also runs unpadded
void launch_rho_pad(int nb, dim3 grid, cudaStream_t st, const DevGeom& g, const float2* mult_pad, float2* spec);
cudaError_t prepare_rho_pad();
void launch_rho_pad_gen(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                        const float2* mult_pad, float2* spec);
cudaError_t prepare_rho_pad_gen(const FftLaunch& L, int nb);
void launch_rho_pass(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                     const float2* mult, float2* spec);
void launch_theta_inv(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                      const float2* spec, float* lp);
void launch_bp_theta_fwd(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                         const float* qg, float2* spec);
void launch_lpc_theta_fwd(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                          const float* data, float2* spec);
void launch_theta_fwd_T(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                        const float* lp, float2* spec);
void launch_theta_inv_fine_T(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                             const float2* spec, float* qbar);
cudaError_t prepare_filter_kernel(const FftLaunch& L);
cudaError_t prepare_out_kernels(int lps);
cudaError_t prepare_prefilter_sino();
void launch_prefilter_sino(int nb, cudaStream_t st, const DevGeom& g, const float* sino, float* qg);
void launch_radon_out(int nb, cudaStream_t st, const DevGeom& g, const float* lp, float* sino);
void launch_bp_out(int nb, cudaStream_t st, const DevGeom& g, const float* lp, float* img);
void launch_sino_filter(const FftLaunch& L, int rows_total, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                        const float* H, const float* in, float* out);

}  // namespace lpr
