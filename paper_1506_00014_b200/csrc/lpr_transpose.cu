// Exact transpose R^T of the GPU Radon transform (lpr_gpu_radon), for the
// adjoint identity <R f, g> = <f, R^T g> (SPEC.md:300-308 with the exact
// discrete adjoint; the oracle's radon_transpose in oracle/lpo.cpp is the
// fp64 counterpart). Stages, each the transpose of a forward stage:
//
//   k_radon_out_T        E_m^T : sinogram rows -> lattice rows of the sector
//                        grids (shared-memory scatter of the rho spline taps)
//   k_theta_fwd_T  (T2)  real theta FFT of the lattice rows (length 2 nts)
//   k_rho_pass  (T3)     rho FFT x conj(zeta / Bhat_rho / (Lf n_rho)) x iFFT
//   k_theta_inv_fine_T   Hermitian theta inverse over the doubled fine
//                        period Lf (zero-filled beyond |k| < nts), then the
//                        transposed fine-grid gather: spline taps scattered
//                        into the apron-extended coefficient image
//   k_prefilter_cols_T / k_prefilter_rows_T   banded transposes of the
//                        FIR prefilter, including the mirror apron.
#include "lpr_kernels.cuh"

namespace lpr {

namespace {
__device__ __forceinline__ void bswT(float a, float w[4]) {
    const float b = 1.0f - a;
    const float a2 = a * a, b2 = b * b;
    w[0] = b2 * b * (1.0f / 6.0f);
    w[1] = fmaf(a2, fmaf(0.5f, a, -1.0f), 2.0f / 3.0f);
    w[2] = fmaf(b2, fmaf(0.5f, b, -1.0f), 2.0f / 3.0f);
    w[3] = a2 * a * (1.0f / 6.0f);
}
}  // namespace

// E_m^T: one block per sinogram row i; the lattice row (m, j) it reads in the
// forward pass receives out_scale * w_a * g(i, c) at taps k0 + a (periodic).
__global__ void k_radon_out_T(DevGeom g, const float* __restrict__ sino, float* __restrict__ lp) {
    extern __shared__ float srow[];
    const int i = blockIdx.x, b = blockIdx.y;
    const int nts = g.nts, n = g.n_rho, N = g.N;
    for (int l = threadIdx.x; l < n; l += blockDim.x) srow[l] = 0.f;
    __syncthreads();
    const int k = (2 * i + nts) / (2 * nts);
    const int m = k % g.M;
    const bool flip = ((k - m) / g.M) & 1;
    const int j = i - k * nts;
    const float cth = __ldg(g.coarse_cos + j + nts / 2) * g.one_m_aR;
    const float sgn = flip ? -1.f : 1.f;
    const float invN = 1.f / float(N);
    const float* in = sino + (size_t(b) * g.n_theta + i) * N;
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
        const float sp = sgn * float(2 * c - N) * invN;  // (x / N exactly for power-of-two N)
        const float rho = logf(fmaf(g.aR, sp, cth));
        const float t = (rho - g.log_ar) * g.inv_drho;
        const float kf = floorf(t);
        float w[4];
        bswT(t - kf, w);
        const int k0 = int(kf) - 1;
        const float v = __ldg(in + c) * g.out_scale;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            int idx = k0 + a;
            idx = idx < 0 ? idx + n : (idx >= n ? idx - n : idx);
            atomicAdd(srow + idx, w[a] * v);
        }
    }
    __syncthreads();
    float* dst = lp + ((size_t(b) * g.M + m) * g.win + (j - g.j0)) * g.lps;
    for (int l = threadIdx.x; l < n; l += blockDim.x) dst[l] = srow[l];
}

// Banded transposes of the prefilter. band[r][j] = Q1[r + A - H + j][r] where
// Q1: R^N -> R^pitch is the apron-extended 1-D FIR prefilter (host-built).
__global__ void k_prefilter_cols_T(DevGeom g, const float* __restrict__ band, int H, const float* __restrict__ qbar,
                                   float* __restrict__ tmp) {
    const int cp = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y, b = blockIdx.z;
    if (cp >= g.pitch) return;
    const float* src = qbar + size_t(b) * g.pitch * g.pitch + cp;
    const float* w = band + size_t(r) * (2 * H + 1);
    float acc = 0.f;
    for (int j = 0; j <= 2 * H; ++j) {
        const int rp = r + kApron - H + j;
        if (rp >= 0 && rp < g.pitch) acc = fmaf(__ldg(w + j), __ldg(src + size_t(rp) * g.pitch), acc);
    }
    tmp[(size_t(b) * g.N + r) * g.pitch + cp] = acc;
}

__global__ void k_prefilter_rows_T(DevGeom g, const float* __restrict__ band, int H, const float* __restrict__ tmp,
                                   float* __restrict__ img, float scale) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y, b = blockIdx.z;
    if (c >= g.N) return;
    const float* src = tmp + (size_t(b) * g.N + r) * g.pitch;
    const float* w = band + size_t(c) * (2 * H + 1);
    float acc = 0.f;
    for (int j = 0; j <= 2 * H; ++j) {
        const int cp = c + kApron - H + j;
        if (cp >= 0 && cp < g.pitch) acc = fmaf(__ldg(w + j), __ldg(src + cp), acc);
    }
    img[(size_t(b) * g.N + r) * g.N + c] = scale * acc;
}

}  // namespace lpr
