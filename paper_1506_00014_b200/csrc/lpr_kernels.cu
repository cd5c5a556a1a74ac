// sm_100a kernels for the log-polar Radon transform R (PAPER.md:433-450,
// Algorithm 1) and back-projection R# (Algorithm 2).
//
// Stage map (DESIGN.md §4 has the HBM layout and byte model of each):
//   R : k_prefilter_rows -> k_prefilter_cols   (Alg.1 step 1, Qf)
//       k_radon_theta_fwd  gather T_m f e^rho on the fine grid Omega_lp,
//                          zero-embed into the doubled theta period, real
//                          theta FFT, keep |k_theta| < nts  (steps 3-6a)
//       k_rho_pass         rho FFT x (zeta / Bhat) x inverse rho FFT (6b)
//       k_theta_inv        Hermitian theta inverse, crop to the sector (6c)
//       k_radon_out        S_m resampling to the sinogram, a_R^-1 (step 7)
//   R#: k_prefilter_sino -> k_bp_theta_fwd -> k_rho_pass -> k_theta_inv
//       -> k_bp_out (sector sum in ascending m, x2)
#include "lpr_kernels.cuh"

namespace lpr {

namespace {

__device__ __forceinline__ int mirror_idx(int i, int n) {
    if (n == 1) return 0;
    const int per = 2 * (n - 1);
    int r = i % per;
    if (r < 0) r += per;
    return r >= n ? per - r : r;
}

__device__ __forceinline__ int wrapi(int i, int n) {
    int r = i % n;
    return r < 0 ? r + n : r;
}

// Cubic B-spline taps for t = k + a: weights of samples k-1, k, k+1, k+2.
__device__ __forceinline__ void bsw(float a, float w[4]) {
    const float b = 1.0f - a;
    const float a2 = a * a, b2 = b * b;
    w[0] = b2 * b * (1.0f / 6.0f);
    w[1] = fmaf(a2, fmaf(0.5f, a, -1.0f), 2.0f / 3.0f);  // (3a^3 - 6a^2 + 4)/6
    w[2] = fmaf(b2, fmaf(0.5f, b, -1.0f), 2.0f / 3.0f);
    w[3] = a2 * a * (1.0f / 6.0f);
}

}  // namespace

// ------------------------------------------------------------- prefilter
// The cubic B-spline prefilter (bspline.cpp:83-130: causal + anticausal IIR
// with pole z = sqrt(3) - 2, mirror extension) has the two-sided impulse
// response h_d = sqrt(3) z^|d|. Truncated at |d| <= 16 (|z|^17 ~ 2e-10) it
// is a 33-tap separable FIR on the mirror-extended line: every output is
// independent, so lines need no sequential scan and both passes coalesce.

// rows: tmp[b][r][c'] for c' in [0, pitch), apron columns mirrored.
__global__ void k_prefilter_rows(DevGeom g, const float* __restrict__ img, float* __restrict__ tmp) {
    const int cp = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y, b = blockIdx.z;
    if (cp >= g.pitch) return;
    const int N = g.N;
    const float* src = img + (size_t(b) * N + r) * N;
    const int c = mirror_idx(cp - kApron, N);
    float acc = 0.f;
#pragma unroll
    for (int d = -kFirHalf; d <= kFirHalf; ++d) acc = fmaf(__ldg(g.fir + d + kFirHalf), __ldg(src + mirror_idx(c + d, N)), acc);
    tmp[(size_t(b) * N + r) * g.pitch + cp] = acc;
}

// cols: qf[b][r'][c'] over the apron-extended raster.
__global__ void k_prefilter_cols(DevGeom g, const float* __restrict__ tmp, float* __restrict__ qf) {
    const int cp = blockIdx.x * blockDim.x + threadIdx.x;
    const int rp = blockIdx.y, b = blockIdx.z;
    if (cp >= g.pitch) return;
    const int N = g.N;
    const float* src = tmp + size_t(b) * N * g.pitch + cp;
    const int r = mirror_idx(rp - kApron, N);
    float acc = 0.f;
#pragma unroll
    for (int d = -kFirHalf; d <= kFirHalf; ++d)
        acc = fmaf(__ldg(g.fir + d + kFirHalf), __ldg(src + size_t(mirror_idx(r + d, N)) * g.pitch), acc);
    qf[(size_t(b) * g.pitch + rp) * g.pitch + cp] = acc;
}

// sinogram rows (R#, Alg. 2 step 1): prefilter along s only.
__global__ void k_prefilter_sino(DevGeom g, const float* __restrict__ sino, float* __restrict__ qg) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, b = blockIdx.z;
    const int N = g.N;
    if (c >= N) return;
    const float* src = sino + (size_t(b) * g.n_theta + i) * N;
    float acc = 0.f;
#pragma unroll
    for (int d = -kFirHalf; d <= kFirHalf; ++d) acc = fmaf(__ldg(g.fir + d + kFirHalf), __ldg(src + mirror_idx(c + d, N)), acc);
    qg[(size_t(b) * g.n_theta + i) * N + c] = acc;
}

// ------------------------------------------------------------- forward R
// Split the packed transform of z = a + i b into the half spectra of the
// two real sequences and store them as columns l0, l0 + 1 of the sector's
// (nts + 1) x n_rho spectral grid. The theta Nyquist row is zeroed
// (|k_theta| < nts low-pass).
__device__ __forceinline__ void store_half_spectra(const float2* a, int L, int nts, int n_rho, int l0,
                                                   float2* __restrict__ out, int gtid, int gsize) {
    for (int k = gtid; k <= nts; k += gsize) {
        float2 A = make_float2(0.f, 0.f), B = A;
        if (k < nts) {
            const float2 z = a[k], zm = a[k == 0 ? 0 : L - k];
            A = make_float2(0.5f * (z.x + zm.x), 0.5f * (z.y - zm.y));
            B = make_float2(0.5f * (z.y + zm.y), -0.5f * (z.x - zm.x));
        }
        float2* row = out + size_t(k) * n_rho;
        row[l0] = A;
        if (l0 + 1 < n_rho) row[l0 + 1] = B;
    }
}

__device__ __forceinline__ float gather_image(const DevGeom& g, const float* __restrict__ q, float cm, float sm,
                                              float er, float ct, float st) {
    const float dx = fmaf(er, ct, -g.one_m_aR), dy = er * st;
    if (fmaf(dx, dx, dy * dy) > g.aR2) return 0.f;  // outside the sector disc D
    const float ux = dx * g.inv_aR, uy = dy * g.inv_aR;
    const float xp = fmaf(cm, ux, -sm * uy), yp = fmaf(sm, ux, cm * uy);  // T_m^{-1}, physical units
    const float half = 0.5f * g.N;
    const float tc = fmaf(xp, half, half), tr = fmaf(yp, half, half);
    const float kc = floorf(tc), kr = floorf(tr);
    float wc[4], wr[4];
    bsw(tc - kc, wc);
    bsw(tr - kr, wr);
    const float* p = q + (int(kr) - 1 + kApron) * g.pitch + (int(kc) - 1 + kApron);
    float acc = 0.f;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const float* row = p + a * g.pitch;
        const float v = fmaf(wc[0], __ldg(row), fmaf(wc[1], __ldg(row + 1), fmaf(wc[2], __ldg(row + 2), wc[3] * __ldg(row + 3))));
        acc = fmaf(wr[a], v, acc);
    }
    return er * acc;
}

__global__ void __launch_bounds__(512) k_radon_theta_fwd(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd, const float* __restrict__ qf, float2* __restrict__ spec) {
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x, T = blockDim.x;
    const int l0 = 2 * blockIdx.x, m = blockIdx.y, b = blockIdx.z;
    const int Lf = g.Lf, nf = g.nf;
    for (int i = tid; i < Lf; i += T) sm[i] = make_float2(0.f, 0.f);
    __syncthreads();
    const float* q = qf + size_t(b) * g.pitch * g.pitch;
    const float cm = g.cosm[m], smm = g.sinm[m];
    const float er0 = __ldg(g.erho + l0);
    const bool two = l0 + 1 < g.n_rho;
    const float er1 = two ? __ldg(g.erho + l0 + 1) : 0.f;
    for (int i = tid; i < nf; i += T) {
        const float ct = __ldg(g.fine_cos + i), st = __ldg(g.fine_sin + i);
        const float h0 = gather_image(g, q, cm, smm, er0, ct, st);
        const float h1 = two ? gather_image(g, q, cm, smm, er1, ct, st) : 0.f;
        const int qq = i - nf / 2;
        sm[qq < 0 ? qq + Lf : qq] = make_float2(h0, h1);
    }
    __syncthreads();
    const float2* res = block_fft<false>(sm, sm + (fd.nb ? fd.nb : fd.n), fd, tid, T);
    float2* out = spec + (size_t(b) * g.M + m) * size_t(g.nts + 1) * g.n_rho;
    store_half_spectra(res, Lf, g.nts, g.n_rho, l0, out, tid, T);
}

// rho pass: for every (item, k_theta) row, FFT along rho, multiply by the
// kernel spectrum row, inverse FFT. One block per row; the multiplier row is
// shared by all items of the batch (grid.y).
__global__ void __launch_bounds__(512) k_rho_pass(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd, const float2* __restrict__ mult, float2* __restrict__ spec) {
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x, T = blockDim.x;
    const int k = blockIdx.x, item = blockIdx.y;
    const int n = g.n_rho;
    float2* row = spec + (size_t(item) * (g.nts + 1) + k) * n;
    const int len = fd.nb ? fd.nb : fd.n;
    for (int j = tid; j < n; j += T) sm[j] = row[j];
    __syncthreads();
    float2* a = block_fft<false>(sm, sm + len, fd, tid, T);
    const float2* mrow = mult + size_t(k) * n;
    for (int j = tid; j < n; j += T) a[j] = cmul(a[j], __ldg(mrow + j));
    __syncthreads();
    a = block_fft<true>(a, a == sm ? sm + len : sm, fd, tid, T);
    for (int j = tid; j < n; j += T) row[j] = a[j];
}

// Hermitian theta inverse: two real columns per complex transform of length
// 2 nts; rows [j0, j0 + win) of the periodic result are kept.
__global__ void __launch_bounds__(512) k_theta_inv(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd, const float2* __restrict__ spec, float* __restrict__ lp) {
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x, T = blockDim.x;
    const int l0 = 2 * blockIdx.x, m = blockIdx.y, b = blockIdx.z;
    const int nts = g.nts, L2 = g.L2, n = g.n_rho;
    const bool two = l0 + 1 < n;
    const size_t item = size_t(b) * g.M + m;
    const float2* in = spec + item * size_t(nts + 1) * n;
    for (int k = tid; k <= nts; k += T) {
        const float2 A = in[size_t(k) * n + l0];
        const float2 B = two ? in[size_t(k) * n + l0 + 1] : make_float2(0.f, 0.f);
        sm[k] = make_float2(A.x - B.y, A.y + B.x);  // A + iB
        if (k > 0 && k < nts) sm[L2 - k] = make_float2(A.x + B.y, B.x - A.y);  // conj(A) + i conj(B)
    }
    __syncthreads();
    const float2* res = block_fft<true>(sm, sm + (fd.nb ? fd.nb : fd.n), fd, tid, T);
    float* out = lp + item * size_t(g.win) * n;
    for (int r = tid; r < g.win; r += T) {
        const float2 z = res[wrapi(g.j0 + r, L2)];
        out[size_t(r) * n + l0] = z.x;
        if (two) out[size_t(r) * n + l0 + 1] = z.y;
    }
}

// S_m resampling to the sinogram (Alg. 1 step 7). Theta residuals land on
// lattice rows (sector centres are polar rows), so each sinogram row needs
// one coefficient row and a 1-D periodic spline along rho; the theta-axis
// spline weights (1/6, 2/3, 1/6) cancel the theta part of 1/Bhat, which the
// multiplier therefore omits.
__global__ void k_radon_out(DevGeom g, const float* __restrict__ lp, float* __restrict__ sino) {
    extern __shared__ float srow[];
    const int i = blockIdx.x, b = blockIdx.y;
    const int nts = g.nts, n = g.n_rho, N = g.N;
    const int k = (2 * i + nts) / (2 * nts);
    const int m = k % g.M;
    const bool flip = ((k - m) / g.M) & 1;
    const int j = i - k * nts;
    const float* src = lp + ((size_t(b) * g.M + m) * g.win + (j - g.j0)) * n;
    for (int l = threadIdx.x; l < n; l += blockDim.x) srow[l] = src[l];
    __syncthreads();
    const float cth = __ldg(g.coarse_cos + j + nts / 2) * g.one_m_aR;
    const float sgn = flip ? -1.f : 1.f;
    float* out = sino + (size_t(b) * g.n_theta + i) * N;
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
        const float sp = sgn * float(2 * c - N) / float(N);
        const float rho = logf(fmaf(g.aR, sp, cth));
        const float t = (rho - g.log_ar) * g.inv_drho;
        const float kf = floorf(t);
        float w[4];
        bsw(t - kf, w);
        const int k0 = int(kf) - 1;
        float acc = 0.f;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            int idx = k0 + a;
            idx = idx < 0 ? idx + n : (idx >= n ? idx - n : idx);
            acc = fmaf(w[a], srow[idx], acc);
        }
        out[c] = acc * g.out_scale;
    }
}

// ------------------------------------------------------------- R#
__device__ __forceinline__ float gather_sino(const float* __restrict__ row, int N, float t) {
    const float kf = floorf(t);
    float w[4];
    bsw(t - kf, w);
    const int k0 = int(kf) - 1;
    float acc = 0.f;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int idx = k0 + a;
        if (idx >= 0 && idx < N) acc = fmaf(w[a], __ldg(row + idx), acc);
    }
    return acc;
}

// g(S_m^{-1}) on Omega_p (Alg. 2 step 3): theta' rows are polar rows, so each
// sample is a 1-D spline along s (zero outside the detector), then the real
// theta FFT of the zero-embedded doubled period.
__global__ void __launch_bounds__(512) k_bp_theta_fwd(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd, const float* __restrict__ qg, float2* __restrict__ spec) {
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x, T = blockDim.x;
    const int l0 = 2 * blockIdx.x, m = blockIdx.y, b = blockIdx.z;
    const int nts = g.nts, L2 = g.L2, N = g.N;
    for (int i = tid; i < L2; i += T) sm[i] = make_float2(0.f, 0.f);
    __syncthreads();
    const bool two = l0 + 1 < g.n_rho;
    const float er0 = __ldg(g.erho + l0);
    const float er1 = two ? __ldg(g.erho + l0 + 1) : 0.f;
    const float halfN = 0.5f * N;
    for (int jj = tid; jj < nts; jj += T) {
        const int j = jj - nts / 2;
        int i = m * nts + j;
        const bool flip = i < 0;
        if (flip) i += g.n_theta;
        const float* row = qg + (size_t(b) * g.n_theta + i) * N;
        const float cth = __ldg(g.coarse_cos + jj) * g.one_m_aR;
        const float sg = flip ? -halfN : halfN;
        // t = (s_raster + 1/2) N with s_raster = (e^rho - (1-aR) cos) / (2 aR)
        const float t0 = fmaf((er0 - cth) * g.inv_aR, sg, halfN);
        const float v0 = gather_sino(row, N, t0);
        float v1 = 0.f;
        if (two) v1 = gather_sino(row, N, fmaf((er1 - cth) * g.inv_aR, sg, halfN));
        sm[j < 0 ? j + L2 : j] = make_float2(v0, v1);
    }
    __syncthreads();
    const float2* res = block_fft<false>(sm, sm + (fd.nb ? fd.nb : fd.n), fd, tid, T);
    float2* out = spec + (size_t(b) * g.M + m) * size_t(nts + 1) * g.n_rho;
    store_half_spectra(res, L2, nts, g.n_rho, l0, out, tid, T);
}

// T_m^{-1} Omega_p -> X resampling and the sector sum (Alg. 2 steps 5-7).
__global__ void k_bp_out(DevGeom g, const float* __restrict__ lp, float* __restrict__ img) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y, b = blockIdx.z;
    const int N = g.N, n = g.n_rho;
    if (c >= N) return;
    const int dxr = 2 * c - N, dyr = 2 * r - N;
    float* out = img + (size_t(b) * N + r) * N + c;
    if (dxr * dxr + dyr * dyr > N * N) {
        *out = 0.f;
        return;
    }
    const float xp = float(dxr) / float(N), yp = float(dyr) / float(N);
    float acc = 0.f;
    for (int m = 0; m < g.M; ++m) {
        const float cm = g.cosm[m], smm = g.sinm[m];
        const float yx = fmaf(g.aR, fmaf(cm, xp, smm * yp), g.one_m_aR);
        const float yy = g.aR * fmaf(-smm, xp, cm * yp);
        const float th = atan2f(yy, yx);
        const float rho = 0.5f * logf(fmaf(yx, yx, yy * yy));
        const float tt = th * g.inv_dtheta_p;
        const float tr = (rho - g.log_ar) * g.inv_drho;
        const float kt = floorf(tt), kr = floorf(tr);
        float wt[4], wr[4];
        bsw(tt - kt, wt);
        bsw(tr - kr, wr);
        const float* base = lp + (size_t(b) * g.M + m) * size_t(g.win) * n;
        const int r0 = int(kt) - 1 - g.j0;
        int cidx[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int idx = int(kr) - 1 + q;
            cidx[q] = idx < 0 ? idx + n : (idx >= n ? idx - n : idx);
        }
        float sacc = 0.f;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const float* row = base + size_t(r0 + a) * n;
            const float v = fmaf(wr[0], __ldg(row + cidx[0]),
                                 fmaf(wr[1], __ldg(row + cidx[1]), fmaf(wr[2], __ldg(row + cidx[2]), wr[3] * __ldg(row + cidx[3]))));
            sacc = fmaf(wt[a], v, sacc);
        }
        acc += sacc;
    }
    *out = 2.f * acc;
}

}  // namespace lpr
