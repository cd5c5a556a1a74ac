// sm_100a kernels for the log-polar Radon transform R (PAPER.md:433-450,
// Algorithm 1) and back-projection R# (Algorithm 2).
//
// Stage map (DESIGN.md §4 has the HBM layout and byte model of each):
//   R : k_prefilter_2d     (Alg.1 step 1, Qf with a mirrored apron)
//       k_radon_theta_fwd  gather T_m f e^rho on the fine grid Omega_lp,
//                          zero-embed into the doubled theta period, real
//                          theta FFT, keep |k_theta| < nts  (steps 3-6a)
//       k_rho_pass         rho FFT x (zeta / Bhat) x inverse rho FFT (6b)
//       k_theta_inv        Hermitian theta inverse, crop to the sector (6c)
//       k_radon_out        S_m resampling to the sinogram, a_R^-1 (step 7)
//   R#: k_prefilter_sino -> k_bp_theta_fwd -> k_rho_pass -> k_theta_inv
//       -> k_bp_out (sector sum in ascending m, x2)
#include <cuda_pipeline.h>

#include <cstdint>
#include <cstdlib>

#include "lpr_fft_ct.cuh"
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


// Cubic B-spline taps for t = k + a: weights of samples k-1, k, k+1, k+2.
__device__ __forceinline__ void bsw(float a, float w[4]) {
    const float b = 1.0f - a;
    const float a2 = a * a, b2 = b * b;
    w[0] = b2 * b * (1.0f / 6.0f);
    w[1] = fmaf(a2, fmaf(0.5f, a, -1.0f), 2.0f / 3.0f);  // (3a^3 - 6a^2 + 4)/6
    w[2] = fmaf(b2, fmaf(0.5f, b, -1.0f), 2.0f / 3.0f);
    w[3] = a2 * a * (1.0f / 6.0f);
}

// Both axes' tap weights at once on the packed fp32x2 pipe: (wx[k], wy[k]) = bsw
// of (ax, ay), the same polynomials as bsw.
__device__ __forceinline__ void bsw2(float2 a, float2 w[4]) {
    const float2 b = __fadd2_rn(make_float2(1.f, 1.f), make_float2(-a.x, -a.y));
    const float2 a2 = __fmul2_rn(a, a), b2 = __fmul2_rn(b, b);
    const float2 sixth = make_float2(1.0f / 6.0f, 1.0f / 6.0f), half = make_float2(0.5f, 0.5f);
    const float2 m1 = make_float2(-1.f, -1.f), two3 = make_float2(2.0f / 3.0f, 2.0f / 3.0f);
    w[0] = __fmul2_rn(__fmul2_rn(b2, b), sixth);
    w[1] = __ffma2_rn(a2, __ffma2_rn(half, a, m1), two3);
    w[2] = __ffma2_rn(b2, __ffma2_rn(half, b, m1), two3);
    w[3] = __fmul2_rn(__fmul2_rn(a2, a), sixth);
}

}  // namespace

// ------------------------------------------------------------- prefilter
// The cubic B-spline prefilter (bspline.cpp:83-130), recursive: a 64 x 64 output
// tile is staged with a 16-sample warm-up margin per side (through the
// mirror map), then each thread runs the causal + anticausal recursion
// (pole z = sqrt(3) - 2, bspline.cpp:93-106) along one row, then along one
// column, 2 FMAs per sample per pass instead of 33. Starting the recursion
// 16 samples early with the steady-state initial value leaves |z|^16 ~ 7e-10
// of the start-up transient, the same truncation as the FIR form.
constexpr int kIT = 64;                   // output tile edge
constexpr int kIW = 16;                   // warm-up samples per side
constexpr int kIR = kIT + 2 * kIW;        // staged rows
constexpr int kIC = kIT + 3 + 2 * kIW;    // staged columns (quad needs 3 more)
constexpr int kICP = kIC + 2;             // odd row pitch (101): row- and column-walks are conflict-free
constexpr int kIQ = (kIC + 3) / 4;        // 16-byte words per staged row on the interior fast path (25)

// Stage R rows of Q float4 (row stride `ld` floats, 16-byte aligned source) into
// shared rows of pitch P floats: every load of the thread issued before any store.
template <int R, int Q, int P, int T>
__device__ __forceinline__ void stage_rows(float* s, const float* __restrict__ src, int ld, int tid) {
    constexpr int TOT = R * Q, PER = (TOT + T - 1) / T;
    float4 v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int idx = tid + u * T;
        if (idx < TOT) v[u] = __ldg(reinterpret_cast<const float4*>(src + size_t(idx / Q) * ld) + idx % Q);
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int idx = tid + u * T;
        if (idx < TOT) {
            float* d = s + (idx / Q) * P + 4 * (idx % Q);
            d[0] = v[u].x;
            d[1] = v[u].y;
            d[2] = v[u].z;
            d[3] = v[u].w;
        }
    }
}

// PITCH > 0: the raster pitch at compile time (N = 2048: 2056), so the store
// loops' row steps are immediates
template <class T, int PITCH = 0>
__global__ void __launch_bounds__(128, 5) k_prefilter_2d_iir(DevGeom g, const float* __restrict__ img, T* __restrict__ q4,
                                                          T* __restrict__ q4t) {
    __shared__ float s[kIR][kICP];
    constexpr float z = -0.26794919243112270647f;
    constexpr float c0 = 6.0f / (1.0f - z), ca = -z / (1.0f - z);
    const int tid = threadIdx.x;
    const int N = g.N, pitch = PITCH ? PITCH : g.pitch;
    const int x0 = blockIdx.x * kIT, y0 = blockIdx.y * kIT, b = blockIdx.z;
    const float* src = img + size_t(b) * N * N;
    const int vx0 = x0 - kApron - kIW, vy0 = y0 - kApron - kIW;
    if (vx0 >= 0 && vx0 + 4 * kIQ <= N && vy0 >= 0 && vy0 + kIR <= N && (N & 3) == 0 &&
        (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        // interior tile (no mirroring): all of a thread's 16-byte loads in flight at once
        stage_rows<kIR, kIQ, kICP, 128>(&s[0][0], src + size_t(vy0) * N + vx0, N, tid);
    } else {
        for (int idx = tid; idx < kIR * kIC; idx += blockDim.x) {
            const int i = idx / kIC, j = idx % kIC;
            s[i][j] = __ldg(src + size_t(mirror_idx(vy0 + i, N)) * N + mirror_idx(vx0 + j, N));
        }
    }
    __syncthreads();
    if (tid < kIR) {  // rows
        float* r = s[tid];
        float c = c0 * r[0];
        r[0] = c;
        for (int k = 1; k < kIC; ++k) r[k] = c = fmaf(z, c, 6.0f * r[k]);
        float d = ca * c;
        r[kIC - 1] = d;
        for (int k = kIC - 2; k >= 0; --k) r[k] = d = z * (d - r[k]);
    }
    __syncthreads();
    if (tid < kIT + 3) {  // columns kIW .. kIW + kIT + 2
        const int j = kIW + tid;
        float c = c0 * s[0][j];
        s[0][j] = c;
        for (int k = 1; k < kIR; ++k) s[k][j] = c = fmaf(z, c, 6.0f * s[k][j]);
        float d = ca * c;
        s[kIR - 1][j] = d;
        for (int k = kIR - 2; k >= 0; --k) s[k][j] = d = z * (d - s[k][j]);
    }
    __syncthreads();
    // stores (128 threads, launch_prefilter_2d): a thread keeps one tile column
    // (row-major quads) or one tile row (transposed quads) and steps the other
    // index by 2, so the index math is hoisted out of the loop
    static_assert(kIT == 64, "the store loops assume 128 threads over 64-wide tiles");
    T* dst = q4 + size_t(b) * pitch * pitch;
    {
        const int j = tid & (kIT - 1);
        if (x0 + j < pitch) {
            T* d = dst + size_t(y0) * pitch + x0 + j;
#pragma unroll 2
            for (int i = tid >> 6; i < kIT; i += 2) {
                if (y0 + i >= pitch) break;
                const float* r = s[kIW + i] + kIW + j;
                if constexpr (sizeof(T) == sizeof(float4)) {
                    d[size_t(i) * pitch] = make_float4(r[0], r[1], r[2], r[3]);
                } else {
                    d[size_t(i) * pitch] = r[0];
                }
            }
        }
    }
    if constexpr (sizeof(T) == sizeof(float4)) {
        if (q4t) {  // transposed quads qt[c][r] = Q[r..r+3][c] (read by sector 0); a warp writes 32 consecutive r
            const int i = tid & (kIT - 1);
            if (y0 + i < pitch) {
                T* dt = q4t + size_t(b) * pitch * pitch + size_t(x0) * pitch + y0 + i;
                const float* r0 = s[kIW + i] + kIW;
#pragma unroll 2
                for (int j = tid >> 6; j < kIT; j += 2) {
                    if (x0 + j >= pitch) break;
                    const float* r = r0 + j;
                    dt[size_t(j) * pitch] = make_float4(r[0], r[kICP], r[2 * kICP], r[3 * kICP]);
                }
            }
        }
    }
}

// quad = false writes the plain fp32 coefficient raster (the texture ablation binds it).
void launch_prefilter_2d(bool quad, int nb, cudaStream_t st, const DevGeom& g, const float* img, void* out,
                         void* out_t) {
    const dim3 grid((g.pitch + kIT - 1) / kIT, (g.pitch + kIT - 1) / kIT, nb);
    if (quad)
        if (g.pitch == 2048 + 2 * kApron)
            k_prefilter_2d_iir<Tap, 2048 + 2 * kApron><<<grid, 128, 0, st>>>(g, img, static_cast<Tap*>(out),
                                                                           static_cast<Tap*>(out_t));
        else
            k_prefilter_2d_iir<Tap><<<grid, 128, 0, st>>>(g, img, static_cast<Tap*>(out), static_cast<Tap*>(out_t));
    else
        k_prefilter_2d_iir<float><<<grid, 128, 0, st>>>(g, img, static_cast<float*>(out), nullptr);
}

// Recursive prefilter along s for R# (Alg. 2 step 1): a 128-row x 64-column
// tile with a 16-sample warm-up per side, every thread running the causal +
// anticausal recursion of one row (96 steps each way; a 32 x 256 tile left
// three of four warps idle through a 288-step recursion: 0.337 -> 0.323 ms
// per 16 slices).
constexpr int kSRows = 128, kSCols = 64, kSP = kSCols + 2 * kIW + 1;  // odd pitch
constexpr size_t kSinoPfSmem = size_t(kSRows) * kSP * sizeof(float);

// LD > 0: n_theta (the Qg^T row stride) at compile time, so the transposed
// store's column steps are immediates (the N = 2048 bench plan: 3072)
template <int LD = 0>
__global__ void __launch_bounds__(128) k_prefilter_sino_iir(DevGeom g, const float* __restrict__ sino,
                                                            float* __restrict__ qg) {
    extern __shared__ float s[];  // [kSRows][kSP]
    constexpr float z = -0.26794919243112270647f;
    constexpr float c0 = 6.0f / (1.0f - z), ca = -z / (1.0f - z);
    constexpr int L = kSCols + 2 * kIW;
    const int tid = threadIdx.x;
    const int N = g.N;
    const int c0col = blockIdx.x * kSCols, i0 = blockIdx.y * kSRows, b = blockIdx.z;
    const int rows = min(kSRows, g.n_theta - i0);
    if (rows == kSRows && c0col - kIW >= 0 && c0col - kIW + L <= N && (N & 3) == 0 &&
        (reinterpret_cast<uintptr_t>(sino) & 15) == 0) {
        stage_rows<kSRows, L / 4, kSP, 128>(s, sino + (size_t(b) * g.n_theta + i0) * N + c0col - kIW, N, tid);
    } else {
        for (int idx = tid; idx < rows * L; idx += blockDim.x) {
            const int i = idx / L, j = idx % L;
            s[i * kSP + j] = __ldg(sino + (size_t(b) * g.n_theta + i0 + i) * N + mirror_idx(c0col - kIW + j, N));
        }
    }
    __syncthreads();
    if (tid < rows) {
        float* r = s + tid * kSP;
        float c = c0 * r[0];
        r[0] = c;
        for (int k = 1; k < L; ++k) r[k] = c = fmaf(z, c, 6.0f * r[k]);
        float d = ca * c;
        r[L - 1] = d;
        for (int k = L - 2; k >= 0; --k) r[k] = d = z * (d - r[k]);
    }
    __syncthreads();
    // transposed store (Qg^T[b][s][theta], see gather_sino): a warp writes 32
    // consecutive theta of one s column; the odd pitch keeps the reads conflict-free
    // (128 threads = kSRows: thread i owns tile row i and steps the s column)
    static_assert(kSRows == 128, "one tile row per thread");
    if (tid < rows) {
        const int ld = LD ? LD : g.n_theta;
        float* d = qg + (size_t(b) * N + c0col) * ld + i0 + tid;
        const float* src = s + tid * kSP + kIW;
        const int cols = min(kSCols, N - c0col);
#pragma unroll 8
        for (int j = 0; j < cols; ++j) d[size_t(j) * ld] = src[j];
    }
}

constexpr int kNThetaSino = 3072;  // the N = 2048 plans' n_theta (k_prefilter_sino_iir<LD>)

cudaError_t prepare_prefilter_sino() {
    cudaError_t e = cudaFuncSetAttribute(k_prefilter_sino_iir<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kSinoPfSmem));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_prefilter_sino_iir<kNThetaSino>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(kSinoPfSmem));
}

void launch_prefilter_sino(int nb, cudaStream_t st, const DevGeom& g, const float* sino, float* qg) {
    const dim3 grid((g.N + kSCols - 1) / kSCols, (g.n_theta + kSRows - 1) / kSRows, nb);
    if (g.n_theta == kNThetaSino)
        k_prefilter_sino_iir<kNThetaSino><<<grid, 128, kSinoPfSmem, st>>>(g, sino, qg);
    else
        k_prefilter_sino_iir<0><<<grid, 128, kSinoPfSmem, st>>>(g, sino, qg);
}

// ------------------------------------------------------------- FFT-policy kernels
// Every kernel with a transform is a template over the FFT policy F
// (lpr_fft_ct.cuh): a compile-time register FFT for the hot lengths or the
// generic runtime Stockham/Bluestein. F::idx maps element i to its shared
// slot. Theta kernels run F::kP transforms per block, one per thread group,
// each on a pair of real columns packed as re/im, so a block touches 4 kP
// contiguous complex columns per spectral row.
template <class F>
struct Group {
    int g, tid, size;
    __device__ __forceinline__ Group() {
        if constexpr (F::kT > 0) {
            size = F::kT;
            g = threadIdx.x / F::kT;
            tid = threadIdx.x % F::kT;
        } else {
            size = blockDim.x;
            g = 0;
            tid = threadIdx.x;
        }
    }
};

#define LPR_LB(F) __launch_bounds__((F::kT > 0 ? F::kT * F::kP : 512), F::kMinBlocks)

template <class F>
__device__ __forceinline__ float2* fft_scratch(float2* sm, const FftDesc& d) {
    return sm + (d.nb ? d.nb : d.n);
}

// The kP transform buffers of a block, addressed arithmetically (an array of
// pointers indexed by a runtime p would live in local memory).
struct Slots {
    float2* base;
    int stride;
    __device__ __forceinline__ float2* operator()(int p) const { return base + p * stride; }
};

// Where the results are: compile-time plans run in place (slot p = smem + p E);
// the generic plan (kP = 1) may finish in its scratch half.
template <class F>
__device__ __forceinline__ Slots result_slots(float2* smem, int E, float2* res) {
    if constexpr (F::kT > 0) return Slots{smem, E};
    return Slots{res, 0};
}

// Pair the block's columns: pair p of the block covers columns l0 + 2p, l0 + 2p + 1.
__device__ __forceinline__ bool col_ok(int l, int n) { return l < n; }

// Split the packed transforms into half spectra and store rows k in [0, nts]
// for all kP pairs of the block; consecutive threads take consecutive pairs of
// one row (float4 each when aligned). The theta Nyquist row is zeroed.
template <class F>
__device__ __forceinline__ void store_half_spectra(Slots res, int L, int nts, int n_rho, int l0,
                                                   float2* __restrict__ out) {
    constexpr int P = F::kP;
    if constexpr (F::kT > 0) {
        // compile-time block size: one pair per thread, rows tid / P + j kT (index math hoisted)
        const int p = threadIdx.x % P, l = l0 + 2 * p;
        if (l >= n_rho) return;
        const float2* x = res(p);
        float2* dst0 = out + l;
        const bool two = l + 1 < n_rho;
        for (int k = threadIdx.x / P; k <= nts; k += F::kT) {
            float2 A = make_float2(0.f, 0.f), B = A;
            if (k < nts) {
                const float2 z = x[F::idx(k)], zm = x[F::idx(k == 0 ? 0 : L - k)];
                A = make_float2(0.5f * (z.x + zm.x), 0.5f * (z.y - zm.y));
                B = make_float2(0.5f * (z.y + zm.y), -0.5f * (z.x - zm.x));
            }
            float2* dst = dst0 + size_t(k) * n_rho;
            if (two && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                *reinterpret_cast<float4*>(dst) = make_float4(A.x, A.y, B.x, B.y);
            } else {
                dst[0] = A;
                if (two) dst[1] = B;
            }
        }
        return;
    }
    for (int e = threadIdx.x; e < (nts + 1) * P; e += blockDim.x) {
        const int k = e / P, p = e % P;
        const int l = l0 + 2 * p;
        if (l >= n_rho) continue;
        float2 A = make_float2(0.f, 0.f), B = A;
        if (k < nts) {
            const float2 z = res(p)[F::idx(k)], zm = res(p)[F::idx(k == 0 ? 0 : L - k)];
            A = make_float2(0.5f * (z.x + zm.x), 0.5f * (z.y - zm.y));
            B = make_float2(0.5f * (z.y + zm.y), -0.5f * (z.x - zm.x));
        }
        float2* dst = out + size_t(k) * n_rho + l;
        if (l + 1 < n_rho && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            *reinterpret_cast<float4*>(dst) = make_float4(A.x, A.y, B.x, B.y);
        } else {
            dst[0] = A;
            if (l + 1 < n_rho) dst[1] = B;
        }
    }
}

// Same, for a plan whose final radix-2 pass (NS = L/2) was not run: only the
// outputs |k| < nts are needed, so each is finished here from the four
// inputs of its two radix-2 butterflies: Z(k) = x[k] + w x[k + L/2] and
// Z(L - k) = x[L/2 - k] + conj(w) x[L - k], w = exp(-2 pi i k / L).
template <class F>
__device__ __forceinline__ void store_half_spectra_r2(Slots res, int L, int nts, int n_rho, int l0b,
                                                      float2* __restrict__ out, float s0 = 1.f, float s1 = 1.f) {
    const float h0 = 0.5f * s0, h1 = 0.5f * s1;  // column scales (P = 1), with the 1/2 of the split
    constexpr int P = F::kP;
    const int H = L / 2;
    for (int e = threadIdx.x; e < (nts + 1) * P; e += (F::kT > 0 ? F::kT * F::kP : int(blockDim.x))) {
        const int k = e / P, p = e % P;
        const int l = l0b + 2 * p;
        if (l >= n_rho) continue;
        float2 A = make_float2(0.f, 0.f), B = A;
        if (k < nts) {
            float sn, cs;
            __sincosf(-6.283185307179586f * (float(k) / float(L)), &sn, &cs);
            const float2 w = make_float2(cs, sn);
            const float2* x = res(p);
            const float2 z = cadd(x[F::idx(k)], cmul(x[F::idx(k + H)], w));
            const float2 zm = k == 0 ? z : cadd(x[F::idx(H - k)], cmulc(x[F::idx(L - k)], w));
            A = make_float2(h0 * (z.x + zm.x), h0 * (z.y - zm.y));
            B = make_float2(h1 * (z.y + zm.y), -h1 * (z.x - zm.x));
        }
        float2* dst = out + size_t(k) * n_rho + l;
        if (l + 1 < n_rho && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            *reinterpret_cast<float4*>(dst) = make_float4(A.x, A.y, B.x, B.y);
        } else {
            dst[0] = A;
            if (l + 1 < n_rho) dst[1] = B;
        }
    }
}

// Load half spectra rows k in [0, kmax) of the block's pairs and rebuild each
// packed Hermitian transform of length L: Z(k) = A + iB, Z(L-k) = conj(A) + i conj(B).
template <class F>
__device__ __forceinline__ void put_packed(Slots sm, int k, int p, int L, float2 A, float2 B) {
    sm(p)[F::idx(k)] = make_float2(A.x - B.y, A.y + B.x);
    if (k > 0) sm(p)[F::idx(L - k)] = make_float2(A.x + B.y, B.x - A.y);
}

template <class F>
__device__ __forceinline__ void load_packed_hermitian(Slots sm, const float2* __restrict__ in, int kmax,
                                                      int L, int n, int l0) {
    constexpr int P = F::kP;
    if constexpr (F::kT > 0) {
        // compile-time block size: a thread keeps one column pair p and walks
        // rows k = tid / P + j RS, so the index math is hoisted out of the loop
        // (the integer pipe was this kernel's busiest)
        constexpr int BT = F::kT * P, RS = BT / P;
        constexpr int U = 8;  // independent 16-byte loads in flight per thread
        const int p = threadIdx.x % P, k0 = threadIdx.x / P;
        const int l = l0 + 2 * p;
        const bool vec = l + 2 <= n && (n % 2) == 0 && (reinterpret_cast<uintptr_t>(in + l) & 15) == 0;
        float2* dst = sm(p);
        if (vec && l0 + 2 * P <= n) {
            const float4* src = reinterpret_cast<const float4*>(in + l);
            const int n4 = n / 2;  // float4 row stride
            for (int kb = k0; kb < kmax; kb += U * RS) {
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = kb + u * RS;
                    if (k < kmax) v[u] = __ldg(src + size_t(k) * n4);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = kb + u * RS;
                    if (k < kmax) {
                        const float2 A = make_float2(v[u].x, v[u].y), B = make_float2(v[u].z, v[u].w);
                        dst[F::idx(k)] = make_float2(A.x - B.y, A.y + B.x);
                        if (k > 0) dst[F::idx(L - k)] = make_float2(A.x + B.y, B.x - A.y);
                    }
                }
            }
            return;
        }
        if (l0 + 2 * P <= n) {
            // odd n (the reference plans' N_rho, e.g. 4333): rows are only 8-byte
            // aligned, so two 8-byte loads per row, still U rows in flight
            const float2* src = in + l;
            for (int kb = k0; kb < kmax; kb += U * RS) {
                float2 a[U], c[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = kb + u * RS;
                    if (k < kmax) {
                        a[u] = __ldg(src + size_t(k) * n);
                        c[u] = __ldg(src + size_t(k) * n + 1);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = kb + u * RS;
                    if (k < kmax) {
                        dst[F::idx(k)] = make_float2(a[u].x - c[u].y, a[u].y + c[u].x);
                        if (k > 0) dst[F::idx(L - k)] = make_float2(a[u].x + c[u].y, c[u].x - a[u].y);
                    }
                }
            }
            return;
        }
    }
#ifndef LPR_HERM_U
#define LPR_HERM_U 8
#endif
    constexpr int U = LPR_HERM_U;  // independent 16-byte loads in flight per thread
    const int total = kmax * P;
    const bool vec = l0 + 2 * P <= n && (n % 2) == 0 && (reinterpret_cast<uintptr_t>(in + l0) & 15) == 0;
    if (vec) {
        for (int base = threadIdx.x; base < total; base += U * blockDim.x) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = base + u * blockDim.x;
                if (e < total)
                    v[u] = __ldg(reinterpret_cast<const float4*>(in + size_t(e / P) * n + l0 + 2 * (e % P)));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = base + u * blockDim.x;
                if (e < total)
                    put_packed<F>(sm, e / P, e % P, L, make_float2(v[u].x, v[u].y), make_float2(v[u].z, v[u].w));
            }
        }
        return;
    }
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int k = e / P, p = e % P;
        const int l = l0 + 2 * p;
        if (l >= n) continue;
        const float2* src = in + size_t(k) * n + l;
        const float2 A = src[0];
        const float2 B = l + 1 < n ? src[1] : make_float2(0.f, 0.f);
        put_packed<F>(sm, k, p, L, A, B);
    }
}

// Fine-grid point -> image sample coordinates. For fine row theta' (ct, st)
// and column radius e^rho = er, T_m^{-1}(er (ct, st)) in pixels is affine in
// er: (tc, tr) = er (uc, ur) + (vc_m, vr_m); the sector-disc test
// |er e^{i theta'} - (1 - aR)|^2 <= aR^2 is er (er - 2 (1 - aR) ct) + 1 - 2 aR <= 0.
struct FineRow {
    float uc, ur, c2;
};

__device__ __forceinline__ FineRow fine_row(const DevGeom& g, float cm, float sm, float ct, float st) {
    const float sc = 0.5f * g.N * g.inv_aR;
    return {sc * fmaf(cm, ct, -sm * st), sc * fmaf(sm, ct, cm * st), 2.f * g.one_m_aR * ct};
}

__device__ __forceinline__ bool fine_pos(const DevGeom& g, const FineRow& r, float vc, float vr, float er, float& tc,
                                         float& tr) {
    if (fmaf(er, er - r.c2, g.mask_k) > 0.f) return false;  // outside the sector disc D
    tc = fmaf(er, r.uc, vc);
    tr = fmaf(er, r.ur, vr);
    return true;
}

// Cubic spline of the prefiltered image at one fine-grid point. The taps come
// from a quad raster: element [a][b] holds Q at four consecutive b. For
// sector 0 (`transposed`) the fine-row arcs run down image columns, so the
// raster is the transposed one (element [c][r] = Q[r..r+3][c]) and a warp's
// 32 consecutive samples again walk along raster rows.
constexpr int kPitch2048 = 2048 + 2 * kApron;  // raster pitch of the N = 2048 plans (the bench size)
constexpr int kNTheta2048 = 3072;              // their angle count (the Qg^T row stride)

// SCALE = false leaves out the e^rho factor (constant along a column: the
// fused kernel applies it to the column's spectrum instead of every sample).
template <int PITCH = 0, bool SCALE = true>  // compile-time raster pitch (0: g.pitch): tap-row offsets as load immediates
__device__ __forceinline__ float gather_image(const DevGeom& g, const Tap* __restrict__ q4, const FineRow& r,
                                              float vc, float vr, float er, bool transposed = false) {
    const int pitch = PITCH ? PITCH : g.pitch;
    float tc, tr;
    if (!fine_pos(g, r, vc, vr, er, tc, tr)) return 0.f;
    const float ta = transposed ? tc : tr, tb = transposed ? tr : tc;  // raster-row and quad axes
    const float ka = floorf(ta), kb = floorf(tb);
    float2 w[4];  // (row-axis, quad-axis) weights
    bsw2(make_float2(ta - ka, tb - kb), w);
    const Tap* p = q4 + ((int(ka) - 1 + kApron) * pitch + (int(kb) - 1 + kApron));
    float acc = 0.f;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const float4 t = __ldg(p + a * pitch);
        acc = fmaf(w[a].x, fmaf(w[0].y, t.x, fmaf(w[1].y, t.y, fmaf(w[2].y, t.z, w[3].y * t.w))), acc);
    }
    return SCALE ? er * acc : acc;
}

// First FFT pass fused with the sample gather, for a real-pair transform of
// length N whose input occupies rows [0, N/2) placed at positions
// p = row + N/4 - ... i.e. [0, N/4) <- rows [N/4, N/2) and [3N/4, N) <- rows
// [0, N/4) (the zero-embedded period), zero elsewhere. Each thread gathers the
// R1 inputs of its first-pass butterflies into registers (the zero half is
// skipped at compile time), does the radix-R1 DFT and writes the pass output:
// no zero fill, no staging store, no first-pass shared read.
template <class F, class Gather>
__device__ __forceinline__ void first_pass_gathered(float2* sm, int tid, Gather&& gather) {
    constexpr int N = F::kN, R1 = F::kR1, B1 = N / R1, T = F::kT;
    static_assert(R1 % 4 == 0, "first radix must split the zero half");
    constexpr int NB1 = (B1 + T - 1) / T;
#pragma unroll
    for (int i = 0; i < NB1; ++i) {
        const int bb = tid + i * T;
        if (bb < B1) {
            float2 v[R1];
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                // gathered rows are bb + B1 j, j = 0 .. R1/2 - 1
                if (r < R1 / 4) {
                    v[r] = gather(bb + B1 * r + N / 4, r + R1 / 4);  // p in [0, N/4)
                } else if (r >= 3 * R1 / 4) {
                    v[r] = gather(bb + B1 * r - 3 * N / 4, r - 3 * R1 / 4);  // p in [3N/4, N)
                } else {
                    v[r] = make_float2(0.f, 0.f);
                }
            }
            Dft<R1, false>::run(v);
            if constexpr (F::kPadWalk1) {  // the R1 outputs stay inside one padding block
                float2* w = sm + F::idx(bb * R1);
#pragma unroll
                for (int r = 0; r < R1; ++r) w[r] = v[Dft<R1, false>::slot(r)];
            } else {
#pragma unroll
                for (int r = 0; r < R1; ++r) sm[F::idx(bb * R1 + r)] = v[Dft<R1, false>::slot(r)];
            }
        }
    }
    __syncthreads();
}

template <class F>
constexpr bool kFusedFirstPass = F::kT > 0 && (F::kN % 4 == 0);

// Texture-filtered ablation of gather_image: the cubic
// spline as two hardware-bilinear lookups per axis, 4 filtered fetches per
// sample from the plain coefficient raster bound as a pitched 2-D texture
// (slice b at rows b * pitch). The texture unit quantises the interpolation
// weights (9-bit fixed point), so this is ~1e-3 accurate, not 1e-4.
__device__ __forceinline__ float gather_tex(const DevGeom& g, const FineRow& r, float vc, float vr, float er, int b) {
    float tc, tr;
    if (!fine_pos(g, r, vc, vr, er, tc, tr)) return 0.f;
    const float kc = floorf(tc), kr = floorf(tr);
    float wc[4], wr[4];
    bsw(tc - kc, wc);
    bsw(tr - kr, wr);
    const float gc0 = wc[0] + wc[1], gc1 = wc[2] + wc[3], gr0 = wr[0] + wr[1], gr1 = wr[2] + wr[3];
    const float x0 = kc + float(kApron - 1) + __fdividef(wc[1], gc0) + 0.5f;
    const float x1 = kc + float(kApron + 1) + __fdividef(wc[3], gc1) + 0.5f;
    const float yb = float(b * g.pitch) + kr + 0.5f;
    const float y0 = yb + float(kApron - 1) + __fdividef(wr[1], gr0);
    const float y1 = yb + float(kApron + 1) + __fdividef(wr[3], gr1);
    const float top = fmaf(gc0, tex2D<float>(g.qtex, x0, y0), gc1 * tex2D<float>(g.qtex, x1, y0));
    const float bot = fmaf(gc0, tex2D<float>(g.qtex, x0, y1), gc1 * tex2D<float>(g.qtex, x1, y1));
    return er * fmaf(gr0, top, gr1 * bot);
}

// Alg. 1 steps 3-6a: gather T_m f e^rho on the fine grid of two rho columns,
// zero-embed into the doubled fine period Lf, real theta FFT, keep |k| < nts.
// Each thread gathers two fine rows per iteration (64 independent tap loads
// in flight) to hide the L2 latency of the spline taps.
// BAND = N/8 (the plan's |k| < nts band when refine = 4) prunes the
// pass before the fused radix-2 store to the outputs that store reads.
template <class F, int TEX = 0, int PITCH = 0, int BAND = 0>
__global__ void LPR_LB(F) k_radon_theta_fwd(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd,
                                            const Tap* __restrict__ qf, const Tap* __restrict__ qft,
                                            float2* __restrict__ spec) {
    extern __shared__ float2 smem[];
    const Group<F> G;
    const int E = F::elems(fd);
    float2* sm = smem + G.g * E;
    const int m = blockIdx.y, b = blockIdx.z;
    const int l0b = 2 * F::kP * blockIdx.x, l0 = l0b + 2 * G.g;
    const int Lf = g.Lf, nf = g.nf;
    const bool tq = m == 0 && qft != nullptr;  // sector 0 reads the transposed raster
    const Tap* q = (tq ? qft : qf) + size_t(b) * g.pitch * g.pitch;
    const float cm = g.cosm[m], smm = g.sinm[m], vc = g.vcm[m], vr = g.vrm[m];
    const bool one = l0 < g.n_rho, two = l0 + 1 < g.n_rho;
    const float er0 = one ? __ldg(g.erho + l0) : 0.f;
    const float er1 = two ? __ldg(g.erho + l0 + 1) : 0.f;
    if constexpr (kFusedFirstPass<F>) {
        if (F::kN == Lf) {
            // the thread's rows are bb + B1 j: (cos, sin) of row bb from the table,
            // the others by an exact-to-fp32 rotation by j B1 dtheta_lp (no dependent load per row)
            constexpr bool kScaleAtStore = TEX == 0 && F::kLast2 && F::kP == 1;
            constexpr int B1 = F::kN / F::kR1;
            const bool rot = B1 <= F::kT && g.fine_b1 == B1;  // one butterfly per thread: bb = G.tid
            const float cb = __ldg(g.fine_cos + G.tid), sb = __ldg(g.fine_sin + G.tid);
            first_pass_gathered<F>(sm, G.tid, [&](int row, int j) {
                float ct, st;
                if (rot) {
                    const float2 w = g.fine_rot[j];
                    ct = fmaf(cb, w.x, -sb * w.y);
                    st = fmaf(sb, w.x, cb * w.y);
                } else {
                    ct = __ldg(g.fine_cos + row);
                    st = __ldg(g.fine_sin + row);
                }
                const FineRow fr = fine_row(g, cm, smm, ct, st);
                if constexpr (TEX == 1)
                    return make_float2(one ? gather_tex(g, fr, vc, vr, er0, b) : 0.f,
                                       two ? gather_tex(g, fr, vc, vr, er1, b) : 0.f);
                else
                    return make_float2(one ? gather_image<PITCH, !kScaleAtStore>(g, q, fr, vc, vr, er0, tq) : 0.f,
                                       two ? gather_image<PITCH, !kScaleAtStore>(g, q, fr, vc, vr, er1, tq) : 0.f);
            });
            if constexpr (BAND > 0)
                F::template run_tail_band<false, BAND>(sm, fd, G.tid);
            else
                F::template run_tail<false>(sm, fd, G.tid);
            float2* out = spec + (size_t(b) * g.M + m) * size_t(g.nts + 1) * g.n_rho;
            if constexpr (F::kLast2)
                store_half_spectra_r2<F>(Slots{smem, E}, Lf, g.nts, g.n_rho, l0b, out,
                                         kScaleAtStore ? er0 : 1.f, kScaleAtStore ? er1 : 1.f);
            else
                store_half_spectra<F>(Slots{smem, E}, Lf, g.nts, g.n_rho, l0b, out);
            return;
        }
    }
    for (int i = G.tid; i < Lf / 4; i += G.size) {  // the zero half [nf/2, Lf - nf/2)
        sm[F::idx(nf / 2 + i)] = make_float2(0.f, 0.f);
        sm[F::idx(nf / 2 + Lf / 4 + i)] = make_float2(0.f, 0.f);
    }
    const int half_rows = nf / 2;
    for (int i = G.tid; i < half_rows; i += G.size) {
        const int i2 = i + half_rows;
        const FineRow r1 = fine_row(g, cm, smm, __ldg(g.fine_cos + i), __ldg(g.fine_sin + i));
        const FineRow r2 = fine_row(g, cm, smm, __ldg(g.fine_cos + i2), __ldg(g.fine_sin + i2));
        float h0, h1, h2, h3;
        if constexpr (TEX == 1) {
            h0 = one ? gather_tex(g, r1, vc, vr, er0, b) : 0.f;
            h1 = two ? gather_tex(g, r1, vc, vr, er1, b) : 0.f;
            h2 = one ? gather_tex(g, r2, vc, vr, er0, b) : 0.f;
            h3 = two ? gather_tex(g, r2, vc, vr, er1, b) : 0.f;
        } else {
            h0 = one ? gather_image(g, q, r1, vc, vr, er0, tq) : 0.f;
            h1 = two ? gather_image(g, q, r1, vc, vr, er1, tq) : 0.f;
            h2 = one ? gather_image(g, q, r2, vc, vr, er0, tq) : 0.f;
            h3 = two ? gather_image(g, q, r2, vc, vr, er1, tq) : 0.f;
        }
        sm[F::idx(i - nf / 2 + Lf)] = make_float2(h0, h1);  // q = i - nf/2 < 0
        sm[F::idx(i2 - nf / 2)] = make_float2(h2, h3);      // q = i2 - nf/2 >= 0
    }
    __syncthreads();
    float2* res = F::template run<false>(sm, fft_scratch<F>(sm, fd), fd, G.tid);
    float2* out = spec + (size_t(b) * g.M + m) * size_t(g.nts + 1) * g.n_rho;
    store_half_spectra<F>(result_slots<F>(smem, E, res), Lf, g.nts, g.n_rho, l0b, out);
}

// rho pass: for every (item, k_theta) row, FFT along rho, multiply by the
// kernel spectrum row, inverse FFT. One transform per block. The row and the
// multiplier row are staged with cp.async (LDGSTS): the row is awaited before
// the forward FFT, the multiplier lands during it. The multiplier rows are
// shared by all items of the batch (grid.y), so they stay L2-resident.
template <class F>
__global__ void LPR_LB(F) k_rho_pass(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd,
                                     const float2* __restrict__ mult, float2* __restrict__ spec) {
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x, T = blockDim.x;
    const int k = blockIdx.x, item = blockIdx.y;
    const int n = g.n_rho;
    float2* ms = sm + F::elems(fd);
    float2* row = spec + (size_t(item) * (g.nts + 1) + k) * n;
    const float2* mrow = mult + size_t(k) * n;
    for (int j = tid; j < n; j += T) __pipeline_memcpy_async(sm + F::idx(j), row + j, sizeof(float2));
    __pipeline_commit();
    for (int j = tid; j < n; j += T) __pipeline_memcpy_async(ms + j, mrow + j, sizeof(float2));
    __pipeline_commit();
    __pipeline_wait_prior(1);
    __syncthreads();
    float2* a = F::template run<false>(sm, fft_scratch<F>(sm, fd), fd, tid);
    __pipeline_wait_prior(0);
    __syncthreads();
    for (int j = tid; j < n; j += T) a[F::idx(j)] = cmul(a[F::idx(j)], ms[j]);
    __syncthreads();
    a = F::template run<true>(a, a == sm ? fft_scratch<F>(sm, fd) : sm, fd, tid);
    for (int j = tid; j < n; j += T) row[j] = a[F::idx(j)];
}

// Padded rho pass for a non-smooth N_rho without a compile-time padded
// kernel (the reference plans at N = 256 / 512 / 1024: N_rho = 541, 1083,
// 2166): the circular convolution of period N_rho as the first N_rho outputs
// of a zero-padded linear one over the 7-smooth length fd.n >= 2 N_rho - 1
// (padded multipliers from rho_pad_multipliers), through the runtime Stockham
// or a compile-time plan of that length: two FFTs of the padded length per
// row instead of Bluestein's four.
// STAGE: the multiplier row is staged in shared memory (cp.async, landing
// during the forward FFT); else it is read from L2 in the multiply (long
// padded rows need all of shared memory for the transform, e.g. 13122).
template <class F, bool STAGE>
__global__ void LPR_LB(F) k_rho_pad_gen(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd,
                                        const float2* __restrict__ mult, float2* __restrict__ spec) {
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x, T = blockDim.x;
    const int k = blockIdx.x, item = blockIdx.y;
    const int n = g.n_rho, nb = F::kT > 0 ? F::kN : fd.n;
    float2* row = spec + (size_t(item) * (g.nts + 1) + k) * n;
    const float2* mrow = mult + size_t(k) * nb;
    float2* ms = sm + F::elems(fd);
    for (int j = tid; j < n; j += T) __pipeline_memcpy_async(sm + F::idx(j), row + j, sizeof(float2));
    __pipeline_commit();
    for (int j = n + tid; j < nb; j += T) sm[F::idx(j)] = make_float2(0.f, 0.f);
    if constexpr (STAGE) {
        for (int j = tid; j < nb; j += T) __pipeline_memcpy_async(ms + j, mrow + j, sizeof(float2));
        __pipeline_commit();
        __pipeline_wait_prior(1);
    } else {
        __pipeline_wait_prior(0);
    }
    __syncthreads();
    float2* a = F::template run<false>(sm, fft_scratch<F>(sm, fd), fd, tid);
    if constexpr (STAGE) __pipeline_wait_prior(0);
    __syncthreads();
    for (int j = tid; j < nb; j += T) a[F::idx(j)] = cmul(a[F::idx(j)], STAGE ? ms[j] : __ldg(mrow + j));
    __syncthreads();
    a = F::template run<true>(a, a == sm ? fft_scratch<F>(sm, fd) : sm, fd, tid);
    for (int j = tid; j < n; j += T) row[j] = a[F::idx(j)];
}

// ---- TMA bulk copies (cp.async.bulk, non-tensor) and mbarriers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// global -> shared, completion counted on bar (bytes % 16 == 0, both ends 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Streamed rho pass (the 7-smooth hot length): a block takes the rows of two
// items at one k_theta. Both rows and their shared multiplier row are
// requested at once by TMA bulk copy into shared memory, so the second row
// lands while the first is transformed; the forward last / inverse first
// butterflies are fused around the multiply and the inverse's last pass
// stores straight from registers to the row in HBM. (Straight-line on
// purpose: in a persistent row loop ptxas keeps every pass's loop-invariant
// state live and spills.)
template <class F>
__global__ void __launch_bounds__(F::kT, 2) k_rho_stream(const __grid_constant__ DevGeom g, const float4* __restrict__ twf,
                                                         const float4* __restrict__ twi, const float2* __restrict__ mult,
                                                         float2* __restrict__ spec, int items) {
    extern __shared__ __align__(16) float2 sm[];
    __shared__ __align__(8) uint64_t bars[2];
    constexpr int E = F::kElems;
    const int tid = threadIdx.x;
    const int n = g.n_rho, ks = g.nts + 1;
    const int pairs = (items + 1) / 2;
    const int k = blockIdx.x / pairs, i0 = 2 * (blockIdx.x % pairs);
    const bool two = i0 + 1 < items;
    float2* ms = sm + 2 * E;
    const uint32_t row_bytes = uint32_t(n) * sizeof(float2);
    float2* row0 = spec + (size_t(i0) * ks + k) * n;
    float2* row1 = row0 + size_t(ks) * n;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&bars[0], 2 * row_bytes);
        bulk_g2s(ms, mult + size_t(k) * n, row_bytes, &bars[0]);
        bulk_g2s(sm, row0, row_bytes, &bars[0]);
        if (two) {
            mbar_expect_tx(&bars[1], row_bytes);
            bulk_g2s(sm + E, row1, row_bytes, &bars[1]);
        }
    }
    __syncthreads();
    mbar_wait(&bars[0], 0);
    F::convolve(sm, twf, twi, ms, row0, tid);
    if (two) {
        mbar_wait(&bars[1], 0);
        F::convolve(sm + E, twf, twi, ms, row1, tid);
    }
}

// Default-plan rho pass (N_rho not 7-smooth, e.g. 4333 = 7 * 619): the
// circular convolution y = IDFT_n(M DFT_n(x)) equals the first n outputs of a
// linear convolution with the n-periodised kernel, done as one zero-padded
// transform pair of the 7-smooth length F::kN >= 2n - 1 with the padded
// multiplier DFT_nb(periodised IDFT_n(M)) / nb (built once per plan on the
// GPU in fp64, rho_pad_multipliers). One row per block, the multiplier read
// from L2 inside the fused middle butterfly; replaces Bluestein (15x slower).
template <class F>
__global__ void __launch_bounds__(F::kT, F::kT > 512 ? 1 : 2) k_rho_pad(const __grid_constant__ DevGeom g,
                                                      const float2* __restrict__ mult_pad, float2* __restrict__ spec) {
    extern __shared__ __align__(16) float2 sm[];
    const int k = blockIdx.x, item = blockIdx.y, n = g.n_rho, tid = threadIdx.x;
    float2* row = spec + (size_t(item) * (g.nts + 1) + k) * n;
    for (int j = tid; j < n; j += F::kT) sm[j] = row[j];  // [n, kN) is zero: the first pass does not read it
    __syncthreads();
    F::convolve(sm, nullptr, nullptr, mult_pad + size_t(k) * F::kN, row, tid, n);
}

size_t rho_direct_length() { return RhoPad8748::kN; }

// padded length for a non-smooth n_rho: 8748 for the N = 2048 default plan
// (4333), 17496 for N = 4096 (8666); 0: none (Bluestein)
size_t rho_pad_length(int n_rho) {
    if (2 * n_rho - 1 <= RhoPad8748::kN && n_rho > 4096) return RhoPad8748::kN;
    if (2 * n_rho - 1 <= RhoPad17496::kN && n_rho > 8192 && n_rho != RhoPad8748::kN) return RhoPad17496::kN;  // 8748: direct
    return 0;
}

void launch_rho_pad(int nb, dim3 grid, cudaStream_t st, const DevGeom& g, const float2* mult_pad, float2* spec) {
    if (nb == RhoPad17496::kN)
        k_rho_pad<RhoPad17496><<<grid, RhoPad17496::kT, sizeof(float2) * RhoPad17496::kElems, st>>>(g, mult_pad, spec);
    else
        k_rho_pad<RhoPad8748><<<grid, RhoPad8748::kT, sizeof(float2) * RhoPad8748::kElems, st>>>(g, mult_pad, spec);
}

cudaError_t prepare_rho_pad() {
    cudaError_t e = cudaFuncSetAttribute((const void*)k_rho_pad<RhoPad8748>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sizeof(float2) * RhoPad8748::kElems));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute((const void*)k_rho_pad<RhoPad17496>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sizeof(float2) * RhoPad17496::kElems));
}

// Hermitian theta inverse: two real columns per complex transform of length
// 2 nts; rows [j0, j0 + win) of the periodic result are kept.
// (A variant with N_rho = 4374 and nts = 1024 at compile time measured slower:
// 0.780 -> 0.943 ms per 16 slices.)
template <class F>
__global__ void LPR_LB(F) k_theta_inv(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd,
                                      const float2* __restrict__ spec, float* __restrict__ lp) {
    extern __shared__ float2 smem[];
    constexpr int P = F::kP;
    const Group<F> G;
    const int E = F::elems(fd);
    const Slots sms{smem, E};
    const int m = blockIdx.y, b = blockIdx.z;
    const int l0b = 2 * P * blockIdx.x;
    const int nts = g.nts, L2 = 2 * nts, n = g.n_rho;
    const int lps = g.lps;
    const int win = g.win, j0 = g.j0;
    const size_t item = size_t(b) * g.M + m;
    if (threadIdx.x < P) sms(threadIdx.x)[F::idx(nts)] = make_float2(0.f, 0.f);  // zeroed band edge
    load_packed_hermitian<F>(sms, spec + item * size_t(nts + 1) * n, nts, L2, n, l0b);
    __syncthreads();
    float2* res = F::template run<true>(sms(G.g), fft_scratch<F>(sms(G.g), fd), fd, G.tid);
    const Slots rs = result_slots<F>(smem, E, res);
    float* out = lp + item * size_t(win) * lps;
    if constexpr (F::kT > 0) {
        // one column pair per thread, rows tid / P + j RS; the window rows
        // r < -j0 come from the top of the period (q + L2)
        constexpr int RS = F::kT;  // = blockDim.x / P
        const int p = threadIdx.x % P, l = l0b + 2 * p;
        if (l < n) {
            const float2* src = rs(p);
            float* dst = out + l;
            const bool pair = l + 1 < n && (reinterpret_cast<uintptr_t>(dst) & 7) == 0 && (lps % 2) == 0;
            const int wrap = -j0;  // rows [0, wrap) read slot j0 + r + L2
            for (int r = threadIdx.x / P; r < win; r += RS) {
                const int q = j0 + r + (r < wrap ? L2 : 0);
                const float2 z = src[F::idx(q)];
                float* d = dst + size_t(r) * lps;
                if (pair) {
                    *reinterpret_cast<float2*>(d) = z;
                } else {
                    d[0] = z.x;
                    if (l + 1 < n) d[1] = z.y;
                }
                if (l < 3) {  // periodic copy of columns 0..2 past the end: rho taps never wrap
                    d[n] = z.x;
                    if (l + 1 < 3) d[n + 1] = z.y;
                }
            }
        }
        return;
    }
    for (int e = threadIdx.x; e < g.win * P; e += blockDim.x) {
        const int r = e / P, p = e % P;
        const int l = l0b + 2 * p;
        if (l >= n) continue;
        const int q = g.j0 + r;  // in (-L2, L2): one conditional add instead of a modulo
        const float2 z = rs(p)[F::idx(q < 0 ? q + L2 : q)];
        float* dst = out + size_t(r) * g.lps + l;
        if (l + 1 < n && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
            *reinterpret_cast<float2*>(dst) = z;
        } else {
            dst[0] = z.x;
            if (l + 1 < n) dst[1] = z.y;
        }
        if (l < 3) {  // periodic copy of columns 0..2 past the end: rho taps never wrap
            dst[n] = z.x;
            if (l + 1 < 3) dst[n + 1] = z.y;
        }
    }
}

// ------------------------------------------------------------- R#
// Qg is stored s-major (Qg^T[b][s][theta], written by k_prefilter_sino_iir):
// the 32 lanes of a warp take 32 consecutive lattice rows at nearly the same
// s, so each tap load is one or two cache lines instead of 32.
// LD > 0: the row stride (n_theta) at compile time, so the four tap rows are
// load immediates off one address (the N = 2048 bench plan: 3072)
template <int LD = 0>
__device__ __forceinline__ float gather_sino(const float* __restrict__ row, int N, float t, int ld_rt) {
    const int ld = LD ? LD : ld_rt;
    const float kf = floorf(t);
    float w[4];
    bsw(t - kf, w);
    const int k0 = int(kf) - 1;
    float acc = 0.f;
    if (k0 >= 0 && k0 + 3 < N) {  // all four taps on the detector (the common case): no per-tap tests
        const float* p = row + size_t(k0) * ld;
#pragma unroll
        for (int a = 0; a < 4; ++a) acc = fmaf(w[a], __ldg(p + a * ld), acc);
        return acc;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int idx = k0 + a;
        if (idx >= 0 && idx < N) acc = fmaf(w[a], __ldg(row + size_t(idx) * ld), acc);
    }
    return acc;
}

// g(S_m^{-1}) on Omega_p (Alg. 2 step 3): theta' rows are polar rows, so each
// sample is a 1-D spline along s (zero outside the detector), then the real
// theta FFT of the zero-embedded doubled period.
template <class F, int LD = 0>
__global__ void LPR_LB(F) k_bp_theta_fwd(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd,
                                         const float* __restrict__ qg, float2* __restrict__ spec) {
    extern __shared__ float2 smem[];
    const Group<F> G;
    const int E = F::elems(fd);
    float2* sm = smem + G.g * E;
    const int m = blockIdx.y, b = blockIdx.z;
    const int l0b = 2 * F::kP * blockIdx.x, l0 = l0b + 2 * G.g;
    const int nts = g.nts, L2 = g.L2, N = g.N;
    const bool one = l0 < g.n_rho, two = l0 + 1 < g.n_rho;
    const float er0 = one ? __ldg(g.erho + l0) : 0.f;
    const float er1 = two ? __ldg(g.erho + l0 + 1) : 0.f;
    const float halfN = 0.5f * N;
    if constexpr (kFusedFirstPass<F>) {
        if (F::kN == L2) {
            first_pass_gathered<F>(sm, G.tid, [&](int jj, int) {
                const int j = jj - nts / 2;
                int i = m * nts + j;
                const bool flip = i < 0;
                if (flip) i += g.n_theta;
                const float* row = qg + size_t(b) * N * g.n_theta + i;
                const float cth = __ldg(g.coarse_cos + jj) * g.one_m_aR;
                const float sg = flip ? -halfN : halfN;
                return make_float2(one ? gather_sino<LD>(row, N, fmaf((er0 - cth) * g.inv_aR, sg, halfN), g.n_theta) : 0.f,
                                   two ? gather_sino<LD>(row, N, fmaf((er1 - cth) * g.inv_aR, sg, halfN), g.n_theta) : 0.f);
            });
            F::template run_tail<false>(sm, fd, G.tid);
            float2* out = spec + (size_t(b) * g.M + m) * size_t(nts + 1) * g.n_rho;
            store_half_spectra<F>(Slots{smem, E}, L2, nts, g.n_rho, l0b, out);
            return;
        }
    }
    for (int i = G.tid; i < nts; i += G.size) sm[F::idx(nts / 2 + i)] = make_float2(0.f, 0.f);
    // two lattice rows per iteration (jj and jj + nts/2) for more loads in flight
    for (int jh = G.tid; jh < nts / 2; jh += G.size) {
        float v[2][2];
        int slot[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int jj = jh + h * (nts / 2);
            const int j = jj - nts / 2;
            int i = m * nts + j;
            const bool flip = i < 0;
            if (flip) i += g.n_theta;
            const float* row = qg + size_t(b) * N * g.n_theta + i;
            const float cth = __ldg(g.coarse_cos + jj) * g.one_m_aR;
            const float sg = flip ? -halfN : halfN;
            // t = (s_raster + 1/2) N with s_raster = (e^rho - (1-aR) cos) / (2 aR)
            v[h][0] = one ? gather_sino(row, N, fmaf((er0 - cth) * g.inv_aR, sg, halfN), g.n_theta) : 0.f;
            v[h][1] = two ? gather_sino(row, N, fmaf((er1 - cth) * g.inv_aR, sg, halfN), g.n_theta) : 0.f;
            slot[h] = j < 0 ? j + L2 : j;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) sm[F::idx(slot[h])] = make_float2(v[h][0], v[h][1]);
    }
    __syncthreads();
    float2* res = F::template run<false>(sm, fft_scratch<F>(sm, fd), fd, G.tid);
    float2* out = spec + (size_t(b) * g.M + m) * size_t(nts + 1) * g.n_rho;
    store_half_spectra<F>(result_slots<F>(smem, E, res), L2, nts, g.n_rho, l0b, out);
}

// R^T stage 2: real theta FFT of the lattice rows [-nts/2, nts/2) held in
// the window buffer (the transpose of the forward theta inverse + crop).
template <class F>
__global__ void LPR_LB(F) k_theta_fwd_T(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd,
                                        const float* __restrict__ lp, float2* __restrict__ spec) {
    extern __shared__ float2 smem[];
    constexpr int P = F::kP;
    const Group<F> G;
    const int E = F::elems(fd);
    const int m = blockIdx.y, b = blockIdx.z;
    const int l0b = 2 * P * blockIdx.x;
    const int nts = g.nts, L2 = g.L2, n = g.n_rho;
    {
        float2* sm = smem + G.g * E;
        for (int i = G.tid; i < nts; i += G.size) sm[F::idx(nts / 2 + i)] = make_float2(0.f, 0.f);
    }
    const float* in = lp + (size_t(b) * g.M + m) * size_t(g.win) * g.lps;
    for (int e = threadIdx.x; e < nts * P; e += blockDim.x) {
        const int jj = e / P, p = e % P;
        const int l = l0b + 2 * p;
        const int j = jj - nts / 2;
        const float* row = in + size_t(j - g.j0) * g.lps;
        const float a = l < n ? row[l] : 0.f, c = l + 1 < n ? row[l + 1] : 0.f;
        smem[p * E + F::idx(j < 0 ? j + L2 : j)] = make_float2(a, c);
    }
    __syncthreads();
    float2* sm = smem + G.g * E;
    float2* res = F::template run<false>(sm, fft_scratch<F>(sm, fd), fd, G.tid);
    float2* out = spec + (size_t(b) * g.M + m) * size_t(nts + 1) * n;
    store_half_spectra<F>(result_slots<F>(smem, E, res), L2, nts, n, l0b, out);
}

// lp_convolve stage 1: theta FFT of a real doubled-grid
// raster (2 nts rows in natural periodic order, n_rho columns, row stride
// n_rho), two columns per complex transform, half spectra k in [0, nts] out.
template <class F>
__global__ void LPR_LB(F) k_lpc_theta_fwd(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd,
                                          const float* __restrict__ data, float2* __restrict__ spec) {
    extern __shared__ float2 smem[];
    constexpr int P = F::kP;
    const Group<F> G;
    const int E = F::elems(fd);
    const int b = blockIdx.z;
    const int l0b = 2 * P * blockIdx.x;
    const int nts = g.nts, L2 = g.L2, n = g.n_rho;
    const float* in = data + size_t(b) * L2 * n;
    for (int e = threadIdx.x; e < L2 * P; e += blockDim.x) {
        const int r = e / P, p = e % P;
        const int l = l0b + 2 * p;
        const float* row = in + size_t(r) * n;
        smem[p * E + F::idx(r)] = make_float2(l < n ? row[l] : 0.f, l + 1 < n ? row[l + 1] : 0.f);
    }
    __syncthreads();
    float2* sm = smem + G.g * E;
    float2* res = F::template run<false>(sm, fft_scratch<F>(sm, fd), fd, G.tid);
    store_half_spectra<F>(result_slots<F>(smem, E, res), L2, nts, n, l0b, spec + size_t(b) * (nts + 1) * n);
}

// R^T stage 4: Hermitian inverse over the doubled fine period (zero beyond
// |k| < nts) and the transposed fine-grid gather G_m^T, scattering the spline
// taps into the apron-extended coefficient image.
template <class F>
__global__ void LPR_LB(F) k_theta_inv_fine_T(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd,
                                             const float2* __restrict__ spec, float* __restrict__ qbar) {
    extern __shared__ float2 smem[];
    constexpr int P = F::kP;
    const Group<F> G;
    const int E = F::elems(fd);
    const Slots sms{smem, E};
    const int m = blockIdx.y, b = blockIdx.z;
    const int l0b = 2 * P * blockIdx.x, l0 = l0b + 2 * G.g;
    const int nts = g.nts, Lf = g.Lf, n = g.n_rho, nf = g.nf;
    const size_t item = size_t(b) * g.M + m;
    for (int k = nts + G.tid; k <= Lf - nts; k += G.size) sms(G.g)[F::idx(k)] = make_float2(0.f, 0.f);
    load_packed_hermitian<F>(sms, spec + item * size_t(nts + 1) * n, nts, Lf, n, l0b);
    __syncthreads();
    const float2* res = F::template run<true>(sms(G.g), fft_scratch<F>(sms(G.g), fd), fd, G.tid);
    float* q = qbar + size_t(b) * g.pitch * g.pitch;
    const float cm = g.cosm[m], smm = g.sinm[m], vc = g.vcm[m], vr = g.vrm[m];
    for (int i = G.tid; i < nf; i += G.size) {
        const int qq = i - nf / 2;
        const float2 z = res[F::idx(qq < 0 ? qq + Lf : qq)];
        const FineRow rw = fine_row(g, cm, smm, __ldg(g.fine_cos + i), __ldg(g.fine_sin + i));
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            if (l0 + c >= n) break;
            const float er = __ldg(g.erho + l0 + c);
            float tc, tr;
            if (!fine_pos(g, rw, vc, vr, er, tc, tr)) continue;
            const float kc = floorf(tc), kr = floorf(tr);
            float wc[4], wr[4];
            bsw(tc - kc, wc);
            bsw(tr - kr, wr);
            const float v = er * (c == 0 ? z.x : z.y);
            float* p = q + (int(kr) - 1 + kApron) * g.pitch + (int(kc) - 1 + kApron);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int e = 0; e < 4; ++e) atomicAdd(p + a * g.pitch + e, v * wr[a] * wc[e]);
        }
    }
}

// FBP filter along s (the caller of R# in fbp):
// two sinogram rows per complex transform of length 2N (zero padded, so the
// circular convolution is the linear one on [0, N)), times the real even
// transfer H (already divided by 2N); both packed rows see the same real H.
template <class F>
__global__ void LPR_LB(F) k_sino_filter(const __grid_constant__ DevGeom g, const __grid_constant__ FftDesc fd,
                                        const float* __restrict__ H, const float* __restrict__ in,
                                        float* __restrict__ out, int rows_total) {
    extern __shared__ float2 smem[];
    const Group<F> G;
    const int E = F::elems(fd);
    float2* sm = smem + G.g * E;
    const int r0 = 2 * (blockIdx.x * F::kP + G.g), N = g.N, L = 2 * N;
    const bool has0 = r0 < rows_total, has1 = r0 + 1 < rows_total;
    for (int j = G.tid; j < L; j += G.size) {
        float a = 0.f, c = 0.f;
        if (j < N) {
            if (has0) a = __ldg(in + size_t(r0) * N + j);
            if (has1) c = __ldg(in + size_t(r0 + 1) * N + j);
        }
        sm[F::idx(j)] = make_float2(a, c);
    }
    __syncthreads();
    float2* a = F::template run<false>(sm, fft_scratch<F>(sm, fd), fd, G.tid);
    for (int j = G.tid; j < L; j += G.size) a[F::idx(j)] = cscale(a[F::idx(j)], __ldg(H + j));
    __syncthreads();
    a = F::template run<true>(a, a == sm ? fft_scratch<F>(sm, fd) : sm, fd, G.tid);
    for (int j = G.tid; j < N; j += G.size) {
        const float2 v = a[F::idx(j)];
        if (has0) out[size_t(r0) * N + j] = v.x;
        if (has1) out[size_t(r0 + 1) * N + j] = v.y;
    }
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
    const float invN = 1.f / float(N);
    const float xp = float(dxr) * invN, yp = float(dyr) * invN;
    float acc = 0.f;
    for (int m = 0; m < g.M; ++m) {
        const float cm = g.cosm[m], smm = g.sinm[m];
        const float yx = fmaf(g.aR, fmaf(cm, xp, smm * yp), g.one_m_aR);
        const float yy = g.aR * fmaf(-smm, xp, cm * yp);
        const float th = atanf(__fdividef(yy, yx));  // yx >= 1 - 2 aR > 0 inside the unit disc
        const float rho = 0.5f * logf(fmaf(yx, yx, yy * yy));
        const float tt = th * g.inv_dtheta_p;
        const float tr = (rho - g.log_ar) * g.inv_drho;
        const float kt = floorf(tt), kr = floorf(tr);
        float wt[4], wr[4];
        {
            float2 w2[4];
            bsw2(make_float2(tt - kt, tr - kr), w2);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                wt[q] = w2[q].x;
                wr[q] = w2[q].y;
            }
        }
        const float* base = lp + (size_t(b) * g.M + m) * size_t(g.win) * g.lps + (int(kt) - 1 - g.j0) * g.lps;
        const int c0 = int(kr) - 1;
        float sacc = 0.f;
        if (g.lptex) {  // four tld4 gathers (2 x 2 texels each, exact fp32)
            const float x0 = float(c0 + 1), x1 = x0 + 2.f;
            const float y0 = float((b * g.M + m) * g.win + int(kt) - 1 - g.j0) + 1.f, y1 = y0 + 2.f;
            const float4 a = tex2Dgather<float4>(g.lptex, x0, y0, 0), e = tex2Dgather<float4>(g.lptex, x1, y0, 0);
            const float4 d = tex2Dgather<float4>(g.lptex, x0, y1, 0), f = tex2Dgather<float4>(g.lptex, x1, y1, 0);
            const float r0 = fmaf(wr[0], a.w, fmaf(wr[1], a.z, fmaf(wr[2], e.w, wr[3] * e.z)));
            const float r1 = fmaf(wr[0], a.x, fmaf(wr[1], a.y, fmaf(wr[2], e.x, wr[3] * e.y)));
            const float r2 = fmaf(wr[0], d.w, fmaf(wr[1], d.z, fmaf(wr[2], f.w, wr[3] * f.z)));
            const float r3 = fmaf(wr[0], d.x, fmaf(wr[1], d.y, fmaf(wr[2], f.x, wr[3] * f.y)));
            acc += fmaf(wt[0], r0, fmaf(wt[1], r1, fmaf(wt[2], r2, wt[3] * r3)));
            continue;
        }
        if (c0 >= 0 && c0 + 3 < n + 3) {  // columns n..n+2 repeat 0..2 (k_theta_inv), so no wrap inside the disc
            const float* row = base + c0;
#pragma unroll
            for (int a = 0; a < 4; ++a, row += g.lps)
                sacc = fmaf(wt[a], fmaf(wr[0], __ldg(row), fmaf(wr[1], __ldg(row + 1), fmaf(wr[2], __ldg(row + 2), wr[3] * __ldg(row + 3)))), sacc);
        } else {
            int cidx[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int idx = c0 + q;
                cidx[q] = idx < 0 ? idx + n : (idx >= n ? idx - n : idx);
            }
            const float* row = base;
#pragma unroll
            for (int a = 0; a < 4; ++a, row += g.lps) {
                const float v = fmaf(wr[0], __ldg(row + cidx[0]),
                                     fmaf(wr[1], __ldg(row + cidx[1]), fmaf(wr[2], __ldg(row + cidx[2]), wr[3] * __ldg(row + cidx[3]))));
                sacc = fmaf(wt[a], v, sacc);
            }
        }
        acc += sacc;
    }
    *out = 2.f * acc;
}

// S_m resampling to the sinogram (Alg. 1 step 7). Theta residuals land on
// lattice rows (sector centres are polar rows), so each sinogram row needs
// one coefficient row and a 1-D periodic spline along rho; the theta-axis
// spline weights (1/6, 2/3, 1/6) cancel the theta part of 1/Bhat, which the
// multiplier therefore omits. SB slices per block: the SB lattice rows are
// staged together and each sinogram bin's rho coordinate (logf) and spline
// weights are computed once for all of them.
template <int SB>
__global__ void __launch_bounds__(256) k_radon_out_b(DevGeom g, const float* __restrict__ lp, float* __restrict__ sino,
                                                     int nb) {
    extern __shared__ float srow[];
    const int i = blockIdx.x, b0 = blockIdx.y * SB;
    const int nts = g.nts, n = g.n_rho, N = g.N, lps = g.lps;
    const int k = (2 * i + nts) / (2 * nts);
    const int m = k % g.M;
    const bool flip = ((k - m) / g.M) & 1;
    const int j = i - k * nts;
    const int ns = min(SB, nb - b0);
    for (int s = 0; s < ns; ++s) {
        const float* src = lp + ((size_t(b0 + s) * g.M + m) * g.win + (j - g.j0)) * lps;
        for (int l = threadIdx.x; l < lps / 4; l += 256)
            reinterpret_cast<float4*>(srow + s * lps)[l] = __ldg(reinterpret_cast<const float4*>(src) + l);
    }
    __syncthreads();
    const float cth = __ldg(g.coarse_cos + j + nts / 2) * g.one_m_aR;
    const float sgn = flip ? -1.f : 1.f;
    const float invN = 1.f / float(N);
    float* out = sino + (size_t(b0) * g.n_theta + i) * N;
    const size_t slice = size_t(g.n_theta) * N;
    for (int c = threadIdx.x; c < N; c += 256) {
        const float sp = sgn * float(2 * c - N) * invN;  // (x / N exactly for power-of-two N)
        const float rho = logf(fmaf(g.aR, sp, cth));
        const float t = (rho - g.log_ar) * g.inv_drho;
        const float kf = floorf(t);
        float w[4];
        bsw(t - kf, w);
        // t in [0, n] so k0 in [-1, n - 1]: only k0 = -1 wraps, and taps past
        // n - 1 read the row's periodic copy of columns 0..2 (k_theta_inv)
        int k0 = int(kf) - 1;
        k0 = k0 < 0 ? k0 + n : k0;
#pragma unroll
        for (int s = 0; s < SB; ++s) {
            if (s < ns) {
                const float* row = srow + s * lps + k0;
                float acc = 0.f;
#pragma unroll
                for (int a = 0; a < 4; ++a) acc = fmaf(w[a], row[a], acc);
                out[s * slice + c] = acc * g.out_scale;
            }
        }
    }
}

// ------------------------------------------------------------- host launchers
// R output resampling: SB = kOutSlices slices per block (k_radon_out_b,
// 0.434 -> 0.373 ms / 16 slices against one slice per block).
// (The same for k_bp_out, SB slices per thread sharing the atan/log
// coordinates, measured 1.107 -> 1.104: that kernel is bound by its tld4 gathers.)
cudaError_t prepare_out_kernels(int lps) {
    return cudaFuncSetAttribute(k_radon_out_b<kOutSlices>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kOutSlices * lps * int(sizeof(float)));
}
void launch_radon_out(int nb, cudaStream_t st, const DevGeom& g, const float* lp, float* sino) {
    k_radon_out_b<kOutSlices><<<dim3(g.n_theta, (nb + kOutSlices - 1) / kOutSlices), 256,
                                size_t(kOutSlices) * g.lps * sizeof(float), st>>>(g, lp, sino, nb);
}
void launch_bp_out(int nb, cudaStream_t st, const DevGeom& g, const float* lp, float* img) {
    // (the sector loop unrolled for M = 3, all 12 tld4 gathers in flight: 1.107 -> 1.106)
    // (taps of rows kt + 1, kt + 2 by direct loads beside two tld4 for rows kt - 1, kt: 1.105 -> 1.125)
    k_bp_out<<<dim3((g.N + 127) / 128, g.N, nb), 128, 0, st>>>(g, lp, img);
}
std::vector<float2> fft_pass_twiddles(int variant) {
    switch (variant) {
        case kFft2048: return Fft2048::pass_twiddles();
        case kFft4096: return Fft4096::pass_twiddles();
        case kFft4374: return Fft4374::pass_twiddles();
        case kFft8192: return Fft8192::pass_twiddles();
        case kFft16384: return Fft16384::pass_twiddles();
        default: return {};
    }
}

int fft_first_radix(int variant) {
    switch (variant) {
        case kFft2048: return Fft2048::kR1;
        case kFft4096: return Fft4096::kR1;
        case kFft4374: return Fft4374::kR1;
        case kFft8192: return Fft8192::kR1;
        case kFft16384: return Fft16384::kR1;
        default: return 0;
    }
}

FftLaunch fft_launch_config(const FftDesc& d) {
    const int gt = GenericFft::threads(d);
    FftLaunch L{kFftGeneric, gt, gt, 1, size_t(GenericFft::elems(d)) * sizeof(float2)};
    if (d.nb != 0) return L;
#define LPR_PICK(F, ID)                                                                                     \
    if (d.n == F::kN)                                                                                       \
        return FftLaunch{ID, F::kT * F::kP, F::kT, F::kP, size_t(F::elems(d)) * sizeof(float2)};
    LPR_PICK(Fft2048, kFft2048)
    LPR_PICK(Fft4096, kFft4096)
    LPR_PICK(Fft4374, kFft4374)
    LPR_PICK(Fft8192, kFft8192)
    LPR_PICK(Fft16384, kFft16384)
#undef LPR_PICK
    return L;
}

#define LPR_FFT_SWITCH(var, CALL)      \
    switch (var) {                     \
        case kFft2048: CALL(Fft2048); break;   \
        case kFft4096: CALL(Fft4096); break;   \
        case kFft4374: CALL(Fft4374); break;   \
        case kFft8192: CALL(Fft8192); break;   \
        case kFft16384: CALL(Fft16384); break; \
        default: CALL(GenericFft); break;      \
    }

// grid.x arrives as the number of column pairs; a block takes per_block of them
static dim3 theta_grid(dim3 grid, const FftLaunch& L) {
    grid.x = (grid.x + L.per_block - 1) / L.per_block;
    return grid;
}

static cudaError_t smem_attr(const void* fn, size_t bytes) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

cudaError_t prepare_fft_kernels(const FftLaunch& fine, const FftLaunch& rho, const FftLaunch& coarse,
                                size_t rho_mult_bytes) {
    cudaError_t e = cudaSuccess;
#define SET(K, L)                                                              \
    do {                                                                       \
        cudaError_t r = smem_attr((const void*)K, L);                          \
        if (r != cudaSuccess) e = r;                                           \
    } while (0)
    if (fine.variant == kFft8192) {
        SET(k_radon_theta_fwd<Fft8192Band>, fine.smem * fine.per_block);
        SET((k_radon_theta_fwd<Fft8192Band, 0, kPitch2048>), fine.smem * fine.per_block);
        SET((k_radon_theta_fwd<Fft8192Band, 0, kPitch2048, 1024>), fine.smem * fine.per_block);
    }
    if (fine.variant == kFft16384) SET((k_radon_theta_fwd<Fft16384Band, 0, 0, 2048>), fine.smem * fine.per_block);
#define FINE(F)                                                   \
    SET(k_radon_theta_fwd<F>, fine.smem * fine.per_block);         \
    SET((k_radon_theta_fwd<F, 1>), fine.smem * fine.per_block);    \
    SET(k_theta_inv_fine_T<F>, fine.smem * fine.per_block)
#define RHO(F) SET(k_rho_pass<F>, rho.smem + rho_mult_bytes)
    if (rho.variant == kFft4374) SET(k_rho_stream<Rho4374>, rho_stream_smem(kFft4374));
#define COARSE(F)                                          \
    SET(k_theta_inv<F>, coarse.smem * coarse.per_block);    \
    SET(k_bp_theta_fwd<F>, coarse.smem * coarse.per_block); \
    SET((k_bp_theta_fwd<F, kNTheta2048>), coarse.smem * coarse.per_block); \
    SET(k_theta_fwd_T<F>, coarse.smem * coarse.per_block);  \
    SET(k_lpc_theta_fwd<F>, coarse.smem * coarse.per_block)
    LPR_FFT_SWITCH(fine.variant, FINE)
    LPR_FFT_SWITCH(rho.variant, RHO)
    LPR_FFT_SWITCH(coarse.variant, COARSE)
#undef FINE
#undef RHO
#undef COARSE
#undef SET
    return e;
}

void launch_radon_theta_fwd(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                            const Tap* qf, const Tap* qft, float2* spec, int tex) {
    if (tex == 1) {
#define CALL(F) k_radon_theta_fwd<F, 1><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(g, fd, qf, qft, spec)
        LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
        return;
    }
#define CALL(F) k_radon_theta_fwd<F><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(g, fd, qf, qft, spec)
    if (L.variant == kFft8192) {
        if (g.pitch == kPitch2048 && g.Lf == 8 * g.nts && g.nts == 1024)
            k_radon_theta_fwd<Fft8192Band, 0, kPitch2048, 1024><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(
                g, fd, qf, qft, spec);
        else if (g.pitch == kPitch2048)
            k_radon_theta_fwd<Fft8192Band, 0, kPitch2048><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(
                g, fd, qf, qft, spec);
        else
            CALL(Fft8192Band);
        return;
    }
    if (L.variant == kFft16384 && g.Lf == 8 * g.nts && g.nts == 2048) {  // N = 4096: band-pruned, radix 2 fused into the store
        k_radon_theta_fwd<Fft16384Band, 0, 0, 2048><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(
            g, fd, qf, qft, spec);
        return;
    }
    LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
}

size_t rho_stream_smem(int variant) {
    return variant == kFft4374 ? size_t(3) * Rho4374::kElems * sizeof(float2) : 0;
}

std::vector<float4> rho_stream_inv_twiddles(int variant) {
    return variant == kFft4374 ? Rho4374::inv_twiddles() : std::vector<float4>{};
}

std::vector<float4> rho_stream_fwd_twiddles(int variant) {
    return variant == kFft4374 ? Rho4374::fwd_twiddles() : std::vector<float4>{};
}

void launch_rho_pass(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                     const float2* mult, float2* spec) {
    if (L.rho_stream && fd.twp_inv != nullptr && fd.twp_sfwd != nullptr) {
        const int items = int(grid.y);
        if (L.variant == kFft4374) {
            k_rho_stream<Rho4374><<<int(grid.x) * ((items + 1) / 2), Rho4374::kT, rho_stream_smem(kFft4374), st>>>(g, fd.twp_sfwd, fd.twp_inv,
                                                                                                mult, spec, items);
            return;
        }
    }
#define CALL(F) k_rho_pass<F><<<grid, L.tpt, L.smem + size_t(g.n_rho) * sizeof(float2), st>>>(g, fd, mult, spec)
    LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
}

void launch_rho_pad_gen(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                        const float2* mult_pad, float2* spec) {
    const size_t staged = L.smem + size_t(fd.n) * sizeof(float2);
    if (staged <= 227 * 1024) {
#define CALL(F) k_rho_pad_gen<F, true><<<grid, L.tpt, staged, st>>>(g, fd, mult_pad, spec)
        LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
    } else {
#define CALL(F) k_rho_pad_gen<F, false><<<grid, L.tpt, L.smem, st>>>(g, fd, mult_pad, spec)
        LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
    }
}

cudaError_t prepare_rho_pad_gen(const FftLaunch& L, int nb) {
    const size_t staged = L.smem + size_t(nb) * sizeof(float2);
    cudaError_t e = cudaSuccess;
#define SETG(F)                                                                                              \
    if (staged <= 227 * 1024)                                                                                \
        e = cudaFuncSetAttribute(k_rho_pad_gen<F, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(staged)); \
    else                                                                                                     \
        e = cudaFuncSetAttribute(k_rho_pad_gen<F, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.smem))
    LPR_FFT_SWITCH(L.variant, SETG)
#undef SETG
    return e;
}

void launch_theta_inv(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                      const float2* spec, float* lp) {
#define CALL(F) k_theta_inv<F><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(g, fd, spec, lp)
    LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
}

void launch_bp_theta_fwd(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                         const float* qg, float2* spec) {
    if (L.variant == kFft2048 && g.n_theta == kNTheta2048) {
        k_bp_theta_fwd<Fft2048, kNTheta2048><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(g, fd, qg, spec);
        return;
    }
#define CALL(F) k_bp_theta_fwd<F><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(g, fd, qg, spec)
    LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
}

void launch_lpc_theta_fwd(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                          const float* data, float2* spec) {
#define CALL(F) k_lpc_theta_fwd<F><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(g, fd, data, spec)
    LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
}

void launch_theta_fwd_T(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                        const float* lp, float2* spec) {
#define CALL(F) k_theta_fwd_T<F><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(g, fd, lp, spec)
    LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
}

cudaError_t prepare_filter_kernel(const FftLaunch& L) {
    cudaError_t e = cudaSuccess;
#define SETF(F)                                                                            \
    do {                                                                                   \
        cudaError_t r = smem_attr((const void*)k_sino_filter<F>, L.smem * L.per_block);    \
        if (r != cudaSuccess) e = r;                                                       \
    } while (0)
    LPR_FFT_SWITCH(L.variant, SETF)
#undef SETF
    return e;
}

void launch_sino_filter(const FftLaunch& L, int rows_total, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                        const float* H, const float* in, float* out) {
    const dim3 grid((((rows_total + 1) / 2) + L.per_block - 1) / L.per_block);
#define CALL(F) k_sino_filter<F><<<grid, L.threads, L.smem * L.per_block, st>>>(g, fd, H, in, out, rows_total)
    LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
}

void launch_theta_inv_fine_T(const FftLaunch& L, dim3 grid, cudaStream_t st, const DevGeom& g, const FftDesc& fd,
                             const float2* spec, float* qbar) {
#define CALL(F) k_theta_inv_fine_T<F><<<theta_grid(grid, L), L.threads, L.smem * L.per_block, st>>>(g, fd, spec, qbar)
    LPR_FFT_SWITCH(L.variant, CALL)
#undef CALL
}

}  // namespace lpr
