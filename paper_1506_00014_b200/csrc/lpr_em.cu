// Elementwise and reduction kernels of the EM reconstruction (SPEC.md:390-446,
// PAPER.md:595-630): f+ = f R#(g / max(Rf, eps)) / R#chi_C, device-resident.
// The operators themselves are the plan's R and R# (lpr_capi.cu, em_chunk);
// these kernels are the glue between them, one pass each over HBM.
#include <cuda_runtime.h>

#include <cstdint>

#include "lpr_em.cuh"

namespace lpr {

namespace {

// float max on non-negative values through the int ordering of their bits
__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
    atomicMax(reinterpret_cast<int*>(addr), __float_as_int(fmaxf(v, 0.f)));
}

template <class T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    T s = 0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : T(0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    return s;
}

}  // namespace

// 1 inside the unit disc (the same integer test as k_bp_out), 0 outside.
__global__ void k_disc_fill(int N, float* __restrict__ img) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y, b = blockIdx.z;
    if (c >= N) return;
    const int dx = 2 * c - N, dy = 2 * r - N;
    img[(size_t(b) * N + r) * N + c] = dx * dx + dy * dy <= N * N ? 1.f : 0.f;
}

__global__ void k_fill(float* __restrict__ x, size_t n, float v) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) x[i] = v;
}

// per-slice max (of max(x, 0)) and a flag for negative or non-finite entries
__global__ void k_slice_max(const float* __restrict__ x, size_t per, float* __restrict__ mx, int* __restrict__ bad) {
    const int b = blockIdx.y;
    const float* s = x + size_t(b) * per;
    float m = 0.f;
    bool neg = false;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < per; i += size_t(gridDim.x) * blockDim.x) {
        const float v = s[i];
        neg |= !(v >= 0.f) || !isfinite(v);
        m = fmaxf(m, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(mx + b, m);
    if (neg) atomicOr(bad, 1);
}

// q = g / Rf where Rf > eps (1e-6 max g of the slice), else 0;
// optionally the Poisson log-likelihood sum(g log Rf - Rf) over Rf > eps
// of this Rf, accumulated into ll[b * ll_stride].
__global__ void k_em_ratio(const float* __restrict__ g, float* __restrict__ rf_q, size_t per,
                           const float* __restrict__ gmax, double* __restrict__ ll, int ll_stride, int write_ratio) {
    __shared__ double sh[32];
    const int b = blockIdx.y;
    const float eps = 1e-6f * gmax[b];
    const float* gs = g + size_t(b) * per;
    float* rs = rf_q + size_t(b) * per;
    double acc = 0.0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < per; i += size_t(gridDim.x) * blockDim.x) {
        const float rf = rs[i], gv = gs[i];
        const bool ok = rf > eps;
        if (ll && ok) acc += double(gv) * log(double(rf)) - double(rf);
        if (write_ratio) rs[i] = ok ? gv / rf : 0.f;
    }
    if (ll) {
        const double s = block_sum(acc, sh);
        if (threadIdx.x == 0) atomicAdd(ll + size_t(b) * ll_stride, s);
    }
}

// f = max(0, f * bp * inv_sens) (inv_sens = 0 outside the unit disc); flags non-finite results
__global__ void k_em_update(float* __restrict__ f, const float* __restrict__ bp, const float* __restrict__ inv_sens,
                            size_t per, int* __restrict__ bad) {
    const int b = blockIdx.y;
    float* fs = f + size_t(b) * per;
    const float* bs = bp + size_t(b) * per;
    bool nf = false;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < per; i += size_t(gridDim.x) * blockDim.x) {
        const float v = fs[i] * bs[i] * inv_sens[i];
        nf |= !isfinite(v);
        fs[i] = fmaxf(v, 0.f);
    }
    if (nf) atomicOr(bad, 2);
}

// 1 / max(s, 1e-6 max s) inside the unit disc, 0 outside
__global__ void k_sens_invert(int N, const float* __restrict__ sens, const float* __restrict__ smax,
                              float* __restrict__ inv) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (c >= N) return;
    const int dx = 2 * c - N, dy = 2 * r - N;
    const size_t i = size_t(r) * N + c;
    inv[i] = dx * dx + dy * dy <= N * N ? 1.f / fmaxf(sens[i], 1e-6f * smax[0]) : 0.f;
}

// launchers
static unsigned grid_for(size_t per) {
    const size_t b = (per + 255) / 256;
    return unsigned(b < 1024 ? b : 1024);
}
void launch_disc_fill(int N, float* img, int batch, cudaStream_t st) {
    k_disc_fill<<<dim3((N + 255) / 256, N, batch), 256, 0, st>>>(N, img);
}
void launch_fill(float* x, size_t n, float v, cudaStream_t st) { k_fill<<<grid_for(n), 256, 0, st>>>(x, n, v); }
void launch_slice_max(const float* x, size_t per, int batch, float* mx, int* bad, cudaStream_t st) {
    cudaMemsetAsync(mx, 0, sizeof(float) * batch, st);
    k_slice_max<<<dim3(grid_for(per), batch), 256, 0, st>>>(x, per, mx, bad);
}
void launch_em_ratio(const float* g, float* rf_q, size_t per, int batch, const float* gmax, double* ll, int ll_stride,
                     bool write_ratio, cudaStream_t st) {
    k_em_ratio<<<dim3(grid_for(per), batch), 256, 0, st>>>(g, rf_q, per, gmax, ll, ll_stride, write_ratio ? 1 : 0);
}
void launch_em_update(float* f, const float* bp, const float* inv_sens, size_t per, int batch, int* bad,
                      cudaStream_t st) {
    k_em_update<<<dim3(grid_for(per), batch), 256, 0, st>>>(f, bp, inv_sens, per, bad);
}
void launch_sens_invert(int N, const float* sens, const float* smax, float* inv, cudaStream_t st) {
    k_sens_invert<<<dim3((N + 255) / 256, N), 256, 0, st>>>(N, sens, smax, inv);
}

}  // namespace lpr
