// Kernel spectra zeta / zeta# on the GPU (plan-time constants, fp64).
//
// Same quadrature as the host restatement (lpr_host.cpp, following
// kernel.cpp:293-429): for every rho frequency v, end-corrected trapezoid
// samples of cos(t)^alpha on [-beta, beta] (alpha = -1 - i y for zeta,
// i y for zeta#, y = 2 pi k_rho / ell), one power-of-two FFT, and the theta
// frequencies mu = -pi k / beta read from it with the (-1)^k phase of the
// interval shift. The host code runs one FFT per column on the CPU threads
// (~10 s per spectrum at N=2048); here the sample generation and the
// scatter into the (2 nts) x n_rho layout are kernels and the FFTs are
// batched double-precision cuFFT transforms, grouped by length.
#include <cufft.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "lpradon_gpu.h"

namespace lpr {

namespace {

constexpr double kPiD = 3.14159265358979323846;

// end-point correction deltas of the first/last seven nodes, / 120960
__constant__ double c_dc[7] = {-23681.0 / 120960, 55688.0 / 120960, -66109.0 / 120960, 57024.0 / 120960,
                               -31523.0 / 120960, 9976.0 / 120960,  -1375.0 / 120960};

__global__ void k_spec_samples(double2* __restrict__ s, const int* __restrict__ cols, int ncol, long n, int kind,
                               double beta, double ell, int n_rho) {
    const long j = blockIdx.x * long(blockDim.x) + threadIdx.x;
    const int c = blockIdx.y;
    if (j >= n || c >= ncol) return;
    const int v = cols[c];
    const long kr = v < (n_rho + 1) / 2 ? v : v - n_rho;  // signed rho frequency
    const double y = 2.0 * kPiD * double(kr) / ell;
    const double ar = kind == 0 ? -1.0 : 0.0, ai = kind == 0 ? -y : y;
    const double h = 2.0 * beta / double(n);
    double w = 1.0;
    if (j == 0) w += 2.0 * c_dc[0];  // both ends meet at node 0 on the circle
    else if (j < 7) w += c_dc[j];
    if (n - j < 7) w += c_dc[n - j];
    const double lc = log(cos(-beta + double(j) * h));
    const double mag = w * exp(ar * lc);
    double sn, cs;
    sincos(ai * lc, &sn, &cs);
    s[size_t(c) * n + j] = make_double2(mag * cs, mag * sn);
}

// out rows r = k mod 2 nts (FFT order), interleaved re/im, row-major over n_rho columns
__global__ void k_spec_scatter(double* __restrict__ out, const double2* __restrict__ s, const int* __restrict__ cols,
                               int ncol, long n, int nts, int n_rho, double beta, int special_col) {
    const int rows = 2 * nts;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= rows || c >= ncol) return;
    const int v = cols[c];
    const long kt = r < nts ? r : r - rows;
    double2 val;
    if (v == special_col) {  // zeta# at k_rho = 0 (alpha = 0): 2 sin(mu beta) / mu
        const double mu = -kPiD * double(kt) / beta;
        val = make_double2(kt == 0 ? 2.0 * beta : 2.0 * sin(mu * beta) / mu, 0.0);
    } else {
        const double h = 2.0 * beta / double(n);
        const double2 z = s[size_t(c) * n + ((kt % n) + n) % n];
        const double sg = (kt & 1) ? -h : h;
        val = make_double2(sg * z.x, sg * z.y);
    }
    double* o = out + 2 * (size_t(r) * n_rho + v);
    o[0] = val.x;
    o[1] = (n_rho % 2 == 0 && v == n_rho / 2) ? 0.0 : val.y;  // real rho-Nyquist column
}

struct CuErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CuErr(std::string(what) + ": " + cudaGetErrorString(e));
}
void ckf(cufftResult r, const char* what) {
    if (r != CUFFT_SUCCESS) throw CuErr(std::string(what) + ": cuFFT error " + std::to_string(int(r)));
}

}  // namespace

// Device spectrum: fills d_out (2 nts x n_rho complex, interleaved doubles) on `stream`.
void spectrum_device(const lpr_geometry& g, int kind, double* d_out, cudaStream_t stream) {
    const long nts = g.nts, cols = g.n_rho;
    const double beta = g.beta, ell = -g.log_ar;
    // FFT length per column (the same rule as the host restatement)
    std::map<long, std::vector<int>> groups;
    int special = -1;
    for (long v = 0; v < cols; ++v) {
        const long kr = v < (cols + 1) / 2 ? v : v - cols;
        if (kind == 1 && kr == 0) {
            special = int(v);
            continue;
        }
        const double y = 2.0 * kPiD * double(kr) / ell;
        const double rate = (kPiD * double(nts) / beta + std::fabs(y) * std::tan(beta)) * beta / kPiD;
        long n = 1;
        while (n < 16 * std::max<long>(32, long(std::ceil(rate)))) n <<= 1;
        groups[n].push_back(int(v));
    }
    const size_t budget = size_t(1) << 30;  // bytes of samples per batch
    double2* buf = nullptr;
    int* dcols = nullptr;
    size_t buf_bytes = 0;
    ck(cudaMalloc(&dcols, sizeof(int) * size_t(cols)), "cudaMalloc");
    try {
        if (special >= 0) {
            ck(cudaMemcpyAsync(dcols, &special, sizeof(int), cudaMemcpyHostToDevice, stream), "H2D");
            k_spec_scatter<<<dim3(unsigned((2 * nts + 255) / 256), 1), 256, 0, stream>>>(d_out, nullptr, dcols, 1, 1, int(nts),
                                                                                      int(cols), beta, special);
            ck(cudaGetLastError(), "spectrum scatter");
            ck(cudaStreamSynchronize(stream), "sync");
        }
        for (auto& [n, vs] : groups) {
            const long per = std::max<long>(1, long(budget / (size_t(n) * sizeof(double2))));
            for (size_t c0 = 0; c0 < vs.size(); c0 += per) {
                const int nc = int(std::min<size_t>(per, vs.size() - c0));
                const size_t need = size_t(nc) * n * sizeof(double2);
                if (need > buf_bytes) {
                    if (buf) cudaFree(buf);
                    buf = nullptr;
                    ck(cudaMalloc(&buf, need), "cudaMalloc");
                    buf_bytes = need;
                }
                ck(cudaMemcpyAsync(dcols, vs.data() + c0, sizeof(int) * nc, cudaMemcpyHostToDevice, stream), "H2D");
                k_spec_samples<<<dim3(unsigned((n + 255) / 256), nc), 256, 0, stream>>>(buf, dcols, nc, n, kind, beta,
                                                                                       ell, int(cols));
                ck(cudaGetLastError(), "spectrum samples");
                cufftHandle plan;
                int len = int(n);
                ckf(cufftPlanMany(&plan, 1, &len, nullptr, 1, len, nullptr, 1, len, CUFFT_Z2Z, nc), "cufftPlanMany");
                cufftResult fr = cufftSetStream(plan, stream);
                if (fr == CUFFT_SUCCESS)
                    fr = cufftExecZ2Z(plan, reinterpret_cast<cufftDoubleComplex*>(buf),
                                      reinterpret_cast<cufftDoubleComplex*>(buf), CUFFT_FORWARD);
                k_spec_scatter<<<dim3(unsigned((2 * nts + 255) / 256), nc), 256, 0, stream>>>(d_out, buf, dcols, nc, n,
                                                                                           int(nts), int(cols), beta, -1);
                const cudaError_t le = cudaGetLastError();
                const cudaError_t se = cudaStreamSynchronize(stream);
                cufftDestroy(plan);
                ckf(fr, "cufftExecZ2Z");
                ck(le, "spectrum scatter");
                ck(se, "sync");
            }
        }
    } catch (...) {
        if (buf) cudaFree(buf);
        cudaFree(dcols);
        throw;
    }
    if (buf) cudaFree(buf);
    cudaFree(dcols);
}

__global__ void k_pad_periodise(const double2* __restrict__ m, double2* __restrict__ mt, int n, int nb) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (t >= nb) return;
    const double2* src = m + size_t(r) * n;
    double2 v = make_double2(0.0, 0.0);
    if (t < n) v = src[t];
    else if (t > nb - n) v = src[t - nb + n];  // negative lags -(nb - t) of the n-periodic kernel
    const double sc = 1.0 / double(nb);
    mt[size_t(r) * nb + t] = make_double2(v.x * sc, v.y * sc);
}

__global__ void k_to_f32(const double2* __restrict__ a, float2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        b[i] = make_float2(float(a[i].x), float(a[i].y));
}

// Padded multipliers of the default-plan rho pass (k_rho_pad): for every row
// of the multiplier M (rows x n, fp64, host), DFT_nb of the n-periodised
// kernel IDFT_n(M) over lags -(n-1)..n-1, divided by nb; fp32 into d_out
// (rows x nb). Double-precision cuFFT (arbitrary n).
void rho_pad_multipliers(int device, int rows, int n, int nb, const double* mult, float2* d_out) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    double2 *dm = nullptr, *dt = nullptr;
    const size_t bm = sizeof(double2) * size_t(rows) * n, bt = sizeof(double2) * size_t(rows) * nb;
    ck(cudaMalloc(&dm, bm), "cudaMalloc");
    if (cudaMalloc(&dt, bt) != cudaSuccess) {
        cudaFree(dm);
        throw CuErr("cudaMalloc: padded multipliers");
    }
    cufftHandle p1 = 0, p2 = 0;
    try {
        ck(cudaMemcpy(dm, mult, bm, cudaMemcpyHostToDevice), "H2D");
        int ln = n, lb = nb;
        ckf(cufftPlanMany(&p1, 1, &ln, nullptr, 1, ln, nullptr, 1, ln, CUFFT_Z2Z, rows), "cufftPlanMany");
        ckf(cufftExecZ2Z(p1, reinterpret_cast<cufftDoubleComplex*>(dm), reinterpret_cast<cufftDoubleComplex*>(dm),
                         CUFFT_INVERSE),
            "cufftExecZ2Z");
        k_pad_periodise<<<dim3((nb + 255) / 256, rows), 256>>>(dm, dt, n, nb);
        ck(cudaGetLastError(), "periodise");
        ckf(cufftPlanMany(&p2, 1, &lb, nullptr, 1, lb, nullptr, 1, lb, CUFFT_Z2Z, rows), "cufftPlanMany");
        ckf(cufftExecZ2Z(p2, reinterpret_cast<cufftDoubleComplex*>(dt), reinterpret_cast<cufftDoubleComplex*>(dt),
                         CUFFT_FORWARD),
            "cufftExecZ2Z");
        k_to_f32<<<1024, 256>>>(dt, d_out, size_t(rows) * nb);
        ck(cudaGetLastError(), "to f32");
        ck(cudaDeviceSynchronize(), "sync");
    } catch (...) {
        if (p1) cufftDestroy(p1);
        if (p2) cufftDestroy(p2);
        cudaFree(dm);
        cudaFree(dt);
        throw;
    }
    cufftDestroy(p1);
    cufftDestroy(p2);
    cudaFree(dm);
    cudaFree(dt);
}

// Host-array form: computes on `device` and copies the (2 nts) x n_rho array back.
void spectrum_gpu(int device, const lpr_geometry& g, int kind, double* out) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    const size_t bytes = sizeof(double) * 2 * size_t(2 * g.nts) * size_t(g.n_rho);
    double* d = nullptr;
    cudaStream_t st = nullptr;
    ck(cudaMalloc(&d, bytes), "cudaMalloc");
    try {
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
        spectrum_device(g, kind, d, st);
        ck(cudaMemcpyAsync(out, d, bytes, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
    } catch (...) {
        if (st) cudaStreamDestroy(st);
        cudaFree(d);
        throw;
    }
    cudaStreamDestroy(st);
    cudaFree(d);
}

}  // namespace lpr
