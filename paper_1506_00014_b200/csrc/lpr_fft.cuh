// Block-cooperative shared-memory FFTs for the log-polar convolution legs.
//
// A transform of length n lives in shared memory as float2. Each pass of
// radix R runs Stockham autosort (Govindaraju et al. 2008 form): butterfly b
// reads x[b + r n/R], twiddles by W_{Ns R}^{(b mod Ns) r}, does an R-point
// DFT in registers and writes y[(b/Ns) Ns R + b mod Ns + r Ns], ping-ponging
// between two n-element shared buffers (one barrier per pass, R live values
// per thread, no register staging).
//
// Lengths must factor into {2,3,4,5,7,8}; other lengths (e.g. the default
// N_rho = 4333 = 7 * 619 at N = 2048) go through Bluestein over a 7-smooth
// length, built from the same passes. Twiddles come from a per-length fp32
// table computed in fp64 on the host.
#pragma once

#include <cuda_runtime.h>

namespace lpr {

constexpr int kMaxPasses = 24;

struct FftDesc {
    int n = 0;
    int npass = 0;
    int radix[kMaxPasses] = {};
    const float2* tw = nullptr;   // tw[j] = exp(-2 pi i j / n)
    const float2* twp = nullptr;  // per-pass twiddles of the compile-time plan (lpr_fft_ct.cuh)
    const float4* twp_sfwd = nullptr;  // streamed rho pass: forward per-pass twiddles of its radix order (tw4 form)
    const float4* twp_inv = nullptr;   // ... and of the reversed order, conjugated (its inverse)
    // Bluestein: when nb > 0 the transform of length n runs through length nb
    int nb = 0;
    int nbpass = 0;
    int bradix[kMaxPasses] = {};
    const float2* btw = nullptr;   // twiddles for nb
    const float2* chirp = nullptr; // c_j = exp(-i pi j^2 / n), j < n
    const float2* bhat = nullptr;  // FFT_nb of conj chirp kernel, times 1/nb
};

// Complex arithmetic on the sm_100 packed fp32x2 pipe (FADD2/FMUL2/FFMA2: one
// instruction per complex add, two per complex multiply; IEEE per lane).
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
// a * b = a.x (b.x, b.y) + a.y (-b.y, b.x); the swizzled operand first and
// the broadcast second, the order in which ptxas folds the swap / partial
// negation and the broadcast into operand modifiers instead of MOVs
#ifndef LPR_CMUL_SWZ_FIRST
#define LPR_CMUL_SWZ_FIRST 1
#endif
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
#if LPR_CMUL_SWZ_FIRST
    return __ffma2_rn(make_float2(-b.y, b.x), make_float2(a.y, a.y), __fmul2_rn(b, make_float2(a.x, a.x)));
#else
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x), __fmul2_rn(make_float2(a.x, a.x), b));
#endif
}
// a * conj(b) = a.x (b.x, -b.y) + a.y (b.y, b.x)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
#if LPR_CMUL_SWZ_FIRST
    return __ffma2_rn(make_float2(b.y, b.x), make_float2(a.y, a.y), __fmul2_rn(make_float2(b.x, -b.y), make_float2(a.x, a.x)));
#else
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(b.y, b.x), __fmul2_rn(make_float2(a.x, a.x), make_float2(b.x, -b.y)));
#endif
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {
    return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// R-point DFT in registers, sign -1 (forward) or +1 (INV). Output k is left
// in register slot(k) (identity here; composite radices permute).
template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<2, INV> {
    __host__ __device__ static constexpr int slot(int k) { return k; }
    __device__ __forceinline__ static void run(float2* v) {
        const float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};

template <bool INV>
struct Dft<4, INV> {
    __host__ __device__ static constexpr int slot(int k) { return k; }
    __device__ __forceinline__ static void run(float2* v) {
        const float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
        const float2 s13 = cadd(v[1], v[3]), d13 = mul_mi<INV>(csub(v[1], v[3]));
        v[0] = cadd(s02, s13);
        v[2] = csub(s02, s13);
        v[1] = cadd(d02, d13);
        v[3] = csub(d02, d13);
    }
};

template <bool INV>
struct Dft<8, INV> {
    __host__ __device__ static constexpr int slot(int k) { return k; }
    __device__ __forceinline__ static void run(float2* v) {
        constexpr float h = 0.70710678118654752f;
        float2 e[4] = {v[0], v[2], v[4], v[6]};
        float2 o[4] = {v[1], v[3], v[5], v[7]};
        Dft<4, INV>::run(e);
        Dft<4, INV>::run(o);
        // twiddles W8^k for k = 0..3; W8^1, W8^3 = h (1 -+ i) applied as
        // e +- h u with u = o (1 -+ i) folded into FFMA2s
        const float2 u1 = INV ? cadd(o[1], make_float2(-o[1].y, o[1].x)) : cadd(o[1], make_float2(o[1].y, -o[1].x));
        const float2 o2 = mul_mi<INV>(o[2]);
        const float2 u3 = INV ? csub(make_float2(-o[3].y, o[3].x), o[3]) : csub(make_float2(o[3].y, -o[3].x), o[3]);
        v[0] = cadd(e[0], o[0]);
        v[4] = csub(e[0], o[0]);
        v[1] = __ffma2_rn(u1, make_float2(h, h), e[1]);
        v[5] = __ffma2_rn(u1, make_float2(-h, -h), e[1]);
        v[2] = cadd(e[2], o2);
        v[6] = csub(e[2], o2);
        v[3] = __ffma2_rn(u3, make_float2(h, h), e[3]);
        v[7] = __ffma2_rn(u3, make_float2(-h, -h), e[3]);
    }
};

// Odd radices: direct O(R^2) DFT with compile-time roots.
template <int R>
struct Roots {
    float c[R], s[R];  // cos / sin(2 pi k / R)
};
__constant__ Roots<3> c_roots3 = {{1.0f, -0.5f, -0.5f}, {0.0f, 0.86602540378443865f, -0.86602540378443865f}};
__constant__ Roots<5> c_roots5 = {{1.0f, 0.30901699437494742f, -0.80901699437494742f, -0.80901699437494742f,
                                    0.30901699437494742f},
                                   {0.0f, 0.95105651629515357f, 0.58778525229247313f, -0.58778525229247313f,
                                    -0.95105651629515357f}};
__constant__ Roots<7> c_roots7 = {{1.0f, 0.62348980185873353f, -0.22252093395631440f, -0.90096886790241913f,
                                    -0.90096886790241913f, -0.22252093395631440f, 0.62348980185873353f},
                                   {0.0f, 0.78183148246802981f, 0.97492791218182361f, 0.43388373911755812f,
                                    -0.43388373911755812f, -0.97492791218182361f, -0.78183148246802981f}};

template <int R>
__device__ __forceinline__ const Roots<R>& roots();
template <>
__device__ __forceinline__ const Roots<3>& roots<3>() { return c_roots3; }
template <>
__device__ __forceinline__ const Roots<5>& roots<5>() { return c_roots5; }
template <>
__device__ __forceinline__ const Roots<7>& roots<7>() { return c_roots7; }

template <int R, bool INV>
struct DftOdd {
    __host__ __device__ static constexpr int slot(int k) { return k; }
    __device__ __forceinline__ static void run(float2* v) {
        const Roots<R>& rt = roots<R>();
        float2 out[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            float2 acc = v[0];
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const int k = (r * q) % R;
                const float c = rt.c[k], s = INV ? rt.s[k] : -rt.s[k];
                acc = __ffma2_rn(make_float2(v[r].x, v[r].x), make_float2(c, s), acc);
                acc = __ffma2_rn(make_float2(v[r].y, v[r].y), make_float2(-s, c), acc);
            }
            out[q] = acc;
        }
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = out[q];
    }
};
// radix 3: X0 = v0 + t1, X1,2 = (v0 - t1/2) -/+ i (sqrt3/2) t2 (forward), t1 = v1 + v2, t2 = v1 - v2
template <bool INV>
struct Dft<3, INV> {
    __host__ __device__ static constexpr int slot(int k) { return k; }
    __device__ __forceinline__ static void run(float2* v) {
        constexpr float s = 0.86602540378443865f;
        const float2 t1 = cadd(v[1], v[2]);
        const float2 t2 = csub(v[1], v[2]);
        const float2 m = __ffma2_rn(t1, make_float2(-0.5f, -0.5f), v[0]);
        // X1,2 = m +- s (-i t2) (forward): two FFMA2 on the swapped t2, no separate product
        const float2 r = INV ? make_float2(-t2.y, t2.x) : make_float2(t2.y, -t2.x);
        v[0] = cadd(v[0], t1);
        v[1] = __ffma2_rn(r, make_float2(s, s), m);
        v[2] = __ffma2_rn(r, make_float2(-s, -s), m);
    }
};
template <bool INV>
struct Dft<5, INV> : DftOdd<5, INV> {};
template <bool INV>
struct Dft<7, INV> : DftOdd<7, INV> {};

// One Stockham pass of radix R from `x` into `y` (length n), executed by a
// thread group (gtid in [0, gsize)); ends with a block barrier, so every
// thread of the block must call it. Out of place, so a butterfly never waits
// for others and only R values are live per thread.
template <int R, bool INV>
__device__ __forceinline__ void fft_pass(const float2* __restrict__ x, float2* __restrict__ y, int n, int ns,
                                         const float2* __restrict__ tw, int gtid, int gsize) {
    const int nbf = n / R;
    const int tstride = n / (ns * R);
    for (int b = gtid; b < nbf; b += gsize) {
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = x[b + r * nbf];
        const int k = b % ns;
        if (ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const float2 w = __ldg(tw + k * r * tstride);
                v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
            }
        }
        Dft<R, INV>::run(v);
        const int base = (b - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) y[base + r * ns] = v[r];
    }
    __syncthreads();
}

// All passes, ping-ponging between x and y; returns the buffer holding the
// result.
template <bool INV>
__device__ __forceinline__ float2* fft_passes(float2* x, float2* y, int n, int npass, const int* radix,
                                              const float2* tw, int gtid, int gsize) {
    int ns = 1;
    for (int p = 0; p < npass; ++p) {
        switch (radix[p]) {
            case 8: fft_pass<8, INV>(x, y, n, ns, tw, gtid, gsize); break;
            case 4: fft_pass<4, INV>(x, y, n, ns, tw, gtid, gsize); break;
            case 2: fft_pass<2, INV>(x, y, n, ns, tw, gtid, gsize); break;
            case 3: fft_pass<3, INV>(x, y, n, ns, tw, gtid, gsize); break;
            case 5: fft_pass<5, INV>(x, y, n, ns, tw, gtid, gsize); break;
            case 7: fft_pass<7, INV>(x, y, n, ns, tw, gtid, gsize); break;
            default: break;
        }
        ns *= radix[p];
        float2* t = x;
        x = y;
        y = t;
    }
    return x;
}

// Shared-memory elements one transform needs (data + ping-pong scratch).
__host__ __device__ inline int fft_smem_elems(const FftDesc& d) { return 2 * (d.nb ? d.nb : d.n); }

// Unnormalised transform of x[0..n); `scratch` must hold fft_smem_elems(d) -
// (nb or n) further elements (the ping-pong partner, and for Bluestein the
// zero-padded tail lives in x[n, nb)). Returns the buffer holding the result
// (x or scratch); ends with a block barrier.
template <bool INV>
__device__ __forceinline__ float2* block_fft(float2* x, float2* scratch, const FftDesc& d, int gtid, int gsize) {
    if (d.nb == 0) return fft_passes<INV>(x, scratch, d.n, d.npass, d.radix, d.tw, gtid, gsize);
    const int n = d.n, nb = d.nb;
    for (int j = gtid; j < nb; j += gsize) {
        if (j < n) {
            const float2 c = __ldg(d.chirp + j);
            x[j] = INV ? cmulc(x[j], c) : cmul(x[j], c);
        } else {
            x[j] = make_float2(0.f, 0.f);
        }
    }
    __syncthreads();
    float2* a = fft_passes<false>(x, scratch, nb, d.nbpass, d.bradix, d.btw, gtid, gsize);
    float2* other = a == x ? scratch : x;
    for (int j = gtid; j < nb; j += gsize) {
        const float2 b = __ldg(d.bhat + j);
        a[j] = INV ? cmulc(a[j], b) : cmul(a[j], b);
    }
    __syncthreads();
    a = fft_passes<true>(a, other, nb, d.nbpass, d.bradix, d.btw, gtid, gsize);
    for (int j = gtid; j < n; j += gsize) {
        const float2 c = __ldg(d.chirp + j);
        a[j] = INV ? cmulc(a[j], c) : cmul(a[j], c);
    }
    __syncthreads();
    return a;
}

}  // namespace lpr
