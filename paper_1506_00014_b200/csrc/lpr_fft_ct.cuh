// Compile-time register FFTs for the plan lengths that dominate the hot path
// (the 2048 / 8192 theta periods and the 7-smooth rho length 4374 of the
// N=2048 bench plan, 16384 for N=4096). A transform runs in place in one
// padded shared buffer: each pass stages all of a thread's butterflies in
// registers between two barriers, with radices of 6..32 so a transform takes
// 3-4 shared-memory round trips, and the index map pad(i) = i + i/16 keeps
// the strided Stockham writes of the early passes (stride R float2) off
// colliding banks (the padding per length is chosen by a bank-conflict
// count of each pass, see ct_pad).
#pragma once

#include <cmath>
#include <type_traits>
#include <vector>

#include "lpr_fft.cuh"

#ifndef LPR_RHO_TW_TABLE
#define LPR_RHO_TW_TABLE 0  // streamed rho pass: 1 = twiddle tables from global, 0 = computed (__sincosf + powers)
#endif

namespace lpr {

// Radix-R roots W_R^j = (c, s) = exp(-2 pi i j / R) in the (c, s, -s, c)
// form of tw_mul (c_wqc: the conjugate, for inverse butterflies), so a
// constant twiddle is one FMUL2 + one FFMA2 on uniform-register pairs.
__constant__ float4 c_wq6[6] = {{1.000000000e+00f, -0.000000000e+00f, 0.000000000e+00f, 1.000000000e+00f}, {5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, 5.000000000e-01f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {-1.000000000e+00f, -1.224646799e-16f, 1.224646799e-16f, -1.000000000e+00f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, 5.000000000e-01f}};
__constant__ float4 c_wqc6[6] = {{1.000000000e+00f, 0.000000000e+00f, -0.000000000e+00f, 1.000000000e+00f}, {5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, 5.000000000e-01f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {-1.000000000e+00f, 1.224646799e-16f, -1.224646799e-16f, -1.000000000e+00f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, 5.000000000e-01f}};
__constant__ float4 c_wq9[9] = {{1.000000000e+00f, -0.000000000e+00f, 0.000000000e+00f, 1.000000000e+00f}, {7.660444431e-01f, -6.427876097e-01f, 6.427876097e-01f, 7.660444431e-01f}, {1.736481777e-01f, -9.848077530e-01f, 9.848077530e-01f, 1.736481777e-01f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {-9.396926208e-01f, -3.420201433e-01f, 3.420201433e-01f, -9.396926208e-01f}, {-9.396926208e-01f, 3.420201433e-01f, -3.420201433e-01f, -9.396926208e-01f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {1.736481777e-01f, 9.848077530e-01f, -9.848077530e-01f, 1.736481777e-01f}, {7.660444431e-01f, 6.427876097e-01f, -6.427876097e-01f, 7.660444431e-01f}};
__constant__ float4 c_wqc9[9] = {{1.000000000e+00f, 0.000000000e+00f, -0.000000000e+00f, 1.000000000e+00f}, {7.660444431e-01f, 6.427876097e-01f, -6.427876097e-01f, 7.660444431e-01f}, {1.736481777e-01f, 9.848077530e-01f, -9.848077530e-01f, 1.736481777e-01f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {-9.396926208e-01f, 3.420201433e-01f, -3.420201433e-01f, -9.396926208e-01f}, {-9.396926208e-01f, -3.420201433e-01f, 3.420201433e-01f, -9.396926208e-01f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {1.736481777e-01f, -9.848077530e-01f, 9.848077530e-01f, 1.736481777e-01f}, {7.660444431e-01f, -6.427876097e-01f, 6.427876097e-01f, 7.660444431e-01f}};
__constant__ float4 c_wq12[12] = {{1.000000000e+00f, -0.000000000e+00f, 0.000000000e+00f, 1.000000000e+00f}, {8.660254038e-01f, -5.000000000e-01f, 5.000000000e-01f, 8.660254038e-01f}, {5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, 5.000000000e-01f}, {6.123233996e-17f, -1.000000000e+00f, 1.000000000e+00f, 6.123233996e-17f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {-8.660254038e-01f, -5.000000000e-01f, 5.000000000e-01f, -8.660254038e-01f}, {-1.000000000e+00f, -1.224646799e-16f, 1.224646799e-16f, -1.000000000e+00f}, {-8.660254038e-01f, 5.000000000e-01f, -5.000000000e-01f, -8.660254038e-01f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {-1.836970199e-16f, 1.000000000e+00f, -1.000000000e+00f, -1.836970199e-16f}, {5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, 5.000000000e-01f}, {8.660254038e-01f, 5.000000000e-01f, -5.000000000e-01f, 8.660254038e-01f}};
__constant__ float4 c_wqc12[12] = {{1.000000000e+00f, 0.000000000e+00f, -0.000000000e+00f, 1.000000000e+00f}, {8.660254038e-01f, 5.000000000e-01f, -5.000000000e-01f, 8.660254038e-01f}, {5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, 5.000000000e-01f}, {6.123233996e-17f, 1.000000000e+00f, -1.000000000e+00f, 6.123233996e-17f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {-8.660254038e-01f, 5.000000000e-01f, -5.000000000e-01f, -8.660254038e-01f}, {-1.000000000e+00f, 1.224646799e-16f, -1.224646799e-16f, -1.000000000e+00f}, {-8.660254038e-01f, -5.000000000e-01f, 5.000000000e-01f, -8.660254038e-01f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {-1.836970199e-16f, -1.000000000e+00f, 1.000000000e+00f, -1.836970199e-16f}, {5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, 5.000000000e-01f}, {8.660254038e-01f, -5.000000000e-01f, 5.000000000e-01f, 8.660254038e-01f}};
__constant__ float4 c_wq16[16] = {{1.000000000e+00f, -0.000000000e+00f, 0.000000000e+00f, 1.000000000e+00f}, {9.238795325e-01f, -3.826834324e-01f, 3.826834324e-01f, 9.238795325e-01f}, {7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f, 7.071067812e-01f}, {3.826834324e-01f, -9.238795325e-01f, 9.238795325e-01f, 3.826834324e-01f}, {6.123233996e-17f, -1.000000000e+00f, 1.000000000e+00f, 6.123233996e-17f}, {-3.826834324e-01f, -9.238795325e-01f, 9.238795325e-01f, -3.826834324e-01f}, {-7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f}, {-9.238795325e-01f, -3.826834324e-01f, 3.826834324e-01f, -9.238795325e-01f}, {-1.000000000e+00f, -1.224646799e-16f, 1.224646799e-16f, -1.000000000e+00f}, {-9.238795325e-01f, 3.826834324e-01f, -3.826834324e-01f, -9.238795325e-01f}, {-7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f, -7.071067812e-01f}, {-3.826834324e-01f, 9.238795325e-01f, -9.238795325e-01f, -3.826834324e-01f}, {-1.836970199e-16f, 1.000000000e+00f, -1.000000000e+00f, -1.836970199e-16f}, {3.826834324e-01f, 9.238795325e-01f, -9.238795325e-01f, 3.826834324e-01f}, {7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f}, {9.238795325e-01f, 3.826834324e-01f, -3.826834324e-01f, 9.238795325e-01f}};
__constant__ float4 c_wqc16[16] = {{1.000000000e+00f, 0.000000000e+00f, -0.000000000e+00f, 1.000000000e+00f}, {9.238795325e-01f, 3.826834324e-01f, -3.826834324e-01f, 9.238795325e-01f}, {7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f}, {3.826834324e-01f, 9.238795325e-01f, -9.238795325e-01f, 3.826834324e-01f}, {6.123233996e-17f, 1.000000000e+00f, -1.000000000e+00f, 6.123233996e-17f}, {-3.826834324e-01f, 9.238795325e-01f, -9.238795325e-01f, -3.826834324e-01f}, {-7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f, -7.071067812e-01f}, {-9.238795325e-01f, 3.826834324e-01f, -3.826834324e-01f, -9.238795325e-01f}, {-1.000000000e+00f, 1.224646799e-16f, -1.224646799e-16f, -1.000000000e+00f}, {-9.238795325e-01f, -3.826834324e-01f, 3.826834324e-01f, -9.238795325e-01f}, {-7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f}, {-3.826834324e-01f, -9.238795325e-01f, 9.238795325e-01f, -3.826834324e-01f}, {-1.836970199e-16f, -1.000000000e+00f, 1.000000000e+00f, -1.836970199e-16f}, {3.826834324e-01f, -9.238795325e-01f, 9.238795325e-01f, 3.826834324e-01f}, {7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f, 7.071067812e-01f}, {9.238795325e-01f, -3.826834324e-01f, 3.826834324e-01f, 9.238795325e-01f}};
__constant__ float4 c_wq18[18] = {{1.000000000e+00f, -0.000000000e+00f, 0.000000000e+00f, 1.000000000e+00f}, {9.396926208e-01f, -3.420201433e-01f, 3.420201433e-01f, 9.396926208e-01f}, {7.660444431e-01f, -6.427876097e-01f, 6.427876097e-01f, 7.660444431e-01f}, {5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, 5.000000000e-01f}, {1.736481777e-01f, -9.848077530e-01f, 9.848077530e-01f, 1.736481777e-01f}, {-1.736481777e-01f, -9.848077530e-01f, 9.848077530e-01f, -1.736481777e-01f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {-7.660444431e-01f, -6.427876097e-01f, 6.427876097e-01f, -7.660444431e-01f}, {-9.396926208e-01f, -3.420201433e-01f, 3.420201433e-01f, -9.396926208e-01f}, {-1.000000000e+00f, -1.224646799e-16f, 1.224646799e-16f, -1.000000000e+00f}, {-9.396926208e-01f, 3.420201433e-01f, -3.420201433e-01f, -9.396926208e-01f}, {-7.660444431e-01f, 6.427876097e-01f, -6.427876097e-01f, -7.660444431e-01f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {-1.736481777e-01f, 9.848077530e-01f, -9.848077530e-01f, -1.736481777e-01f}, {1.736481777e-01f, 9.848077530e-01f, -9.848077530e-01f, 1.736481777e-01f}, {5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, 5.000000000e-01f}, {7.660444431e-01f, 6.427876097e-01f, -6.427876097e-01f, 7.660444431e-01f}, {9.396926208e-01f, 3.420201433e-01f, -3.420201433e-01f, 9.396926208e-01f}};
__constant__ float4 c_wqc18[18] = {{1.000000000e+00f, 0.000000000e+00f, -0.000000000e+00f, 1.000000000e+00f}, {9.396926208e-01f, 3.420201433e-01f, -3.420201433e-01f, 9.396926208e-01f}, {7.660444431e-01f, 6.427876097e-01f, -6.427876097e-01f, 7.660444431e-01f}, {5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, 5.000000000e-01f}, {1.736481777e-01f, 9.848077530e-01f, -9.848077530e-01f, 1.736481777e-01f}, {-1.736481777e-01f, 9.848077530e-01f, -9.848077530e-01f, -1.736481777e-01f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {-7.660444431e-01f, 6.427876097e-01f, -6.427876097e-01f, -7.660444431e-01f}, {-9.396926208e-01f, 3.420201433e-01f, -3.420201433e-01f, -9.396926208e-01f}, {-1.000000000e+00f, 1.224646799e-16f, -1.224646799e-16f, -1.000000000e+00f}, {-9.396926208e-01f, -3.420201433e-01f, 3.420201433e-01f, -9.396926208e-01f}, {-7.660444431e-01f, -6.427876097e-01f, 6.427876097e-01f, -7.660444431e-01f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {-1.736481777e-01f, -9.848077530e-01f, 9.848077530e-01f, -1.736481777e-01f}, {1.736481777e-01f, -9.848077530e-01f, 9.848077530e-01f, 1.736481777e-01f}, {5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, 5.000000000e-01f}, {7.660444431e-01f, -6.427876097e-01f, 6.427876097e-01f, 7.660444431e-01f}, {9.396926208e-01f, -3.420201433e-01f, 3.420201433e-01f, 9.396926208e-01f}};
__constant__ float4 c_wq27[27] = {{1.000000000e+00f, -0.000000000e+00f, 0.000000000e+00f, 1.000000000e+00f}, {9.730448706e-01f, -2.306158707e-01f, 2.306158707e-01f, 9.730448706e-01f}, {8.936326403e-01f, -4.487991802e-01f, 4.487991802e-01f, 8.936326403e-01f}, {7.660444431e-01f, -6.427876097e-01f, 6.427876097e-01f, 7.660444431e-01f}, {5.971585917e-01f, -8.021231928e-01f, 8.021231928e-01f, 5.971585917e-01f}, {3.960797660e-01f, -9.182161069e-01f, 9.182161069e-01f, 3.960797660e-01f}, {1.736481777e-01f, -9.848077530e-01f, 9.848077530e-01f, 1.736481777e-01f}, {-5.814482891e-02f, -9.983081583e-01f, 9.983081583e-01f, -5.814482891e-02f}, {-2.868032327e-01f, -9.579895123e-01f, 9.579895123e-01f, -2.868032327e-01f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {-6.862416379e-01f, -7.273736416e-01f, 7.273736416e-01f, -6.862416379e-01f}, {-8.354878114e-01f, -5.495089781e-01f, 5.495089781e-01f, -8.354878114e-01f}, {-9.396926208e-01f, -3.420201433e-01f, 3.420201433e-01f, -9.396926208e-01f}, {-9.932383577e-01f, -1.160929141e-01f, 1.160929141e-01f, -9.932383577e-01f}, {-9.932383577e-01f, 1.160929141e-01f, -1.160929141e-01f, -9.932383577e-01f}, {-9.396926208e-01f, 3.420201433e-01f, -3.420201433e-01f, -9.396926208e-01f}, {-8.354878114e-01f, 5.495089781e-01f, -5.495089781e-01f, -8.354878114e-01f}, {-6.862416379e-01f, 7.273736416e-01f, -7.273736416e-01f, -6.862416379e-01f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {-2.868032327e-01f, 9.579895123e-01f, -9.579895123e-01f, -2.868032327e-01f}, {-5.814482891e-02f, 9.983081583e-01f, -9.983081583e-01f, -5.814482891e-02f}, {1.736481777e-01f, 9.848077530e-01f, -9.848077530e-01f, 1.736481777e-01f}, {3.960797660e-01f, 9.182161069e-01f, -9.182161069e-01f, 3.960797660e-01f}, {5.971585917e-01f, 8.021231928e-01f, -8.021231928e-01f, 5.971585917e-01f}, {7.660444431e-01f, 6.427876097e-01f, -6.427876097e-01f, 7.660444431e-01f}, {8.936326403e-01f, 4.487991802e-01f, -4.487991802e-01f, 8.936326403e-01f}, {9.730448706e-01f, 2.306158707e-01f, -2.306158707e-01f, 9.730448706e-01f}};
__constant__ float4 c_wqc27[27] = {{1.000000000e+00f, 0.000000000e+00f, -0.000000000e+00f, 1.000000000e+00f}, {9.730448706e-01f, 2.306158707e-01f, -2.306158707e-01f, 9.730448706e-01f}, {8.936326403e-01f, 4.487991802e-01f, -4.487991802e-01f, 8.936326403e-01f}, {7.660444431e-01f, 6.427876097e-01f, -6.427876097e-01f, 7.660444431e-01f}, {5.971585917e-01f, 8.021231928e-01f, -8.021231928e-01f, 5.971585917e-01f}, {3.960797660e-01f, 9.182161069e-01f, -9.182161069e-01f, 3.960797660e-01f}, {1.736481777e-01f, 9.848077530e-01f, -9.848077530e-01f, 1.736481777e-01f}, {-5.814482891e-02f, 9.983081583e-01f, -9.983081583e-01f, -5.814482891e-02f}, {-2.868032327e-01f, 9.579895123e-01f, -9.579895123e-01f, -2.868032327e-01f}, {-5.000000000e-01f, 8.660254038e-01f, -8.660254038e-01f, -5.000000000e-01f}, {-6.862416379e-01f, 7.273736416e-01f, -7.273736416e-01f, -6.862416379e-01f}, {-8.354878114e-01f, 5.495089781e-01f, -5.495089781e-01f, -8.354878114e-01f}, {-9.396926208e-01f, 3.420201433e-01f, -3.420201433e-01f, -9.396926208e-01f}, {-9.932383577e-01f, 1.160929141e-01f, -1.160929141e-01f, -9.932383577e-01f}, {-9.932383577e-01f, -1.160929141e-01f, 1.160929141e-01f, -9.932383577e-01f}, {-9.396926208e-01f, -3.420201433e-01f, 3.420201433e-01f, -9.396926208e-01f}, {-8.354878114e-01f, -5.495089781e-01f, 5.495089781e-01f, -8.354878114e-01f}, {-6.862416379e-01f, -7.273736416e-01f, 7.273736416e-01f, -6.862416379e-01f}, {-5.000000000e-01f, -8.660254038e-01f, 8.660254038e-01f, -5.000000000e-01f}, {-2.868032327e-01f, -9.579895123e-01f, 9.579895123e-01f, -2.868032327e-01f}, {-5.814482891e-02f, -9.983081583e-01f, 9.983081583e-01f, -5.814482891e-02f}, {1.736481777e-01f, -9.848077530e-01f, 9.848077530e-01f, 1.736481777e-01f}, {3.960797660e-01f, -9.182161069e-01f, 9.182161069e-01f, 3.960797660e-01f}, {5.971585917e-01f, -8.021231928e-01f, 8.021231928e-01f, 5.971585917e-01f}, {7.660444431e-01f, -6.427876097e-01f, 6.427876097e-01f, 7.660444431e-01f}, {8.936326403e-01f, -4.487991802e-01f, 4.487991802e-01f, 8.936326403e-01f}, {9.730448706e-01f, -2.306158707e-01f, 2.306158707e-01f, 9.730448706e-01f}};
__constant__ float4 c_wq32[32] = {{1.000000000e+00f, -0.000000000e+00f, 0.000000000e+00f, 1.000000000e+00f}, {9.807852804e-01f, -1.950903220e-01f, 1.950903220e-01f, 9.807852804e-01f}, {9.238795325e-01f, -3.826834324e-01f, 3.826834324e-01f, 9.238795325e-01f}, {8.314696123e-01f, -5.555702330e-01f, 5.555702330e-01f, 8.314696123e-01f}, {7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f, 7.071067812e-01f}, {5.555702330e-01f, -8.314696123e-01f, 8.314696123e-01f, 5.555702330e-01f}, {3.826834324e-01f, -9.238795325e-01f, 9.238795325e-01f, 3.826834324e-01f}, {1.950903220e-01f, -9.807852804e-01f, 9.807852804e-01f, 1.950903220e-01f}, {6.123233996e-17f, -1.000000000e+00f, 1.000000000e+00f, 6.123233996e-17f}, {-1.950903220e-01f, -9.807852804e-01f, 9.807852804e-01f, -1.950903220e-01f}, {-3.826834324e-01f, -9.238795325e-01f, 9.238795325e-01f, -3.826834324e-01f}, {-5.555702330e-01f, -8.314696123e-01f, 8.314696123e-01f, -5.555702330e-01f}, {-7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f}, {-8.314696123e-01f, -5.555702330e-01f, 5.555702330e-01f, -8.314696123e-01f}, {-9.238795325e-01f, -3.826834324e-01f, 3.826834324e-01f, -9.238795325e-01f}, {-9.807852804e-01f, -1.950903220e-01f, 1.950903220e-01f, -9.807852804e-01f}, {-1.000000000e+00f, -1.224646799e-16f, 1.224646799e-16f, -1.000000000e+00f}, {-9.807852804e-01f, 1.950903220e-01f, -1.950903220e-01f, -9.807852804e-01f}, {-9.238795325e-01f, 3.826834324e-01f, -3.826834324e-01f, -9.238795325e-01f}, {-8.314696123e-01f, 5.555702330e-01f, -5.555702330e-01f, -8.314696123e-01f}, {-7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f, -7.071067812e-01f}, {-5.555702330e-01f, 8.314696123e-01f, -8.314696123e-01f, -5.555702330e-01f}, {-3.826834324e-01f, 9.238795325e-01f, -9.238795325e-01f, -3.826834324e-01f}, {-1.950903220e-01f, 9.807852804e-01f, -9.807852804e-01f, -1.950903220e-01f}, {-1.836970199e-16f, 1.000000000e+00f, -1.000000000e+00f, -1.836970199e-16f}, {1.950903220e-01f, 9.807852804e-01f, -9.807852804e-01f, 1.950903220e-01f}, {3.826834324e-01f, 9.238795325e-01f, -9.238795325e-01f, 3.826834324e-01f}, {5.555702330e-01f, 8.314696123e-01f, -8.314696123e-01f, 5.555702330e-01f}, {7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f}, {8.314696123e-01f, 5.555702330e-01f, -5.555702330e-01f, 8.314696123e-01f}, {9.238795325e-01f, 3.826834324e-01f, -3.826834324e-01f, 9.238795325e-01f}, {9.807852804e-01f, 1.950903220e-01f, -1.950903220e-01f, 9.807852804e-01f}};
__constant__ float4 c_wqc32[32] = {{1.000000000e+00f, 0.000000000e+00f, -0.000000000e+00f, 1.000000000e+00f}, {9.807852804e-01f, 1.950903220e-01f, -1.950903220e-01f, 9.807852804e-01f}, {9.238795325e-01f, 3.826834324e-01f, -3.826834324e-01f, 9.238795325e-01f}, {8.314696123e-01f, 5.555702330e-01f, -5.555702330e-01f, 8.314696123e-01f}, {7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f}, {5.555702330e-01f, 8.314696123e-01f, -8.314696123e-01f, 5.555702330e-01f}, {3.826834324e-01f, 9.238795325e-01f, -9.238795325e-01f, 3.826834324e-01f}, {1.950903220e-01f, 9.807852804e-01f, -9.807852804e-01f, 1.950903220e-01f}, {6.123233996e-17f, 1.000000000e+00f, -1.000000000e+00f, 6.123233996e-17f}, {-1.950903220e-01f, 9.807852804e-01f, -9.807852804e-01f, -1.950903220e-01f}, {-3.826834324e-01f, 9.238795325e-01f, -9.238795325e-01f, -3.826834324e-01f}, {-5.555702330e-01f, 8.314696123e-01f, -8.314696123e-01f, -5.555702330e-01f}, {-7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f, -7.071067812e-01f}, {-8.314696123e-01f, 5.555702330e-01f, -5.555702330e-01f, -8.314696123e-01f}, {-9.238795325e-01f, 3.826834324e-01f, -3.826834324e-01f, -9.238795325e-01f}, {-9.807852804e-01f, 1.950903220e-01f, -1.950903220e-01f, -9.807852804e-01f}, {-1.000000000e+00f, 1.224646799e-16f, -1.224646799e-16f, -1.000000000e+00f}, {-9.807852804e-01f, -1.950903220e-01f, 1.950903220e-01f, -9.807852804e-01f}, {-9.238795325e-01f, -3.826834324e-01f, 3.826834324e-01f, -9.238795325e-01f}, {-8.314696123e-01f, -5.555702330e-01f, 5.555702330e-01f, -8.314696123e-01f}, {-7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f, -7.071067812e-01f}, {-5.555702330e-01f, -8.314696123e-01f, 8.314696123e-01f, -5.555702330e-01f}, {-3.826834324e-01f, -9.238795325e-01f, 9.238795325e-01f, -3.826834324e-01f}, {-1.950903220e-01f, -9.807852804e-01f, 9.807852804e-01f, -1.950903220e-01f}, {-1.836970199e-16f, -1.000000000e+00f, 1.000000000e+00f, -1.836970199e-16f}, {1.950903220e-01f, -9.807852804e-01f, 9.807852804e-01f, 1.950903220e-01f}, {3.826834324e-01f, -9.238795325e-01f, 9.238795325e-01f, 3.826834324e-01f}, {5.555702330e-01f, -8.314696123e-01f, 8.314696123e-01f, 5.555702330e-01f}, {7.071067812e-01f, -7.071067812e-01f, 7.071067812e-01f, 7.071067812e-01f}, {8.314696123e-01f, -5.555702330e-01f, 5.555702330e-01f, 8.314696123e-01f}, {9.238795325e-01f, -3.826834324e-01f, 3.826834324e-01f, 9.238795325e-01f}, {9.807852804e-01f, -1.950903220e-01f, 1.950903220e-01f, 9.807852804e-01f}};


// A twiddle-row pointer the compiler cannot hoist above the preceding barrier
// (in persistent loops it otherwise pulls every pass's table loads to the top
// of the row body and spills).
template <class P>
__device__ __forceinline__ const P* pinned(const P* p) {
    asm volatile("mov.b64 %0, %0;" : "+l"(p)::"memory");
    return p;
}

template <int R, bool INV>
__device__ __forceinline__ float4 wq(int j);
#define LPR_WQ(R)                                                                                          \
    template <>                                                                                            \
    __device__ __forceinline__ float4 wq<R, false>(int j) { return c_wq##R[j]; }                            \
    template <>                                                                                            \
    __device__ __forceinline__ float4 wq<R, true>(int j) { return c_wqc##R[j]; }
LPR_WQ(6)
LPR_WQ(9)
LPR_WQ(12)
LPR_WQ(16)
LPR_WQ(18)
LPR_WQ(27)
LPR_WQ(32)
#undef LPR_WQ

// a * w for a (c, s, -s, c) entry
__device__ __forceinline__ float2 cmul_q(float2 a, float4 w) {
#if LPR_CMUL_SWZ_FIRST
    return __ffma2_rn(make_float2(w.z, w.w), make_float2(a.y, a.y), __fmul2_rn(make_float2(w.x, w.y), make_float2(a.x, a.x)));
#else
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(w.z, w.w), __fmul2_rn(make_float2(a.x, a.x), make_float2(w.x, w.y)));
#endif
}

// Composite radix R = P * Q in registers, natural order in and out:
// x[Q n1 + n2] -> P-point DFTs over n1, twiddle W_R^{n2 k1}, Q-point DFTs over n2
// -> X[k1 + P k2].
template <int P, int Q, bool INV>
__device__ __forceinline__ void dft_pq(float2* v) {
    constexpr int R = P * Q;
    // in place: P-point DFTs over n1 leave Y(n2, k1) in v[Q k1 + n2]
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) {
        float2 t[P];
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) t[n1] = v[Q * n1 + n2];
        Dft<P, INV>::run(t);
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) v[Q * k1 + n2] = t[Dft<P, INV>::slot(k1)];
    }
#pragma unroll
    for (int k1 = 1; k1 < P; ++k1)
#pragma unroll
        for (int n2 = 1; n2 < Q; ++n2) {
            v[Q * k1 + n2] = cmul_q(v[Q * k1 + n2], wq<R, INV>((n2 * k1) % R));
        }
    // Q-point DFTs over n2: X(k1 + P k2) -> v[Q k1 + k2]
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) {
        float2 t[Q];
#pragma unroll
        for (int n2 = 0; n2 < Q; ++n2) t[n2] = v[Q * k1 + n2];
        Dft<Q, INV>::run(t);
#pragma unroll
        for (int k2 = 0; k2 < Q; ++k2) v[Q * k1 + k2] = t[Dft<Q, INV>::slot(k2)];
    }
}

// Composite radix R = P Q, in place: output k sits in slot Q (k mod P) + k / P.
#define LPR_DFT_PQ(RR, PP, QQ)                                                               \
    template <bool INV>                                                                      \
    struct Dft<RR, INV> {                                                                    \
        __host__ __device__ static constexpr int slot(int k) { return QQ * (k % PP) + k / PP; } \
        __device__ __forceinline__ static void run(float2* v) { dft_pq<PP, QQ, INV>(v); }    \
    };
LPR_DFT_PQ(6, 2, 3)
LPR_DFT_PQ(9, 3, 3)
LPR_DFT_PQ(12, 4, 3)
LPR_DFT_PQ(16, 4, 4)
LPR_DFT_PQ(18, 2, 9)
LPR_DFT_PQ(27, 3, 9)
LPR_DFT_PQ(32, 4, 8)
#undef LPR_DFT_PQ

// Padded shared index: one spare slot every 2^S elements (S = 0: none). The
// best S per plan comes from a bank-conflict count of every pass's read and
// write pattern (64-bit accesses, half-warp phases): i/16 for 2048 and 4096,
// i/32 for 8192 and 16384, none for 4374 (radix 6/9 strides).
template <int S>
__host__ __device__ constexpr int ct_pad(int i) { return S ? i + (i >> S) : i; }

// Per-pass twiddle tables: pass (R, NS) stores W_{NS R}^{k r}, r = 1..R-1, at
// OFF + (r - 1) NS + k, so for each r the butterflies of a warp (consecutive
// k) read consecutive float2: two fully used wavefronts per load. (Indexing
// one length-N table by k r N/(NS R) scatters a warp over up to 32 cache
// lines per load; a [k][r] layout still strides lanes by R float2.)
__host__ __device__ constexpr int tw_rs(int R) { return R - 1; }

// Twiddle multiply by a table entry. float2 tables hold w = (c, s) and the
// inverse uses conj(w); float4 tables hold (c, s, -s, c) of the entry already
// conjugated for an inverse table, so the product is one FMUL2 + one FFMA2
// with no operand swaps or negations: a w = a.x (c, s) + a.y (-s, c).
template <bool INV>
__device__ __forceinline__ float2 tw_mul(float2 a, const float2* p) {
    const float2 w = __ldg(p);
    return INV ? cmulc(a, w) : cmul(a, w);
}
template <bool INV>
__device__ __forceinline__ float2 tw_mul(float2 a, const float4* p) {
    return cmul_q(a, __ldg(p));
}

// Computed twiddles (no table): w = exp(-+2 pi i k / L) from one fast
// __sincosf (|angle| < 2 pi / R, abs error ~4e-7) and its powers w^2..w^(R-1)
// by complex products of depth <= 3. Used where the shared-memory carve-out
// leaves too little L1 for the tables (the streamed rho pass); the twiddle
// error (< 4e-6) is far below the 1e-4 parity bar.
struct TwSincos {};

template <int R, bool INV>
__device__ __forceinline__ void tw_apply_sincos(float2* v, int k, int L) {
    float sn, cs;
    __sincosf((INV ? 6.283185307179586f : -6.283185307179586f) * (float(k) / float(L)), &sn, &cs);
    float2 p[R];
    p[1] = make_float2(cs, sn);
#pragma unroll
    for (int r = 2; r < R; ++r) p[r] = cmul(p[r / 2], p[r - r / 2]);
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], p[r]);
}

// Band pruning of the pass before a final radix-2 (NS R = N/2) whose caller
// needs only the outputs k with k mod N/2 in [0, BAND) or (N/2 - BAND, N/2):
// output r of a butterfly lands at k + r NS (mod N/2), k < NS, so only the
// r with r NS < BAND or r NS + NS - 1 > N/2 - BAND are stored (the dead
// outputs' butterfly arithmetic is then dropped by the compiler).
template <int N, int R, int NS, int BAND>
__host__ __device__ constexpr bool band_keep(int r) {
    return BAND == 0 || r * NS < BAND || r * NS + NS - 1 > N / 2 - BAND;
}

// Shared-memory store of one complex value. ptxas otherwise copies many
// packed-FP results into a fresh register pair before each STS.64 (two MOVs
// per store in the rho FFT); the asm store takes the pair as it is.
#ifndef LPR_STS_ASM
#define LPR_STS_ASM 1
#endif
__device__ __forceinline__ void sts2(float2* p, float2 v) {
#if LPR_STS_ASM
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(p))), "f"(v.x),
                 "f"(v.y));
#else
    *p = v;
#endif
}

// Padded walks: elements base + r STRIDE, r < R, of a buffer padded by
// ct_pad<S> sit at ct_pad<S>(base) + r STRIDE + (r STRIDE >> S) whenever
// STRIDE is a multiple of 2^S, or STRIDE = 1 with R dividing 2^S and base a
// multiple of R (the walk stays inside one 2^S block). Then one padded base
// per butterfly and compile-time offsets replace a shift-add per access.
template <int S, int STRIDE, int R>
__host__ __device__ constexpr bool pad_walk_ok() {
    return S == 0 || STRIDE % (1 << S) == 0 || (STRIDE == 1 && (1 << S) % R == 0);
}
template <int S, int STRIDE>
__host__ __device__ constexpr int pad_walk_off(int r) {
    return r * STRIDE + (S ? (r * STRIDE) >> S : 0);
}

// One in-place pass of radix R at Stockham stride NS over a padded buffer.
// PIN (first pass of a zero-padded transform): elements at or past n_in are
// zero and are neither read nor required to be in the buffer.
template <int N, int T, int S, int R, int NS, int OFF, bool INV, int BAND = 0, bool PIN = false, class TW>
__device__ __forceinline__ void ct_pass(float2* x, const TW* __restrict__ twp, int tid, int n_in = N) {
    static_assert(BAND == 0 || NS * R * 2 == N, "band pruning applies to the pass before a final radix 2");
    constexpr int B = N / R;
    constexpr int NB = (B + T - 1) / T;
    float2 v[NB][R];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int b = tid + i * T;
        if (b < B) {
            if constexpr (PIN) {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    v[i][r] = b + r * B < n_in ? x[ct_pad<S>(b + r * B)] : make_float2(0.f, 0.f);
            } else if constexpr (pad_walk_ok<S, B, R>()) {
                const float2* xb = x + ct_pad<S>(b);
#pragma unroll
                for (int r = 0; r < R; ++r) v[i][r] = xb[pad_walk_off<S, B>(r)];
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) v[i][r] = x[ct_pad<S>(b + r * B)];
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int b = tid + i * T;
        if (b < B) {
            const int k = b % NS;
            if constexpr (NS > 1 && std::is_same<TW, TwSincos>::value) {
                tw_apply_sincos<R, INV>(v[i], k, NS * R);
            } else if constexpr (NS > 1) {
                const TW* tw = pinned(twp + (OFF + k));  // one base; the r offsets fold into the loads
#pragma unroll
                for (int r = 1; r < R; ++r) v[i][r] = tw_mul<INV>(v[i][r], tw + (r - 1) * NS);
            }
            Dft<R, INV>::run(v[i]);
            const int base = (b - k) * R + k;
            if constexpr (pad_walk_ok<S, NS, R>()) {
                float2* xw = x + ct_pad<S>(base);
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (band_keep<N, R, NS, BAND>(r)) sts2(xw + pad_walk_off<S, NS>(r), v[i][Dft<R, INV>::slot(r)]);
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (band_keep<N, R, NS, BAND>(r)) sts2(x + ct_pad<S>(base + r * NS), v[i][Dft<R, INV>::slot(r)]);
            }
        }
    }
    __syncthreads();
}

template <int N, int T, int S, bool INV, int NS, int OFF, int R, int... Rest, class TW>
__device__ __forceinline__ void ct_run(float2* x, const TW* twp, int tid) {
    ct_pass<N, T, S, R, NS, OFF, INV>(x, twp, tid);
    if constexpr (sizeof...(Rest) > 0)
        ct_run<N, T, S, INV, NS * R, OFF + (NS > 1 ? NS * tw_rs(R) : 0), Rest...>(x, twp, tid);
}
template <int N, int T, int S, bool INV, int BAND, int NS, int OFF, int R, int... Rest, class TW>
__device__ __forceinline__ void ct_run_band(float2* x, const TW* twp, int tid) {
    if constexpr (sizeof...(Rest) > 0) {
        ct_pass<N, T, S, R, NS, OFF, INV>(x, twp, tid);
        ct_run_band<N, T, S, INV, BAND, NS * R, OFF + (NS > 1 ? NS * tw_rs(R) : 0), Rest...>(x, twp, tid);
    } else {
        ct_pass<N, T, S, R, NS, OFF, INV, BAND>(x, twp, tid);
    }
}

// Host side: the per-pass table in exactly the order ct_run consumes it.
template <int N, int NS, int R, int... Rest>
void ct_twiddles(std::vector<float2>& out) {
    if (NS > 1) {
        const int rs = tw_rs(R);
        const size_t off = out.size();
        out.resize(off + size_t(NS) * rs, make_float2(0.f, 0.f));
        for (int k = 0; k < NS; ++k)
            for (int r = 1; r < R; ++r) {
                const double a = -2.0 * 3.14159265358979323846 * double(k) * double(r) / double(NS * R);
                out[off + size_t(r - 1) * NS + k] = make_float2(float(std::cos(a)), float(std::sin(a)));
            }
    }
    if constexpr (sizeof...(Rest) > 0) ct_twiddles<N, NS * R, Rest...>(out);
}

// float4 form of a float2 table for tw_mul: (c, s, -s, c) of w, or of conj(w)
// for a table read by inverse passes.
inline std::vector<float4> tw4(const std::vector<float2>& t, bool conj) {
    std::vector<float4> o(t.size());
    for (size_t i = 0; i < t.size(); ++i) {
        const float c = t[i].x, s = conj ? -t[i].y : t[i].y;
        o[i] = make_float4(c, s, -s, c);
    }
    return o;
}

// Twiddle source of the compile-time plans: the per-pass table, or computed
// (LPR_CT_TW_SINCOS) so the tables do not compete with the gather for L1.
#ifndef LPR_CT_TW_SINCOS
#define LPR_CT_TW_SINCOS 1
#endif
__device__ __forceinline__ auto ct_tw(const FftDesc& d) {
#if LPR_CT_TW_SINCOS
    (void)d;
    return static_cast<const TwSincos*>(nullptr);
#else
    return d.twp;
#endif
}

template <int R1, int... Rest>
struct RadixPack {
    static constexpr int first = R1;
    template <int N, int T, int S, bool INV, class TW>
    __device__ __forceinline__ static void tail(float2* x, const TW* twp, int tid) {
        if constexpr (sizeof...(Rest) > 0) ct_run<N, T, S, INV, R1, 0, Rest...>(x, twp, tid);
    }
    template <int N, int T, int S, bool INV, int BAND, class TW>
    __device__ __forceinline__ static void tail_band(float2* x, const TW* twp, int tid) {
        if constexpr (sizeof...(Rest) > 0) ct_run_band<N, T, S, INV, BAND, R1, 0, Rest...>(x, twp, tid);
    }
};

// FFT policies: idx() (the buffer slot of element i), elems() (shared
// float2 slots one transform needs), kT threads per transform and kP
// transforms per block (the theta kernels give each transform two real
// columns, so kP pairs make 4 kP contiguous columns per global row access),
// kMinBlocks for __launch_bounds__, and run() on the calling thread group
// (gtid in [0, kT); every thread of the block must call it).
template <int N, int T, int P, int MINB, int S, int... R>
struct CtFft {
    static constexpr int kN = N;
    static constexpr int kT = T;
    static constexpr int kP = P;
    static constexpr int kMinBlocks = MINB;
    // radices covering only N/2: the final radix-2 pass is left to the caller
    // (the fine theta kernel fuses it into its band-limited store)
    static constexpr bool kLast2 = (R * ...) * 2 == N;
    // per-transform slots, rounded to 4 mod 16 so the kP buffers of a block
    // start on different banks (row loads spread consecutive lanes over them)
    static constexpr int kElems = (ct_pad<S>(N - 1) + 1 + 12) / 16 * 16 + 4;
    __device__ __forceinline__ static int idx(int i) { return ct_pad<S>(i); }
    __host__ __device__ static int elems(const FftDesc&) { return kElems; }
    template <bool INV>
    __device__ __forceinline__ static float2* run(float2* x, float2*, const FftDesc& d, int gtid) {
        ct_run<N, T, S, INV, 1, 0, R...>(x, ct_tw(d), gtid);
        return x;
    }
    // first radix, and the remaining passes for kernels that run the first
    // (twiddle-free, NS = 1) pass themselves straight from gathered registers
    static constexpr int kR1 = RadixPack<R...>::first;
    static constexpr bool kPadWalk1 = pad_walk_ok<S, 1, kR1>();  // first-pass outputs bb R1 + r: one padded base
    template <bool INV>
    __device__ __forceinline__ static void run_tail(float2* x, const FftDesc& d, int gtid) {
        RadixPack<R...>::template tail<N, T, S, INV>(x, ct_tw(d), gtid);
    }
    // same, storing only what a band-limited final radix-2 reads (band_keep)
    template <bool INV, int BAND>
    __device__ __forceinline__ static void run_tail_band(float2* x, const FftDesc& d, int gtid) {
        RadixPack<R...>::template tail_band<N, T, S, INV, BAND>(x, ct_tw(d), gtid);
    }
    static std::vector<float2> pass_twiddles() {
        std::vector<float2> t;
        ct_twiddles<N, 1, R...>(t);
        if (t.empty()) t.push_back(make_float2(1.f, 0.f));
        return t;
    }
};

// ---- pieces of the streamed rho pass (k_rho_stream): forward radices
// R1, R2, R3 and the inverse in the reversed order R3, R2, R1, so the
// forward's last butterfly and the inverse's first (twiddle-free, NS = 1)
// butterfly see the same R3 elements: they are fused in registers with the
// spectral multiply between them (one shared round trip instead of three).

// Forward last pass (radix R at NS = N / R) x multiplier x inverse first pass.
template <int N, int T, int S, int R, int OFF, class TW>
__device__ __forceinline__ void ct_mid_fused(float2* x, const TW* __restrict__ twp, const float2* ms, int tid) {
    constexpr int B = N / R;
    constexpr int NB = (B + T - 1) / T;
    float2 v[NB][R];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int b = tid + i * T;
        if (b < B) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[i][r] = x[ct_pad<S>(b + r * B)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int b = tid + i * T;
        if (b < B) {
            if constexpr (std::is_same<TW, TwSincos>::value) {
                tw_apply_sincos<R, false>(v[i], b, N);
            } else {
                const TW* tw = pinned(twp + (OFF + b));
#pragma unroll
                for (int r = 1; r < R; ++r) v[i][r] = tw_mul<false>(v[i][r], tw + (r - 1) * B);
            }
            Dft<R, false>::run(v[i]);
            float2 u[R];
#pragma unroll
            for (int r = 0; r < R; ++r) u[r] = cmul(v[i][Dft<R, false>::slot(r)], ms[b + r * B]);
            Dft<R, true>::run(u);
            if constexpr (S == 0 && R % 2 == 0) {  // R consecutive outputs: 16-byte stores, conflict-free
                float4* dst = reinterpret_cast<float4*>(x + R * b);
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    const float2 a = u[Dft<R, true>::slot(r)], c = u[Dft<R, true>::slot(r + 1)];
                    dst[r / 2] = make_float4(a.x, a.y, c.x, c.y);
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) sts2(x + ct_pad<S>(R * b + r), u[Dft<R, true>::slot(r)]);
            }
        }
    }
    __syncthreads();
}

// Inverse last pass (radix R at NS = N / R) straight from registers to a
// global row: butterfly b writes out[b + r NS], coalesced across the warp.
// The buffer is free for the next TMA load once this returns.
template <int N, int T, int S, int R, int OFF, class TW>
__device__ __forceinline__ void ct_last_to_global(const float2* x, const TW* __restrict__ twp,
                                                  float2* __restrict__ out, int tid, int n_out = N) {
    constexpr int B = N / R;
    constexpr int NB = (B + T - 1) / T;
    float2 v[NB][R];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int b = tid + i * T;
        if (b < B) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[i][r] = x[ct_pad<S>(b + r * B)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int b = tid + i * T;
        if (b < B) {
            if constexpr (std::is_same<TW, TwSincos>::value) {
                tw_apply_sincos<R, true>(v[i], b, N);
            } else {
                const TW* tw = pinned(twp + (OFF + b));
#pragma unroll
                for (int r = 1; r < R; ++r) v[i][r] = tw_mul<true>(v[i][r], tw + (r - 1) * B);
            }
            Dft<R, true>::run(v[i]);
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (N == n_out || b + r * B < n_out) out[b + r * B] = v[i][Dft<R, true>::slot(r)];
        }
    }
}

// Streamed rho-pass plan: length N = R1 R2 R3, T threads per row.
template <int N, int T, int S, int R1, int R2, int R3>
struct RhoStream {
    static constexpr int kN = N;
    static constexpr int kT = T;
    static constexpr int kElems = (ct_pad<S>(N - 1) + 2) / 2 * 2;  // even: every buffer starts 16-byte aligned
    // forward (R1, R2, R3 + fused) then inverse (R2, R1 to global); the whole
    // per-row convolution on a buffer whose row has landed
    __device__ __forceinline__ static void convolve(float2* x, const float4* twf4, const float4* twi4, const float2* ms,
                                                    float2* out, int tid) {
#if LPR_RHO_TW_TABLE
        const float4 *twf = twf4, *twi = twi4;
#else
        const TwSincos *twf = nullptr, *twi = nullptr;
#endif
        ct_pass<N, T, S, R1, 1, 0, false>(x, twf, tid);
        ct_pass<N, T, S, R2, R1, 0, false>(x, twf, tid);
        ct_mid_fused<N, T, S, R3, R1 * (R2 - 1)>(x, twf, ms, tid);
        ct_pass<N, T, S, R2, R3, 0, true>(x, twi, tid);
        ct_last_to_global<N, T, S, R1, R3 * (R2 - 1)>(x, twi, out, tid);
    }
    static std::vector<float4> fwd_twiddles() {
        std::vector<float2> t;
        ct_twiddles<N, 1, R1, R2, R3>(t);
        return tw4(t, false);
    }
    static std::vector<float4> inv_twiddles() {
        std::vector<float2> t;
        ct_twiddles<N, 1, R3, R2, R1>(t);
        return tw4(t, true);
    }
};

// Same with four radices: forward R1..R3 + fused R4, inverse R3, R2 + R1 to global.
// Smaller radices give more butterflies per pass, so more threads (warps) per row.
template <int N, int T, int S, int R1, int R2, int R3, int R4>
struct RhoStream4 {
    static constexpr int kN = N;
    static constexpr int kT = T;
    static constexpr int kElems = (ct_pad<S>(N - 1) + 2) / 2 * 2;
    __device__ __forceinline__ static void convolve(float2* x, const float4* twf4, const float4* twi4, const float2* ms,
                                                    float2* out, int tid, int n_out = N) {
#if LPR_RHO_TW_TABLE
        const float4 *twf = twf4, *twi = twi4;
#else
        const TwSincos *twf = nullptr, *twi = nullptr;
#endif
        // the first pass reads only the n_out data elements: a zero-padded
        // convolution (k_rho_pad) leaves the rest of the buffer unwritten
        ct_pass<N, T, S, R1, 1, 0, false, 0, true>(x, twf, tid, n_out);
        ct_pass<N, T, S, R2, R1, 0, false>(x, twf, tid);
        ct_pass<N, T, S, R3, R1 * R2, R1 * (R2 - 1), false>(x, twf, tid);
        ct_mid_fused<N, T, S, R4, R1 * (R2 - 1) + R1 * R2 * (R3 - 1)>(x, twf, ms, tid);
        ct_pass<N, T, S, R3, R4, 0, true>(x, twi, tid);
        ct_pass<N, T, S, R2, R4 * R3, R4 * (R3 - 1), true>(x, twi, tid);
        ct_last_to_global<N, T, S, R1, R4 * (R3 - 1) + R4 * R3 * (R2 - 1)>(x, twi, out, tid, n_out);
    }
    static std::vector<float4> fwd_twiddles() {
        std::vector<float2> t;
        ct_twiddles<N, 1, R1, R2, R3, R4>(t);
        return tw4(t, false);
    }
    static std::vector<float4> inv_twiddles() {
        std::vector<float2> t;
        ct_twiddles<N, 1, R4, R3, R2, R1>(t);
        return tw4(t, true);
    }
};

struct GenericFft {
    static constexpr int kN = 0;
    static constexpr bool kPadWalk1 = false;
    static constexpr int kT = 0;  // runtime: threads(d)
    static constexpr int kP = 1;
    static constexpr int kMinBlocks = 1;
    __device__ __forceinline__ static int idx(int i) { return i; }
    __host__ __device__ static int elems(const FftDesc& d) { return fft_smem_elems(d); }
    static int threads(const FftDesc& d) {
        const long len = d.nb ? d.nb : d.n;
        long t = (len / 16 + 31) / 32 * 32;
        return int(t < 64 ? 64 : (t > 512 ? 512 : t));
    }
    template <bool INV>
    __device__ __forceinline__ static float2* run(float2* x, float2* scratch, const FftDesc& d, int gtid) {
        return block_fft<INV>(x, scratch, d, gtid, blockDim.x);
    }
};

// The compile-time shapes, by length (host-side selection in lpr_capi.cu).
//                   N      T   P  minB pad radices
using Fft2048 = CtFft<2048, 128, 4, 2, 4, 16, 16, 8>;
using Fft4096 = CtFft<4096, 256, 2, 1, 4, 16, 16, 16>;
using Fft4374 = CtFft<4374, 192, 1, 2, 0, 27, 27, 6>;
#ifndef LPR_FFT8192_P
#define LPR_FFT8192_P 1  // column pairs per block of the fine theta kernels (A/B knob)
#endif
#ifndef LPR_FFT8192_MINB
#define LPR_FFT8192_MINB (LPR_FFT8192_P == 1 ? 2 : 1)
#endif
using Fft8192 = CtFft<8192, 512, LPR_FFT8192_P, LPR_FFT8192_MINB, 4, 16, 16, 16, 2>;
// the fine theta forward of R: same plan without the last radix-2 pass
using Fft8192Band = CtFft<8192, 512, LPR_FFT8192_P, LPR_FFT8192_MINB, 4, 16, 16, 16>;
using Fft16384 = CtFft<16384, 512, 1, 1, 5, 32, 32, 16>;
// the fine theta forward of R at N = 4096: last radix 2 fused into the band store
using Fft16384Band = CtFft<16384, 512, 1, 1, 5, 32, 32, 8>;
// streamed rho pass for N_rho = 4374 (2 rows in flight per block, 2 blocks per SM)
// default-plan rho pass (N_rho = 4333 = 7 * 619): the circular convolution as
// a zero-padded linear one over 8748 = 2^2 3^7 >= 2 N_rho - 1 (k_rho_pad)
using RhoPad8748 = RhoStream4<8748, 486, 0, 9, 9, 9, 12>;  // 486 threads: two radix-9 butterflies each (512: 2.99, 486: 2.92 ms)
// the reference's N = 4096 plan (N_rho = 8666 = 2 * 7 * 619) the same way over
// 17496 = 2^3 3^7 >= 2 * 8666 - 1: one 140 KB row per block
// 972 threads: exactly 1 / 3 / 2 butterflies per thread in the radix-18 / 6 / 9 passes (1024: 3.58, 972: 3.47 ms per 4 slices)
using RhoPad17496 = RhoStream4<17496, 972, 0, 18, 18, 6, 9>;
// (radix 27,27,6 at 192 threads: 1.44 ms / 16 slices; 9,9,9,6 at 512 threads: 1.49)
#ifndef LPR_RHO_T
#define LPR_RHO_T 192
#endif
#if defined(LPR_RHO_R18)
using Rho4374 = RhoStream<4374, LPR_RHO_T, 0, 9, 27, 18>;
#elif !defined(LPR_RHO_RADIX9)
using Rho4374 = RhoStream<4374, LPR_RHO_T, 0, 27, 27, 6>;
#else
using Rho4374 = RhoStream4<4374, 512, 0, 9, 9, 9, 6>;
#endif

}  // namespace lpr
