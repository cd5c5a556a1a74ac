// Launchers of the EM glue kernels (lpr_em.cu); the orchestration is em_chunk
// in lpr_capi.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace lpr {

void launch_disc_fill(int N, float* img, int batch, cudaStream_t st);
void launch_fill(float* x, size_t n, float v, cudaStream_t st);
void launch_slice_max(const float* x, size_t per, int batch, float* mx, int* bad, cudaStream_t st);
void launch_em_ratio(const float* g, float* rf_q, size_t per, int batch, const float* gmax, double* ll, int ll_stride,
                     bool write_ratio, cudaStream_t st);
void launch_em_update(float* f, const float* bp, const float* inv_sens, size_t per, int batch, int* bad,
                      cudaStream_t st);
void launch_sens_invert(int N, const float* sens, const float* smax, float* inv, cudaStream_t st);

}  // namespace lpr
