// Exact transpose R^T of the GPU Radon transform (placeholder until the
// transpose kernels land; lpr_gpu_radon_transpose reports not-built).
#include "lpr_kernels.cuh"
