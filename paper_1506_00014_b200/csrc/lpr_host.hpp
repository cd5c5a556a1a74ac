#pragma once

#include "lpradon_gpu.h"

namespace lpr::host {

int minimal_n_rho(int N, int M);
int smooth_n_rho(int N, int M);
lpr_geometry make_geometry(int N, int M, int n_theta, int n_rho);
void spectrum(const lpr_geometry& g, int kind, double* out_re_im);

}  // namespace lpr::host
