#pragma once

#include "lpradon_gpu.h"

namespace lpr::host {

int minimal_n_rho(int N, int M);
int smooth_n_rho(int N, int M);
lpr_geometry make_geometry(int N, int M, int n_theta, int n_rho);
void spectrum(const lpr_geometry& g, int kind, double* out_re_im);

// on-disk spectrum cache (lpr_cache.cpp)
bool spectrum_cache_load(const lpr_geometry& g, int kind, double* out_re_im);
void spectrum_cache_store(const lpr_geometry& g, int kind, const double* re_im);
void set_spectrum_cache_dir(const char* dir);
long long spectrum_cache_hits();
long long spectrum_cache_stores();

}  // namespace lpr::host
