// lp_ops.hpp — the fast log-polar operators of the reference's (specified,
// unimplemented) lp_ops module, as a drop-in for
// proj/src/lp_ops.cpp:1-2 (empty namespace upstream). The declarations follow
// SPEC.md:267-308 and the reference's value-type conventions
// (proj/include/lpradon/types.hpp:10-74): Image / Sinogram returned by value,
// preconditions via require() -> std::invalid_argument, device failures ->
// std::runtime_error.
//
// The implementation (paper_1506_00014_b200/csrc/dropin/lp_ops.cpp) is a thin
// C++ layer over the C ABI in lpradon_gpu.h: fp64 rasters are staged to fp32,
// the plan owns the uploaded spectra (zeta_spectrum / zeta_bp_spectrum from
// the reference's kernel.cpp) and every operator runs on the B200. Include
// this from a tree that provides the reference headers (lpradon/types.hpp,
// geometry.hpp, kernel.hpp).
#pragma once

#include <memory>
#include <vector>

#include "lpradon/geometry.hpp"
#include "lpradon/kernel.hpp"
#include "lpradon/types.hpp"

struct lpr_gpu_plan;

namespace lpr {

/// geometry + both kernel spectra + the device plan.
/// Immutable after construction and shareable; one plan per device.
struct RadonPlan {
    GeometryPlan geom;
    KernelSpectrum zeta, zeta_bp;
    int device = 0;
    int max_batch = 1;
    std::shared_ptr<lpr_gpu_plan> gpu;
};

RadonPlan make_radon_plan(const GeometryPlan& geom, KernelMethod method = KernelMethod::quadrature,
                          int device = 0, int max_batch = 1);

/// lp_convolve: Re IFFT2(FFT2(data) * spectrum [/ Bhat]) on the doubled grid
/// (2 N_theta_sector x N_rho, rows in periodic order), on the plan's device; the spectrum's
/// theta-Nyquist row is treated as zero, as Algorithms 1-2 do. Shape mismatch: invalid_argument.
Array2D<double> lp_convolve(const Array2D<double>& data, const KernelSpectrum& spectrum, bool divide_bspline,
                            const RadonPlan& plan);

/// Algorithm 1.
Sinogram fast_radon(const Image& image, const RadonPlan& plan);
/// Algorithm 2.
Image fast_backprojection(const Sinogram& sino, const RadonPlan& plan);
/// Exact discrete adjoint of fast_radon under the adjoint_gap inner products.
Image radon_transpose(const Sinogram& sino, const RadonPlan& plan);
/// max over `trials` random pairs of |<Rf,g> - <f,R#g>| / (|f||g|).
double adjoint_gap(const RadonPlan& plan, int trials);

/// FBP filters along s and fbp = c_norm R#(filter(g)).
enum class FilterKind { ramp, shepp_logan, cosine };
Image fbp(const Sinogram& sino, const RadonPlan& plan, FilterKind kind = FilterKind::ramp);

/// EM: the sensitivity R# chi_C, one step, and a run.
struct EmState {
    Image estimate;                      ///< >= 0, zero outside the unit disc
    int iteration = 0;
    Image sensitivity;                   ///< R# chi_C
    std::vector<double> loglik_history;  ///< Poisson log-likelihood after each step
};
Image sensitivity_image(const RadonPlan& plan);
/// f+ = f R#(g / max(Rf, eps)) / R# chi_C; appends the log-likelihood of f+.
EmState em_step(EmState state, const Sinogram& g, const RadonPlan& plan);
/// iters steps from f0 (default: 1 inside the unit disc); the history goes to *history when given.
Image em_run(const Sinogram& g, const RadonPlan& plan, int iters, const Image* f0 = nullptr,
             std::vector<double>* history = nullptr);

}  // namespace lpr
