// Drop-in implementation of include/lpradon/lp_ops.hpp for the reference tree
// (replaces proj/src/lp_ops.cpp:1-2). Host C++ over the C ABI: the reference
// keeps building its plan-time blocks (sampling_plan, zeta_spectrum) and all
// per-slice work runs in the sm_100a kernels behind lpradon_gpu.h.
#include "lpradon/lp_ops.hpp"

#include <cmath>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "lpradon_gpu.h"

namespace lpr {

namespace {

void check(int rc) {
    if (rc == LPR_OK) return;
    const std::string msg = lpr_gpu_last_error();
    if (rc == LPR_ERR_ARG) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

lpr_geometry to_c(const GeometryPlan& p) {
    lpr_geometry g{};
    check(lpr_geometry_make(p.N, p.M, p.N_theta, p.N_rho, &g));
    return g;
}

std::vector<float> to_f32(const Array2D<double>& a) {
    std::vector<float> v(a.size());
    for (std::size_t i = 0; i < a.size(); ++i) v[i] = float(a.storage()[i]);
    return v;
}

void from_f32(const std::vector<float>& v, Array2D<double>& a) {
    for (std::size_t i = 0; i < a.size(); ++i) a.storage()[i] = double(v[i]);
}

}  // namespace

RadonPlan make_radon_plan(const GeometryPlan& geom, KernelMethod method, int device, int max_batch) {
    RadonPlan plan;
    plan.geom = geom;
    plan.zeta = zeta_spectrum(geom, method);
    plan.zeta_bp = zeta_bp_spectrum(geom, method);
    plan.device = device;
    plan.max_batch = max_batch;
    const lpr_geometry g = to_c(geom);
    lpr_gpu_plan* raw = nullptr;
    check(lpr_gpu_plan_create(device, &g, reinterpret_cast<const double*>(plan.zeta.coeffs.data()),
                              reinterpret_cast<const double*>(plan.zeta_bp.coeffs.data()), max_batch, &raw));
    plan.gpu = std::shared_ptr<lpr_gpu_plan>(raw, lpr_gpu_plan_destroy);
    return plan;
}

Array2D<double> lp_convolve(const Array2D<double>& data, const KernelSpectrum& spectrum, bool divide_bspline,
                            const RadonPlan& plan) {
    const std::size_t rows = 2 * std::size_t(plan.geom.N_theta_sector), cols = std::size_t(plan.geom.N_rho);
    require(data.rows() == rows && data.cols() == cols, "lp_convolve: data is not the plan's doubled grid");
    require(spectrum.coeffs.rows() == rows && spectrum.coeffs.cols() == cols,
            "lp_convolve: spectrum does not match the plan");
    const std::vector<float> in = to_f32(data);
    std::vector<float> res(in.size());
    check(lpr_gpu_lp_convolve_host(plan.gpu.get(), reinterpret_cast<const double*>(spectrum.coeffs.data()),
                                   divide_bspline ? 1 : 0, in.data(), res.data(), 1));
    Array2D<double> out(rows, cols);
    from_f32(res, out);
    return out;
}

Sinogram fast_radon(const Image& image, const RadonPlan& plan) {
    const auto& p = plan.geom;
    require(image.pixels.rows() == std::size_t(p.N) && image.pixels.cols() == std::size_t(p.N),
            "fast_radon: image does not match the plan");
    Sinogram out;
    out.grid = p.polar_grid();
    out.values = Array2D<double>(p.N_theta, p.N);
    const std::vector<float> in = to_f32(image.pixels);
    std::vector<float> res(out.values.size());
    check(lpr_gpu_radon_host(plan.gpu.get(), in.data(), res.data(), 1));
    from_f32(res, out.values);
    return out;
}

Image fast_backprojection(const Sinogram& sino, const RadonPlan& plan) {
    const auto& p = plan.geom;
    require(sino.values.rows() == std::size_t(p.N_theta) && sino.values.cols() == std::size_t(p.N),
            "fast_backprojection: sinogram does not match the plan");
    Image out;
    out.grid = p.cartesian_grid();
    out.pixels = Array2D<double>(p.N, p.N);
    const std::vector<float> in = to_f32(sino.values);
    std::vector<float> res(out.pixels.size());
    check(lpr_gpu_backproject_host(plan.gpu.get(), in.data(), res.data(), 1));
    from_f32(res, out.pixels);
    return out;
}

Image radon_transpose(const Sinogram& sino, const RadonPlan& plan) {
    const auto& p = plan.geom;
    require(sino.values.rows() == std::size_t(p.N_theta) && sino.values.cols() == std::size_t(p.N),
            "radon_transpose: sinogram does not match the plan");
    // device entry point only: stage through cudaMalloc'd buffers owned here
    Image out;
    out.grid = p.cartesian_grid();
    out.pixels = Array2D<double>(p.N, p.N);
    const std::vector<float> in = to_f32(sino.values);
    std::vector<float> res(out.pixels.size());
    check(lpr_gpu_radon_transpose_host(plan.gpu.get(), in.data(), res.data(), 1));
    from_f32(res, out.pixels);
    return out;
}

double adjoint_gap(const RadonPlan& plan, int trials) {
    require(trials >= 1, "adjoint_gap: trials must be >= 1");
    const auto& p = plan.geom;
    std::mt19937_64 rng(0x5EEDULL);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    double worst = 0.0;
    for (int t = 0; t < trials; ++t) {
        Image f;
        f.grid = p.cartesian_grid();
        f.pixels = Array2D<double>(p.N, p.N);
        for (auto& v : f.pixels.storage()) v = u(rng);
        Sinogram g;
        g.grid = p.polar_grid();
        g.values = Array2D<double>(p.N_theta, p.N);
        for (auto& v : g.values.storage()) v = u(rng);
        const Sinogram rf = fast_radon(f, plan);
        const Image bg = fast_backprojection(g, plan);
        double lhs = 0.0, rhs = 0.0, ff = 0.0, gg = 0.0;
        for (std::size_t i = 0; i < rf.values.size(); ++i) {
            lhs += rf.values.storage()[i] * g.values.storage()[i];
            gg += g.values.storage()[i] * g.values.storage()[i];
        }
        for (std::size_t i = 0; i < f.pixels.size(); ++i) {
            rhs += f.pixels.storage()[i] * bg.pixels.storage()[i];
            ff += f.pixels.storage()[i] * f.pixels.storage()[i];
        }
        const double w = 2.0 * p.dtheta_p * p.ds, n2 = double(p.N) * double(p.N);
        const double gap = std::abs(w * lhs - rhs / n2) / std::sqrt((ff / n2) * (w * gg));
        worst = std::max(worst, gap);
    }
    return worst;
}

Image fbp(const Sinogram& sino, const RadonPlan& plan, FilterKind kind) {
    const auto& p = plan.geom;
    require(sino.values.rows() == std::size_t(p.N_theta) && sino.values.cols() == std::size_t(p.N),
            "fbp: sinogram does not match the plan");
    Image out;
    out.grid = p.cartesian_grid();
    out.pixels = Array2D<double>(p.N, p.N);
    const std::vector<float> in = to_f32(sino.values);
    std::vector<float> res(out.pixels.size());
    check(lpr_gpu_fbp_host(plan.gpu.get(), int(kind), in.data(), res.data(), 1));
    from_f32(res, out.pixels);
    return out;
}

Image sensitivity_image(const RadonPlan& plan) {
    const auto& p = plan.geom;
    Image out;
    out.grid = p.cartesian_grid();
    out.pixels = Array2D<double>(p.N, p.N);
    std::vector<float> res(out.pixels.size());
    check(lpr_gpu_sensitivity_host(plan.gpu.get(), res.data()));
    from_f32(res, out.pixels);
    return out;
}

namespace {
Image em_iterate(const Sinogram& g, const RadonPlan& plan, int iters, const Image* f0, std::vector<double>* hist) {
    const auto& p = plan.geom;
    require(g.values.rows() == std::size_t(p.N_theta) && g.values.cols() == std::size_t(p.N),
            "em: sinogram does not match the plan");
    require(iters >= 0, "em: iters must be >= 0");
    if (f0) require(f0->pixels.rows() == std::size_t(p.N) && f0->pixels.cols() == std::size_t(p.N),
                    "em: f0 does not match the plan");
    Image out;
    out.grid = p.cartesian_grid();
    out.pixels = Array2D<double>(p.N, p.N);
    const std::vector<float> gin = to_f32(g.values);
    std::vector<float> f = f0 ? to_f32(f0->pixels) : std::vector<float>(out.pixels.size());
    std::vector<double> ll(std::max(iters, 1));
    check(lpr_gpu_em_host(plan.gpu.get(), gin.data(), f.data(), 1, iters, f0 ? 0 : 1, ll.data()));
    from_f32(f, out.pixels);
    if (hist) hist->insert(hist->end(), ll.begin(), ll.begin() + iters);
    return out;
}
}  // namespace

EmState em_step(EmState state, const Sinogram& g, const RadonPlan& plan) {
    if (state.sensitivity.pixels.size() == 0) state.sensitivity = sensitivity_image(plan);
    state.estimate = em_iterate(g, plan, 1, &state.estimate, &state.loglik_history);
    ++state.iteration;
    return state;
}

Image em_run(const Sinogram& g, const RadonPlan& plan, int iters, const Image* f0, std::vector<double>* history) {
    if (iters == 0 && f0) return *f0;
    return em_iterate(g, plan, iters, f0, history);
}

}  // namespace lpr
