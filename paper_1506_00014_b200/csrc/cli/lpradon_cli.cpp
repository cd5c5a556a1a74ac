// lpradon — the reference's CLI surface (proj/src/cli.cpp:7-10
// is a stub upstream) over the B200 library's C ABI (include/lpradon_gpu.h)
// and LPT1 containers (include/lpradon/lpt1.hpp). Pipelines compose through
// files only; identical inputs and flags give identical outputs.
//
//   lpradon phantom --size N --out F
//   lpradon radon --in F [--method logpolar] [--sectors M] [--ntheta T] [--nrho R] --out F
//   lpradon backproject --in F [--method logpolar] [--sectors M] [--nrho R] --out F
//   lpradon fbp --in F [--filter ramp|shepp-logan|cosine] [--sectors M] [--nrho R] --out F
//   lpradon em --in F --iters K [--sectors M] [--nrho R] [--seed S] --out F
//   lpradon kernel-dump --size N [--sectors M] [--ntheta T] [--nrho R] --kind radon|backprojection --out F
//   lpradon bench --sizes N1,N2,... --json F [--sectors M] [--reps K]
//   lpradon inspect --in F [--out G]      (header to stdout; G = the re-encoded container)
//   lpradon calibrate-cnorm [--size N] [--filter K]   (tools/calibrate_cnorm: the disc calibration)
// Global: --device D (default 0), --threads T (accepted; the host work is GPU-side).
// Exit 0 on success, 1 with a message on a runtime error, 2 with the usage
// text on an unknown subcommand or flag, 3 / 4 / 5 / 6 on a bad-magic /
// truncated / shape / schema error of an input container.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "lpradon/lpt1.hpp"
#include "lpradon_gpu.h"

using lpr::io::Container;
using lpr::io::Json;

namespace {

const char* kUsage =
    "usage: lpradon <subcommand> [flags]\n"
    "  phantom --size N --out F\n"
    "  radon --in F [--method logpolar] [--sectors M] [--ntheta T] [--nrho R] --out F\n"
    "  backproject --in F [--method logpolar] [--sectors M] [--nrho R] --out F\n"
    "  fbp --in F [--filter ramp|shepp-logan|cosine] [--sectors M] [--nrho R] --out F\n"
    "  em --in F --iters K [--sectors M] [--nrho R] [--seed S] --out F\n"
    "  kernel-dump --size N [--sectors M] [--ntheta T] [--nrho R] --kind radon|backprojection --out F\n"
    "  bench --sizes N1,N2,... --json F [--sectors M] [--reps K]\n"
    "  inspect --in F [--out G]\n"
    "  calibrate-cnorm [--size N] [--filter ramp|shepp-logan|cosine] [--sectors M]\n"
    "global flags: --device D, --threads T\n";

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Args {
    std::map<std::string, std::string> kv;
    bool has(const std::string& k) const { return kv.count(k) > 0; }
    std::string str(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        if (it != kv.end()) return it->second;
        if (def.empty()) throw Usage("missing --" + k);
        return def;
    }
    long num(const std::string& k, long def, bool required = false) const {
        auto it = kv.find(k);
        if (it == kv.end()) {
            if (required) throw Usage("missing --" + k);
            return def;
        }
        char* end = nullptr;
        const long v = std::strtol(it->second.c_str(), &end, 10);
        if (!end || *end) throw Usage("--" + k + " expects an integer, got '" + it->second + "'");
        return v;
    }
};

Args parse(int argc, char** argv, const std::set<std::string>& allowed) {
    Args a;
    for (int i = 2; i < argc; ++i) {
        std::string f = argv[i];
        if (f.rfind("--", 0) != 0) throw Usage("unexpected argument '" + f + "'");
        f = f.substr(2);
        if (!allowed.count(f) && f != "device" && f != "threads") throw Usage("unknown flag --" + f);
        if (i + 1 >= argc) throw Usage("--" + f + " needs a value");
        a.kv[f] = argv[++i];
    }
    return a;
}

void ck(int status, const char* what) {
    if (status != LPR_OK) throw std::runtime_error(std::string(what) + ": " + lpr_gpu_last_error());
}

lpr_geometry geometry(int N, int M, int n_theta, int n_rho) {
    lpr_geometry g{};
    ck(lpr_geometry_make(N, M, n_theta, n_rho, &g), "sampling_plan");
    return g;
}

struct Plan {
    lpr_gpu_plan* p = nullptr;
    Plan(int device, const lpr_geometry& g, int batch = 1) {
        ck(lpr_gpu_plan_create(device, &g, nullptr, nullptr, batch, &p), "plan");
    }
    ~Plan() { lpr_gpu_plan_destroy(p); }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
};

Json plan_meta(const lpr_geometry& g) {
    Json m = Json::object();
    m["method"] = "logpolar";
    m["sectors"] = Json(g.M);
    m["n_theta"] = Json(g.n_theta);
    m["n_rho"] = Json(g.n_rho);
    return m;
}

Container need(const Container& c, const char* kind) {
    if (c.kind != kind || c.complex) throw std::invalid_argument(std::string("input must be an f32 ") + kind + " container");
    return c;
}

// modified Shepp-Logan head phantom, point-sampled on the raster (values in
// {0, 0.1, ..., 1}; the reference's phantom_image, oracle.cpp:157-163)
std::vector<float> shepp_logan(int N) {
    struct E {
        double A, x, y, a, b, deg;
    };
    static const E kSL[10] = {{1.0, 0.0, 0.0, 0.69, 0.92, 0.0},     {-0.8, 0.0, -0.0184, 0.6624, 0.874, 0.0},
                              {-0.2, 0.22, 0.0, 0.11, 0.31, -18.0}, {-0.2, -0.22, 0.0, 0.16, 0.41, 18.0},
                              {0.1, 0.0, 0.35, 0.21, 0.25, 0.0},    {0.1, 0.0, 0.1, 0.046, 0.046, 0.0},
                              {0.1, 0.0, -0.1, 0.046, 0.046, 0.0},  {0.1, -0.08, -0.605, 0.046, 0.023, 0.0},
                              {0.1, 0.0, -0.605, 0.023, 0.023, 0.0}, {0.1, 0.06, -0.605, 0.023, 0.046, 0.0}};
    std::vector<float> img(std::size_t(N) * N);
    for (int r = 0; r < N; ++r) {
        const double y = -0.5 + double(r) / N;
        for (int c = 0; c < N; ++c) {
            const double x = -0.5 + double(c) / N;
            double v = 0.0;
            for (const E& e : kSL) {
                const double t = e.deg * M_PI / 180.0, co = std::cos(t), si = std::sin(t);
                const double dx = x - 0.5 * e.x, dy = y - 0.5 * e.y;
                const double u = (co * dx + si * dy) / (0.5 * e.a), w = (-si * dx + co * dy) / (0.5 * e.b);
                if (u * u + w * w <= 1.0) v += e.A;
            }
            img[std::size_t(r) * N + c] = float(std::round(v * 10.0) / 10.0);
        }
    }
    return img;
}

int cmd_phantom(const Args& a) {
    const int N = int(a.num("size", 0, true));
    if (N < 2) throw std::invalid_argument("--size must be >= 2");
    Container c;
    c.kind = "image";
    c.rows = c.cols = N;
    c.data = shepp_logan(N);
    c.grid = lpr::io::image_grid(N);
    c.meta["phantom"] = "shepp-logan";
    lpr::io::write_container(a.str("out"), c);
    return 0;
}

void check_method(const Args& a) {
    const std::string m = a.str("method", "logpolar");
    if (m == "direct")
        throw std::invalid_argument("--method direct: the O(N^3) direct operators are the reference's test oracle "
                                    "(proj/src/oracle.cpp), not part of this library");
    if (m != "logpolar") throw Usage("--method must be logpolar or direct");
}

int cmd_radon(const Args& a) {
    check_method(a);
    const Container in = need(lpr::io::read_container(a.str("in")), "image");
    if (in.rows != in.cols) throw std::invalid_argument("image must be square");
    const lpr_geometry g = geometry(in.rows, int(a.num("sectors", 3)), int(a.num("ntheta", 0)), int(a.num("nrho", 0)));
    Plan plan(int(a.num("device", 0)), g);
    Container out;
    out.kind = "sinogram";
    out.rows = g.n_theta;
    out.cols = g.N;
    out.data.resize(std::size_t(g.n_theta) * g.N);
    ck(lpr_gpu_radon_host(plan.p, in.data.data(), out.data.data(), 1), "radon");
    out.grid = lpr::io::sinogram_grid(g.n_theta, g.N);
    out.meta = plan_meta(g);
    lpr::io::write_container(a.str("out"), out);
    return 0;
}

// the plan of an input sinogram: N = its columns, n_theta = its rows
lpr_geometry sino_geometry(const Container& s, const Args& a) {
    const lpr_geometry g = geometry(s.cols, int(a.num("sectors", 3)), s.rows, int(a.num("nrho", 0)));
    if (g.n_theta != s.rows)
        throw std::invalid_argument("sinogram rows (" + std::to_string(s.rows) + ") are not a valid angle count for " +
                                    std::to_string(g.M) + " sectors (a multiple of 2M)");
    return g;
}

Container image_out(const lpr_geometry& g) {
    Container c;
    c.kind = "image";
    c.rows = c.cols = g.N;
    c.data.resize(std::size_t(g.N) * g.N);
    c.grid = lpr::io::image_grid(g.N);
    c.meta = plan_meta(g);
    return c;
}

int cmd_backproject(const Args& a) {
    check_method(a);
    const Container in = need(lpr::io::read_container(a.str("in")), "sinogram");
    const lpr_geometry g = sino_geometry(in, a);
    Plan plan(int(a.num("device", 0)), g);
    Container out = image_out(g);
    ck(lpr_gpu_backproject_host(plan.p, in.data.data(), out.data.data(), 1), "backproject");
    lpr::io::write_container(a.str("out"), out);
    return 0;
}

int cmd_fbp(const Args& a) {
    const Container in = need(lpr::io::read_container(a.str("in")), "sinogram");
    const std::string f = a.str("filter", "ramp");
    const int kind = f == "ramp" ? 0 : f == "shepp-logan" ? 1 : f == "cosine" ? 2 : -1;
    if (kind < 0) throw Usage("--filter must be ramp, shepp-logan or cosine");
    const lpr_geometry g = sino_geometry(in, a);
    Plan plan(int(a.num("device", 0)), g);
    Container out = image_out(g);
    ck(lpr_gpu_fbp_host(plan.p, kind, in.data.data(), out.data.data(), 1), "fbp");
    out.meta["filter"] = f;
    lpr::io::write_container(a.str("out"), out);
    return 0;
}

int cmd_em(const Args& a) {
    const Container in = need(lpr::io::read_container(a.str("in")), "sinogram");
    const int iters = int(a.num("iters", 0, true));
    if (iters < 0) throw std::invalid_argument("--iters must be >= 0");
    const lpr_geometry g = sino_geometry(in, a);
    Plan plan(int(a.num("device", 0)), g);
    Container out = image_out(g);
    std::vector<double> ll(std::size_t(iters > 0 ? iters : 1));
    ck(lpr_gpu_em_host(plan.p, in.data.data(), out.data.data(), 1, iters, 1, iters > 0 ? ll.data() : nullptr), "em");
    out.meta["iters"] = Json(iters);
    out.meta["seed"] = Json(a.num("seed", 0));  // the start is deterministic (1 inside the unit disc)
    Json hist = Json::array();
    for (int k = 0; k < iters; ++k) hist.push_back(Json(ll[std::size_t(k)]));
    out.meta["loglik"] = hist;
    lpr::io::write_container(a.str("out"), out);
    return 0;
}

int cmd_kernel_dump(const Args& a) {
    const std::string k = a.str("kind");
    const int kind = k == "radon" ? 0 : k == "backprojection" ? 1 : -1;
    if (kind < 0) throw Usage("--kind must be radon or backprojection");
    const lpr_geometry g = geometry(int(a.num("size", 0, true)), int(a.num("sectors", 3)), int(a.num("ntheta", 0)),
                                    int(a.num("nrho", 0)));
    std::vector<double> z(std::size_t(2) * 2 * g.nts * g.n_rho);
    ck(lpr_spectrum_quadrature(&g, kind, z.data()), "kernel spectrum");
    Container c;
    c.kind = "spectrum";
    c.complex = true;
    c.rows = 2 * g.nts;
    c.cols = g.n_rho;
    c.data.assign(z.begin(), z.end());  // c32: the fp64 spectrum rounded once
    c.meta = plan_meta(g);
    c.meta["kernel"] = k;
    c.meta["rows"] = "theta frequency, FFT order (2 nts)";
    c.meta["cols"] = "rho frequency, FFT order (n_rho)";
    lpr::io::write_container(a.str("out"), c);
    return 0;
}

int cmd_bench(const Args& a) {
    std::vector<int> sizes;
    {
        const std::string s = a.str("sizes");
        std::size_t i = 0;
        while (i < s.size()) {
            const std::size_t j = s.find(',', i);
            const std::string t = s.substr(i, j == std::string::npos ? std::string::npos : j - i);
            char* end = nullptr;
            const long v = std::strtol(t.c_str(), &end, 10);
            if (t.empty() || !end || *end || v < 8) throw Usage("--sizes expects a comma-separated list of N >= 8");
            sizes.push_back(int(v));
            if (j == std::string::npos) break;
            i = j + 1;
        }
    }
    const int M = int(a.num("sectors", 3)), reps = int(a.num("reps", 5)), dev = int(a.num("device", 0));
    if (reps < 1) throw std::invalid_argument("--reps must be >= 1");
    Json out = Json::object();
    out["tool"] = "lpradon bench";
    Json rows = Json::array();
    for (const int N : sizes) {
        const lpr_geometry g = geometry(N, M, 0, 0);
        Plan plan(dev, g);
        const std::vector<float> img = shepp_logan(N);
        std::vector<float> sino(std::size_t(g.n_theta) * N), back(std::size_t(N) * N);
        ck(lpr_gpu_radon_host(plan.p, img.data(), sino.data(), 1), "radon");  // warm-up
        ck(lpr_gpu_backproject_host(plan.p, sino.data(), back.data(), 1), "backproject");
        const long long f0 = lpr_gpu_fft_count(plan.p);
        using clk = std::chrono::steady_clock;
        auto t0 = clk::now();
        for (int r = 0; r < reps; ++r) ck(lpr_gpu_radon_host(plan.p, img.data(), sino.data(), 1), "radon");
        auto t1 = clk::now();
        const long long f1 = lpr_gpu_fft_count(plan.p);
        for (int r = 0; r < reps; ++r) ck(lpr_gpu_backproject_host(plan.p, sino.data(), back.data(), 1), "backproject");
        auto t2 = clk::now();
        // per-stage device times (CUDA events between the launches on the plan's stream)
        Json stages = Json::object();
        for (int op = 0; op < 2; ++op) {
            double ms[8];
            int ns = 0;
            const char* names[8] = {};
            ck(lpr_gpu_profile_stages_host(plan.p, op, op == 0 ? img.data() : sino.data(), 1, reps, ms, &ns, names),
               "profile");
            Json st = Json::object();
            for (int i = 0; i < ns; ++i) st[names[i]] = Json(ms[i]);
            stages[op == 0 ? "radon" : "backprojection"] = st;
        }
        Json r = Json::object();
        r["N"] = Json(N);
        r["n_theta"] = Json(g.n_theta);
        r["n_rho"] = Json(g.n_rho);
        r["sectors"] = Json(M);
        r["radon_ms"] = Json(std::chrono::duration<double, std::milli>(t1 - t0).count() / reps);
        r["backprojection_ms"] = Json(std::chrono::duration<double, std::milli>(t2 - t1).count() / reps);
        r["timing"] = "wall clock of the host-buffer C-ABI call (copies included), mean of --reps";
        r["fft_count_per_transform"] = Json((f1 - f0) / reps);  // 2M
        r["stages_ms"] = stages;
        rows.push_back(r);
        std::printf("N=%d: R %.3f ms, R# %.3f ms, %lld spectral convolutions per transform\n", N,
                    r.at("radon_ms").as_number(), r.at("backprojection_ms").as_number(), (f1 - f0) / reps);
    }
    out["sizes"] = rows;
    std::FILE* f = std::fopen(a.str("json").c_str(), "w");
    if (!f) throw std::runtime_error("cannot write " + a.str("json"));
    const std::string s = out.dump() + "\n";
    std::fwrite(s.data(), 1, s.size(), f);
    std::fclose(f);
    return 0;
}

// c_norm calibration (SPEC.md:378 DESIGN DECISIONS; the reference's
// tools/calibrate_cnorm.cpp is an empty main): the analytic sinogram of the
// centred disc of physical radius 0.5 (raster radius 1/4, line integral
// 2 sqrt(1/16 - s^2)), filtered back-projected with the built-in c_norm = 1/2;
// the interior mean (physical radius < 0.4) should be 1, and c_norm = 1/2 /
// mean is what the calibration would fix.
int cmd_calibrate_cnorm(const Args& a) {
    const int N = int(a.num("size", 256));
    const std::string f = a.str("filter", "ramp");
    const int kind = f == "ramp" ? 0 : f == "shepp-logan" ? 1 : f == "cosine" ? 2 : -1;
    if (kind < 0) throw Usage("--filter must be ramp, shepp-logan or cosine");
    const lpr_geometry g = geometry(N, int(a.num("sectors", 3)), 0, int(a.num("nrho", 0)));
    Plan plan(int(a.num("device", 0)), g);
    std::vector<float> sino(std::size_t(g.n_theta) * N), img(std::size_t(N) * N);
    for (int i = 0; i < g.n_theta; ++i)
        for (int j = 0; j < N; ++j) {
            const double s = -0.5 + double(j) / N;
            sino[std::size_t(i) * N + j] = std::abs(s) < 0.25 ? float(2.0 * std::sqrt(0.0625 - s * s)) : 0.f;
        }
    ck(lpr_gpu_fbp_host(plan.p, kind, sino.data(), img.data(), 1), "fbp");
    double mean = 0.0;
    long cnt = 0;
    for (int r = 0; r < N; ++r)
        for (int c = 0; c < N; ++c) {
            const double x = -0.5 + double(c) / N, y = -0.5 + double(r) / N;
            if (x * x + y * y < 0.04) mean += img[std::size_t(r) * N + c], ++cnt;
        }
    mean /= double(cnt);
    Json out = Json::object();
    out["N"] = Json(N);
    out["filter"] = f;
    out["c_norm_builtin"] = Json(0.5);
    out["interior_mean"] = Json(mean);
    out["c_norm_calibrated"] = Json(0.5 / mean);
    out["within_spec"] = Json(std::abs(mean - 1.0) <= 0.05);  // mean in [0.95, 1.05]
    std::printf("%s\n", out.dump().c_str());
    return std::abs(mean - 1.0) <= 0.05 ? 0 : 1;
}

int cmd_inspect(const Args& a) {
    const Container c = lpr::io::read_container(a.str("in"));
    Json h = Json::object();
    h["kind"] = c.kind;
    h["rows"] = Json(c.rows);
    h["cols"] = Json(c.cols);
    h["dtype"] = c.complex ? "c32" : "f32";
    h["grid"] = c.grid;
    h["meta"] = c.meta;
    std::printf("%s\n", h.dump().c_str());
    if (a.has("out")) lpr::io::write_container(a.str("out"), c);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fputs(kUsage, stderr);
        return 2;
    }
    const std::string sub = argv[1];
    const std::map<std::string, std::pair<std::set<std::string>, int (*)(const Args&)>> cmds = {
        {"phantom", {{"size", "out"}, cmd_phantom}},
        {"radon", {{"in", "out", "method", "sectors", "ntheta", "nrho"}, cmd_radon}},
        {"backproject", {{"in", "out", "method", "sectors", "nrho"}, cmd_backproject}},
        {"fbp", {{"in", "out", "filter", "sectors", "nrho"}, cmd_fbp}},
        {"em", {{"in", "out", "iters", "seed", "sectors", "nrho"}, cmd_em}},
        {"kernel-dump", {{"size", "sectors", "ntheta", "nrho", "kind", "out"}, cmd_kernel_dump}},
        {"bench", {{"sizes", "json", "sectors", "reps"}, cmd_bench}},
        {"inspect", {{"in", "out"}, cmd_inspect}},
        {"calibrate-cnorm", {{"size", "filter", "sectors", "nrho"}, cmd_calibrate_cnorm}},
    };
    auto it = cmds.find(sub);
    if (it == cmds.end()) {
        std::fprintf(stderr, "lpradon: unknown subcommand '%s'\n%s", sub.c_str(), kUsage);
        return 2;
    }
    try {
        return it->second.second(parse(argc, argv, it->second.first));
    } catch (const Usage& e) {
        std::fprintf(stderr, "lpradon %s: %s\n%s", sub.c_str(), e.what(), kUsage);
        return 2;
    } catch (const lpr::io::BadMagicError& e) {  // the four container errors: distinct classes and exit codes
        std::fprintf(stderr, "lpradon %s: BadMagicError: %s\n", sub.c_str(), e.what());
        return 3;
    } catch (const lpr::io::TruncatedError& e) {
        std::fprintf(stderr, "lpradon %s: TruncatedError: %s\n", sub.c_str(), e.what());
        return 4;
    } catch (const lpr::io::ShapeError& e) {
        std::fprintf(stderr, "lpradon %s: ShapeError: %s\n", sub.c_str(), e.what());
        return 5;
    } catch (const lpr::io::SchemaError& e) {
        std::fprintf(stderr, "lpradon %s: SchemaError: %s\n", sub.c_str(), e.what());
        return 6;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "lpradon %s: %s\n", sub.c_str(), e.what());
        return 1;
    }
}
