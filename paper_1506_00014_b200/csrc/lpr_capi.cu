// C ABI (include/lpradon_gpu.h): plan construction, table upload and the
// launch sequences of R, R# and R^T. Host orchestration only; the compute
// is in lpr_kernels.cu / lpr_transpose.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <complex>
#include <mutex>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "lpr_host.hpp"
#include "lpr_em.cuh"
#include "lpr_kernels.cuh"
#include "lpradon_gpu.h"

namespace lpr {

// plan-time spectra on the GPU (lpr_spectrum.cu)
void spectrum_gpu(int device, const lpr_geometry& g, int kind, double* out);
void rho_pad_multipliers(int device, int rows, int n, int nb, const double* mult, float2* d_out);

// kernels (lpr_kernels.cu, lpr_transpose.cu)
__global__ void k_radon_out_T(DevGeom g, const float* sino, float* lp);
__global__ void k_prefilter_cols_T(DevGeom g, const float* band, int H, const float* qbar, float* tmp);
__global__ void k_prefilter_rows_T(DevGeom g, const float* band, int H, const float* tmp, float* img, float scale);

namespace {

thread_local std::string g_last_error;

struct Error : std::runtime_error {
    lpr_status code;
    Error(lpr_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    cudaGetLastError();  // a non-sticky error must not resurface at the next launch check
    const lpr_status c = e == cudaErrorMemoryAllocation ? LPR_ERR_OOM : LPR_ERR_CUDA;
    throw Error(c, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return LPR_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return LPR_ERR_ARG;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LPR_ERR_CUDA;
    }
}

using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;

std::vector<int> radices(long n) {
    std::vector<int> r;
    for (int f : {8, 4, 2, 3, 5, 7})
        while (n % f == 0) {
            r.push_back(f);
            n /= f;
        }
    if (n != 1) r.clear();
    return r;
}

long smooth_at_least(long n) {
    while (radices(n).empty()) ++n;
    return n;
}

// Host mixed-radix DFT (fp64) for the Bluestein kernel transform.
void host_fft(std::vector<cd>& x) {
    const long n = long(x.size());
    if (n == 1) return;
    long p = 0;
    for (long f : {2L, 3L, 5L, 7L})
        if (n % f == 0) {
            p = f;
            break;
        }
    if (p == 0) throw std::logic_error("host_fft: length not 7-smooth");
    const long m = n / p;
    std::vector<std::vector<cd>> sub(p, std::vector<cd>(m));
    for (long r = 0; r < p; ++r)
        for (long j = 0; j < m; ++j) sub[r][j] = x[j * p + r];
    for (auto& s : sub) host_fft(s);
    for (long k = 0; k < n; ++k) {
        cd acc = 0;
        for (long r = 0; r < p; ++r) acc += sub[r][k % m] * std::polar(1.0, -2.0 * kPi * double(r * k % n) / double(n));
        x[k] = acc;
    }
}


}  // namespace
}  // namespace lpr

using namespace lpr;

#ifndef LPR_HOST_CHUNKS
#define LPR_HOST_CHUNKS 8  // pipeline depth of the pinned host path (chunks per call)
#endif
#ifndef LPR_HOST_SLOTS
#define LPR_HOST_SLOTS 4  // device staging slots of the pinned host path
#endif

struct lpr_gpu_plan {
    int device = 0;
    lpr_geometry geo{};
    int max_batch = 1;
    DevGeom g{};
    FftDesc d_fine{}, d_rho{}, d_coarse{}, d_filt{};
    FftLaunch l_fine{}, l_rho{}, l_coarse{}, l_filt{};
    float* filt_tab = nullptr;  // 2 x 3 transfer functions of length 2N: [fbp?][kind][k], / 2N (fbp: x c_norm)
    float* fsino = nullptr;     // filtered sinograms for fbp
    float2* mult_R = nullptr;
    float2* mult_B = nullptr;
    float2* mult_RT = nullptr;   // conj(mult_R): the transposed rho multiplier
    int rho_pad = 0;             // padded rho-convolution length (non-smooth N_rho), 0: none
    bool rho_direct = false;     // N_rho == that compile-time length: same kernel, plain multipliers
    bool rho_pad_gen = false;    // rho_pad without a compile-time padded kernel: k_rho_pad_gen over d_rho_pad
    FftDesc d_rho_pad{};
    FftLaunch l_rho_pad{};
    float2 *pad_R = nullptr, *pad_B = nullptr, *pad_RT = nullptr;  // its multipliers, (nts + 1) x rho_pad
    float2* lpc_mult = nullptr;  // lp_convolve: the call's multipliers ((nts + 1) x (rho_pad or n_rho))
    float* lpc_out = nullptr;    // lp_convolve: theta-inverse output, max_batch x 2 nts x lps
    float *lpc_din = nullptr, *lpc_dout = nullptr;  // lp_convolve host path: device staging, max_batch rasters each
    float* band = nullptr;       // banded transpose of the apron-extended 1-D prefilter
    int band_h = 0;
    float *qf = nullptr, *tmp = nullptr, *qg = nullptr, *lp = nullptr;
    Tap* q4 = nullptr;  // coefficient raster read by the R gather; qf aliases it as the R^T scatter target
    Tap* q4t = nullptr; // transposed quad raster for sector 0
    float2* spec = nullptr;
    float *d_in = nullptr, *d_out = nullptr;   // staging for the *_host entry points
    float *h_in = nullptr, *h_out = nullptr;   // pinned
    cudaStream_t stream = nullptr;
    cudaStream_t s_in = nullptr, s_out = nullptr;  // host-path copy streams
    static constexpr int kHostChunks = LPR_HOST_CHUNKS;  // chunks per host call (round 2, 4 paired runs: 8 -> 949 vs 16 -> 921 e2e slices/s)
    // Calls share the scratch above, so they are serialised: the mutex covers
    // the host side of a call (enqueue, host staging), and ev_done, recorded on
    // the stream of the call that last used the scratch, orders its device work
    // before the next call's (which may come on another stream).
    std::recursive_mutex mu;
    cudaEvent_t ev_done = nullptr;
    bool has_done = false;
    static constexpr int kHostSlots = LPR_HOST_SLOTS;  // device staging slots of the pinned host pipeline
    cudaEvent_t ev_h2d[kHostSlots] = {}, ev_comp[kHostSlots] = {}, ev_d2h[kHostSlots] = {};
    cudaEvent_t ev_mid[kHostSlots] = {};  // R done in a slot (radon_backproject_host: its sinograms may go out)
    float* d_back = nullptr;              // radon_backproject_host: back-projection staging (max_batch images)
    cudaEvent_t* prof = nullptr;  // per-stage profiling events (lpr_gpu_profile_stages)
    bool tex_gather = false;      // LPR_PLAN_TEXTURE_GATHER ablation
    int tex_mode = 0;             // gather path of the R fine grid: 0 quad taps, 1 hardware bilinear (ablation)
    cudaTextureObject_t qtex = 0;
    cudaTextureObject_t lptex = 0;  // tld4 view of lp for the R# output resampling (0: direct loads)
    std::vector<void*> allocs;
    long long launches = 0, ffts = 0;
    // EM state (allocated on first use): Rf / ratio sinograms, R# images, the
    // inverted sensitivity R# chi_C, per-slice max g, flags, log-likelihoods
    float *em_rf = nullptr, *em_bp = nullptr, *em_inv_sens = nullptr, *em_gmax = nullptr;
    int* em_bad = nullptr;

    template <class T>
    T* dalloc(size_t count) {
        void* p = nullptr;
        ck(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
    template <class T>
    T* upload(const std::vector<T>& v) {
        T* p = dalloc<T>(v.size());
        ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
        return p;
    }

    // staged_row: the rho pass also stages one multiplier row (n float2) in shared memory
    void build_desc(long n, FftDesc& d, FftLaunch& launch, bool staged_row = false) {
        d = FftDesc{};
        d.n = int(n);
        auto rad = radices(n);
        auto twiddles = [&](long len) {
            std::vector<float2> tw(len);
            for (long j = 0; j < len; ++j) {
                const double a = -2.0 * kPi * double(j) / double(len);
                tw[j] = make_float2(float(std::cos(a)), float(std::sin(a)));
            }
            return upload(tw);
        };
        if (!rad.empty()) {
            if (rad.size() > size_t(kMaxPasses)) throw std::invalid_argument("fft: too many passes");
            d.npass = int(rad.size());
            std::copy(rad.begin(), rad.end(), d.radix);
            d.tw = twiddles(n);
        } else {
            const long nb = smooth_at_least(2 * n - 1);
            auto brad = radices(nb);
            d.nb = int(nb);
            d.nbpass = int(brad.size());
            std::copy(brad.begin(), brad.end(), d.bradix);
            d.btw = twiddles(nb);
            std::vector<float2> chirp(n);
            std::vector<cd> kern(nb, cd(0.0));
            for (long j = 0; j < n; ++j) {
                const long jj = (j * j) % (2 * n);
                const cd c = std::polar(1.0, -kPi * double(jj) / double(n));
                chirp[j] = make_float2(float(c.real()), float(c.imag()));
                kern[j] = std::conj(c);
                if (j) kern[nb - j] = std::conj(c);
            }
            host_fft(kern);
            std::vector<float2> bh(nb);
            for (long j = 0; j < nb; ++j) bh[j] = make_float2(float(kern[j].real() / nb), float(kern[j].imag() / nb));
            d.chirp = upload(chirp);
            d.bhat = upload(bh);
        }
        launch = fft_launch_config(d);
        if (launch.variant != kFftGeneric) d.twp = upload(fft_pass_twiddles(launch.variant));
        // rho pass: the TMA-streamed kernel where one exists for this length
        if (staged_row && rho_stream_smem(launch.variant) > 0 && (n * sizeof(float2)) % 16 == 0) {
            d.twp_sfwd = upload(rho_stream_fwd_twiddles(launch.variant));
            d.twp_inv = upload(rho_stream_inv_twiddles(launch.variant));
            launch.rho_stream = 1;
        }
        // a non-smooth rho length runs padded (k_rho_pad / k_rho_pad_gen), never through this descriptor
        const bool padded = staged_row && launch.variant == kFftGeneric && d.nb != 0;
        if (!padded && (launch.smem * launch.per_block > 227 * 1024 ||
                        (staged_row && launch.smem + size_t(n) * sizeof(float2) > 227 * 1024)))
            throw std::invalid_argument("fft: a length-" + std::to_string(n) + " transform does not fit in shared memory (for a non-7-smooth n_rho this large, use the 7-smooth plan: lpr_smooth_n_rho)");
    }

    ~lpr_gpu_plan() {
        if (qtex) cudaDestroyTextureObject(qtex);
        if (lptex) cudaDestroyTextureObject(lptex);
        for (void* p : allocs) cudaFree(p);
        if (h_in) cudaFreeHost(h_in);
        if (h_out) cudaFreeHost(h_out);
        for (int i = 0; i < kHostSlots; ++i) {
            if (ev_h2d[i]) cudaEventDestroy(ev_h2d[i]);
            if (ev_comp[i]) cudaEventDestroy(ev_comp[i]);
            if (ev_d2h[i]) cudaEventDestroy(ev_d2h[i]);
            if (ev_mid[i]) cudaEventDestroy(ev_mid[i]);
        }
        if (ev_done) cudaEventDestroy(ev_done);
        if (s_in) cudaStreamDestroy(s_in);
        if (s_out) cudaStreamDestroy(s_out);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

void set_smem(const void* fn, size_t bytes) {
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)), "smem attribute");
}

inline int cdiv(long a, long b) { return int((a + b - 1) / b); }

void check_launch(const char* what) { ck(cudaGetLastError(), what); }

void init_plan(lpr_gpu_plan* p, const double* zeta, const double* zeta_bp) {
    const lpr_geometry& G = p->geo;
    if (G.M > kMaxSectors) throw std::invalid_argument("plan: M above the device limit");
    ck(cudaSetDevice(p->device), "cudaSetDevice");
    int major = 0;
    ck(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, p->device), "device query");
    if (major < 10) throw Error(LPR_ERR_CUDA, "plan: the kernels are built for sm_100a (B200)");
    DevGeom& g = p->g;
    g.N = G.N;
    g.M = G.M;
    g.n_theta = G.n_theta;
    g.nts = G.nts;
    g.n_rho = G.n_rho;
    g.refine = G.refine;
    g.nf = G.refine * G.nts;
    g.Lf = 2 * g.nf;
    g.L2 = 2 * G.nts;
    g.win = G.nts + 8;
    g.lps = lp_stride(G.n_rho);
    g.j0 = -G.nts / 2 - 4;
    g.pitch = G.N + 2 * kApron;
    g.aR = float(G.a_R);
    g.inv_aR = float(1.0 / G.a_R);
    g.one_m_aR = float(1.0 - G.a_R);
    g.aR2 = float(G.a_R * G.a_R);
    g.log_ar = float(G.log_ar);
    g.inv_drho = float(1.0 / G.drho);
    g.inv_dtheta_p = float(1.0 / G.dtheta_p);
    g.out_scale = float(1.0 / (2.0 * G.a_R));
    g.mask_k = float(1.0 - 2.0 * G.a_R);
    for (int m = 0; m < G.M; ++m) {
        g.cosm[m] = float(std::cos(m * G.beta));
        g.sinm[m] = float(std::sin(m * G.beta));
        g.vcm[m] = float(0.5 * G.N * (1.0 - std::cos(m * G.beta) * (1.0 - G.a_R) / G.a_R));
        g.vrm[m] = float(0.5 * G.N * (1.0 - std::sin(m * G.beta) * (1.0 - G.a_R) / G.a_R));
    }
    std::vector<float> fc(g.nf), fs(g.nf), cc(G.nts), er(G.n_rho), fir(2 * kFirHalf + 1);
    for (int i = 0; i < g.nf; ++i) {
        const double th = double(i - g.nf / 2) * G.dtheta_lp;
        fc[i] = float(std::cos(th));
        fs[i] = float(std::sin(th));
    }
    for (int jj = 0; jj < G.nts; ++jj) cc[jj] = float(std::cos(double(jj - G.nts / 2) * G.dtheta_p));
    for (int l = 0; l < G.n_rho; ++l) er[l] = float(std::exp(G.log_ar + double(l) * G.drho));
    const double z = std::sqrt(3.0) - 2.0;
    for (int d = -kFirHalf; d <= kFirHalf; ++d) fir[d + kFirHalf] = float(std::sqrt(3.0) * std::pow(z, std::abs(d)));
    g.fine_cos = p->upload(fc);
    g.fine_sin = p->upload(fs);
    g.coarse_cos = p->upload(cc);
    g.erho = p->upload(er);
    g.fir = p->upload(fir);

    p->build_desc(g.Lf, p->d_fine, p->l_fine);
    {  // row rotations of the fused fine first pass (k_radon_theta_fwd)
        const int r1 = fft_first_radix(p->l_fine.variant);
        g.fine_b1 = 0;
        if (r1 > 0 && g.Lf % r1 == 0 && r1 / 2 <= 16) {
            g.fine_b1 = g.Lf / r1;
            for (int j = 0; j < 16; ++j) {
                const double a = double(j) * g.fine_b1 * G.dtheta_lp;
                g.fine_rot[j] = make_float2(float(std::cos(a)), float(std::sin(a)));
            }
        }
    }
    p->build_desc(G.n_rho, p->d_rho, p->l_rho, true);
    p->build_desc(g.L2, p->d_coarse, p->l_coarse);
    p->build_desc(2L * G.N, p->d_filt, p->l_filt);

    // spectral multipliers on the half theta spectrum k in [0, nts]
    const long nts = G.nts, nr = G.n_rho, rows = 2 * nts;
    std::vector<double> zbuf, zbbuf;
    auto computed = [&](int kind, std::vector<double>& buf) {  // on-disk cache, else the GPU quadrature
        buf.resize(2 * rows * nr);
        if (!host::spectrum_cache_load(G, kind, buf.data())) {
            spectrum_gpu(p->device, G, kind, buf.data());
            host::spectrum_cache_store(G, kind, buf.data());
        }
        return buf.data();
    };
    if (!zeta) zeta = computed(0, zbuf);
    if (!zeta_bp) zeta_bp = computed(1, zbbuf);
    auto bhat = [](long k, long n) { return (2.0 + std::cos(2.0 * kPi * double(k) / double(n))) / 3.0; };
    std::vector<float2> mr((nts + 1) * nr), mb((nts + 1) * nr);
    const double sr = 1.0 / (double(g.Lf) * double(nr)), sb = 1.0 / (double(rows) * double(nr));
    for (long k = 0; k <= nts; ++k)
        for (long v = 0; v < nr; ++v) {
            const long i = k * nr + v;
            if (k == nts) {
                mr[i] = mb[i] = make_float2(0.f, 0.f);
                continue;
            }
            const cd zr(zeta[2 * i], zeta[2 * i + 1]), zb(zeta_bp[2 * i], zeta_bp[2 * i + 1]);
            const cd a = zr * (sr / bhat(v, nr));                  // theta Bhat cancels at lattice rows
            const cd b = zb * (sb / (bhat(k, rows) * bhat(v, nr)));
            mr[i] = make_float2(float(a.real()), float(a.imag()));
            mb[i] = make_float2(float(b.real()), float(b.imag()));
        }
    p->mult_R = p->upload(mr);
    p->mult_B = p->upload(mb);
    for (auto& v : mr) v.y = -v.y;
    p->mult_RT = p->upload(mr);
    // non-7-smooth N_rho with a compile-time padded plan: the rho pass runs as a
    // zero-padded linear convolution (k_rho_pad) with these padded multipliers
    p->rho_pad = p->l_rho.variant == kFftGeneric ? int(rho_pad_length(int(nr))) : 0;
    // N_rho equal to the padded plan's length (8748: the N = 4096 bench plan):
    // the same compile-time kernel runs the circular convolution directly with
    // the plain multipliers (no padding)
    p->rho_direct = p->l_rho.variant == kFftGeneric && rho_direct_length() == size_t(nr);
    if (p->rho_direct) ck(prepare_rho_pad(), "rho pad smem attribute");
    // a runtime-radix length within a factor ~2 of the compile-time 4374 = 2 3^7 (e.g. 2187 = 3^7,
    // the N = 1024 plans) also runs padded: the compile-time transform of twice the length measured
    // faster than the runtime Stockham (R# at N = 1024: 1.70e-4 -> 1.54e-4 s per slice)
    const bool near_ct = 2 * nr - 1 <= 4374 && 4374 <= 2.05 * double(nr);
    if (p->l_rho.variant == kFftGeneric && !p->rho_pad && !p->rho_direct && (p->d_rho.nb != 0 || near_ct)) {
        // any other non-smooth N_rho (Bluestein otherwise): padded over the next 7-smooth length
        p->rho_pad = near_ct ? 4374 : int(smooth_at_least(2 * nr - 1));
        p->rho_pad_gen = true;
        p->build_desc(p->rho_pad, p->d_rho_pad, p->l_rho_pad);  // one row per block, multiplier from L2
        ck(prepare_rho_pad_gen(p->l_rho_pad, p->rho_pad), "rho pad smem attribute");
    }
    if (p->rho_pad) {
        const long rr = nts + 1, nb = p->rho_pad;
        std::vector<double> m64(2 * rr * nr);
        auto build = [&](int which) {  // 0: R, 1: R#, 2: R^T (conjugate of R's)
            for (long k = 0; k <= nts; ++k)
                for (long v = 0; v < nr; ++v) {
                    const long i = k * nr + v;
                    cd z(0.0, 0.0);
                    if (k < nts) {
                        if (which == 1) z = cd(zeta_bp[2 * i], zeta_bp[2 * i + 1]) * (sb / (bhat(k, rows) * bhat(v, nr)));
                        else z = cd(zeta[2 * i], zeta[2 * i + 1]) * (sr / bhat(v, nr));
                        if (which == 2) z = std::conj(z);
                    }
                    m64[2 * i] = z.real();
                    m64[2 * i + 1] = z.imag();
                }
        };
        float2** dst[3] = {&p->pad_R, &p->pad_B, &p->pad_RT};
        for (int w = 0; w < 3; ++w) {
            build(w);
            *dst[w] = p->dalloc<float2>(size_t(rr) * nb);
            rho_pad_multipliers(p->device, int(rr), int(nr), int(nb), m64.data(), *dst[w]);
        }
        if (!p->rho_pad_gen) ck(prepare_rho_pad(), "rho pad smem attribute");
    }

    // FBP transfer functions: DFT of the band-limited discrete
    // ramp kernel h(0) = 1/(4 ds^2), h(odd n) = -1/(n pi ds)^2 times ds, windowed
    // by sinc(sigma/N) (Shepp-Logan) or cos(pi sigma/N) (cosine); / 2N for the
    // unnormalised inverse; the fbp copy also carries c_norm = 1/2 (R# integrates
    // over all lines, the inversion over a half turn).
    {
        const long N = G.N, L = 2 * N;
        const double ds = 1.0 / double(N);
        std::vector<double> h(L, 0.0), ramp(L, 0.0);
        for (long n = 0; n < L; ++n) {
            const long lag = n < N ? n : n - L;
            if (lag == 0) h[n] = 1.0 / (4.0 * ds * ds);
            else if (lag % 2) h[n] = -1.0 / ((kPi * double(lag) * ds) * (kPi * double(lag) * ds));
        }
        for (long k = 0; k < L; ++k) {  // real, even kernel: cosine transform
            double acc = 0.0;
            for (long n = 0; n < L; ++n) acc += h[n] * std::cos(2.0 * kPi * double((k * n) % L) / double(L));
            ramp[k] = acc * ds;
        }
        std::vector<float> tab(6 * L);
        for (int kind = 0; kind < 3; ++kind)
            for (long k = 0; k < L; ++k) {
                const double sigma = double(k <= N ? k : L - k) / (double(L) * ds);
                double w = 1.0;
                if (kind == 1) {
                    const double x = sigma / double(N);
                    w = x == 0.0 ? 1.0 : std::sin(kPi * x) / (kPi * x);
                } else if (kind == 2) {
                    w = std::cos(kPi * sigma / double(N));
                }
                const double v = ramp[k] * w / double(L);
                tab[kind * L + k] = float(v);
                tab[(3 + kind) * L + k] = float(0.5 * v);
            }
        p->filt_tab = p->upload(tab);
    }

    // Q1 (pitch x N): apron-extended FIR prefilter as the forward kernels apply
    // it (fp32 taps); band[c][j] = Q1[c + A - H + j][c] holds its transpose.
    {
        const int N = G.N, pitch = g.pitch, H = kFirHalf + kApron + 8;
        auto mir = [](int i, int n) {
            if (n == 1) return 0;
            const int per = 2 * (n - 1);
            int r = i % per;
            if (r < 0) r += per;
            return r >= n ? per - r : r;
        };
        std::vector<double> q1(size_t(pitch) * N, 0.0);
        for (int cp = 0; cp < pitch; ++cp)
            for (int d = -kFirHalf; d <= kFirHalf; ++d)
                q1[size_t(cp) * N + mir(mir(cp - kApron, N) + d, N)] += double(fir[d + kFirHalf]);
        std::vector<float> band(size_t(N) * (2 * H + 1), 0.f);
        for (int cp = 0; cp < pitch; ++cp)
            for (int c = 0; c < N; ++c) {
                const double v = q1[size_t(cp) * N + c];
                if (v == 0.0) continue;
                const int j = cp - (c + kApron - H);
                if (j < 0 || j > 2 * H) throw std::invalid_argument("plan: prefilter transpose band too narrow for N");
                band[size_t(c) * (2 * H + 1) + j] = float(v);
            }
        p->band = p->upload(band);
        p->band_h = H;
    }

    const size_t B = size_t(p->max_batch);
    p->tmp = p->dalloc<float>(B * G.N * g.pitch);
    p->q4 = p->dalloc<Tap>(B * g.pitch * g.pitch);
    if (p->tex_mode == 0) p->q4t = p->dalloc<Tap>(B * g.pitch * g.pitch);
    p->qf = reinterpret_cast<float*>(p->q4);
    p->qg = p->dalloc<float>(B * G.n_theta * G.N);
    p->fsino = p->dalloc<float>(B * G.n_theta * G.N);
    p->spec = p->dalloc<float2>(B * G.M * (nts + 1) * nr);
    p->lp = p->dalloc<float>(B * G.M * g.win * size_t(g.lps));
    const size_t io = B * std::max<size_t>(size_t(G.N) * G.N, size_t(G.n_theta) * G.N);
    p->d_in = p->dalloc<float>(io);
    p->d_out = p->dalloc<float>(io);
    ck(cudaHostAlloc(&p->h_in, io * sizeof(float), cudaHostAllocDefault), "cudaHostAlloc");
    ck(cudaHostAlloc(&p->h_out, io * sizeof(float), cudaHostAllocDefault), "cudaHostAlloc");
    ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming), "cudaEventCreate");
    for (int i = 0; i < lpr_gpu_plan::kHostSlots; ++i) {
        ck(cudaEventCreateWithFlags(&p->ev_h2d[i], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&p->ev_d2h[i], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&p->ev_mid[i], cudaEventDisableTiming), "cudaEventCreate");
    }

    ck(prepare_filter_kernel(p->l_filt), "filter smem attribute");
    {
        // a plan whose rho pass runs in k_rho_pad never launches the generic rho kernel
        // (whose Bluestein buffer would not fit, e.g. N_rho = 8666)
        FftLaunch lr = p->l_rho;
        const bool padded = p->rho_pad || p->rho_direct;
        if (padded) lr.smem = 0;
        ck(prepare_fft_kernels(p->l_fine, lr, p->l_coarse, padded ? 0 : size_t(G.n_rho) * sizeof(float2)),
           "fft smem attributes");
    }
    if (p->tex_mode) {
        // the plain coefficient rasters of the whole batch as one tall pitched
        // 2-D texture with hardware bilinear filtering
        int align = 0;
        ck(cudaDeviceGetAttribute(&align, cudaDevAttrTexturePitchAlignment, p->device), "device query");
        const size_t pitch_bytes = size_t(g.pitch) * sizeof(float);
        if (align <= 0 || pitch_bytes % size_t(align) != 0)
            throw std::invalid_argument("texture gather: image row pitch not texture-aligned (use N divisible by 8)");
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypePitch2D;
        rd.res.pitch2D.devPtr = p->qf;
        rd.res.pitch2D.desc = cudaCreateChannelDesc<float>();
        rd.res.pitch2D.width = size_t(g.pitch);
        rd.res.pitch2D.height = size_t(g.pitch) * B;
        rd.res.pitch2D.pitchInBytes = pitch_bytes;
        cudaTextureDesc td{};
        td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModeLinear;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        ck(cudaCreateTextureObject(&p->qtex, &rd, &td, nullptr), "cudaCreateTextureObject");
        p->g.qtex = p->qtex;
    }
    {
        // R# output resampling taps through the texture path (four exact tld4
        // gathers per sample instead of 16 scalar loads; measured 1.51 -> 1.11 ms
        // per 16 slices), when the window buffer fits one pitched 2-D texture
        const size_t h = size_t(B) * G.M * g.win;
        int max_h = 0, max_w = 0;
        ck(cudaDeviceGetAttribute(&max_h, cudaDevAttrMaxTexture2DLinearHeight, p->device), "device query");
        ck(cudaDeviceGetAttribute(&max_w, cudaDevAttrMaxTexture2DLinearWidth, p->device), "device query");
        if (h <= size_t(max_h) && g.lps <= max_w) {
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypePitch2D;
            rd.res.pitch2D.devPtr = p->lp;
            rd.res.pitch2D.desc = cudaCreateChannelDesc<float>();
            rd.res.pitch2D.width = size_t(g.lps);
            rd.res.pitch2D.height = h;
            rd.res.pitch2D.pitchInBytes = size_t(g.lps) * sizeof(float);
            cudaTextureDesc td{};
            td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
            td.filterMode = cudaFilterModePoint;
            td.readMode = cudaReadModeElementType;
            ck(cudaCreateTextureObject(&p->lptex, &rd, &td, nullptr), "cudaCreateTextureObject(lp)");
            p->g.lptex = p->lptex;
        }
    }
    ck(prepare_out_kernels(g.lps), "cudaFuncSetAttribute(out kernels)");
    ck(prepare_prefilter_sino(), "cudaFuncSetAttribute(prefilter_sino)");
    set_smem((const void*)k_radon_out_T, size_t(nr) * sizeof(float));

}

// The rho convolution of every (k_theta, item) row: which = 0 (R), 1 (R#), 2 (R^T).
void rho_chunk(lpr_gpu_plan* p, int which, int nb, cudaStream_t st, const DevGeom& g, float2* spec) {
    const dim3 grid(g.nts + 1, nb * g.M);
    if (p->rho_pad) {
        const float2* m = which == 0 ? p->pad_R : which == 1 ? p->pad_B : p->pad_RT;
        if (p->rho_pad_gen)
            launch_rho_pad_gen(p->l_rho_pad, grid, st, g, p->d_rho_pad, m, spec);
        else
            launch_rho_pad(p->rho_pad, grid, st, g, m, spec);
        return;
    }
    if (p->rho_direct) {
        launch_rho_pad(int(rho_direct_length()), grid, st, g, which == 0 ? p->mult_R : which == 1 ? p->mult_B : p->mult_RT, spec);
        return;
    }
    launch_rho_pass(p->l_rho, grid, st, g, p->d_rho, which == 0 ? p->mult_R : which == 1 ? p->mult_B : p->mult_RT, spec);
}

// One call on a plan. Calls share the plan's scratch, so they are serialised
// (ADVICE r1): the plan mutex is held for the whole host side of the call, and
// the call's stream first waits for the device work of the previous call
// (ev_done, recorded on whichever stream that call used), so a device call on
// a user stream and a host call on the plan's own stream cannot overlap on
// the same buffers.
struct Call {
    lpr_gpu_plan* p;
    cudaStream_t st;
    std::unique_lock<std::recursive_mutex> lk;
    Call(lpr_gpu_plan* plan, cudaStream_t s) : p(plan), st(s), lk(plan->mu) {
        ck(cudaSetDevice(p->device), "cudaSetDevice");
        if (p->has_done) ck(cudaStreamWaitEvent(st, p->ev_done, 0), "cudaStreamWaitEvent");
    }
    ~Call() {
        if (cudaEventRecord(p->ev_done, st) == cudaSuccess) p->has_done = true;
    }
};

// Optional per-stage profiling: when p->prof is set, an event is recorded
// before the first and after every launch (lpr_gpu_profile_stages).
inline void mark(lpr_gpu_plan* p, int i, cudaStream_t st) {
    if (p->prof) ck(cudaEventRecord(p->prof[i], st), "profile event");
}

void radon_chunk(lpr_gpu_plan* p, const float* img, float* sino, int nb, cudaStream_t st) {
    const DevGeom& g = p->g;
    mark(p, 0, st);
    launch_prefilter_2d(p->tex_mode == 0, nb, st, g, img, p->q4, p->q4t);
    mark(p, 1, st);
    launch_radon_theta_fwd(p->l_fine, dim3(cdiv(g.n_rho, 2), g.M, nb), st, g, p->d_fine, p->q4, p->q4t, p->spec,
                           p->tex_mode);
    mark(p, 2, st);
    rho_chunk(p, 0, nb, st, g, p->spec);
    mark(p, 3, st);
    launch_theta_inv(p->l_coarse, dim3(cdiv(g.n_rho, 2), g.M, nb), st, g, p->d_coarse, p->spec, p->lp);
    mark(p, 4, st);
    launch_radon_out(nb, st, g, p->lp, sino);
    mark(p, 5, st);
    check_launch("radon launch");
    p->launches += 5;
    p->ffts += 2LL * g.M * nb;
}
const char* const kRadonStages[] = {"prefilter_2d", "radon_theta_fwd", "rho_pass", "theta_inv", "radon_out"};

void backproject_chunk(lpr_gpu_plan* p, const float* sino, float* img, int nb, cudaStream_t st) {
    const DevGeom& g = p->g;
    mark(p, 0, st);
    launch_prefilter_sino(nb, st, g, sino, p->qg);
    mark(p, 1, st);
    launch_bp_theta_fwd(p->l_coarse, dim3(cdiv(g.n_rho, 2), g.M, nb), st, g, p->d_coarse, p->qg, p->spec);
    mark(p, 2, st);
    rho_chunk(p, 1, nb, st, g, p->spec);
    mark(p, 3, st);
    launch_theta_inv(p->l_coarse, dim3(cdiv(g.n_rho, 2), g.M, nb), st, g, p->d_coarse, p->spec, p->lp);
    mark(p, 4, st);
    launch_bp_out(nb, st, g, p->lp, img);
    mark(p, 5, st);
    check_launch("backprojection launch");
    p->launches += 5;
    p->ffts += 2LL * g.M * nb;
}
void transpose_chunk(lpr_gpu_plan* p, const float* sino, float* img, int nb, cudaStream_t st) {
    if (p->tex_gather) throw std::invalid_argument("radon_transpose: not defined for a texture-gather plan");
    const DevGeom& g = p->g;
    k_radon_out_T<<<dim3(g.n_theta, nb), 256, g.n_rho * sizeof(float), st>>>(g, sino, p->lp);
    launch_theta_fwd_T(p->l_coarse, dim3(cdiv(g.n_rho, 2), g.M, nb), st, g, p->d_coarse, p->lp, p->spec);
    rho_chunk(p, 2, nb, st, g, p->spec);
    ck(cudaMemsetAsync(p->qf, 0, sizeof(float) * size_t(nb) * g.pitch * g.pitch, st), "memset");
    launch_theta_inv_fine_T(p->l_fine, dim3(cdiv(g.n_rho, 2), g.M, nb), st, g, p->d_fine, p->spec, p->qf);
    k_prefilter_cols_T<<<dim3(cdiv(g.pitch, 256), g.N, nb), 256, 0, st>>>(g, p->band, p->band_h, p->qf, p->tmp);
    const float scale = float(2.0 * p->geo.dtheta_p * p->geo.ds * double(g.N) * double(g.N));
    k_prefilter_rows_T<<<dim3(cdiv(g.N, 256), g.N, nb), 256, 0, st>>>(g, p->band, p->band_h, p->tmp, img, scale);
    check_launch("radon transpose launch");
    p->launches += 6;
    p->ffts += 2LL * g.M * nb;
}

// FBP pieces: filter along s, then Algorithm 2.
template <int KIND, bool FBP>
void filter_chunk(lpr_gpu_plan* p, const float* sino, float* out, int nb, cudaStream_t st) {
    const DevGeom& g = p->g;
    const float* H = p->filt_tab + size_t((FBP ? 3 : 0) + KIND) * 2 * g.N;
    launch_sino_filter(p->l_filt, nb * g.n_theta, st, g, p->d_filt, H, sino, out);
    check_launch("filter launch");
    p->launches += 1;
}

template <int KIND>
void fbp_chunk(lpr_gpu_plan* p, const float* sino, float* img, int nb, cudaStream_t st) {
    filter_chunk<KIND, true>(p, sino, p->fsino, nb, st);
    backproject_chunk(p, p->fsino, img, nb, st);
}

const char* const kBackprojectStages[] = {"prefilter_sino", "bp_theta_fwd", "rho_pass", "theta_inv", "bp_out"};

// ---- EM: f+ = f R#(g / max(Rf, eps)) / R#chi_C
void em_buffers(lpr_gpu_plan* p) {
    if (p->em_rf) return;
    const lpr_geometry& G = p->geo;
    p->em_rf = p->dalloc<float>(size_t(p->max_batch) * G.n_theta * G.N);
    p->em_bp = p->dalloc<float>(size_t(p->max_batch) * G.N * G.N);
    p->em_inv_sens = p->dalloc<float>(size_t(G.N) * G.N);
    p->em_gmax = p->dalloc<float>(size_t(p->max_batch) + 1);
    p->em_bad = p->dalloc<int>(1);
    // sensitivity R# chi_C: chi_C = 1 on every bin (|s| <= 1/2 covers the detector)
    cudaStream_t st = p->stream;
    if (p->has_done) ck(cudaStreamWaitEvent(st, p->ev_done, 0), "cudaStreamWaitEvent");  // the scratch is free
    launch_fill(p->em_rf, size_t(G.n_theta) * G.N, 1.f, st);
    backproject_chunk(p, p->em_rf, p->em_bp, 1, st);
    launch_slice_max(p->em_bp, size_t(G.N) * G.N, 1, p->em_gmax, p->em_bad, st);
    launch_sens_invert(G.N, p->em_bp, p->em_gmax, p->em_inv_sens, st);
    check_launch("em sensitivity");
    ck(cudaStreamSynchronize(st), "sync");
}

// iters EM steps on nb slices: f (device, in/out), g (device); ll (device,
// nb x iters doubles, zeroed) receives the log-likelihood of every iterate
// f^1..f^iters (appended after each step).
void em_chunk(lpr_gpu_plan* p, const float* g, float* f, int nb, int iters, double* ll, cudaStream_t st) {
    const lpr_geometry& G = p->geo;
    const size_t ps = size_t(G.n_theta) * G.N, pi = size_t(G.N) * G.N;
    ck(cudaMemsetAsync(p->em_bad, 0, sizeof(int), st), "memset");
    launch_slice_max(g, ps, nb, p->em_gmax, p->em_bad, st);
    radon_chunk(p, f, p->em_rf, nb, st);
    for (int k = 0; k < iters; ++k) {
        // ratio for this step; its pass also scores the current iterate f^k (k >= 1)
        launch_em_ratio(g, p->em_rf, ps, nb, p->em_gmax, k > 0 ? ll + (k - 1) : nullptr, iters, true, st);
        backproject_chunk(p, p->em_rf, p->em_bp, nb, st);
        launch_em_update(f, p->em_bp, p->em_inv_sens, pi, nb, p->em_bad, st);
        radon_chunk(p, f, p->em_rf, nb, st);
    }
    if (iters > 0) launch_em_ratio(g, p->em_rf, ps, nb, p->em_gmax, ll + (iters - 1), iters, false, st);
    check_launch("em launch");
    p->launches += 2 + 3LL * iters;
}

using ChunkFn = void (*)(lpr_gpu_plan*, const float*, float*, int, cudaStream_t);

void run_device(lpr_gpu_plan* p, ChunkFn fn, const float* in, float* out, int batch, size_t in_sz, size_t out_sz,
                void* stream) {
    if (!p) throw std::invalid_argument("null plan");
    if (batch < 0 || (batch > 0 && (!in || !out))) throw std::invalid_argument("bad buffers or batch");
    ck(cudaSetDevice(p->device), "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Call call(p, st);
    for (int b0 = 0; b0 < batch; b0 += p->max_batch) {
        const int nb = std::min(p->max_batch, batch - b0);
        fn(p, in + size_t(b0) * in_sz, out + size_t(b0) * out_sz, nb, st);
    }
}

// lp_convolve on nb doubled-grid rasters with the
// multipliers set in p->lpc_mult: theta FFT -> rho pass -> Hermitian theta
// inverse over all 2 nts rows -> compaction to row stride n_rho.
void lpc_chunk(lpr_gpu_plan* p, const float* in, float* out, int nb, cudaStream_t st) {
    DevGeom g = p->g;
    g.M = 1;  // one item per raster
    const int nr = g.n_rho, rows = g.L2;
    launch_lpc_theta_fwd(p->l_coarse, dim3(cdiv(nr, 2), 1, nb), st, g, p->d_coarse, in, p->spec);
    const dim3 grid(g.nts + 1, nb);
    if (p->rho_pad_gen)
        launch_rho_pad_gen(p->l_rho_pad, grid, st, g, p->d_rho_pad, p->lpc_mult, p->spec);
    else if (p->rho_pad)
        launch_rho_pad(p->rho_pad, grid, st, g, p->lpc_mult, p->spec);
    else if (p->rho_direct)
        launch_rho_pad(int(rho_direct_length()), grid, st, g, p->lpc_mult, p->spec);
    else
        launch_rho_pass(p->l_rho, grid, st, g, p->d_rho, p->lpc_mult, p->spec);
    g.win = rows;  // every row of the period, in natural order
    g.j0 = 0;
    launch_theta_inv(p->l_coarse, dim3(cdiv(nr, 2), 1, nb), st, g, p->d_coarse, p->spec, p->lpc_out);
    ck(cudaMemcpy2DAsync(out, size_t(nr) * sizeof(float), p->lpc_out, size_t(g.lps) * sizeof(float),
                         size_t(nr) * sizeof(float), size_t(rows) * nb, cudaMemcpyDeviceToDevice, st),
       "lp_convolve compaction");
    check_launch("lp_convolve launch");
    p->launches += 3;
    p->ffts += nb;
}

bool is_pinned(const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Host-buffer path. With pinned user buffers the batch is cut into chunks
// that flow through a three-stream pipeline (H2D of chunk i+1 and D2H of
// chunk i-1 overlap the compute of chunk i; two device slots, events order
// slot reuse). Pageable buffers are staged through the plan's pinned buffers
// one chunk at a time.
void run_host(lpr_gpu_plan* p, ChunkFn fn, const float* hin, float* hout, int batch, size_t in_sz, size_t out_sz) {
    if (!p) throw std::invalid_argument("null plan");
    if (batch < 0 || (batch > 0 && (!hin || !hout))) throw std::invalid_argument("bad buffers or batch");
    ck(cudaSetDevice(p->device), "cudaSetDevice");
    const bool pin_in = is_pinned(hin), pin_out = is_pinned(hout);
    cudaStream_t st = p->stream;
    const Call call(p, st);
    if (pin_in && pin_out && batch > 1 && p->max_batch > 1) {
        // ~8 chunks: the exposed pipeline fill (first H2D) and drain (last D2H) shrink with the chunk
        const int c = std::max(1, std::min(p->max_batch / 2, (batch + lpr_gpu_plan::kHostChunks - 1) / lpr_gpu_plan::kHostChunks));
        const int chunks = (batch + c - 1) / c;
        // up to kHostSlots chunks in flight: a copy waits only for the compute
        // (or D2H) of the chunk kHostSlots back, so jitter from other work on
        // the device or the link (a concurrent call on another plan) is absorbed
        const int slots = std::min(lpr_gpu_plan::kHostSlots, p->max_batch / c);
        for (int i = 0; i < chunks; ++i) {
            const int slot = i % slots, b0 = i * c, nb = std::min(c, batch - b0);
            float* din = p->d_in + size_t(slot) * c * in_sz;
            float* dout = p->d_out + size_t(slot) * c * out_sz;
            if (i >= slots) ck(cudaStreamWaitEvent(p->s_in, p->ev_comp[slot], 0), "wait");
            ck(cudaMemcpyAsync(din, hin + size_t(b0) * in_sz, size_t(nb) * in_sz * sizeof(float),
                               cudaMemcpyHostToDevice, p->s_in), "H2D");
            ck(cudaEventRecord(p->ev_h2d[slot], p->s_in), "event");
            ck(cudaStreamWaitEvent(st, p->ev_h2d[slot], 0), "wait");
            if (i >= slots) ck(cudaStreamWaitEvent(st, p->ev_d2h[slot], 0), "wait");
            fn(p, din, dout, nb, st);
            ck(cudaEventRecord(p->ev_comp[slot], st), "event");
            ck(cudaStreamWaitEvent(p->s_out, p->ev_comp[slot], 0), "wait");
            ck(cudaMemcpyAsync(hout + size_t(b0) * out_sz, dout, size_t(nb) * out_sz * sizeof(float),
                               cudaMemcpyDeviceToHost, p->s_out), "D2H");
            ck(cudaEventRecord(p->ev_d2h[slot], p->s_out), "event");
        }
        ck(cudaStreamSynchronize(p->s_out), "stream sync");
        ck(cudaStreamSynchronize(st), "stream sync");
        return;
    }
    for (int b0 = 0; b0 < batch; b0 += p->max_batch) {
        const int nb = std::min(p->max_batch, batch - b0);
        const float* src = hin + size_t(b0) * in_sz;
        float* dst = hout + size_t(b0) * out_sz;
        const size_t ib = size_t(nb) * in_sz * sizeof(float), ob = size_t(nb) * out_sz * sizeof(float);
        if (!pin_in) {
            std::memcpy(p->h_in, src, ib);
            src = p->h_in;
        }
        ck(cudaMemcpyAsync(p->d_in, src, ib, cudaMemcpyHostToDevice, st), "H2D");
        fn(p, p->d_in, p->d_out, nb, st);
        ck(cudaMemcpyAsync(pin_out ? dst : p->h_out, p->d_out, ob, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "stream sync");
        if (!pin_out) std::memcpy(dst, p->h_out, ob);
    }
}

// lp_convolve's multipliers on the half theta spectrum: S(k, v) [/ (Bhat(k) Bhat(v))] / (2 nts n_rho),
// the theta-Nyquist row zero as in Algorithms 1-2; padded like the plan's own when its rho pass is.
// The caller holds the plan mutex until its kernels are enqueued.
void set_lpc_multipliers(lpr_gpu_plan* p, const double* spectrum, int divide_bspline) {
    if (!spectrum) throw std::invalid_argument("lp_convolve: null spectrum");
    const lpr_geometry& G = p->geo;
    const long nts = G.nts, nr = G.n_rho, rows = 2 * nts;
    ck(cudaSetDevice(p->device), "cudaSetDevice");
    if (p->has_done) ck(cudaEventSynchronize(p->ev_done), "cudaEventSynchronize");  // lpc_mult is free
    auto bhat = [](long k, long n) { return (2.0 + std::cos(2.0 * kPi * double(k) / double(n))) / 3.0; };
    std::vector<double> m64(2 * (nts + 1) * nr, 0.0);
    const double sc = 1.0 / (double(rows) * double(nr));
    for (long k = 0; k < nts; ++k)
        for (long v = 0; v < nr; ++v) {
            const double d = divide_bspline ? sc / (bhat(k, rows) * bhat(v, nr)) : sc;
            m64[2 * (k * nr + v)] = spectrum[2 * (k * nr + v)] * d;
            m64[2 * (k * nr + v) + 1] = spectrum[2 * (k * nr + v) + 1] * d;
        }
    const long cols = p->rho_pad ? p->rho_pad : nr;
    if (!p->lpc_mult) {
        p->lpc_mult = p->dalloc<float2>(size_t(nts + 1) * cols);
        p->lpc_out = p->dalloc<float>(size_t(p->max_batch) * rows * p->g.lps);
    }
    if (p->rho_pad) {
        rho_pad_multipliers(p->device, int(nts + 1), int(nr), int(p->rho_pad), m64.data(), p->lpc_mult);
    } else {
        std::vector<float2> m32((nts + 1) * nr);
        for (size_t i = 0; i < m32.size(); ++i) m32[i] = make_float2(float(m64[2 * i]), float(m64[2 * i + 1]));
        ck(cudaMemcpy(p->lpc_mult, m32.data(), m32.size() * sizeof(float2), cudaMemcpyHostToDevice),
           "upload lp_convolve multipliers");
    }
}

// One step of the normal operator on host buffers: R of each chunk of
// images, its sinograms out to the host, R# of the same sinograms straight
// from device memory, the back-projections out; H2D / compute / D2H of
// successive chunks overlap on three streams (chunks of c slices, up to
// kHostSlots in flight, as run_host). The sinograms never come back in.
void run_host_normal(lpr_gpu_plan* p, const float* h_img, float* h_sino, float* h_back, int batch) {
    if (!p) throw std::invalid_argument("null plan");
    if (batch < 0 || (batch > 0 && (!h_img || !h_sino || !h_back))) throw std::invalid_argument("bad buffers or batch");
    ck(cudaSetDevice(p->device), "cudaSetDevice");
    const size_t isz = size_t(p->geo.N) * p->geo.N, ssz = size_t(p->geo.n_theta) * p->geo.N;
    cudaStream_t st = p->stream;
    const Call call(p, st);
    if (!p->d_back) p->d_back = p->dalloc<float>(size_t(p->max_batch) * isz);
    const bool pinned = is_pinned(h_img) && is_pinned(h_sino) && is_pinned(h_back);
    const int c = pinned ? std::max(1, std::min(p->max_batch / 2, (batch + lpr_gpu_plan::kHostChunks - 1) /
                                                                      lpr_gpu_plan::kHostChunks))
                         : p->max_batch;
    const int slots = pinned ? std::min(lpr_gpu_plan::kHostSlots, p->max_batch / c) : 1;
    const int chunks = (batch + c - 1) / c;
    for (int i = 0; i < chunks; ++i) {
        const int slot = i % slots, b0 = i * c, nb = std::min(c, batch - b0);
        float* di = p->d_in + size_t(slot) * c * isz;
        float* ds = p->d_out + size_t(slot) * c * ssz;
        float* db = p->d_back + size_t(slot) * c * isz;
        if (i >= slots) ck(cudaStreamWaitEvent(p->s_in, p->ev_comp[slot], 0), "wait");
        ck(cudaMemcpyAsync(di, h_img + size_t(b0) * isz, size_t(nb) * isz * sizeof(float), cudaMemcpyHostToDevice,
                           p->s_in), "H2D");
        ck(cudaEventRecord(p->ev_h2d[slot], p->s_in), "event");
        ck(cudaStreamWaitEvent(st, p->ev_h2d[slot], 0), "wait");
        if (i >= slots) ck(cudaStreamWaitEvent(st, p->ev_d2h[slot], 0), "wait");
        radon_chunk(p, di, ds, nb, st);
        ck(cudaEventRecord(p->ev_mid[slot], st), "event");
        backproject_chunk(p, ds, db, nb, st);
        ck(cudaEventRecord(p->ev_comp[slot], st), "event");
        ck(cudaStreamWaitEvent(p->s_out, p->ev_mid[slot], 0), "wait");
        ck(cudaMemcpyAsync(h_sino + size_t(b0) * ssz, ds, size_t(nb) * ssz * sizeof(float), cudaMemcpyDeviceToHost,
                           p->s_out), "D2H");
        ck(cudaStreamWaitEvent(p->s_out, p->ev_comp[slot], 0), "wait");
        ck(cudaMemcpyAsync(h_back + size_t(b0) * isz, db, size_t(nb) * isz * sizeof(float), cudaMemcpyDeviceToHost,
                           p->s_out), "D2H");
        ck(cudaEventRecord(p->ev_d2h[slot], p->s_out), "event");
        if (!pinned) ck(cudaStreamSynchronize(p->s_out), "stream sync");  // pageable: one chunk at a time
    }
    ck(cudaStreamSynchronize(p->s_out), "stream sync");
    ck(cudaStreamSynchronize(st), "stream sync");
}

}  // namespace

extern "C" {

const char* lpr_gpu_last_error(void) { return g_last_error.c_str(); }

int lpr_geometry_make(int N, int M, int n_theta, int n_rho, lpr_geometry* out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output");
        *out = host::make_geometry(N, M, n_theta, n_rho);
    });
}

int lpr_smooth_n_rho(int N, int M) {
    try {
        return host::smooth_n_rho(N, M);
    } catch (...) {
        return -1;
    }
}

int lpr_spectrum_quadrature(const lpr_geometry* geom, int kind, double* out) {
    return guard([&] {
        if (!geom || !out || (kind != 0 && kind != 1)) throw std::invalid_argument("bad spectrum arguments");
        const lpr_geometry G = host::make_geometry(geom->N, geom->M, geom->n_theta, geom->n_rho);
        if (host::spectrum_cache_load(G, kind, out)) return;
        host::spectrum(G, kind, out);
        host::spectrum_cache_store(G, kind, out);
    });
}

int lpr_gpu_spectrum_quadrature(int device, const lpr_geometry* geom, int kind, double* out) {
    return guard([&] {
        if (!geom || !out || (kind != 0 && kind != 1)) throw std::invalid_argument("bad spectrum arguments");
        const lpr_geometry G = host::make_geometry(geom->N, geom->M, geom->n_theta, geom->n_rho);
        if (host::spectrum_cache_load(G, kind, out)) return;
        spectrum_gpu(device, G, kind, out);
        host::spectrum_cache_store(G, kind, out);
    });
}

int lpr_spectrum_cache_dir(const char* dir) {
    return guard([&] { host::set_spectrum_cache_dir(dir); });
}

long long lpr_spectrum_cache_hits(void) { return host::spectrum_cache_hits(); }
long long lpr_spectrum_cache_stores(void) { return host::spectrum_cache_stores(); }

int lpr_gpu_plan_create(int device, const lpr_geometry* geom, const double* zeta, const double* zeta_bp,
                        int max_batch, lpr_gpu_plan** out) {
    return lpr_gpu_plan_create_ex(device, geom, zeta, zeta_bp, max_batch, 0u, out);
}

int lpr_gpu_plan_create_ex(int device, const lpr_geometry* geom, const double* zeta, const double* zeta_bp,
                           int max_batch, unsigned flags, lpr_gpu_plan** out) {
    return guard([&] {
        if (flags & ~unsigned(LPR_PLAN_TEXTURE_GATHER)) throw std::invalid_argument("plan: unknown flags");
        if (!geom || !out) throw std::invalid_argument("null argument");
        if (max_batch < 1) throw std::invalid_argument("max_batch must be >= 1");
        // re-derive so a hand-edited struct cannot desynchronise the tables
        const lpr_geometry G = host::make_geometry(geom->N, geom->M, geom->n_theta, geom->n_rho);
        if (G.n_theta != geom->n_theta || G.nts != geom->nts)
            throw std::invalid_argument("plan: geometry does not match sampling_plan");
        auto* p = new lpr_gpu_plan();
        p->device = device;
        p->geo = G;
        p->max_batch = max_batch;
        p->tex_gather = (flags & LPR_PLAN_TEXTURE_GATHER) != 0;
        p->tex_mode = p->tex_gather ? 1 : 0;
        try {
            init_plan(p, zeta, zeta_bp);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

void lpr_gpu_plan_destroy(lpr_gpu_plan* plan) { delete plan; }

int lpr_gpu_sensitivity(lpr_gpu_plan* p, float* d_img, void* stream) {
    return guard([&] {
        if (!p || !d_img) throw std::invalid_argument("null argument");
        ck(cudaSetDevice(p->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const Call call(p, st);
        em_buffers(p);
        launch_fill(p->em_rf, size_t(p->geo.n_theta) * p->geo.N, 1.f, st);
        backproject_chunk(p, p->em_rf, d_img, 1, st);
        check_launch("sensitivity");
    });
}

int lpr_gpu_sensitivity_host(lpr_gpu_plan* p, float* h_img) {
    return guard([&] {
        if (!p || !h_img) throw std::invalid_argument("null argument");
        ck(cudaSetDevice(p->device), "cudaSetDevice");
        cudaStream_t st = p->stream;
        const Call call(p, st);
        em_buffers(p);
        launch_fill(p->em_rf, size_t(p->geo.n_theta) * p->geo.N, 1.f, st);
        backproject_chunk(p, p->em_rf, p->em_bp, 1, st);
        check_launch("sensitivity");
        ck(cudaMemcpyAsync(h_img, p->em_bp, sizeof(float) * size_t(p->geo.N) * p->geo.N, cudaMemcpyDeviceToHost, st),
           "D2H");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

int lpr_gpu_em(lpr_gpu_plan* p, const float* d_sino, float* d_img, int batch, int iters, int init, double* h_loglik,
               void* stream) {
    return guard([&] {
        if (!p) throw std::invalid_argument("null plan");
        if (batch < 0 || iters < 0 || (batch > 0 && (!d_sino || !d_img)))
            throw std::invalid_argument("em: bad buffers, batch or iters");
        ck(cudaSetDevice(p->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const Call call(p, st);
        em_buffers(p);
        const lpr_geometry& G = p->geo;
        const size_t ps = size_t(G.n_theta) * G.N, pi = size_t(G.N) * G.N;
        double* ll = nullptr;
        ck(cudaMalloc(&ll, sizeof(double) * std::max<size_t>(1, size_t(p->max_batch) * std::max(iters, 1))), "cudaMalloc");
        try {
            for (int b0 = 0; b0 < batch; b0 += p->max_batch) {
                const int nb = std::min(p->max_batch, batch - b0);
                float* f = d_img + size_t(b0) * pi;
                if (init) launch_disc_fill(G.N, f, nb, st);  // f0 = 1 inside the unit disc
                ck(cudaMemsetAsync(ll, 0, sizeof(double) * size_t(nb) * std::max(iters, 1), st), "memset");
                em_chunk(p, d_sino + size_t(b0) * ps, f, nb, iters, ll, st);
                int bad = 0;
                ck(cudaMemcpyAsync(&bad, p->em_bad, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
                if (h_loglik && iters > 0)
                    ck(cudaMemcpyAsync(h_loglik + size_t(b0) * iters, ll, sizeof(double) * size_t(nb) * iters,
                                       cudaMemcpyDeviceToHost, st),
                       "D2H");
                ck(cudaStreamSynchronize(st), "sync");
                if (bad & 1) throw std::invalid_argument("em: the sinogram must be finite and nonnegative");
                if (bad & 2) throw std::runtime_error("em: non-finite estimate");
            }
        } catch (...) {
            cudaFree(ll);
            throw;
        }
        cudaFree(ll);
    });
}

int lpr_gpu_em_host(lpr_gpu_plan* p, const float* h_sino, float* h_img, int batch, int iters, int init,
                    double* h_loglik) {
    return guard([&] {
        if (!p) throw std::invalid_argument("null plan");
        if (batch < 0 || (batch > 0 && (!h_sino || !h_img))) throw std::invalid_argument("em: bad buffers or batch");
        ck(cudaSetDevice(p->device), "cudaSetDevice");
        const lpr_geometry& G = p->geo;
        const size_t ps = size_t(G.n_theta) * G.N, pi = size_t(G.N) * G.N;
        float *dg = nullptr, *df = nullptr;
        ck(cudaMalloc(&dg, sizeof(float) * ps * std::max(batch, 1)), "cudaMalloc");
        if (cudaMalloc(&df, sizeof(float) * pi * std::max(batch, 1)) != cudaSuccess) {
            cudaFree(dg);
            throw Error(LPR_ERR_OOM, "cudaMalloc");
        }
        int rc = LPR_OK;
        cudaStream_t st = p->stream;
        const Call call(p, st);
        try {
            ck(cudaMemcpyAsync(dg, h_sino, sizeof(float) * ps * batch, cudaMemcpyHostToDevice, st), "H2D");
            if (!init) ck(cudaMemcpyAsync(df, h_img, sizeof(float) * pi * batch, cudaMemcpyHostToDevice, st), "H2D");
            rc = lpr_gpu_em(p, dg, df, batch, iters, init, h_loglik, st);
            if (rc == LPR_OK) {
                ck(cudaMemcpyAsync(h_img, df, sizeof(float) * pi * batch, cudaMemcpyDeviceToHost, st), "D2H");
                ck(cudaStreamSynchronize(st), "sync");
            }
        } catch (...) {
            cudaFree(dg);
            cudaFree(df);
            throw;
        }
        cudaFree(dg);
        cudaFree(df);
        if (rc != LPR_OK) throw Error(lpr_status(rc), g_last_error);
    });
}

int lpr_gpu_radon(lpr_gpu_plan* p, const float* d_img, float* d_sino, int batch, void* stream) {
    return guard([&] {
        run_device(p, radon_chunk, d_img, d_sino, batch, size_t(p ? p->geo.N : 0) * (p ? p->geo.N : 0),
                   size_t(p ? p->geo.n_theta : 0) * (p ? p->geo.N : 0), stream);
    });
}

int lpr_gpu_backproject(lpr_gpu_plan* p, const float* d_sino, float* d_img, int batch, void* stream) {
    return guard([&] {
        run_device(p, backproject_chunk, d_sino, d_img, batch, size_t(p ? p->geo.n_theta : 0) * (p ? p->geo.N : 0),
                   size_t(p ? p->geo.N : 0) * (p ? p->geo.N : 0), stream);
    });
}

int lpr_gpu_radon_host(lpr_gpu_plan* p, const float* h_img, float* h_sino, int batch) {
    return guard([&] {
        run_host(p, radon_chunk, h_img, h_sino, batch, size_t(p ? p->geo.N : 0) * (p ? p->geo.N : 0),
                 size_t(p ? p->geo.n_theta : 0) * (p ? p->geo.N : 0));
    });
}

int lpr_gpu_radon_backproject_host(lpr_gpu_plan* p, const float* h_img, float* h_sino, float* h_back, int batch) {
    return guard([&] { run_host_normal(p, h_img, h_sino, h_back, batch); });
}

int lpr_gpu_backproject_host(lpr_gpu_plan* p, const float* h_sino, float* h_img, int batch) {
    return guard([&] {
        run_host(p, backproject_chunk, h_sino, h_img, batch, size_t(p ? p->geo.n_theta : 0) * (p ? p->geo.N : 0),
                 size_t(p ? p->geo.N : 0) * (p ? p->geo.N : 0));
    });
}

namespace {
ChunkFn filter_fn(int kind, bool fbp) {
    switch (kind) {
        case 0: return fbp ? fbp_chunk<0> : filter_chunk<0, false>;
        case 1: return fbp ? fbp_chunk<1> : filter_chunk<1, false>;
        case 2: return fbp ? fbp_chunk<2> : filter_chunk<2, false>;
        default: throw std::invalid_argument("filter kind must be 0 (ramp), 1 (shepp-logan) or 2 (cosine)");
    }
}
}  // namespace

int lpr_gpu_filter(lpr_gpu_plan* p, int kind, const float* d_in, float* d_out, int batch, void* stream) {
    return guard([&] {
        const size_t sz = size_t(p ? p->geo.n_theta : 0) * (p ? p->geo.N : 0);
        run_device(p, filter_fn(kind, false), d_in, d_out, batch, sz, sz, stream);
    });
}

int lpr_gpu_fbp(lpr_gpu_plan* p, int kind, const float* d_sino, float* d_img, int batch, void* stream) {
    return guard([&] {
        run_device(p, filter_fn(kind, true), d_sino, d_img, batch, size_t(p ? p->geo.n_theta : 0) * (p ? p->geo.N : 0),
                   size_t(p ? p->geo.N : 0) * (p ? p->geo.N : 0), stream);
    });
}

int lpr_gpu_fbp_host(lpr_gpu_plan* p, int kind, const float* h_sino, float* h_img, int batch) {
    return guard([&] {
        run_host(p, filter_fn(kind, true), h_sino, h_img, batch, size_t(p ? p->geo.n_theta : 0) * (p ? p->geo.N : 0),
                 size_t(p ? p->geo.N : 0) * (p ? p->geo.N : 0));
    });
}

int lpr_gpu_radon_transpose_host(lpr_gpu_plan* p, const float* h_sino, float* h_img, int batch) {
    return guard([&] {
        run_host(p, transpose_chunk, h_sino, h_img, batch, size_t(p ? p->geo.n_theta : 0) * (p ? p->geo.N : 0),
                 size_t(p ? p->geo.N : 0) * (p ? p->geo.N : 0));
    });
}

int lpr_gpu_radon_transpose(lpr_gpu_plan* p, const float* d_sino, float* d_img, int batch, void* stream) {
    return guard([&] {
        run_device(p, transpose_chunk, d_sino, d_img, batch, size_t(p ? p->geo.n_theta : 0) * (p ? p->geo.N : 0),
                   size_t(p ? p->geo.N : 0) * (p ? p->geo.N : 0), stream);
    });
}

int lpr_gpu_profile_stages(lpr_gpu_plan* p, int op, const float* d_in, float* d_out, int batch, int reps,
                           double* ms, int* nstages, const char** names) {
    return guard([&] {
        if (!p || !d_in || !d_out || !ms || !nstages || batch < 1 || batch > p->max_batch || reps < 1)
            throw std::invalid_argument("profile: bad arguments");
        if (op != 0 && op != 1) throw std::invalid_argument("profile: op must be 0 (R) or 1 (R#)");
        ck(cudaSetDevice(p->device), "cudaSetDevice");
        const int ns = 5;
        std::vector<cudaEvent_t> ev(ns + 1);
        for (auto& e : ev) ck(cudaEventCreate(&e), "cudaEventCreate");
        std::vector<double> acc(ns, 0.0);
        cudaStream_t st = p->stream;
        const Call call(p, st);
        for (int r = 0; r < reps; ++r) {
            p->prof = ev.data();
            try {
                (op == 0 ? radon_chunk : backproject_chunk)(p, d_in, d_out, batch, st);
            } catch (...) {
                p->prof = nullptr;
                throw;
            }
            p->prof = nullptr;
            ck(cudaStreamSynchronize(st), "profile sync");
            for (int i = 0; i < ns; ++i) {
                float t = 0.f;
                ck(cudaEventElapsedTime(&t, ev[i], ev[i + 1]), "cudaEventElapsedTime");
                acc[i] += t;
            }
        }
        for (auto& e : ev) cudaEventDestroy(e);
        for (int i = 0; i < ns; ++i) ms[i] = acc[i] / reps;
        *nstages = ns;
        if (names)
            for (int i = 0; i < ns; ++i) names[i] = op == 0 ? kRadonStages[i] : kBackprojectStages[i];
    });
}

int lpr_gpu_lp_convolve(lpr_gpu_plan* p, const double* spectrum, int divide_bspline, const float* d_in, float* d_out,
                        int batch, void* stream) {
    return guard([&] {
        if (!p) throw std::invalid_argument("null plan");
        // held until the kernels are enqueued: another call must not replace the
        // multipliers in between (run_device's Call re-locks the recursive mutex)
        const std::lock_guard<std::recursive_mutex> lk(p->mu);
        set_lpc_multipliers(p, spectrum, divide_bspline);
        const size_t sz = size_t(2 * p->geo.nts) * p->geo.n_rho;
        run_device(p, lpc_chunk, d_in, d_out, batch, sz, sz, stream);
    });
}

int lpr_gpu_lp_convolve_host(lpr_gpu_plan* p, const double* spectrum, int divide_bspline, const float* h_in,
                             float* h_out, int batch) {
    return guard([&] {
        if (!p) throw std::invalid_argument("null plan");
        if (batch < 0 || (batch > 0 && (!h_in || !h_out))) throw std::invalid_argument("bad buffers or batch");
        const std::lock_guard<std::recursive_mutex> lk(p->mu);
        set_lpc_multipliers(p, spectrum, divide_bspline);
        // doubled-grid rasters are larger than the plan's image / sinogram staging: own device buffers
        const size_t sz = size_t(2 * p->geo.nts) * p->geo.n_rho;
        if (!p->lpc_din) {
            p->lpc_din = p->dalloc<float>(size_t(p->max_batch) * sz);
            p->lpc_dout = p->dalloc<float>(size_t(p->max_batch) * sz);
        }
        cudaStream_t st = p->stream;
        const Call call(p, st);
        for (int b0 = 0; b0 < batch; b0 += p->max_batch) {
            const int nb = std::min(p->max_batch, batch - b0);
            const size_t bytes = size_t(nb) * sz * sizeof(float);
            ck(cudaMemcpyAsync(p->lpc_din, h_in + size_t(b0) * sz, bytes, cudaMemcpyHostToDevice, st), "H2D");
            lpc_chunk(p, p->lpc_din, p->lpc_dout, nb, st);
            ck(cudaMemcpyAsync(h_out + size_t(b0) * sz, p->lpc_dout, bytes, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "stream sync");
        }
    });
}

int lpr_gpu_profile_stages_host(lpr_gpu_plan* p, int op, const float* h_in, int batch, int reps, double* ms,
                                int* nstages, const char** names) {
    return guard([&] {
        if (!p || !h_in || batch < 1 || batch > p->max_batch) throw std::invalid_argument("profile: bad arguments");
        const lpr_geometry& G = p->geo;
        const size_t n = size_t(batch) * (op == 0 ? size_t(G.N) * G.N : size_t(G.n_theta) * G.N);
        const std::lock_guard<std::recursive_mutex> lk(p->mu);  // the staged input stays ours through the profile
        {
            ck(cudaSetDevice(p->device), "cudaSetDevice");
            if (p->has_done) ck(cudaStreamWaitEvent(p->stream, p->ev_done, 0), "cudaStreamWaitEvent");
            ck(cudaMemcpyAsync(p->d_in, h_in, n * sizeof(float), cudaMemcpyHostToDevice, p->stream), "H2D");
            ck(cudaStreamSynchronize(p->stream), "stream sync");
        }
        const int rc = lpr_gpu_profile_stages(p, op, p->d_in, p->d_out, batch, reps, ms, nstages, names);
        if (rc != LPR_OK) throw Error(lpr_status(rc), g_last_error);
    });
}

long long lpr_gpu_launch_count(const lpr_gpu_plan* p) { return p ? p->launches : -1; }
long long lpr_gpu_fft_count(const lpr_gpu_plan* p) { return p ? p->ffts : -1; }

}  // extern "C"
