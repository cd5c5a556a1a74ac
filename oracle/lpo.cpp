// ORACLE — test infrastructure only (see lpo.hpp). fp64 restatement of the
// reference's building blocks and of paper Algorithms 1-2.
#include "lpo.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>

namespace lpo {

namespace {

constexpr double kPi = 3.14159265358979323846;

inline long wrap(long i, long n) {
    long r = i % n;
    return r < 0 ? r + n : r;
}

}  // namespace

// =================================================================== geometry

int min_n_rho(int N, int M) {
    // Eq. (vrho) with the reference's log1p form (geometry.cpp:85-87).
    const double beta = kPi / M;
    const double sh = std::sin(0.5 * beta), ch = std::cos(0.5 * beta);
    const double aR = sh / (1.0 + sh), ar = (ch - sh) / (1.0 + sh);
    return int(std::ceil(std::log(ar) / std::log1p(-2.0 * aR / N)));
}

Plan make_plan(int N, int M, int n_theta, int n_rho) {
    if (N < 16 || (N & 1)) throw std::invalid_argument("make_plan: N must be even and >= 16");
    if (M < 3) throw std::invalid_argument("make_plan: M must be >= 3");
    Plan p;
    p.N = N;
    p.M = M;
    p.beta = kPi / M;
    const double sh = std::sin(0.5 * p.beta), ch = std::cos(0.5 * p.beta);
    p.aR = sh / (1.0 + sh);
    p.ar = (ch - sh) / (1.0 + sh);
    p.log_ar = std::log(p.ar);
    if (n_theta <= 0) n_theta = int(std::ceil(1.5 * N));
    if (n_theta < 2 * M) throw std::invalid_argument("make_plan: n_theta too small");
    const int q = 2 * M;
    p.n_theta = (n_theta + q - 1) / q * q;  // sector centres land on polar rows
    p.nts = p.n_theta / M;
    p.ds = 1.0 / N;
    p.dtheta_p = kPi / p.n_theta;
    const int nmin = min_n_rho(N, M);
    if (n_rho <= 0) n_rho = nmin;
    if (n_rho < nmin) throw std::invalid_argument("make_plan: n_rho below the sampling bound");
    p.n_rho = n_rho;
    p.drho = -p.log_ar / n_rho;
    p.refine = int(std::ceil(p.dtheta_p * N / (2.0 * p.aR) - 1e-12));
    p.dtheta_lp = p.dtheta_p / p.refine;
    return p;
}

// =================================================================== FFT
// Mixed-radix decimation-in-time recursion for lengths whose prime factors
// are <= 13; Bluestein (chirp-z) through a power-of-two length otherwise.

namespace {

struct FftPlan {
    long n = 0;
    std::vector<int> radix;
    std::vector<cd> w;  // w[j] = exp(-2 pi i j / n)
    bool chirp = false;
    long nb = 0;                  // Bluestein power-of-two length
    std::vector<cd> c;            // c[j] = exp(-i pi j^2 / n)
    std::vector<cd> bhat;         // FFT_nb of conj chirp, wrapped
};

std::shared_ptr<const FftPlan> get_plan(long n);

void dit(const cd* in, long istride, cd* out, long n, const int* rad, const cd* w,
         long wstride, int sign, cd* tmp) {
    if (n == 1) {
        out[0] = in[0];
        return;
    }
    const long p = rad[0];
    const long m = n / p;
    for (long r = 0; r < p; ++r) dit(in + r * istride, istride * p, out + r * m, m, rad + 1, w, wstride * p, sign, tmp);
    const long n0 = n * wstride;  // root length of the table
    for (long k = 0; k < m; ++k) {
        for (long r = 0; r < p; ++r) {
            cd t = w[(r * k % n) * wstride];
            if (sign > 0) t = std::conj(t);
            tmp[r] = out[r * m + k] * t;
        }
        for (long q = 0; q < p; ++q) {
            cd acc = 0.0;
            for (long r = 0; r < p; ++r) {
                cd t = w[((r * q) % p) * (n0 / p)];
                if (sign > 0) t = std::conj(t);
                acc += tmp[r] * t;
            }
            out[k + q * m] = acc;
        }
    }
}

void run_plan(const FftPlan& pl, cd* x, int sign) {
    const long n = pl.n;
    if (n == 1) return;
    if (!pl.chirp) {
        std::vector<cd> out(n), tmp(16);
        dit(x, 1, out.data(), n, pl.radix.data(), pl.w.data(), 1, sign, tmp.data());
        std::copy(out.begin(), out.end(), x);
        return;
    }
    // X_k = conj?(c_k) sum_j (x_j c_j) conj(c)_{k-j}; sign +1 uses conj chirps.
    auto sub = get_plan(pl.nb);
    std::vector<cd> a(pl.nb, cd(0.0));
    for (long j = 0; j < n; ++j) a[j] = x[j] * (sign < 0 ? pl.c[j] : std::conj(pl.c[j]));
    run_plan(*sub, a.data(), -1);
    // the chirp kernel is even, so its transform is even: conj serves sign +1
    for (long j = 0; j < pl.nb; ++j) a[j] *= (sign < 0 ? pl.bhat[j] : std::conj(pl.bhat[j]));
    run_plan(*sub, a.data(), +1);
    const double inv = 1.0 / double(pl.nb);
    for (long k = 0; k < n; ++k) x[k] = a[k] * inv * (sign < 0 ? pl.c[k] : std::conj(pl.c[k]));
}

std::shared_ptr<const FftPlan> make_fft_plan(long n) {
    auto pl = std::make_shared<FftPlan>();
    pl->n = n;
    long r = n;
    for (int f : {4, 2, 3, 5, 7, 11, 13}) {
        while (r % f == 0) {
            pl->radix.push_back(f);
            r /= f;
        }
    }
    if (r != 1) {
        pl->chirp = true;
        long nb = 1;
        while (nb < 2 * n - 1) nb <<= 1;
        pl->nb = nb;
        pl->c.resize(n);
        for (long j = 0; j < n; ++j) {
            // j^2 mod 2n keeps the phase argument small
            const long jj = (j * j) % (2 * n);
            pl->c[j] = std::polar(1.0, -kPi * double(jj) / double(n));
        }
        std::vector<cd> b(nb, cd(0.0));
        b[0] = std::conj(pl->c[0]);
        for (long j = 1; j < n; ++j) b[j] = b[nb - j] = std::conj(pl->c[j]);
        auto sub = get_plan(nb);
        run_plan(*sub, b.data(), -1);
        pl->bhat = std::move(b);
        return pl;
    }
    pl->w.resize(n);
    for (long j = 0; j < n; ++j) pl->w[j] = std::polar(1.0, -2.0 * kPi * double(j) / double(n));
    return pl;
}

std::mutex g_plan_mu;
std::map<long, std::shared_ptr<const FftPlan>> g_plans;
std::atomic<std::uint64_t> g_count2d{0};

std::shared_ptr<const FftPlan> get_plan(long n) {
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        auto it = g_plans.find(n);
        if (it != g_plans.end()) return it->second;
    }
    auto pl = make_fft_plan(n);
    std::lock_guard<std::mutex> lk(g_plan_mu);
    g_plans.emplace(n, pl);
    return pl;
}

}  // namespace

void fft1d(cd* x, long n, int sign) {
    if (n <= 0) throw std::invalid_argument("fft: empty transform");
    if (sign != -1 && sign != 1) throw std::invalid_argument("fft: bad sign");
    run_plan(*get_plan(n), x, sign);
}

void fft2d(cd* x, long rows, long cols, int sign) {
    if (rows <= 0 || cols <= 0) throw std::invalid_argument("fft: empty transform");
    if (sign != -1 && sign != 1) throw std::invalid_argument("fft: bad sign");
    auto pr = get_plan(cols), pc = get_plan(rows);
#pragma omp parallel for schedule(dynamic, 4)
    for (long r = 0; r < rows; ++r) run_plan(*pr, x + r * cols, sign);
#pragma omp parallel
    {
        std::vector<cd> col(rows);
#pragma omp for schedule(dynamic, 4)
        for (long c = 0; c < cols; ++c) {
            for (long r = 0; r < rows; ++r) col[r] = x[r * cols + c];
            run_plan(*pc, col.data(), sign);
            for (long r = 0; r < rows; ++r) x[r * cols + c] = col[r];
        }
    }
    g_count2d.fetch_add(1);
}

std::uint64_t fft2d_count() { return g_count2d.load(); }
void fft2d_count_reset() { g_count2d.store(0); }

// =================================================================== B-spline

namespace {
constexpr double kZ = -0.26794919243112270647;  // sqrt(3) - 2
constexpr long kMargin = 32;                     // steady-state start, |z|^32 ~ 5e-19

long mirror_index(long i, long n) {
    if (n == 1) return 0;
    const long per = 2 * (n - 1);
    long r = wrap(i, per);
    return r >= n ? per - r : r;
}

inline double bhat(long k, long n) { return (2.0 + std::cos(2.0 * kPi * double(k) / double(n))) / 3.0; }
}  // namespace

void bspline_weights(double a, double w[4]) {
    const double b = 1.0 - a;
    w[0] = b * b * b / 6.0;                               // tap k-1: B(a+1)
    w[1] = (3.0 * a * a * a - 6.0 * a * a + 4.0) / 6.0;   // tap k:   B(a)
    w[2] = (3.0 * b * b * b - 6.0 * b * b + 4.0) / 6.0;   // tap k+1: B(1-a)
    w[3] = a * a * a / 6.0;                               // tap k+2: B(2-a)
}

void prefilter_1d(double* x, long n, long stride) {
    if (n < 4) throw std::invalid_argument("prefilter_1d: length must be >= 4");
    const long len = n + 2 * kMargin;
    std::vector<double> e(len);
    for (long i = 0; i < len; ++i) e[i] = x[mirror_index(i - kMargin, n) * stride];
    double acc = 6.0 * e[0] / (1.0 - kZ);
    e[0] = acc;
    for (long k = 1; k < len; ++k) e[k] = acc = 6.0 * e[k] + kZ * acc;
    acc = -kZ / (1.0 - kZ) * e[len - 1];
    e[len - 1] = acc;
    for (long k = len - 2; k >= 0; --k) e[k] = acc = kZ * (acc - e[k]);
    for (long k = 0; k < n; ++k) x[k * stride] = e[k + kMargin];
}

void prefilter_2d(double* img, long rows, long cols) {
#pragma omp parallel for schedule(static)
    for (long r = 0; r < rows; ++r) prefilter_1d(img + r * cols, cols, 1);
#pragma omp parallel for schedule(static)
    for (long c = 0; c < cols; ++c) prefilter_1d(img + c, rows, cols);
}

namespace {
// Transpose (reverse-mode) of prefilter_1d: x <- Q^T x.
void prefilter_1d_T(double* x, long n, long stride) {
    const long len = n + 2 * kMargin;
    std::vector<double> d(len, 0.0), c(len, 0.0), e(len, 0.0);
    for (long k = 0; k < n; ++k) d[k + kMargin] = x[k * stride];
    // anticausal pass, reversed
    for (long k = 0; k <= len - 2; ++k) {
        d[k + 1] += kZ * d[k];
        c[k] += -kZ * d[k];
    }
    c[len - 1] += -kZ / (1.0 - kZ) * d[len - 1];
    // causal pass, reversed
    for (long k = len - 1; k >= 1; --k) {
        e[k] += 6.0 * c[k];
        c[k - 1] += kZ * c[k];
    }
    e[0] += 6.0 / (1.0 - kZ) * c[0];
    for (long k = 0; k < n; ++k) x[k * stride] = 0.0;
    for (long i = 0; i < len; ++i) x[mirror_index(i - kMargin, n) * stride] += e[i];
}

void prefilter_2d_T(double* img, long rows, long cols) {
#pragma omp parallel for schedule(static)
    for (long c = 0; c < cols; ++c) prefilter_1d_T(img + c, rows, cols);
#pragma omp parallel for schedule(static)
    for (long r = 0; r < rows; ++r) prefilter_1d_T(img + r * cols, cols, 1);
}
}  // namespace

double eval_mirror_2d(const double* c, long rows, long cols, double tr, double tc) {
    if (!(tr >= -2.0 && tr <= rows + 1.0 && tc >= -2.0 && tc <= cols + 1.0))
        throw std::out_of_range("eval_mirror_2d: beyond the extension margin");
    const long kr = long(std::floor(tr)), kc = long(std::floor(tc));
    double wr[4], wc[4];
    bspline_weights(tr - kr, wr);
    bspline_weights(tc - kc, wc);
    double acc = 0.0;
    for (int a = 0; a < 4; ++a) {
        const long rr = mirror_index(kr - 1 + a, rows);
        double row = 0.0;
        for (int b = 0; b < 4; ++b) row += wc[b] * c[rr * cols + mirror_index(kc - 1 + b, cols)];
        acc += wr[a] * row;
    }
    return acc;
}

double eval_periodic_2d(const double* c, long rows, long cols, double tr, double tc) {
    const long kr = long(std::floor(tr)), kc = long(std::floor(tc));
    double wr[4], wc[4];
    bspline_weights(tr - kr, wr);
    bspline_weights(tc - kc, wc);
    double acc = 0.0;
    for (int a = 0; a < 4; ++a) {
        const long rr = wrap(kr - 1 + a, rows);
        double row = 0.0;
        for (int b = 0; b < 4; ++b) row += wc[b] * c[rr * cols + wrap(kc - 1 + b, cols)];
        acc += wr[a] * row;
    }
    return acc;
}

double eval_periodic_1d(const double* c, long n, double t) {
    const long k = long(std::floor(t));
    double w[4];
    bspline_weights(t - k, w);
    double acc = 0.0;
    for (int b = 0; b < 4; ++b) acc += w[b] * c[wrap(k - 1 + b, n)];
    return acc;
}

double eval_zero_1d(const double* c, long n, double t) {
    const long k = long(std::floor(t));
    double w[4];
    bspline_weights(t - k, w);
    double acc = 0.0;
    for (int b = 0; b < 4; ++b) {
        const long i = k - 1 + b;
        if (i >= 0 && i < n) acc += w[b] * c[i];
    }
    return acc;
}

// =================================================================== spectra
// Restates the FFT-trapezoid path of kernel.cpp:293-429: for each rho
// frequency the integral P(mu, alpha, beta) = int_{-beta}^{beta} e^{i mu t}
// cos(t)^alpha dt is evaluated at every mu = -pi k / beta at once by one FFT
// of end-corrected trapezoid samples (PAPER.md:162-168 weights).

void spectrum(const Plan& p, int kind, cd* out) {
    static const double corr[7] = {-23681.0, 55688.0, -66109.0, 57024.0, -31523.0, 9976.0, -1375.0};
    const long nts = p.nts, rows = 2 * nts, cols = p.n_rho;
    const double beta = p.beta, ell = -p.log_ar;
#pragma omp parallel for schedule(dynamic, 1)
    for (long v = 0; v < cols; ++v) {
        const long kr = v < (cols + 1) / 2 ? v : v - cols;
        const double y = 2.0 * kPi * double(kr) / ell;
        if (kind == 1 && kr == 0) {
            for (long kt = -nts; kt < nts; ++kt) {
                const double mu = -kPi * double(kt) / beta;
                out[wrap(kt, rows) * cols + v] = kt == 0 ? cd(2.0 * beta) : cd(2.0 * std::sin(mu * beta) / mu);
            }
            continue;
        }
        const cd alpha = kind == 0 ? cd(-1.0, -y) : cd(0.0, y);
        const double rate = (kPi * double(nts) / beta + std::abs(y) * std::tan(beta)) * beta / kPi;
        const long base = std::max<long>(32, long(std::ceil(rate)));
        long n = 1;
        while (n < 16 * base) n <<= 1;
        const double h = 2.0 * beta / double(n);
        std::vector<cd> g(n);
        for (long j = 0; j < n; ++j) {
            double wt = 1.0;
            if (j == 0) wt += 2.0 * corr[0] / 120960.0;  // nodes 0 and n coincide
            else if (j < 7) wt += corr[j] / 120960.0;
            if (j > n - 7) wt += corr[n - j] / 120960.0;
            const double th = -beta + double(j) * h;
            g[j] = wt * std::exp(alpha * std::log(std::cos(th)));
        }
        fft1d(g.data(), n, -1);
        for (long kt = -nts; kt < nts; ++kt) {
            const cd val = h * g[wrap(kt, n)];
            out[wrap(kt, rows) * cols + v] = (kt & 1) ? -val : val;
        }
    }
    if (cols % 2 == 0) {
        for (long t = 0; t < rows; ++t) out[t * cols + cols / 2] = cd(out[t * cols + cols / 2].real(), 0.0);
    }
}

// =================================================================== operators

void lp_convolve(const cd* spec, bool divide_bspline, double* data, long rows, long cols) {
    std::vector<cd> buf(rows * cols);
    for (long i = 0; i < rows * cols; ++i) buf[i] = data[i];
    fft2d(buf.data(), rows, cols, -1);
    const double scale = 1.0 / double(rows * cols);
    for (long r = 0; r < rows; ++r)
        for (long c = 0; c < cols; ++c) {
            double d = scale;
            if (divide_bspline) d /= bhat(r, rows) * bhat(c, cols);
            buf[r * cols + c] *= spec[r * cols + c] * d;
        }
    fft2d(buf.data(), rows, cols, +1);
    for (long i = 0; i < rows * cols; ++i) data[i] = buf[i].real();
}

namespace {

struct SectorMap {
    double cm, sm;  // cos / sin (m beta)
};

// Gather of T_m f * e^rho on the fine grid Omega_lp, zero-embedded into the
// doubled theta period: row (q mod L) holds theta' = q * dtheta_lp,
// q in [-nf/2, nf/2). Points outside the sector disc D contribute zero
// (SPEC.md:317). Alg. 1 steps 3 and 5.
void radon_gather(const Plan& p, const double* qf, int m, cd* F) {
    const long N = p.N, nf = long(p.refine) * p.nts, L = 2 * nf, nr = p.n_rho;
    const SectorMap sm{std::cos(m * p.beta), std::sin(m * p.beta)};
    std::fill(F, F + L * nr, cd(0.0));
#pragma omp parallel for schedule(static)
    for (long i = 0; i < nf; ++i) {
        const long q = i - nf / 2;
        const double th = double(q) * p.dtheta_lp;
        const double ct = std::cos(th), st = std::sin(th);
        cd* row = F + wrap(q, L) * nr;
        for (long l = 0; l < nr; ++l) {
            const double er = std::exp(p.log_ar + double(l) * p.drho);
            const double dx = er * ct - (1.0 - p.aR), dy = er * st;
            if (dx * dx + dy * dy > p.aR * p.aR) continue;
            const double ux = dx / p.aR, uy = dy / p.aR;
            const double xp = sm.cm * ux - sm.sm * uy, yp = sm.sm * ux + sm.cm * uy;
            const double tc = (0.5 * xp + 0.5) * N, tr = (0.5 * yp + 0.5) * N;
            row[l] = er * eval_mirror_2d(qf, N, N, tr, tc);
        }
    }
}

// Spectral multiplier of the Radon leg at (kt, v): zeta / Bhat2 / (L n_rho).
inline cd radon_mult(const Plan& p, const cd* zeta, long kt, long v, long L) {
    const long rows = 2 * p.nts, nr = p.n_rho;
    return zeta[wrap(kt, rows) * nr + v] / (bhat(kt, rows) * bhat(v, nr) * double(L) * double(nr));
}

// Sinogram row i -> (sector m, coarse row j in [-nts/2, nts/2), flip).
// Integer form of line_to_sector (geometry.cpp:134-142) with the residual
// half-open on [-beta/2, beta/2).
inline void row_sector(const Plan& p, long i, int& m, long& j, bool& flip) {
    const long k = (2 * i + p.nts) / (2 * p.nts);
    m = int(k % p.M);
    flip = ((k - m) / p.M) % 2 == 1;
    j = i - k * p.nts;
}

}  // namespace

void radon_sector_coeffs(const Plan& p, const cd* zeta, const double* qf, int m, double* out) {
    const long nf = long(p.refine) * p.nts, L = 2 * nf, nr = p.n_rho, nts = p.nts;
    std::vector<cd> F(L * nr);
    radon_gather(p, qf, m, F.data());
    fft2d(F.data(), L, nr, -1);
    for (long kt = 0; kt <= nts; ++kt)
        for (long v = 0; v < nr; ++v) {
            const cd val = kt == nts ? cd(0.0) : F[wrap(kt, L) * nr + v] * radon_mult(p, zeta, kt, v, L);
            out[2 * (kt * nr + v)] = val.real();
            out[2 * (kt * nr + v) + 1] = val.imag();
        }
}

void fast_radon(const Plan& p, const cd* zeta, const double* img, double* sino) {
    const long N = p.N, nts = p.nts, rows = 2 * nts, nr = p.n_rho;
    const long nf = long(p.refine) * nts, L = 2 * nf;
    std::vector<double> qf(img, img + N * N);
    prefilter_2d(qf.data(), N, N);  // Alg. 1 step 1
    std::vector<std::vector<double>> coef(p.M, std::vector<double>(rows * nr));
    std::vector<cd> F(L * nr), G(rows * nr);
    for (int m = 0; m < p.M; ++m) {
        radon_gather(p, qf.data(), m, F.data());                  // steps 3, 5
        fft2d(F.data(), L, nr, -1);                                // step 6 forward
        // step 4: theta low-pass = keep |k_theta| < nts of the doubled period
        for (long kt = -nts; kt < nts; ++kt)
            for (long v = 0; v < nr; ++v)
                G[wrap(kt, rows) * nr + v] =
                    kt == -nts ? cd(0.0) : F[wrap(kt, L) * nr + v] * radon_mult(p, zeta, kt, v, L);
        fft2d(G.data(), rows, nr, +1);                             // step 6 inverse
        for (long i = 0; i < rows * nr; ++i) coef[m][i] = G[i].real();
    }
    // step 7: resample S_m^{-1} Omega_p -> Sigma, scale a_R^{-1} (Eq. 12) and
    // 1/2 for the raster units (s_phys = 2 s_raster, length_phys = 2 length).
#pragma omp parallel for schedule(static)
    for (long i = 0; i < p.n_theta; ++i) {
        int m;
        long j;
        bool flip;
        row_sector(p, i, m, j, flip);
        const double cth = std::cos(double(j) * p.dtheta_p);
        for (long c = 0; c < N; ++c) {
            const double sr = -0.5 + double(c) / N;
            const double sp = 2.0 * (flip ? -sr : sr);
            const double rho = std::log(p.aR * sp + (1.0 - p.aR) * cth);
            const double t = (rho - p.log_ar) / p.drho;
            sino[i * N + c] = eval_periodic_2d(coef[m].data(), rows, nr, double(j), t) / (2.0 * p.aR);
        }
    }
}

void radon_transpose(const Plan& p, const cd* zeta, const double* sino, double* img) {
    const long N = p.N, nts = p.nts, rows = 2 * nts, nr = p.n_rho;
    const long nf = long(p.refine) * nts, L = 2 * nf;
    std::vector<double> acc(N * N, 0.0);
    for (int m = 0; m < p.M; ++m) {
        // E_m^T: scatter the sector's sinogram bins into the coefficient grid.
        std::vector<double> coef(rows * nr, 0.0);
        for (long i = 0; i < p.n_theta; ++i) {
            int mm;
            long j;
            bool flip;
            row_sector(p, i, mm, j, flip);
            if (mm != m) continue;
            const double cth = std::cos(double(j) * p.dtheta_p);
            double wr[4];
            bspline_weights(0.0, wr);
            for (long c = 0; c < N; ++c) {
                const double sr = -0.5 + double(c) / N;
                const double sp = 2.0 * (flip ? -sr : sr);
                const double rho = std::log(p.aR * sp + (1.0 - p.aR) * cth);
                const double t = (rho - p.log_ar) / p.drho;
                const long kc = long(std::floor(t));
                double wc[4];
                bspline_weights(t - kc, wc);
                const double v = sino[i * N + c] / (2.0 * p.aR);
                for (int a = 0; a < 4; ++a)
                    for (int b = 0; b < 4; ++b)
                        coef[wrap(j - 1 + a, rows) * nr + wrap(kc - 1 + b, nr)] += v * wr[a] * wc[b];
            }
        }
        // C_m^T = Re( FFT+_L( zero-fill( conj(S) * FFT-_rows(y) ) ) ) on fine rows.
        std::vector<cd> G(rows * nr), F(L * nr, cd(0.0));
        for (long i = 0; i < rows * nr; ++i) G[i] = coef[i];
        fft2d(G.data(), rows, nr, -1);
        for (long kt = -nts + 1; kt < nts; ++kt)
            for (long v = 0; v < nr; ++v)
                F[wrap(kt, L) * nr + v] = G[wrap(kt, rows) * nr + v] * std::conj(radon_mult(p, zeta, kt, v, L));
        fft2d(F.data(), L, nr, +1);
        // G_m^T: scatter fine-grid adjoints into the coefficient image (mirror).
        const double cmb = std::cos(m * p.beta), smb = std::sin(m * p.beta);
        for (long i = 0; i < nf; ++i) {
            const long q = i - nf / 2;
            const double th = double(q) * p.dtheta_lp;
            const double ct = std::cos(th), st = std::sin(th);
            const cd* row = F.data() + wrap(q, L) * nr;
            for (long l = 0; l < nr; ++l) {
                const double er = std::exp(p.log_ar + double(l) * p.drho);
                const double dx = er * ct - (1.0 - p.aR), dy = er * st;
                if (dx * dx + dy * dy > p.aR * p.aR) continue;
                const double ux = dx / p.aR, uy = dy / p.aR;
                const double xp = cmb * ux - smb * uy, yp = smb * ux + cmb * uy;
                const double tc = (0.5 * xp + 0.5) * N, tr = (0.5 * yp + 0.5) * N;
                const long kr = long(std::floor(tr)), kc = long(std::floor(tc));
                double wr[4], wc[4];
                bspline_weights(tr - kr, wr);
                bspline_weights(tc - kc, wc);
                const double v = er * row[l].real();
                for (int a = 0; a < 4; ++a) {
                    const long rr = mirror_index(kr - 1 + a, N);
                    for (int b = 0; b < 4; ++b) acc[rr * N + mirror_index(kc - 1 + b, N)] += v * wr[a] * wc[b];
                }
            }
        }
    }
    prefilter_2d_T(acc.data(), N, N);
    const double scale = 2.0 * p.dtheta_p * p.ds * double(N) * double(N);
    for (long i = 0; i < N * N; ++i) img[i] = scale * acc[i];
}

void fast_backprojection(const Plan& p, const cd* zeta_bp, const double* sino, double* img) {
    const long N = p.N, nts = p.nts, rows = 2 * nts, nr = p.n_rho;
    std::vector<double> qg(sino, sino + p.n_theta * N);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < p.n_theta; ++i) prefilter_1d(qg.data() + i * N, N, 1);  // Alg. 2 step 1 (along s)
    std::vector<std::vector<double>> coef(p.M, std::vector<double>(rows * nr));
    std::vector<cd> G(rows * nr);
    for (int m = 0; m < p.M; ++m) {
        // step 3: g(S_m^{-1}) on Omega_p; theta' rows are polar rows, so the
        // resampling is one-dimensional along s with zero extension.
        std::fill(G.begin(), G.end(), cd(0.0));
#pragma omp parallel for schedule(static)
        for (long j = -nts / 2; j < nts / 2; ++j) {
            long i = long(m) * nts + j;
            const bool flip = i < 0;
            if (flip) i += p.n_theta;
            const double cth = std::cos(double(j) * p.dtheta_p);
            cd* row = G.data() + wrap(j, rows) * nr;
            for (long l = 0; l < nr; ++l) {
                const double er = std::exp(p.log_ar + double(l) * p.drho);
                double sr = 0.5 * (er - (1.0 - p.aR) * cth) / p.aR;
                if (flip) sr = -sr;
                row[l] = eval_zero_1d(qg.data() + i * N, N, (sr + 0.5) * N);
            }
        }
        // step 4: spectral convolution with zeta# / Bhat
        fft2d(G.data(), rows, nr, -1);
        const double scale = 1.0 / (double(rows) * double(nr));
        for (long kt = -nts; kt < nts; ++kt)
            for (long v = 0; v < nr; ++v) {
                const long idx = wrap(kt, rows) * nr + v;
                G[idx] = kt == -nts ? cd(0.0) : G[idx] * zeta_bp[idx] * (scale / (bhat(kt, rows) * bhat(v, nr)));
            }
        fft2d(G.data(), rows, nr, +1);
        for (long i = 0; i < rows * nr; ++i) coef[m][i] = G[i].real();
    }
    // steps 5-7: resample T_m^{-1} Omega_p -> X, sum sectors ascending, x2.
#pragma omp parallel for schedule(static)
    for (long r = 0; r < N; ++r) {
        for (long c = 0; c < N; ++c) {
            const long dxr = 2 * c - N, dyr = 2 * r - N;
            if (dxr * dxr + dyr * dyr > N * N) {  // outside the unit disc
                img[r * N + c] = 0.0;
                continue;
            }
            const double xp = double(dxr) / N, yp = double(dyr) / N;  // physical units
            double acc = 0.0;
            for (int m = 0; m < p.M; ++m) {
                const double cm = std::cos(m * p.beta), sm = std::sin(m * p.beta);
                const double yx = p.aR * (cm * xp + sm * yp) + (1.0 - p.aR);
                const double yy = p.aR * (-sm * xp + cm * yp);
                const double th = std::atan2(yy, yx);
                const double rho = 0.5 * std::log(yx * yx + yy * yy);
                acc += eval_periodic_2d(coef[m].data(), rows, nr, th / p.dtheta_p, (rho - p.log_ar) / p.drho);
            }
            img[r * N + c] = 2.0 * acc;
        }
    }
}

// =================================================================== direct
// Restated brute-force operators (oracle.cpp:193-265) and the modified
// Shepp-Logan phantom (oracle.cpp:95-191).

namespace {
double bilinear_zero(const double* img, long N, double x, double y) {
    const double fr = (y + 0.5) * N, fc = (x + 0.5) * N;
    const long r0 = long(std::floor(fr)), c0 = long(std::floor(fc));
    const double wr = fr - r0, wc = fc - c0;
    auto at = [&](long r, long c) { return (r < 0 || r >= N || c < 0 || c >= N) ? 0.0 : img[r * N + c]; };
    return (1 - wr) * ((1 - wc) * at(r0, c0) + wc * at(r0, c0 + 1)) + wr * ((1 - wc) * at(r0 + 1, c0) + wc * at(r0 + 1, c0 + 1));
}

struct Ell {
    double A, x, y, a, b, deg;
};
// Toft's modified Shepp-Logan table on [-1,1]^2 (the widely used variant).
const Ell kSL[10] = {{1.0, 0.0, 0.0, 0.69, 0.92, 0.0},         {-0.8, 0.0, -0.0184, 0.6624, 0.874, 0.0},
                     {-0.2, 0.22, 0.0, 0.11, 0.31, -18.0},     {-0.2, -0.22, 0.0, 0.16, 0.41, 18.0},
                     {0.1, 0.0, 0.35, 0.21, 0.25, 0.0},        {0.1, 0.0, 0.1, 0.046, 0.046, 0.0},
                     {0.1, 0.0, -0.1, 0.046, 0.046, 0.0},      {0.1, -0.08, -0.605, 0.046, 0.023, 0.0},
                     {0.1, 0.0, -0.605, 0.023, 0.023, 0.0},    {0.1, 0.06, -0.605, 0.023, 0.046, 0.0}};
}  // namespace

void direct_radon(const Plan& p, const double* img, double* sino) {
    const long N = p.N;
    const double h = 1.0 / (2.0 * N);
    const long K = 3 * N;
#pragma omp parallel for schedule(static)
    for (long i = 0; i < p.n_theta; ++i) {
        const double th = i * p.dtheta_p, ct = std::cos(th), st = std::sin(th);
        for (long j = 0; j < N; ++j) {
            const double s = -0.5 + double(j) / N;
            double acc = 0.0;
            for (long k = 0; k <= K; ++k) {
                const double t = -0.75 + k * h;
                const double f = bilinear_zero(img, N, s * ct - t * st, s * st + t * ct);
                acc += (k == 0 || k == K) ? 0.5 * f : f;
            }
            sino[i * N + j] = acc * h;
        }
    }
}

void direct_backprojection(const Plan& p, const double* sino, double* img) {
    const long N = p.N, nt = p.n_theta;
#pragma omp parallel for schedule(static)
    for (long r = 0; r < N; ++r) {
        const double y = -0.5 + double(r) / N;
        for (long c = 0; c < N; ++c) {
            const double x = -0.5 + double(c) / N;
            double acc = 0.0;
            for (long i = 0; i < nt; ++i) {
                const double th = i * p.dtheta_p;
                const double fj = (x * std::cos(th) + y * std::sin(th) + 0.5) * N;
                const long j0 = long(std::floor(fj));
                const double w = fj - j0;
                const double* g = sino + i * N;
                if (j0 >= 0 && j0 + 1 < N) acc += (1 - w) * g[j0] + w * g[j0 + 1];
                else if (j0 == -1) acc += w * g[0];
                else if (j0 == N - 1) acc += (1 - w) * g[N - 1];
            }
            img[r * N + c] = 2.0 * p.dtheta_p * acc;
        }
    }
}

void phantom_image(int N, double* img) {
    for (long r = 0; r < N; ++r) {
        const double y = -0.5 + double(r) / N;
        for (long c = 0; c < N; ++c) {
            const double x = -0.5 + double(c) / N;
            double v = 0.0;
            for (const Ell& e : kSL) {
                const double rot = e.deg * kPi / 180.0, co = std::cos(rot), si = std::sin(rot);
                const double dx = x - 0.5 * e.x, dy = y - 0.5 * e.y;
                const double u = (co * dx + si * dy) / (0.5 * e.a), w = (-si * dx + co * dy) / (0.5 * e.b);
                if (u * u + w * w <= 1.0) v += e.A;
            }
            img[r * N + c] = std::round(v * 10.0) / 10.0;
        }
    }
}

void phantom_sinogram(const Plan& p, double* sino) {
    const long N = p.N;
    for (long i = 0; i < p.n_theta; ++i) {
        const double th = i * p.dtheta_p, ct = std::cos(th), st = std::sin(th);
        for (long j = 0; j < N; ++j) {
            const double s = -0.5 + double(j) / N;
            double v = 0.0;
            for (const Ell& e : kSL) {
                const double a = 0.5 * e.a, b = 0.5 * e.b, rot = e.deg * kPi / 180.0;
                const double sp = s - (0.5 * e.x * ct + 0.5 * e.y * st);
                const double cp = std::cos(th - rot), spn = std::sin(th - rot);
                const double w2 = a * a * cp * cp + b * b * spn * spn;
                const double rad = w2 - sp * sp;
                if (rad > 0.0) v += 2.0 * e.A * a * b * std::sqrt(rad) / w2;
            }
            sino[i * N + j] = v;
        }
    }
}

}  // namespace lpo
