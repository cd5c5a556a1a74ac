// On-disk cache of the kernel spectra ("Spectra are computed once
// per plan and cached; cache keyed by (N, M, N_theta, N_rho)").
//
// One file per (kind, N, M, n_theta, n_rho) in the cache directory:
//   "LPSC" | uint32 version | int32 kind, N, M, n_theta, n_rho | uint64 count |
//   count fp64 values (the (2 nts) x n_rho complex spectrum, re/im interleaved)
// little endian. The spectrum is cached at full fp64 precision (the plan
// folds it with 1/Bhat and rounds to fp32 once, as without the cache). A file
// whose key, size or magic does not match is ignored and rewritten; writes go
// to a temporary name and are renamed into place, so concurrent plan
// creations never read a partial file. The directory comes from
// lpr_spectrum_cache_dir() or, when that was never called, the environment
// variable LPR_SPECTRUM_CACHE; unset = no caching.
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unistd.h>

#include "lpr_host.hpp"

namespace lpr::host {

namespace {

constexpr char kMagic[4] = {'L', 'P', 'S', 'C'};
constexpr std::uint32_t kVersion = 1;

std::mutex g_mu;
bool g_set = false;  // lpr_spectrum_cache_dir was called (overrides the environment)
std::string g_dir;
std::atomic<long long> g_hits{0}, g_stores{0}, g_tmp_seq{0};

std::string cache_dir() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_set) return g_dir;
    const char* e = std::getenv("LPR_SPECTRUM_CACHE");
    return e ? std::string(e) : std::string();
}

std::string cache_path(const std::string& dir, const lpr_geometry& g, int kind) {
    char name[128];
    std::snprintf(name, sizeof(name), "/zeta%d_N%d_M%d_T%d_R%d.lpsc", kind, g.N, g.M, g.n_theta, g.n_rho);
    return dir + name;
}

struct Header {
    char magic[4];
    std::uint32_t version;
    std::int32_t kind, N, M, n_theta, n_rho;
    std::uint64_t count;
};

std::uint64_t spectrum_count(const lpr_geometry& g) { return 2ull * 2ull * std::uint64_t(g.nts) * std::uint64_t(g.n_rho); }

}  // namespace

bool spectrum_cache_load(const lpr_geometry& g, int kind, double* out) {
    const std::string dir = cache_dir();
    if (dir.empty()) return false;
    std::FILE* f = std::fopen(cache_path(dir, g, kind).c_str(), "rb");
    if (!f) return false;
    Header h{};
    const std::uint64_t n = spectrum_count(g);
    bool ok = std::fread(&h, sizeof(h), 1, f) == 1 && std::memcmp(h.magic, kMagic, 4) == 0 &&
              h.version == kVersion && h.kind == kind && h.N == g.N && h.M == g.M && h.n_theta == g.n_theta &&
              h.n_rho == g.n_rho && h.count == n && std::fread(out, sizeof(double), n, f) == n;
    if (ok) {  // exactly the expected length: no trailing bytes
        char extra;
        ok = std::fread(&extra, 1, 1, f) == 0;
    }
    std::fclose(f);
    if (ok) ++g_hits;
    return ok;
}

void spectrum_cache_store(const lpr_geometry& g, int kind, const double* data) {
    const std::string dir = cache_dir();
    if (dir.empty()) return;
    const std::string path = cache_path(dir, g, kind);
    // unique per process and per call, so concurrent stores (threads or ranks) never share a temporary
    const std::string tmp = path + ".tmp" + std::to_string(long(getpid())) + "_" + std::to_string(g_tmp_seq.fetch_add(1));
    std::FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) return;  // an unwritable cache directory only costs the recomputation
    Header h{};
    std::memcpy(h.magic, kMagic, 4);
    h.version = kVersion;
    h.kind = kind;
    h.N = g.N;
    h.M = g.M;
    h.n_theta = g.n_theta;
    h.n_rho = g.n_rho;
    h.count = spectrum_count(g);
    const bool ok = std::fwrite(&h, sizeof(h), 1, f) == 1 && std::fwrite(data, sizeof(double), h.count, f) == h.count;
    if (std::fclose(f) != 0 || !ok || std::rename(tmp.c_str(), path.c_str()) != 0) {
        std::remove(tmp.c_str());
        return;
    }
    ++g_stores;
}

void set_spectrum_cache_dir(const char* dir) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_set = true;
    g_dir = dir ? std::string(dir) : std::string();
}

long long spectrum_cache_hits() { return g_hits.load(); }
long long spectrum_cache_stores() { return g_stores.load(); }

}  // namespace lpr::host
