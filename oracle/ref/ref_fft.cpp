// ORACLE bridge — test infrastructure only. Implements the reference's
// lpr::fft interface (proj/include/lpradon/fft.hpp) on top of the oracle's
// own FFT, replacing FFTW, which this image does not have. The reference's
// test_fft.cpp (roundtrip, impulse, single frequency, Parseval, counter,
// argument errors) runs unchanged against it via oracle/_ref/ref_tests.
#include "lpradon/fft.hpp"

#include <atomic>
#include <stdexcept>

#include "../lpo.hpp"

namespace lpr::fft {

namespace {
std::atomic<std::uint64_t> n2d{0};
void check(std::size_t n, int sign) {
    if (n == 0) throw std::invalid_argument("fft: empty transform");
    if (sign != forward && sign != backward) throw std::invalid_argument("fft: bad sign");
}
}  // namespace

void c2c_2d(std::complex<double>* data, std::size_t rows, std::size_t cols, int sign) {
    check(rows * cols, sign);
    lpo::fft2d(data, long(rows), long(cols), sign);
    n2d.fetch_add(1);
}

void c2c_1d(std::complex<double>* data, std::size_t n, int sign) {
    check(n, sign);
    lpo::fft1d(data, long(n), sign);
}

std::uint64_t transform_count_2d() { return n2d.load(); }
void reset_transform_count_2d() { n2d.store(0); }

}  // namespace lpr::fft
