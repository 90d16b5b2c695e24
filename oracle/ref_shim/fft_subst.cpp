// ORACLE / TEST INFRASTRUCTURE ONLY.
// Substitute for the reference's FFTW3-backed src/fft.cpp (FFTW3 is absent from
// this image and cannot be installed).  Implements the unchanged interface
// include/ofdmradar/fft.hpp:13-29 (unscaled; forward e^{-j}, inverse e^{+j}) on top
// of the oracle's own double-precision FFT (oracle/oracle.c orc_fft: radix-2 for
// powers of two, Bluestein otherwise).  Every CPU figure built on this is labelled
// "reference sources + substitute FFT".
#include "ofdmradar/fft.hpp"

#include <vector>

extern "C" void orc_fft(double* data, std::size_t n, int sign);

namespace ofdmradar::fft {
namespace {

void run(cplx* data, std::size_t n, std::size_t howmany, std::size_t stride, std::size_t dist, int sign) {
    if (n == 0 || howmany == 0) return;
    if (stride == 1) {
        for (std::size_t h = 0; h < howmany; ++h)
            orc_fft(reinterpret_cast<double*>(data + h * dist), n, sign);
        return;
    }
    thread_local std::vector<cplx> buf;
    buf.resize(n);
    for (std::size_t h = 0; h < howmany; ++h) {
        cplx* base = data + h * dist;
        for (std::size_t i = 0; i < n; ++i) buf[i] = base[i * stride];
        orc_fft(reinterpret_cast<double*>(buf.data()), n, sign);
        for (std::size_t i = 0; i < n; ++i) base[i * stride] = buf[i];
    }
}

}  // namespace

void forward(cplx* data, std::size_t n) { run(data, n, 1, 1, n, -1); }
void inverse(cplx* data, std::size_t n) { run(data, n, 1, 1, n, +1); }
void forward_copy(const cplx* in, cplx* out, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i) out[i] = in[i];
    run(out, n, 1, 1, n, -1);
}
void forward_rows(cplx* data, std::size_t rows, std::size_t cols) { run(data, cols, rows, 1, cols, -1); }
void inverse_rows(cplx* data, std::size_t rows, std::size_t cols) { run(data, cols, rows, 1, cols, +1); }
void forward_cols(cplx* data, std::size_t rows, std::size_t cols) { run(data, rows, cols, cols, 1, -1); }
void inverse_cols(cplx* data, std::size_t rows, std::size_t cols) { run(data, rows, cols, cols, 1, +1); }

}  // namespace ofdmradar::fft
