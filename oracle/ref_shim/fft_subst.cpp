// ORACLE / TEST INFRASTRUCTURE ONLY.
// Substitute for the reference's FFTW3-backed src/fft.cpp (FFTW3 is absent from this image
// and cannot be installed).  Implements the unchanged interface include/ofdmradar/fft.hpp:13-29
// (unscaled; forward e^{-j}, inverse e^{+j}) for the reference's own receiver sources, so that
// the CPU baseline ("reference sources + substitute FFT") is not handicapped by a slow FFT:
//
//  * plans cached per (n, sign) for the life of the process, like the reference's FFTW plan
//    cache (fft.cpp:17-43): per-stage twiddle tables, computed once;
//  * power-of-two n: iterative radix-4 Stockham autosort (no bit reversal, natural order out,
//    one radix-2 stage when log2 n is odd), ping-ponging with a thread-local work vector;
//  * other n: Bluestein chirp-z on the cached power-of-two plans (chirp and kernel transform
//    cached too);
//  * strided batches (the column passes) gathered / scattered in blocks of adjacent columns
//    so every cache line of the row-major grid is touched once per block, like FFTW's
//    vector loops in plan_many_dft.
//
// Every CPU figure built on it is labelled "reference sources + substitute FFT".  The C
// restatement's own FFT (oracle.c orc_fft) is separate and unchanged (it is bit-pinned against
// the golden vectors and mirrored by the GPU FPS-SFT).
#include "ofdmradar/fft.hpp"

#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

namespace ofdmradar::fft {
namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

struct Stage {
    std::size_t len;           // sub-transform length at this stage (4 or 2 for the last radix-2)
    std::vector<cplx> tw;      // radix-4: 3 twiddles per p (W^p, W^2p, W^3p), p < len/4
};

struct Plan {
    std::size_t n = 0;
    int sign = -1;
    std::vector<Stage> stages;     // power-of-two plans
    // Bluestein (n not a power of two)
    std::size_t m = 0;
    std::vector<cplx> chirp, kernel;
    const Plan* inner_fwd = nullptr;
    const Plan* inner_inv = nullptr;
};

const Plan* get_plan(std::size_t n, int sign);

Plan* make_pow2(std::size_t n, int sign) {
    auto* p = new Plan;
    p->n = n;
    p->sign = sign;
    for (std::size_t len = n; len >= 4; len /= 4) {
        Stage st;
        st.len = len;
        const std::size_t q = len / 4;
        st.tw.resize(3 * q);
        for (std::size_t k = 0; k < q; ++k)
            for (std::size_t r = 1; r <= 3; ++r) {
                const double a = double(sign) * kTwoPi * double(r * k) / double(len);
                st.tw[3 * k + r - 1] = cplx(std::cos(a), std::sin(a));
            }
        p->stages.push_back(std::move(st));
        if (len / 4 < 4) {
            if (len / 4 == 2) p->stages.push_back(Stage{2, {}});
            break;
        }
    }
    if (n == 2) p->stages.push_back(Stage{2, {}});
    return p;
}

// y <- radix-4 Stockham step of x (sub-transform length len, stride s), see make_pow2.  Real
// arithmetic written out (std::complex's operator* goes through __muldc3's inf/nan handling
// without -ffast-math, which FFTW's codelets do not pay either).
template <bool INV>
inline __attribute__((always_inline)) void radix4(const cplx* xc, cplx* yc, std::size_t len, std::size_t s, const cplx* twc) {
    const double* x = reinterpret_cast<const double*>(xc);
    double* y = reinterpret_cast<double*>(yc);
    const double* tw = reinterpret_cast<const double*>(twc);
    const std::size_t q = len / 4;
    for (std::size_t p = 0; p < q; ++p) {
        const double w1r = tw[6 * p], w1i = tw[6 * p + 1], w2r = tw[6 * p + 2], w2i = tw[6 * p + 3];
        const double w3r = tw[6 * p + 4], w3i = tw[6 * p + 5];
        const double* xa = x + 2 * s * p;
        double* ya = y + 2 * s * 4 * p;
        const std::size_t o1 = 2 * s * q, o2 = 4 * s * q, o3 = 6 * s * q;
        for (std::size_t i = 0; i < 2 * s; i += 2) {
            const double ar = xa[i], ai = xa[i + 1], br = xa[i + o1], bi = xa[i + o1 + 1];
            const double cr = xa[i + o2], ci = xa[i + o2 + 1], dr = xa[i + o3], di = xa[i + o3 + 1];
            const double apcr = ar + cr, apci = ai + ci, amcr = ar - cr, amci = ai - ci;
            const double bpdr = br + dr, bpdi = bi + di, bmdr = br - dr, bmdi = bi - di;
            // forward: (a - c) - j (b - d) for r = 1; inverse: (a - c) + j (b - d)
            const double jbr = INV ? -bmdi : bmdi, jbi = INV ? bmdr : -bmdr;
            const double t1r = amcr + jbr, t1i = amci + jbi;
            const double t2r = apcr - bpdr, t2i = apci - bpdi;
            const double t3r = amcr - jbr, t3i = amci - jbi;
            ya[i] = apcr + bpdr;
            ya[i + 1] = apci + bpdi;
            ya[i + 2 * s] = w1r * t1r - w1i * t1i;
            ya[i + 2 * s + 1] = w1r * t1i + w1i * t1r;
            ya[i + 4 * s] = w2r * t2r - w2i * t2i;
            ya[i + 4 * s + 1] = w2r * t2i + w2i * t2r;
            ya[i + 6 * s] = w3r * t3r - w3i * t3i;
            ya[i + 6 * s + 1] = w3r * t3i + w3i * t3r;
        }
    }
}

// AVX2/FMA and baseline x86-64 clones, picked at load time (FFTW also dispatches its SIMD
// codelets at run time)
__attribute__((target_clones("avx2,fma", "default"))) void radix4_fwd(const cplx* x, cplx* y, std::size_t len,
                                                                    std::size_t s, const cplx* tw) {
    radix4<false>(x, y, len, s, tw);
}
__attribute__((target_clones("avx2,fma", "default"))) void radix4_inv(const cplx* x, cplx* y, std::size_t len,
                                                                    std::size_t s, const cplx* tw) {
    radix4<true>(x, y, len, s, tw);
}

void run_pow2(const Plan& p, cplx* data) {
    const std::size_t n = p.n;
    thread_local std::vector<cplx> work;
    if (work.size() < n) work.resize(n);
    cplx* cur = data;
    cplx* nxt = work.data();
    std::size_t s = 1;
    for (const Stage& st : p.stages) {
        if (st.len == 2) {
            for (std::size_t i = 0; i < s; ++i) {
                const cplx a = cur[i], b = cur[i + s];
                nxt[i] = a + b;
                nxt[i + s] = a - b;
            }
            s *= 2;
        } else {
            if (p.sign > 0) radix4_inv(cur, nxt, st.len, s, st.tw.data());
            else radix4_fwd(cur, nxt, st.len, s, st.tw.data());
            s *= 4;
        }
        std::swap(cur, nxt);
    }
    if (cur != data)
        for (std::size_t i = 0; i < n; ++i) data[i] = cur[i];
}

Plan* make_bluestein(std::size_t n, int sign) {
    auto* p = new Plan;
    p->n = n;
    p->sign = sign;
    std::size_t m = 1;
    while (m < 2 * n - 1) m <<= 1;
    p->m = m;
    p->chirp.resize(n);
    for (std::size_t k = 0; k < n; ++k) {
        const unsigned long long k2 = (static_cast<unsigned long long>(k) * k) % (2ULL * n);
        const double a = double(sign) * kTwoPi * 0.5 * double(k2) / double(n);
        p->chirp[k] = cplx(std::cos(a), std::sin(a));
    }
    p->kernel.assign(m, cplx(0.0, 0.0));
    p->kernel[0] = std::conj(p->chirp[0]);
    for (std::size_t k = 1; k < n; ++k) p->kernel[k] = p->kernel[m - k] = std::conj(p->chirp[k]);
    p->inner_fwd = get_plan(m, -1);
    p->inner_inv = get_plan(m, +1);
    run_pow2(*p->inner_fwd, p->kernel.data());
    return p;
}

void run_bluestein(const Plan& p, cplx* data) {
    thread_local std::vector<cplx> a;
    a.assign(p.m, cplx(0.0, 0.0));
    auto mul = [](cplx u, cplx v) {
        return cplx(u.real() * v.real() - u.imag() * v.imag(), u.real() * v.imag() + u.imag() * v.real());
    };
    for (std::size_t k = 0; k < p.n; ++k) a[k] = mul(data[k], p.chirp[k]);
    run_pow2(*p.inner_fwd, a.data());
    for (std::size_t k = 0; k < p.m; ++k) a[k] = mul(a[k], p.kernel[k]);
    run_pow2(*p.inner_inv, a.data());
    const double inv_m = 1.0 / double(p.m);
    for (std::size_t k = 0; k < p.n; ++k) data[k] = mul(a[k] * inv_m, p.chirp[k]);
}

const Plan* get_plan(std::size_t n, int sign) {
    static std::map<std::pair<std::size_t, int>, std::unique_ptr<Plan>> cache;
    static std::recursive_mutex mtx;  // Bluestein plans create their inner plans under the lock
    std::lock_guard<std::recursive_mutex> lock(mtx);
    auto it = cache.find({n, sign});
    if (it != cache.end()) return it->second.get();
    Plan* p = (n & (n - 1)) == 0 ? make_pow2(n, sign) : make_bluestein(n, sign);
    cache.emplace(std::make_pair(n, sign), std::unique_ptr<Plan>(p));
    return p;
}

void transform(const Plan& p, cplx* v) {
    if (p.m) run_bluestein(p, v);
    else run_pow2(p, v);
}

void run(cplx* data, std::size_t n, std::size_t howmany, std::size_t stride, std::size_t dist, int sign) {
    if (n == 0 || howmany == 0) return;
    if (n == 1) return;
    const Plan& p = *get_plan(n, sign);
    if (stride == 1) {
        for (std::size_t h = 0; h < howmany; ++h) transform(p, data + h * dist);
        return;
    }
    // strided vectors: gather a block of B vectors (adjacent when dist == 1) row by row
    constexpr std::size_t B = 8;
    thread_local std::vector<cplx> buf;
    buf.resize(B * n);
    for (std::size_t h0 = 0; h0 < howmany; h0 += B) {
        const std::size_t nb = std::min(B, howmany - h0);
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t b = 0; b < nb; ++b) buf[b * n + i] = data[(h0 + b) * dist + i * stride];
        for (std::size_t b = 0; b < nb; ++b) transform(p, buf.data() + b * n);
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t b = 0; b < nb; ++b) data[(h0 + b) * dist + i * stride] = buf[b * n + i];
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
