// Seeded synthetic frame generator (input side of the receiver hot path).
//
// This is NOT the product path and NOT the oracle: it manufactures the c64
// (Y, x_tx) frame pairs that both the CUDA receiver and the CPU oracle consume,
// so both see identical bytes (SURVEY.md §8d "Inputs").  The arithmetic restates
// the reference's signal model in the same operation order so frames match the
// reference generator bit-for-bit before the c64 quantisation:
//   - Rng / derive_seed ............ include/ofdmradar/rng.hpp:11-66
//   - make_random_frame ............ src/waveform.cpp:88-131 (Gray QAM, pilots)
//   - zc_sequence / precode (D = N)  src/zadoffchu.cpp:58-87,98-119,133-136
//   - apply_channel (no validity) .. src/channel.cpp:14-31,65-98
// The model-validity check (channel.cpp:51-63) is deliberately skipped: the
// BASELINE scenes violate it and parity is judged at the
// receiver boundary.
//
// Scene draws (target count, range, velocity per target, SNR) use the stream
// Rng(derive_seed(frame_seed, 0x7363656e)) — a builder choice.

#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

#include "../../include/ofdmr_gen.h"

namespace {

using cplx = std::complex<double>;
constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kC = 3.0e8;

std::uint64_t derive_seed(std::uint64_t base, std::uint64_t stream) {
    std::uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

class Rng {
public:
    explicit Rng(std::uint64_t seed) : e_(seed) {}
    std::uint64_t next_u64() { return e_(); }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    std::uint64_t uniform_int(std::uint64_t n) {
        const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        std::uint64_t v;
        do { v = next_u64(); } while (v >= limit);
        return v % n;
    }
    double normal() {
        if (have_) { have_ = false; return spare_; }
        double u1, u2;
        do { u1 = uniform(); } while (u1 <= 0.0);
        u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = kTwoPi * u2;
        spare_ = r * std::sin(a);
        have_ = true;
        return r * std::cos(a);
    }
private:
    std::mt19937_64 e_;
    double spare_ = 0.0;
    bool have_ = false;
};

int bits_per_symbol(int order) {
    switch (order) {
        case 4: return 2;
        case 16: return 4;
        case 64: return 6;
        case 256: return 8;
        default: return -1;
    }
}

int gray_decode(unsigned g) {
    unsigned b = 0;
    for (; g; g >>= 1) b ^= g;
    return static_cast<int>(b);
}

std::vector<cplx> constellation(int order) {
    const int m = bits_per_symbol(order);
    const int half = m / 2;
    const int levels = 1 << half;
    const double scale = 1.0 / std::sqrt(2.0 * (double(levels) * levels - 1.0) / 3.0);
    std::vector<cplx> pts(static_cast<std::size_t>(order));
    for (int w = 0; w < order; ++w) {
        const unsigned gi = static_cast<unsigned>(w) >> half;
        const unsigned gq = static_cast<unsigned>(w) & ((1u << half) - 1u);
        const double li = double(levels - 1) - 2.0 * gray_decode(gi);
        const double lq = double(levels - 1) - 2.0 * gray_decode(gq);
        pts[static_cast<std::size_t>(w)] = cplx(li * scale, lq * scale);
    }
    return pts;
}

}  // namespace

extern "C" {

/// Generator parameters: include/ofdmr_gen.h

uint64_t ofdmr_derive_seed(uint64_t base, uint64_t stream) { return derive_seed(base, stream); }

}  // extern "C"

namespace {

struct ZcCache {
    std::mutex mtx;
    std::map<std::pair<int, long long>, std::vector<cplx>> mats;
};
ZcCache& zc_cache() {
    static ZcCache c;
    return c;
}

// zadoffchu.cpp:98-119 (even/odd forms), reshaped row-major into D x D with D = N.
const std::vector<cplx>& zc_matrix(int n, long long root) {
    auto& c = zc_cache();
    std::lock_guard<std::mutex> lock(c.mtx);
    auto key = std::make_pair(n, root);
    auto it = c.mats.find(key);
    if (it != c.mats.end()) return it->second;
    const long long l = (long long)n * (long long)n;
    std::vector<cplx> seq(static_cast<std::size_t>(l));
    const double rl = double(root) / double(l);
    for (long long k = 0; k < l; ++k) {
        const double kk = double(k);
        double cycles;
        if (l % 2 == 0) cycles = rl * (kk * kk / 2.0 + 0.0 * kk);
        else cycles = rl * (kk * (kk + 1.0) / 2.0 + 0.0 * kk);
        cycles -= std::floor(cycles);
        seq[static_cast<std::size_t>(k)] = std::polar(1.0, kTwoPi * cycles);
    }
    return c.mats.emplace(key, std::move(seq)).first->second;
}

struct Scene {
    std::vector<double> range, vel;
    double snr_db;
};

Scene draw_scene(const ofdmr_gen_params& p, std::uint64_t frame_seed) {
    Rng rng(derive_seed(frame_seed, 0x7363656e));
    Scene s;
    int count = p.targets_min;
    if (p.targets_max > p.targets_min)
        count += int(rng.uniform_int(std::uint64_t(p.targets_max - p.targets_min + 1)));
    for (int t = 0; t < count; ++t) {
        s.range.push_back(rng.uniform(p.range_lo, p.range_hi));
        s.vel.push_back(rng.uniform(p.vel_lo, p.vel_hi));
    }
    s.snr_db = p.snr_lo_db;
    if (p.snr_hi_db != p.snr_lo_db && std::isfinite(p.snr_lo_db))
        s.snr_db = rng.uniform(p.snr_lo_db, p.snr_hi_db);
    return s;
}

// waveform.cpp:125-131 make_random_frame: pilots in column 0, Gray-QAM payload.
std::vector<cplx> make_random_frame(const ofdmr_gen_params& p, std::uint64_t seed) {
    const std::size_t n = std::size_t(p.n), m = std::size_t(p.m);
    Rng pilot_rng(derive_seed(seed, 0));
    Rng payload_rng(derive_seed(seed, 1));
    static const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
    std::vector<cplx> pilots(n);
    for (auto& v : pilots) {
        const std::uint64_t b = pilot_rng.uniform_int(4);
        v = cplx((b & 1) ? -inv_sqrt2 : inv_sqrt2, (b & 2) ? -inv_sqrt2 : inv_sqrt2);
    }
    const int bps = bits_per_symbol(p.qam_order);
    const auto table = constellation(p.qam_order);
    const std::size_t n_syms = n * (m - 1);
    std::vector<std::uint8_t> bits(n_syms * std::size_t(bps));
    for (auto& b : bits) b = static_cast<std::uint8_t>(payload_rng.uniform_int(2));
    std::vector<cplx> x(n * m);
    std::size_t bp = 0;
    std::vector<cplx> payload(n_syms);
    for (auto& sym : payload) {
        unsigned w = 0;
        for (int b = 0; b < bps; ++b) w = (w << 1) | (bits[bp++] & 1u);
        sym = table[w];
    }
    for (std::size_t k = 0; k < n; ++k) {
        x[k * m] = pilots[k];
        for (std::size_t l = 1; l < m; ++l) x[k * m + l] = payload[k * (m - 1) + (l - 1)];
    }
    return x;
}

// zadoffchu.cpp:58-87 apply_matrix with d == n (plain matrix-vector per column).
std::vector<cplx> precode_direct(const std::vector<cplx>& x, int n, int m, long long root) {
    const auto& zm = zc_matrix(n, root);
    std::vector<cplx> out(x.size());
    std::vector<cplx> col(static_cast<std::size_t>(n)), res(static_cast<std::size_t>(n));
    for (int l = 0; l < m; ++l) {
        for (int k = 0; k < n; ++k) col[std::size_t(k)] = x[std::size_t(k) * m + l];
        for (int i = 0; i < n; ++i) {
            const cplx* zrow = &zm[std::size_t(i) * n];
            cplx acc(0, 0);
            for (int mm = 0; mm < n; ++mm) acc += zrow[mm] * col[std::size_t(mm)];
            res[std::size_t(i)] = acc;
        }
        for (int k = 0; k < n; ++k) out[std::size_t(k) * m + l] = res[std::size_t(k)];
    }
    return out;
}

double mean_power(const std::vector<cplx>& g) {
    if (g.empty()) return 0.0;
    double acc = 0.0;
    for (const auto& v : g) acc += std::norm(v);
    return acc / static_cast<double>(g.size());
}

// channel.cpp:65-98 apply_channel, Normalized amplitudes, random phases, AWGN.
std::vector<cplx> apply_channel(const std::vector<cplx>& x, const Scene& sc, const ofdmr_gen_params& p,
                                std::uint64_t seed, double* sigma2_out) {
    const std::size_t n = std::size_t(p.n), m = std::size_t(p.m);
    const double df = p.df_hz;
    const double t_useful = 1.0 / df;
    const double ts = t_useful + double(p.n_cp) * (t_useful / double(p.n));
    Rng phase_rng(derive_seed(seed, 0x70686173));
    struct Tp { double gain, delay, doppler, phase; };
    std::vector<Tp> tps;
    double total_gain2 = 0.0;
    for (std::size_t t = 0; t < sc.range.size(); ++t) {
        Tp tp;
        tp.gain = 1.0;
        tp.delay = 2.0 * sc.range[t] / kC;
        tp.doppler = 2.0 * sc.vel[t] * p.fc_hz / kC;
        tp.phase = phase_rng.uniform(0.0, kTwoPi);
        total_gain2 += tp.gain * tp.gain;
        tps.push_back(tp);
    }
    std::vector<cplx> y(n * m, cplx(0.0, 0.0));
    std::vector<cplx> dph(n), fph(m);
    for (const auto& tp : tps) {
        for (std::size_t k = 0; k < n; ++k) dph[k] = std::polar(1.0, -kTwoPi * double(k) * df * tp.delay);
        for (std::size_t l = 0; l < m; ++l) fph[l] = std::polar(1.0, kTwoPi * double(l) * ts * tp.doppler);
        const cplx b = std::polar(tp.gain, tp.phase);
        for (std::size_t k = 0; k < n; ++k) {
            const cplx row = b * dph[k];
            for (std::size_t l = 0; l < m; ++l) y[k * m + l] += row * fph[l] * x[k * m + l];
        }
    }
    double sigma2 = 0.0;
    if (std::isfinite(sc.snr_db)) {
        const double snr_lin = std::pow(10.0, sc.snr_db / 10.0);
        const double ref_gain2 = tps.empty() ? 1.0 : total_gain2;
        sigma2 = ref_gain2 * mean_power(x) / snr_lin;
        const double sd = std::sqrt(sigma2 / 2.0);
        Rng noise_rng(derive_seed(seed, 0x6e6f6973));
        // same expression as channel.cpp:94 so the (unspecified) argument
        // evaluation order matches the reference build's compiler
        for (auto& v : y) v += cplx(sd * noise_rng.normal(), sd * noise_rng.normal());
    }
    *sigma2_out = sigma2;
    return y;
}

void store_c64(const std::vector<cplx>& g, float* out) {
    for (std::size_t i = 0; i < g.size(); ++i) {
        out[2 * i] = static_cast<float>(g[i].real());
        out[2 * i + 1] = static_cast<float>(g[i].imag());
    }
}

template <typename F>
void parallel_for(int64_t count, int nthreads, F&& f) {
    if (nthreads <= 1 || count <= 1) {
        for (int64_t i = 0; i < count; ++i) f(i);
        return;
    }
    std::vector<std::thread> pool;
    std::atomic<int64_t> next{0};
    for (int t = 0; t < nthreads; ++t)
        pool.emplace_back([&]() {
            for (;;) {
                const int64_t i = next.fetch_add(1);
                if (i >= count) break;
                f(i);
            }
        });
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

/// One frame: frame_seed = derive_seed(base_seed, frame_index).
/// y, x: N*M interleaved float (c64).  targets_*: up to max_targets entries.
int ofdmr_gen_frame(const ofdmr_gen_params* p, uint64_t base_seed, int64_t frame_index, float* y,
                    float* x_tx, double* sigma2, int32_t* n_targets, double* ranges, double* vels,
                    double* snr_db, int32_t max_targets) {
    if (!p || p->n <= 0 || p->m <= 1 || bits_per_symbol(p->qam_order) < 0) return 2;
    const std::uint64_t fs = derive_seed(base_seed, std::uint64_t(frame_index));
    const Scene sc = draw_scene(*p, fs);
    std::vector<cplx> x = make_random_frame(*p, derive_seed(fs, 0x667261));
    if (p->zc_precode) x = precode_direct(x, p->n, p->m, p->zc_root);
    double s2 = 0.0;
    const std::vector<cplx> yv = apply_channel(x, sc, *p, fs, &s2);
    store_c64(yv, y);
    store_c64(x, x_tx);
    if (sigma2) *sigma2 = s2;
    if (n_targets) *n_targets = int32_t(sc.range.size());
    for (int t = 0; t < int(sc.range.size()) && t < max_targets; ++t) {
        if (ranges) ranges[t] = sc.range[std::size_t(t)];
        if (vels) vels[t] = sc.vel[std::size_t(t)];
    }
    if (snr_db) *snr_db = sc.snr_db;
    return 0;
}

/// run_pipeline's generator half (pipeline.cpp:65-71) for an explicit target list:
/// x = make_random_frame(w, derive_seed(seed, 0x667261)); y = apply_channel(x, targets,
/// snr, seed) — output in fp64 (c128) so it can be pinned bit-exactly to the reference.
int ofdmr_gen_frame_explicit(const ofdmr_gen_params* p, const double* ranges, const double* vels, int32_t count,
                             double snr_db, uint64_t seed, double* y_out, double* x_out, double* sigma2) {
    if (!p || p->n <= 0 || p->m <= 1 || bits_per_symbol(p->qam_order) < 0) return 2;
    Scene sc;
    for (int i = 0; i < count; ++i) {
        sc.range.push_back(ranges[i]);
        sc.vel.push_back(vels[i]);
    }
    sc.snr_db = snr_db;
    std::vector<cplx> x = make_random_frame(*p, derive_seed(seed, 0x667261));
    if (p->zc_precode) x = precode_direct(x, p->n, p->m, p->zc_root);
    double s2 = 0.0;
    const std::vector<cplx> y = apply_channel(x, sc, *p, seed, &s2);
    for (std::size_t i = 0; i < y.size(); ++i) {
        y_out[2 * i] = y[i].real();
        y_out[2 * i + 1] = y[i].imag();
        x_out[2 * i] = x[i].real();
        x_out[2 * i + 1] = x[i].imag();
    }
    *sigma2 = s2;
    return 0;
}

/// Batch of frames [first, first+count) on nthreads host threads.
int ofdmr_gen_batch(const ofdmr_gen_params* p, uint64_t base_seed, int64_t first, int64_t count,
                    float* y, float* x_tx, double* sigma2, int32_t* n_targets, double* ranges,
                    double* vels, double* snr_db, int32_t max_targets, int nthreads) {
    if (!p) return 2;
    const std::size_t cells = std::size_t(p->n) * std::size_t(p->m);
    if (p->zc_precode) zc_matrix(p->n, p->zc_root);  // build once before fan-out
    std::atomic<int> rc{0};
    parallel_for(count, nthreads, [&](int64_t i) {
        const int r = ofdmr_gen_frame(p, base_seed, first + i, y + 2 * cells * std::size_t(i),
                                      x_tx + 2 * cells * std::size_t(i), sigma2 ? sigma2 + i : nullptr,
                                      n_targets ? n_targets + i : nullptr,
                                      ranges ? ranges + i * max_targets : nullptr,
                                      vels ? vels + i * max_targets : nullptr,
                                      snr_db ? snr_db + i : nullptr, max_targets);
        if (r) rc = r;
    });
    return rc.load();
}

/// On-grid sparse channel estimate for the FPS-SFT path (cfg3):
/// H[a,b] = sum_p A_p e^{j2pi(a k_p/N + b l_p/M)} + CN(0, sigma2), distinct k and
/// distinct l per tone, |A| = 1, uniform phase (make_sparse, tests/test_sft.cpp:20-50),
/// sigma2 = K / 10^(snr/10) (apply_channel's convention with unit |X|).
int ofdmr_gen_sparse(int32_t n, int32_t m, int32_t k_count, double snr_db, uint64_t base_seed,
                     int64_t frame_index, float* h, double* sigma2, int32_t* tk, int32_t* tl,
                     double* amp_re, double* amp_im) {
    if (n <= 0 || m <= 0 || k_count < 0 || k_count > n || k_count > m) return 2;
    const std::uint64_t fs = derive_seed(base_seed, std::uint64_t(frame_index));
    Rng rng(derive_seed(fs, 0x73706172));
    std::vector<int> ks, ls;
    std::vector<cplx> amps;
    std::vector<char> used_k(static_cast<std::size_t>(n), 0), used_l(static_cast<std::size_t>(m), 0);
    while (int(ks.size()) < k_count) {
        const int k = int(rng.uniform_int(std::uint64_t(n)));
        const int l = int(rng.uniform_int(std::uint64_t(m)));
        if (used_k[std::size_t(k)] || used_l[std::size_t(l)]) continue;
        used_k[std::size_t(k)] = 1;
        used_l[std::size_t(l)] = 1;
        ks.push_back(k);
        ls.push_back(l);
        amps.push_back(std::polar(1.0, rng.uniform(0.0, kTwoPi)));
    }
    std::vector<cplx> g(std::size_t(n) * std::size_t(m), cplx(0, 0));
    std::vector<cplx> rowph(static_cast<std::size_t>(n)), colph(static_cast<std::size_t>(m));
    for (int t = 0; t < k_count; ++t) {
        for (int a = 0; a < n; ++a)
            rowph[std::size_t(a)] = std::polar(1.0, kTwoPi * double((long long)a * ks[std::size_t(t)] % n) / double(n));
        for (int b = 0; b < m; ++b)
            colph[std::size_t(b)] = std::polar(1.0, kTwoPi * double((long long)b * ls[std::size_t(t)] % m) / double(m));
        for (int a = 0; a < n; ++a) {
            const cplx r = amps[std::size_t(t)] * rowph[std::size_t(a)];
            for (int b = 0; b < m; ++b) g[std::size_t(a) * m + b] += r * colph[std::size_t(b)];
        }
    }
    double s2 = 0.0;
    if (std::isfinite(snr_db)) {
        s2 = double(k_count > 0 ? k_count : 1) / std::pow(10.0, snr_db / 10.0);
        const double sd = std::sqrt(s2 / 2.0);
        for (auto& v : g) v += cplx(sd * rng.normal(), sd * rng.normal());
    }
    store_c64(g, h);
    if (sigma2) *sigma2 = s2;
    for (int t = 0; t < k_count; ++t) {
        if (tk) tk[t] = ks[std::size_t(t)];
        if (tl) tl[t] = ls[std::size_t(t)];
        if (amp_re) amp_re[t] = amps[std::size_t(t)].real();
        if (amp_im) amp_im[t] = amps[std::size_t(t)].imag();
    }
    return 0;
}

int ofdmr_gen_sparse_batch(int32_t n, int32_t m, int32_t k_count, double snr_db, uint64_t base_seed,
                           int64_t first, int64_t count, float* h, double* sigma2, int32_t* tk,
                           int32_t* tl, int nthreads) {
    const std::size_t cells = std::size_t(n) * std::size_t(m);
    std::atomic<int> rc{0};
    parallel_for(count, nthreads, [&](int64_t i) {
        const int r = ofdmr_gen_sparse(n, m, k_count, snr_db, base_seed, first + i,
                                       h + 2 * cells * std::size_t(i), sigma2 ? sigma2 + i : nullptr,
                                       tk ? tk + i * k_count : nullptr, tl ? tl + i * k_count : nullptr,
                                       nullptr, nullptr);
        if (r) rc = r;
    });
    return rc.load();
}

/// Complex AWGN grid CN(0, sigma2) from Rng(seed) (noise_grid, tests/test_periodogram.cpp:31-37).
int ofdmr_gen_noise_grid(int32_t n, int32_t m, double sigma2, uint64_t seed, double* out) {
    Rng rng(seed);
    const double sd = std::sqrt(sigma2 / 2.0);
    for (std::size_t i = 0; i < std::size_t(n) * std::size_t(m); ++i) {
        const cplx v(sd * rng.normal(), sd * rng.normal());
        out[2 * i] = v.real();
        out[2 * i + 1] = v.imag();
    }
    return 0;
}

/// Raw Rng draws for pinning the MT19937-64 stream (tests).
void ofdmr_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
    Rng rng(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = rng.next_u64();
}

}  // extern "C"
