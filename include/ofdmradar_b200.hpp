// ofdmradar_b200.hpp — header-only C++ shim that re-exposes the reference receiver
// signatures (namespace ofdmradar, /root/reference/proj/include/ofdmradar/*.hpp) on top of
// the C-ABI in ofdmr_b200.h, so reference callers can switch by namespace:
//
//     ofdmradar::periodogram(h, w, np, mp)      ->  ofdmradar::b200::periodogram(h, w, np, mp)
//
// Value semantics as in the reference: inputs are host ComplexGrid (complex<double>),
// quantised once to complex64 for the device; results come back as fp64 containers.
// Errors: OFDMR_ERR_CONFIG -> ofdmradar::ConfigError (errors.hpp:9-12), CUDA errors ->
// std::runtime_error.  One cached device context per (shape, window, estimator, L, K,
// pfa) and host thread (the reference functions are reentrant).
#pragma once

#include <cuda_runtime.h>

#include <complex>
#include <cstdint>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "ofdmr_b200.h"
#include "ofdmradar/errors.hpp"
#include "ofdmradar/grid.hpp"
#include "ofdmradar/periodogram.hpp"
#include "ofdmradar/sft.hpp"
#include "ofdmradar/waveform.hpp"

namespace ofdmradar::b200 {
namespace detail {

inline void check(int rc) {
    if (rc == OFDMR_OK) return;
    if (rc == OFDMR_ERR_CONFIG) throw ConfigError(ofdmr_last_error());
    throw std::runtime_error(std::string("ofdmr: ") + ofdmr_last_error());
}
inline void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + cudaGetErrorString(e));
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(std::size_t n) { cuda(cudaMalloc(&p, sizeof(T) * (n ? n : 1))); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

struct Ctx {
    ofdmr_context* c = nullptr;
    explicit Ctx(const ofdmr_config& cfg) { check(ofdmr_create(&cfg, &c)); }
    ~Ctx() { ofdmr_destroy(c); }
};

inline ofdmr_context* context(int32_t n, int32_t m, int32_t np, int32_t mp, int32_t window, int32_t estimator,
                              int32_t n_cp, int32_t k, double pfa) {
    thread_local std::map<std::tuple<int, int, int, int, int, int, int, int, double>, std::unique_ptr<Ctx>> cache;
    const auto key = std::make_tuple(n, m, np, mp, window, estimator, n_cp, k, pfa);
    auto it = cache.find(key);
    if (it == cache.end()) {
        ofdmr_config cfg{n, m, np, mp, window, estimator, n_cp, k, pfa, 0, 0};
        it = cache.emplace(key, std::make_unique<Ctx>(cfg)).first;
    }
    return it->second->c;
}

inline std::vector<float> to_c64(const ComplexGrid& g) {
    std::vector<float> v(2 * g.size());
    for (std::size_t i = 0; i < g.size(); ++i) {
        v[2 * i] = static_cast<float>(g.storage()[i].real());
        v[2 * i + 1] = static_cast<float>(g.storage()[i].imag());
    }
    return v;
}

inline ComplexGrid from_c64(const std::vector<float>& v, std::size_t n, std::size_t m, AxisTag tag) {
    std::vector<cplx> d(n * m);
    for (std::size_t i = 0; i < n * m; ++i) d[i] = cplx(v[2 * i], v[2 * i + 1]);
    return ComplexGrid(n, m, tag, std::move(d));
}

inline int32_t window_kind(const Window2d& w) {
    for (double v : w.subcarrier)
        if (v != 1.0) return OFDMR_WINDOW_HAMMING;
    for (double v : w.symbol)
        if (v != 1.0) return OFDMR_WINDOW_HAMMING;
    return OFDMR_WINDOW_RECT;
}

}  // namespace detail

// estimation.hpp:9 — H = Y / X; ConfigError on shape mismatch or a zero X cell.
inline ComplexGrid spectral_division(const ComplexGrid& y, const ComplexGrid& x) {
    using namespace detail;
    if (y.rows() != x.rows() || y.cols() != x.cols()) throw ConfigError("spectral_division: shape mismatch");
    const int32_t n = int32_t(y.rows()), m = int32_t(y.cols());
    ofdmr_context* c = context(n, m, n, m, OFDMR_WINDOW_RECT, OFDMR_EST_LS, 0, 1, 1e-2);
    const auto yh = to_c64(y), xh = to_c64(x);
    DevBuf<float> yd(yh.size()), xd(xh.size()), hd(yh.size());
    DevBuf<int32_t> st(1);
    cuda(cudaMemcpy(yd.p, yh.data(), sizeof(float) * yh.size(), cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(xd.p, xh.data(), sizeof(float) * xh.size(), cudaMemcpyHostToDevice));
    check(ofdmr_spectral_division(c, yd.p, xd.p, hd.p, st.p, 1));
    int32_t status = 0;
    std::vector<float> hh(yh.size());
    cuda(cudaMemcpy(&status, st.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(hh.data(), hd.p, sizeof(float) * hh.size(), cudaMemcpyDeviceToHost));
    if (status & 1) throw ConfigError("spectral_division: zero cell in X");
    return from_c64(hh, y.rows(), y.cols(), AxisTag::SubcarrierSymbol);
}

// estimation.hpp:14 — DFT-CE with truncation length n_cp.
inline ComplexGrid dft_ce(const ComplexGrid& h, std::size_t n_cp) {
    using namespace detail;
    if (n_cp > h.rows()) throw ConfigError("dft_ce: truncation length exceeds N");
    const int32_t n = int32_t(h.rows()), m = int32_t(h.cols());
    ofdmr_context* c = context(n, m, n, m, OFDMR_WINDOW_RECT, OFDMR_EST_DFT_CE, int32_t(n_cp), 1, 1e-2);
    const auto hh = to_c64(h);
    DevBuf<float> hd(hh.size()), od(hh.size());
    cuda(cudaMemcpy(hd.p, hh.data(), sizeof(float) * hh.size(), cudaMemcpyHostToDevice));
    check(ofdmr_dft_ce(c, hd.p, od.p, 1));
    std::vector<float> oh(hh.size());
    cuda(cudaMemcpy(oh.data(), od.p, sizeof(float) * oh.size(), cudaMemcpyDeviceToHost));
    return from_c64(oh, h.rows(), h.cols(), h.tag());
}

// periodogram.hpp:39-40 — N' x M' map, Doppler fft-shifted, |.|^2/(NM).
inline RealGrid periodogram(const ComplexGrid& h, const Window2d& window, std::size_t n_prime, std::size_t m_prime) {
    using namespace detail;
    if (n_prime < h.rows() || m_prime < h.cols()) throw ConfigError("periodogram: N' >= N and M' >= M required");
    if (window.subcarrier.size() != h.rows() || window.symbol.size() != h.cols())
        throw ConfigError("periodogram: window shape mismatch");
    const int32_t n = int32_t(h.rows()), m = int32_t(h.cols());
    ofdmr_context* c = context(n, m, int32_t(n_prime), int32_t(m_prime), window_kind(window), OFDMR_EST_LS, 0, 1, 1e-2);
    const auto hh = to_c64(h);
    DevBuf<float> hd(hh.size()), pd(n_prime * m_prime);
    cuda(cudaMemcpy(hd.p, hh.data(), sizeof(float) * hh.size(), cudaMemcpyHostToDevice));
    check(ofdmr_periodogram(c, hd.p, pd.p, 1));
    std::vector<float> ph(n_prime * m_prime);
    cuda(cudaMemcpy(ph.data(), pd.p, sizeof(float) * ph.size(), cudaMemcpyDeviceToHost));
    RealGrid p(n_prime, m_prime);
    for (std::size_t i = 0; i < ph.size(); ++i) p.storage()[i] = ph[i];
    return p;
}

// periodogram.hpp:60-61 — greedy strict 3x3 peaks on a threshold mask.  The device entry
// point takes the threshold; for a mask produced by threshold_mask (P >= eta) the smallest
// masked value reproduces it exactly.
inline std::vector<Detection> extract_peaks(const RealGrid& p, const std::vector<std::uint8_t>& mask,
                                            std::size_t max_targets, const WaveformConfig& cfg) {
    using namespace detail;
    if (mask.size() != p.size()) throw ConfigError("extract_peaks: mask shape mismatch");
    double eta = 0.0;
    bool any = false;
    for (std::size_t i = 0; i < p.size(); ++i)
        if (mask[i] && (!any || p.storage()[i] < eta)) {
            eta = p.storage()[i];
            any = true;
        }
    if (!any || max_targets == 0) return {};
    const int32_t k = int32_t(max_targets > 64 ? 64 : max_targets);
    const int32_t np = int32_t(p.rows()), mp = int32_t(p.cols());
    ofdmr_context* c = context(np, mp, np, mp, OFDMR_WINDOW_RECT, OFDMR_EST_LS, 0, k, 1e-2);
    std::vector<float> ph(p.size());
    for (std::size_t i = 0; i < p.size(); ++i) ph[i] = static_cast<float>(p.storage()[i]);
    DevBuf<float> pd(ph.size()), pw(k);
    DevBuf<double> ed(1);
    DevBuf<int32_t> dd(k), vd(k), cn(1);
    cuda(cudaMemcpy(pd.p, ph.data(), sizeof(float) * ph.size(), cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(ed.p, &eta, sizeof(double), cudaMemcpyHostToDevice));
    check(ofdmr_extract_peaks(c, pd.p, ed.p, nullptr, dd.p, vd.p, pw.p, cn.p, 1));
    int32_t cnt = 0;
    std::vector<int32_t> dh(k), vh(k);
    std::vector<float> wh(k);
    cuda(cudaMemcpy(&cnt, cn.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(dh.data(), dd.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(vh.data(), vd.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(wh.data(), pw.p, sizeof(float) * k, cudaMemcpyDeviceToHost));
    std::vector<Detection> out(static_cast<std::size_t>(cnt));
    for (int32_t i = 0; i < cnt; ++i) {
        out[i].delay_bin = dh[i];
        out[i].doppler_bin = vh[i];
        out[i].peak_power = p.at(std::size_t(dh[i]), std::size_t(vh[i] + mp / 2));  // exact fp64 value of the cell
        bins_to_physics(out[i], cfg);  // reference host formula (periodogram.cpp:138-144)
    }
    return out;
}

// periodogram.hpp (estimate_noise_power, periodogram.cpp:146-152) — median cell / ln 2 /
// window power factor.  The map is quantised to fp32 on the device, so the selected order
// statistic is the fp32 rounding of the reference's (relative difference <= 2^-24).
inline double estimate_noise_power(const RealGrid& p, double window_power_factor) {
    using namespace detail;
    const int32_t np = int32_t(p.rows()), mp = int32_t(p.cols());
    ofdmr_context* c = context(np, mp, np, mp, OFDMR_WINDOW_RECT, OFDMR_EST_LS, 0, 1, 1e-2);  // pf = 1
    std::vector<float> ph(p.size());
    for (std::size_t i = 0; i < p.size(); ++i) ph[i] = static_cast<float>(p.storage()[i]);
    DevBuf<float> pd(ph.size());
    DevBuf<double> sd(1);
    cuda(cudaMemcpy(pd.p, ph.data(), sizeof(float) * ph.size(), cudaMemcpyHostToDevice));
    check(ofdmr_estimate_noise_power(c, pd.p, sd.p, 1));
    double s2 = 0.0;
    cuda(cudaMemcpy(&s2, sd.p, sizeof(double), cudaMemcpyDeviceToHost));
    return s2 / window_power_factor;  // (v / ln 2 / 1) / pf == v / ln 2 / pf
}

// waveform.hpp:81 — CP strip + forward DFT per symbol.
inline ComplexGrid ofdm_demodulate(std::span<const cplx> stream, const WaveformConfig& cfg) {
    using namespace detail;
    const std::size_t n = cfg.n_subcarriers, m = cfg.n_symbols, ns = cfg.samples_per_symbol();
    if (stream.size() != m * ns) throw ConfigError("stream length must be M*(N+Ncp)");
    ofdmr_context* c = context(int32_t(n), int32_t(m), int32_t(n), int32_t(m), OFDMR_WINDOW_RECT, OFDMR_EST_LS,
                               int32_t(cfg.n_cp), 1, 1e-2);
    std::vector<float> sh(2 * stream.size());
    for (std::size_t i = 0; i < stream.size(); ++i) {
        sh[2 * i] = static_cast<float>(stream[i].real());
        sh[2 * i + 1] = static_cast<float>(stream[i].imag());
    }
    DevBuf<float> sd(sh.size()), gd(2 * n * m);
    cuda(cudaMemcpy(sd.p, sh.data(), sizeof(float) * sh.size(), cudaMemcpyHostToDevice));
    check(ofdmr_ofdm_demodulate(c, sd.p, gd.p, 1));
    std::vector<float> gh(2 * n * m);
    cuda(cudaMemcpy(gh.data(), gd.p, sizeof(float) * gh.size(), cudaMemcpyDeviceToHost));
    return from_c64(gh, n, m, AxisTag::SubcarrierSymbol);
}

// waveform.hpp:78 — per-symbol inverse DFT (1/N) with cyclic prefix.
inline std::vector<cplx> ofdm_modulate(const ComplexGrid& x, const WaveformConfig& cfg) {
    using namespace detail;
    const std::size_t n = cfg.n_subcarriers, m = cfg.n_symbols, ns = cfg.samples_per_symbol();
    if (x.rows() != n || x.cols() != m) throw ConfigError("grid shape does not match config");
    ofdmr_context* c = context(int32_t(n), int32_t(m), int32_t(n), int32_t(m), OFDMR_WINDOW_RECT, OFDMR_EST_LS,
                               int32_t(cfg.n_cp), 1, 1e-2);
    const auto xh = to_c64(x);
    DevBuf<float> xd(xh.size()), sd(2 * m * ns);
    cuda(cudaMemcpy(xd.p, xh.data(), sizeof(float) * xh.size(), cudaMemcpyHostToDevice));
    check(ofdmr_ofdm_modulate(c, xd.p, sd.p, 1));
    std::vector<float> sh(2 * m * ns);
    cuda(cudaMemcpy(sh.data(), sd.p, sizeof(float) * sh.size(), cudaMemcpyDeviceToHost));
    std::vector<cplx> out(m * ns);
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = cplx(sh[2 * i], sh[2 * i + 1]);
    return out;
}

// sft.hpp:62 — FPS-SFT on the GPU (power-of-two N, M with lcm <= 2048).
inline SparseSpectrum sft_iterate(const ComplexGrid& h, const SftConfig& cfg) {
    using namespace detail;
    if (h.rows() == 0 || h.cols() == 0) throw ConfigError("sft_iterate: empty grid");
    const int32_t n = int32_t(h.rows()), m = int32_t(h.cols());
    ofdmr_context* c = context(16, 16, 16, 16, OFDMR_WINDOW_RECT, OFDMR_EST_LS, 0, 1, 1e-2);
    ofdmr_sft_config sc{int32_t(cfg.i_max), cfg.detect_threshold, cfg.pfa, int32_t(cfg.decimation), cfg.frac_tol,
                        cfg.amp_tol, 64};
    const auto hh = to_c64(h);
    DevBuf<float> hd(hh.size());
    DevBuf<int32_t> kd(64), ld(64), ne(1), it(1), cv(1);
    DevBuf<double> ad(128), rs(1);
    DevBuf<int64_t> su(1);
    cuda(cudaMemcpy(hd.p, hh.data(), sizeof(float) * hh.size(), cudaMemcpyHostToDevice));
    const uint64_t seed = cfg.seed;
    const double s2 = cfg.sigma2;
    check(ofdmr_sft(c, hd.p, n, m, &sc, &seed, &s2, kd.p, ld.p, ad.p, ne.p, it.p, su.p, cv.p, rs.p, nullptr, 1));
    cuda(cudaDeviceSynchronize());
    int32_t nent = 0, iters = 0, conv = 0;
    int64_t used = 0;
    double resid = 0.0;
    std::vector<int32_t> kh(64), lh(64);
    std::vector<double> ah(128);
    cuda(cudaMemcpy(&nent, ne.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(&iters, it.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(&conv, cv.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(&used, su.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(&resid, rs.p, sizeof(double), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(kh.data(), kd.p, sizeof(int32_t) * 64, cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(lh.data(), ld.p, sizeof(int32_t) * 64, cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(ah.data(), ad.p, sizeof(double) * 128, cudaMemcpyDeviceToHost));
    SparseSpectrum s;
    for (int32_t i = 0; i < nent && i < 64; ++i) s.entries.push_back({kh[i], lh[i], cplx(ah[2 * i], ah[2 * i + 1])});
    s.residual_energy = resid;
    s.converged = conv != 0;
    s.iterations = std::size_t(iters);
    s.samples_used = std::size_t(used);
    return s;
}

namespace detail {
// Detection records of an FPS-SFT entry set: peak_power recomputed in fp64 from the matching
// entry (the device record carries it in fp32), physics as sft.cpp:476-479.
inline std::vector<Detection> sft_records(const std::vector<int32_t>& dh, const std::vector<int32_t>& vh,
                                          int32_t cnt, const SparseSpectrum& spec, std::size_t n, std::size_t m,
                                          const WaveformConfig& cfg) {
    std::vector<Detection> out(static_cast<std::size_t>(cnt));
    const double nm = double(n) * double(m);
    for (int32_t i = 0; i < cnt; ++i) {
        Detection& d = out[i];
        d.delay_bin = dh[i];
        d.doppler_bin = vh[i];
        const long k = (long(n) - d.delay_bin) % long(n), l = ((d.doppler_bin % long(m)) + long(m)) % long(m);
        for (const auto& e : spec.entries)
            if (long(e.k) == k && long(e.l) == l) d.peak_power = std::norm(e.amplitude) * nm;
        d.range_m = kSpeedOfLight * double(d.delay_bin) / (2.0 * double(n) * cfg.subcarrier_spacing_hz);
        d.velocity_mps =
            kSpeedOfLight * double(d.doppler_bin) / (2.0 * cfg.carrier_hz * double(m) * cfg.symbol_time());
    }
    return out;
}
}  // namespace detail

// sft.hpp:67-70 — detections_from_spectrum through the device entry point (ofdmr_sft_detections):
// threshold, bin mapping and the (power, delay, Doppler) ranking run on the GPU in fp64.
inline std::vector<Detection> detections_from_spectrum(const SparseSpectrum& spec, std::size_t n, std::size_t m,
                                                       const WaveformConfig& cfg, double sigma2, double pfa,
                                                       std::size_t max_targets) {
    using namespace detail;
    if (sigma2 < 0.0) throw ConfigError("threshold: sigma2 must be >= 0");
    if (!(pfa > 0.0 && pfa <= 1.0)) throw ConfigError("threshold: pfa must lie in (0,1]");
    if (spec.entries.empty() || max_targets == 0) return {};
    if (spec.entries.size() > 64) throw ConfigError("detections_from_spectrum: at most 64 entries on the GPU path");
    const int32_t k = int32_t(max_targets > 64 ? 64 : max_targets);
    const int32_t ne = int32_t(spec.entries.size());
    ofdmr_context* c = context(16, 16, 16, 16, OFDMR_WINDOW_RECT, OFDMR_EST_LS, 0, k, 1e-2);
    std::vector<int32_t> kh(ne), lh(ne);
    std::vector<double> ah(2 * ne);
    for (int32_t i = 0; i < ne; ++i) {
        kh[i] = int32_t(spec.entries[i].k);
        lh[i] = int32_t(spec.entries[i].l);
        ah[2 * i] = spec.entries[i].amplitude.real();
        ah[2 * i + 1] = spec.entries[i].amplitude.imag();
    }
    DevBuf<int32_t> kd(ne), ld(ne), nd(1), dd(k), vd(k), cn(1);
    DevBuf<double> ad(2 * ne), sd(1);
    DevBuf<float> pw(k);
    cuda(cudaMemcpy(kd.p, kh.data(), sizeof(int32_t) * ne, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(ld.p, lh.data(), sizeof(int32_t) * ne, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(ad.p, ah.data(), sizeof(double) * 2 * ne, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(nd.p, &ne, sizeof(int32_t), cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(sd.p, &sigma2, sizeof(double), cudaMemcpyHostToDevice));
    check(ofdmr_sft_detections(c, kd.p, ld.p, ad.p, nd.p, ne, int32_t(n), int32_t(m), sd.p, pfa, nullptr, dd.p, vd.p,
                               pw.p, cn.p, 1));
    int32_t cnt = 0;
    std::vector<int32_t> dh(k), vh(k);
    cuda(cudaMemcpy(&cnt, cn.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(dh.data(), dd.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(vh.data(), vd.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost));
    return sft_records(dh, vh, cnt, spec, n, m, cfg);
}

// sft.hpp:73-75 — sft_detect (sft.cpp:492-500): sigma2 / pfa fill the SftConfig when unset.
inline std::vector<Detection> sft_detect(const ComplexGrid& h, const WaveformConfig& cfg, const SftConfig& sft_cfg,
                                         double sigma2, double pfa, std::size_t max_targets) {
    SftConfig scfg = sft_cfg;
    if (scfg.sigma2 == 0.0) scfg.sigma2 = sigma2;
    if (scfg.pfa <= 0.0) scfg.pfa = pfa;
    const SparseSpectrum spec = b200::sft_iterate(h, scfg);
    return b200::detections_from_spectrum(spec, h.rows(), h.cols(), cfg, sigma2, pfa, max_targets);
}

}  // namespace ofdmradar::b200
