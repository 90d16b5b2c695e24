// ORACLE / TEST INFRASTRUCTURE ONLY.
// extern "C" entry points over the reference's OWN receiver sources (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libofdmref.so) so the
// Python tests can (a) pin the C restatement oracle/oracle.c against the reference
// and (b) time the reference as the CPU baseline.  No reference source is copied:
// these are thin adapters that call ofdmradar:: functions.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "ofdmradar/channel.hpp"
#include "ofdmradar/errors.hpp"
#include "ofdmradar/config.hpp"
#include "ofdmradar/estimation.hpp"
#include "ofdmradar/metrics.hpp"
#include "ofdmradar/periodogram.hpp"
#include "ofdmradar/pipeline.hpp"
#include "ofdmradar/rng.hpp"
#include "ofdmradar/sft.hpp"
#include "ofdmradar/waveform.hpp"

using namespace ofdmradar;

namespace {

ComplexGrid grid_from(const double* v, std::size_t n, std::size_t m) {
    std::vector<cplx> d(n * m);
    for (std::size_t i = 0; i < n * m; ++i) d[i] = cplx(v[2 * i], v[2 * i + 1]);
    return ComplexGrid(n, m, AxisTag::SubcarrierSymbol, std::move(d));
}
ComplexGrid grid_from32(const float* v, std::size_t n, std::size_t m) {
    std::vector<cplx> d(n * m);
    for (std::size_t i = 0; i < n * m; ++i) d[i] = cplx(double(v[2 * i]), double(v[2 * i + 1]));
    return ComplexGrid(n, m, AxisTag::SubcarrierSymbol, std::move(d));
}
void grid_to(const ComplexGrid& g, double* out) {
    for (std::size_t i = 0; i < g.size(); ++i) {
        out[2 * i] = g.storage()[i].real();
        out[2 * i + 1] = g.storage()[i].imag();
    }
}

WaveformConfig make_wave(std::size_t n, std::size_t m, std::size_t np, std::size_t mp, double df, double fc,
                         std::size_t n_cp, int window, double pfa) {
    WaveformConfig w;
    w.n_subcarriers = n;
    w.n_symbols = m;
    w.subcarrier_spacing_hz = df;
    w.carrier_hz = fc;
    w.n_cp = n_cp;
    w.qam_order = 4;
    w.n_prime = np;
    w.m_prime = mp;
    w.window = window ? WindowKind::Hamming : WindowKind::Rectangular;
    w.pfa = pfa;
    return w;
}

// pipeline.cpp:18-23 division_noise_power lives in an anonymous namespace there; this is
// the same three-line formula so the adapter can reproduce run_pipeline's receiver half.
double division_noise_power(double sigma2, const ComplexGrid& x_tx) {
    if (sigma2 <= 0.0) return 0.0;
    double inv_acc = 0.0;
    for (const auto& v : x_tx.storage()) inv_acc += 1.0 / std::norm(v);
    return sigma2 * inv_acc / double(x_tx.size());
}

}  // namespace

extern "C" {

int ref_spectral_division(const double* y, const double* x, double* h, int64_t n, int64_t m) {
    try {
        grid_to(spectral_division(grid_from(y, n, m), grid_from(x, n, m)), h);
        return 0;
    } catch (const ConfigError&) { return 2; }
}

int ref_dft_ce(const double* h, double* out, int64_t n, int64_t m, int64_t n_cp) {
    try {
        grid_to(dft_ce(grid_from(h, n, m), std::size_t(n_cp)), out);
        return 0;
    } catch (const ConfigError&) { return 2; }
}

int ref_periodogram(const double* h, int64_t n, int64_t m, int window, int64_t np, int64_t mp, double* p) {
    try {
        const auto win = make_window(window ? WindowKind::Hamming : WindowKind::Rectangular, n, m);
        const RealGrid g = periodogram(grid_from(h, n, m), win, np, mp);
        for (std::size_t i = 0; i < g.size(); ++i) p[i] = g.storage()[i];
        return 0;
    } catch (const ConfigError&) { return 2; }
}

double ref_estimate_noise_power(const double* p, int64_t rows, int64_t cols, double pf) {
    RealGrid g(rows, cols);
    for (int64_t i = 0; i < rows * cols; ++i) g.storage()[i] = p[i];
    return estimate_noise_power(g, pf);
}

int ref_ofdm_modulate(const double* x, int64_t n, int64_t m, int64_t n_cp, double* stream) {
    try {
        const WaveformConfig w = make_wave(n, m, n, m, 1.0, 1.0, n_cp, 0, 0.01);
        const std::vector<cplx> s = ofdm_modulate(grid_from(x, n, m), w);
        for (std::size_t i = 0; i < s.size(); ++i) {
            stream[2 * i] = s[i].real();
            stream[2 * i + 1] = s[i].imag();
        }
        return 0;
    } catch (const ConfigError&) { return 2; }
}

int ref_ofdm_demodulate(const double* stream, int64_t n, int64_t m, int64_t n_cp, double* x) {
    try {
        const WaveformConfig w = make_wave(n, m, n, m, 1.0, 1.0, n_cp, 0, 0.01);
        std::vector<cplx> s(std::size_t(m * (n + n_cp)));
        for (std::size_t i = 0; i < s.size(); ++i) s[i] = cplx(stream[2 * i], stream[2 * i + 1]);
        grid_to(ofdm_demodulate(s, w), x);
        return 0;
    } catch (const ConfigError&) { return 2; }
}

double ref_window_power_factor(int window, int64_t n, int64_t m) {
    return make_window(window ? WindowKind::Hamming : WindowKind::Rectangular, n, m).power_factor();
}

int ref_detection_threshold(double sigma2, double pfa, double pf, double* eta) {
    try {
        *eta = detection_threshold(sigma2, pfa, pf);
        return 0;
    } catch (const ConfigError&) { return 2; }
}

long ref_extract_peaks(const double* p, int64_t rows, int64_t cols, double eta, int64_t max_targets, long* delay,
                       long* doppler, double* power) {
    RealGrid g(rows, cols);
    for (std::size_t i = 0; i < g.size(); ++i) g.storage()[i] = p[i];
    const auto mask = threshold_mask(g, eta);
    WaveformConfig w = make_wave(std::size_t(rows), std::size_t(cols), rows, cols, 240e3, 77e9, rows / 4, 0, 1e-2);
    const auto dets = extract_peaks(g, mask, std::size_t(max_targets), w);
    for (std::size_t i = 0; i < dets.size(); ++i) {
        delay[i] = dets[i].delay_bin;
        doppler[i] = dets[i].doppler_bin;
        power[i] = dets[i].peak_power;
    }
    return long(dets.size());
}

void ref_bins_to_physics(long delay_bin, long doppler_bin, int64_t n, int64_t m, int64_t np, int64_t mp, double df,
                         double fc, int64_t n_cp, double* range_m, double* vel) {
    WaveformConfig w = make_wave(n, m, np, mp, df, fc, n_cp, 0, 1e-2);
    Detection d;
    d.delay_bin = delay_bin;
    d.doppler_bin = doppler_bin;
    bins_to_physics(d, w);
    *range_m = d.range_m;
    *vel = d.velocity_mps;
}

/// Receiver half of run_pipeline (pipeline.cpp:72-96) on c64 frames upcast to fp64.
int ref_receive_frame(int64_t n, int64_t m, int64_t np, int64_t mp, int estimator, int64_t n_cp, int window,
                      double pfa, const float* y32, const float* x32, double sigma2, int64_t max_targets,
                      long* delay, long* doppler, double* power, long* count, double* s2h_out, double* eta_out,
                      double* p_out) {
    try {
        SimulationConfig cfg;
        cfg.waveform = make_wave(n, m, np, mp, 240e3, 77e9, n_cp, window, pfa);
        cfg.estimator.kind = estimator ? EstimatorKind::DftCe : EstimatorKind::Ls;
        const ComplexGrid y = grid_from32(y32, n, m);
        const ComplexGrid x = grid_from32(x32, n, m);
        const ComplexGrid h = estimate_channel(y, x, cfg);
        const double s2h = division_noise_power(sigma2, x);
        const Window2d win = make_window(cfg.waveform.window, n, m);
        const RealGrid p = periodogram(h, win, np, mp);
        const double eta = detection_threshold(s2h, pfa, win.power_factor());
        const auto mask = threshold_mask(p, eta);
        const auto dets = extract_peaks(p, mask, std::size_t(max_targets), cfg.waveform);
        for (std::size_t i = 0; i < dets.size(); ++i) {
            delay[i] = dets[i].delay_bin;
            doppler[i] = dets[i].doppler_bin;
            power[i] = dets[i].peak_power;
        }
        *count = long(dets.size());
        if (s2h_out) *s2h_out = s2h;
        if (eta_out) *eta_out = eta;
        if (p_out)
            for (std::size_t i = 0; i < p.size(); ++i) p_out[i] = p.storage()[i];
        return 0;
    } catch (const ConfigError&) { return 2; }
}

/// Batch of frames, one frame per host thread (reference is reentrant).
int ref_receive_batch(int64_t n, int64_t m, int64_t np, int64_t mp, int estimator, int64_t n_cp, int window,
                      double pfa, const float* y, const float* x, const double* sigma2, int64_t frames,
                      const int32_t* k_per_frame, int64_t k_max, long* delay, long* doppler, double* power,
                      long* count, int nthreads) {
    std::atomic<int64_t> next{0};
    std::atomic<int> rc{0};
    const std::size_t cells = std::size_t(n) * std::size_t(m);
    auto work = [&]() {
        for (;;) {
            const int64_t f = next.fetch_add(1);
            if (f >= frames) break;
            const int64_t kf = k_per_frame ? k_per_frame[f] : k_max;
            const int r = ref_receive_frame(n, m, np, mp, estimator, n_cp, window, pfa, y + 2 * cells * f,
                                            x + 2 * cells * f, sigma2[f], kf, delay + f * k_max,
                                            doppler + f * k_max, power + f * k_max, count + f, nullptr, nullptr,
                                            nullptr);
            if (r) rc = r;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < (nthreads > 0 ? nthreads : 1); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    return rc.load();
}

/// sft_iterate (sft.cpp:185-459) on an fp64 grid.
int ref_sft_iterate(const double* h, int64_t n, int64_t m, int64_t i_max, double detect_threshold, uint64_t seed,
                    double sigma2, double pfa, int64_t decimation, double frac_tol, double amp_tol,
                    int64_t max_entries, long* ek, long* el, double* ea_re, double* ea_im, int64_t* n_entries,
                    double* residual, int32_t* converged, int64_t* iterations, int64_t* samples_used) {
    try {
        SftConfig c;
        c.i_max = std::size_t(i_max);
        c.detect_threshold = detect_threshold;
        c.seed = seed;
        c.sigma2 = sigma2;
        c.pfa = pfa;
        c.decimation = std::size_t(decimation);
        c.frac_tol = frac_tol;
        c.amp_tol = amp_tol;
        const SparseSpectrum s = sft_iterate(grid_from(h, n, m), c);
        *n_entries = int64_t(s.entries.size());
        for (std::size_t i = 0; i < s.entries.size() && int64_t(i) < max_entries; ++i) {
            ek[i] = s.entries[i].k;
            el[i] = s.entries[i].l;
            ea_re[i] = s.entries[i].amplitude.real();
            ea_im[i] = s.entries[i].amplitude.imag();
        }
        *residual = s.residual_energy;
        *converged = s.converged ? 1 : 0;
        *iterations = int64_t(s.iterations);
        *samples_used = int64_t(s.samples_used);
        return 0;
    } catch (const ConfigError&) { return 2; }
}

int ref_sft_batch_c64(const float* h, int64_t n, int64_t m, int64_t frames, int64_t i_max, const uint64_t* seeds,
                      const double* sigma2, double pfa, int64_t decimation, int64_t max_entries, long* ek, long* el,
                      double* ea_re, double* ea_im, int64_t* n_entries, int nthreads) {
    std::atomic<int64_t> next{0};
    std::atomic<int> rc{0};
    const std::size_t cells = std::size_t(n) * std::size_t(m);
    auto work = [&]() {
        for (;;) {
            const int64_t f = next.fetch_add(1);
            if (f >= frames) break;
            SftConfig c;
            c.i_max = std::size_t(i_max);
            c.seed = seeds[f];
            c.sigma2 = sigma2[f];
            c.pfa = pfa;
            c.decimation = std::size_t(decimation);
            try {
                const SparseSpectrum s = sft_iterate(grid_from32(h + 2 * cells * f, n, m), c);
                n_entries[f] = int64_t(s.entries.size());
                for (std::size_t i = 0; i < s.entries.size() && int64_t(i) < max_entries; ++i) {
                    ek[f * max_entries + i] = s.entries[i].k;
                    el[f * max_entries + i] = s.entries[i].l;
                    ea_re[f * max_entries + i] = s.entries[i].amplitude.real();
                    ea_im[f * max_entries + i] = s.entries[i].amplitude.imag();
                }
            } catch (const ConfigError&) { rc = 2; }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < (nthreads > 0 ? nthreads : 1); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    return rc.load();
}

/// make_random_frame + apply_channel (validity-checked) for pinning the generator.
int ref_make_frame_pair(int64_t n, int64_t m, double df, double fc, int64_t n_cp, int qam, const double* ranges,
                        const double* vels, int64_t n_targets, double snr_db, uint64_t seed, double* y_out,
                        double* x_out, double* sigma2) {
    try {
        WaveformConfig w = make_wave(n, m, n, m, df, fc, n_cp, 0, 1e-2);
        w.qam_order = qam;
        std::vector<RadarTarget> t(static_cast<std::size_t>(n_targets));
        for (int64_t i = 0; i < n_targets; ++i) {
            t[std::size_t(i)].range_m = ranges[i];
            t[std::size_t(i)].velocity_mps = vels[i];
        }
        const ComplexGrid x = make_random_frame(w, derive_seed(seed, 0x667261));
        auto [y, real] = apply_channel(x, t, w, snr_db, seed);
        grid_to(y, y_out);
        grid_to(x, x_out);
        *sigma2 = real.sigma2;
        return 0;
    } catch (const ConfigError&) { return 2; } catch (const ModelValidityError&) { return 3; }
}

void ref_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
    Rng r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

namespace {
SimulationConfig scenario(int64_t n, int64_t m, int64_t np, int64_t mp, double df, double fc, int64_t n_cp,
                          int window, double pfa, int estimator, const double* ranges, const double* vels,
                          int32_t count) {
    SimulationConfig cfg;
    cfg.waveform = make_wave(std::size_t(n), std::size_t(m), std::size_t(np), std::size_t(mp), df, fc,
                             std::size_t(n_cp), window, pfa);
    for (int i = 0; i < count; ++i) {
        RadarTarget t{};
        t.range_m = ranges[i];
        t.velocity_mps = vels[i];
        cfg.targets.push_back(t);
    }
    cfg.estimator.kind = estimator == 1 ? EstimatorKind::DftCe : EstimatorKind::Ls;
    cfg.detector.max_targets = std::size_t(count);
    return cfg;
}
}  // namespace

/// One run of the reference's run_pipeline (pipeline.cpp:60-115) on that scenario with the
/// given run seed and SNR; detections as (delay_bin, doppler_bin, range_m, velocity_mps).
int ref_run_pipeline(int64_t n, int64_t m, int64_t np, int64_t mp, double df, double fc, int64_t n_cp, int window,
                     double pfa, int estimator, const double* ranges, const double* vels, int32_t count,
                     double snr_db, uint64_t seed, long* delay, long* doppler, double* range_m, double* vel_mps,
                     long* n_det) {
    try {
        SimulationConfig cfg = scenario(n, m, np, mp, df, fc, n_cp, window, pfa, estimator, ranges, vels, count);
        cfg.channel.snr_db = snr_db;
        const auto res = run_pipeline(cfg, seed);
        for (std::size_t i = 0; i < res.detections.size(); ++i) {
            delay[i] = res.detections[i].delay_bin;
            doppler[i] = res.detections[i].doppler_bin;
            range_m[i] = res.detections[i].range_m;
            vel_mps[i] = res.detections[i].velocity_mps;
        }
        *n_det = long(res.detections.size());
        return 0;
    } catch (const ConfigError&) {
        return 2;
    } catch (...) {  // ModelValidityError (scene outside the CP / ICI bounds) and the rest
        return 3;
    }
}

/// run_pipeline (pipeline.cpp:60-115) with the FPS-SFT detector (DetectorKind::FpsSft, sft_i_max,
/// optionally estimate_noise) on a scenario whose frames ref_make_frame_pair rebuilds with the same
/// seed: detections (delay, Doppler, peak power) and PipelineResult::sigma2_used.
int ref_run_pipeline_sft(int64_t n, int64_t m, double df, double fc, int64_t n_cp, int qam, int estimator,
                         const double* ranges, const double* vels, int32_t count, double snr_db, uint64_t seed,
                         int estimate_noise, int64_t i_max, int64_t max_targets, long* delay, long* doppler,
                         double* power, long* n_det, double* sigma2_used) {
    try {
        SimulationConfig cfg = scenario(n, m, n, m, df, fc, n_cp, 0, 0.01, estimator, ranges, vels, count);
        cfg.waveform.qam_order = std::size_t(qam);
        cfg.channel.snr_db = snr_db;
        cfg.detector.kind = DetectorKind::FpsSft;
        cfg.detector.estimate_noise = estimate_noise != 0;
        cfg.detector.sft_i_max = std::size_t(i_max);
        cfg.detector.max_targets = std::size_t(max_targets);
        const auto res = run_pipeline(cfg, seed);
        for (std::size_t i = 0; i < res.detections.size(); ++i) {
            delay[i] = res.detections[i].delay_bin;
            doppler[i] = res.detections[i].doppler_bin;
            power[i] = res.detections[i].peak_power;
        }
        *n_det = long(res.detections.size());
        *sigma2_used = res.sigma2_used;
        return 0;
    } catch (const ConfigError&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

/// ref_run_pipeline with an explicit QAM order (table1 / fig8 use 16-QAM).
int ref_run_pipeline_q(int64_t n, int64_t m, int64_t np, int64_t mp, double df, double fc, int64_t n_cp, int window,
                       double pfa, int estimator, const double* ranges, const double* vels, int32_t count, int qam,
                       double snr_db, uint64_t seed, long* delay, long* doppler, long* n_det) {
    try {
        SimulationConfig cfg = scenario(n, m, np, mp, df, fc, n_cp, window, pfa, estimator, ranges, vels, count);
        cfg.waveform.qam_order = std::size_t(qam);
        cfg.channel.snr_db = snr_db;
        const auto res = run_pipeline(cfg, seed);
        for (std::size_t i = 0; i < res.detections.size(); ++i) {
            delay[i] = res.detections[i].delay_bin;
            doppler[i] = res.detections[i].doppler_bin;
        }
        *n_det = long(res.detections.size());
        return 0;
    } catch (const ConfigError&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

/// The reference's own bench_estimators (metrics.cpp:145-253) on a base waveform; rows out as
/// arrays (periodogram_ms, sft_ms, speedup, samples_used) per size.  Returns 4 when the
/// reference's support precondition throws.
int ref_bench_estimators(int64_t n, int64_t m, double df, double fc, int qam, int window, double pfa, double snr_db,
                         const int64_t* sizes, int32_t count, int64_t k, int64_t repeats, uint64_t seed, double* pg_ms,
                         double* sft_ms, double* speedup, int64_t* samples) {
    try {
        SimulationConfig cfg;
        cfg.waveform = make_wave(std::size_t(n), std::size_t(m), std::size_t(n), std::size_t(m), df, fc,
                                 std::size_t(n / 4), window, pfa);
        cfg.waveform.qam_order = std::size_t(qam);
        cfg.channel.snr_db = snr_db;
        std::vector<std::size_t> sz(sizes, sizes + count);
        const auto rows = bench_estimators(cfg, sz, std::size_t(k), std::size_t(repeats), seed);
        for (std::size_t i = 0; i < rows.size(); ++i) {
            pg_ms[i] = rows[i].periodogram_ms;
            sft_ms[i] = rows[i].sft_ms;
            speedup[i] = rows[i].speedup;
            samples[i] = int64_t(rows[i].samples_used);
        }
        return 0;
    } catch (const ConfigError&) {
        return 2;
    } catch (const std::runtime_error&) {
        return 4;
    } catch (...) {
        return 3;
    }
}

/// run_pipeline (pipeline.cpp:60-115) with the FPS-SFT detector in estimate-noise mode: the
/// reference's own sigma2_used (= estimate_noise_from_slice(h, derive_seed(seed, 0x6e6573)),
/// an anonymous-namespace function) and the channel estimate h it was computed from, rebuilt
/// with the same public calls run_pipeline makes (pipeline.cpp:65-72).
int ref_sft_noise_case(int64_t n, int64_t m, double df, double fc, int64_t n_cp, const double* ranges,
                       const double* vels, int32_t count, double snr_db, uint64_t seed, double* h_out,
                       double* sigma2_used) {
    try {
        SimulationConfig cfg = scenario(n, m, n, m, df, fc, n_cp, 0, 0.01, 0, ranges, vels, count);
        cfg.channel.snr_db = snr_db;
        cfg.detector.kind = DetectorKind::FpsSft;
        cfg.detector.estimate_noise = true;
        const auto res = run_pipeline(cfg, seed);
        *sigma2_used = res.sigma2_used;
        const WaveformConfig& w = cfg.waveform;
        const ComplexGrid x = make_random_frame(w, derive_seed(seed, 0x667261));
        auto [y, realization] = apply_channel(x, cfg.targets, w, cfg.channel.snr_db, seed, cfg.channel.amplitude_mode);
        (void)realization;
        grid_to(estimate_channel(y, x, cfg), h_out);
        return 0;
    } catch (const ConfigError&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

/// The reference's own Monte-Carlo RMSE sweep (metrics.cpp:92-120) on a scenario built from
/// plain parameters: QPSK, normalized gains, random phases, targets (ranges, vels),
/// estimator 0 LS / 1 DFT-CE.  rows[i] = {range_rmse_m, velocity_rmse_mps, miss_rate}.
int ref_rmse_sweep(int64_t n, int64_t m, int64_t np, int64_t mp, double df, double fc, int64_t n_cp, int window,
                   double pfa, int estimator, const double* ranges, const double* vels, int32_t count,
                   const double* snr_grid, int32_t n_snr, int64_t trials, uint64_t seed, double* rows) {
    try {
        SimulationConfig cfg = scenario(n, m, np, mp, df, fc, n_cp, window, pfa, estimator, ranges, vels, count);
        const EstimatorKind kind = cfg.estimator.kind;
        std::vector<double> grid(snr_grid, snr_grid + n_snr);
        const auto out = rmse_sweep(cfg, kind, grid, std::size_t(trials), seed);
        for (std::size_t i = 0; i < out.size(); ++i) {
            rows[3 * i] = out[i].range_rmse_m;
            rows[3 * i + 1] = out[i].velocity_rmse_mps;
            rows[3 * i + 2] = out[i].miss_rate;
        }
        return 0;
    } catch (const ConfigError&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

/// The reference's mse_sweep (metrics.cpp:122-143) on the same scenario; rows[i] = MSE.
int ref_mse_sweep(int64_t n, int64_t m, int64_t np, int64_t mp, double df, double fc, int64_t n_cp, int window,
                  double pfa, int estimator, const double* ranges, const double* vels, int32_t count,
                  const double* snr_grid, int32_t n_snr, int64_t trials, uint64_t seed, double* rows) {
    try {
        SimulationConfig cfg = scenario(n, m, np, mp, df, fc, n_cp, window, pfa, estimator, ranges, vels, count);
        std::vector<double> grid(snr_grid, snr_grid + n_snr);
        const auto out = mse_sweep(cfg, cfg.estimator.kind, grid, std::size_t(trials), seed);
        for (std::size_t i = 0; i < out.size(); ++i) rows[i] = out[i].channel_mse;
        return 0;
    } catch (const ConfigError&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

}  // extern "C"
