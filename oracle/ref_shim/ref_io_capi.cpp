// ORACLE / TEST INFRASTRUCTURE ONLY.
// extern "C" adapters over the reference's OWN output writers (io.cpp:28-110), compiled
// where they lie by oracle/Makefile into oracle/_ref/libofdmref_io.so, so the golden
// fixtures hold the bytes the reference writes for a given map / detection list.
#include <cstdint>
#include <string>
#include <vector>

#include <cmath>
#include <limits>

#include "ofdmradar/config.hpp"
#include "ofdmradar/io.hpp"

using namespace ofdmradar;

namespace {
RealGrid real_grid(const double* p, int64_t rows, int64_t cols) {
    RealGrid g(rows, cols);
    for (int64_t i = 0; i < rows * cols; ++i) g.storage()[i] = p[i];
    return g;
}
}  // namespace

extern "C" {

int ref_write_map_csv(const double* p, int64_t rows, int64_t cols, const char* path) {
    try {
        write_map_csv(path, real_grid(p, rows, cols));
        return 0;
    } catch (...) { return 2; }
}

int ref_write_map_pgm(const double* p, int64_t rows, int64_t cols, const char* path) {
    try {
        write_map_pgm(path, real_grid(p, rows, cols));
        return 0;
    } catch (...) { return 2; }
}

int ref_write_detections_csv(const long* delay, const long* doppler, const double* power, const double* range_m,
                             const double* velocity, int64_t n, const char* path) {
    try {
        std::vector<Detection> d(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            d[i].delay_bin = delay[i];
            d[i].doppler_bin = doppler[i];
            d[i].peak_power = power[i];
            d[i].range_m = range_m[i];
            d[i].velocity_mps = velocity[i];
        }
        write_detections_csv(path, d);
        return 0;
    } catch (...) { return 2; }
}

// write_run_manifest (io.cpp:112-122) on a config assembled from plain parameters.
int ref_write_run_manifest(const char* path, const char* command, uint64_t seed, int64_t n, int64_t m, double df,
                           double fc, int64_t n_cp, int32_t qam, int64_t np, int64_t mp, int32_t window, double pfa,
                           int32_t estimator, int32_t detector, int64_t max_targets, int32_t estimate_noise,
                           int64_t i_max, const double* ranges, const double* vels, const double* phases,
                           int32_t count, double snr_db, const char* const* extra_k, const char* const* extra_v,
                           int32_t n_extra, double wall_ms) {
    try {
        RunManifest man;
        man.command = command;
        man.seed = seed;
        SimulationConfig& c = man.config;
        c.waveform.n_subcarriers = std::size_t(n);
        c.waveform.n_symbols = std::size_t(m);
        c.waveform.subcarrier_spacing_hz = df;
        c.waveform.carrier_hz = fc;
        c.waveform.n_cp = std::size_t(n_cp);
        c.waveform.qam_order = qam;
        c.waveform.n_prime = std::size_t(np);
        c.waveform.m_prime = std::size_t(mp);
        c.waveform.window = window ? WindowKind::Hamming : WindowKind::Rectangular;
        c.waveform.pfa = pfa;
        for (int32_t i = 0; i < count; ++i) {
            RadarTarget t{};
            t.range_m = ranges[i];
            t.velocity_mps = vels[i];
            t.phase_rad = phases ? phases[i] : std::numeric_limits<double>::quiet_NaN();
            c.targets.push_back(t);
        }
        c.channel.snr_db = snr_db;
        c.channel.seed = seed;
        c.estimator.kind = estimator == 1 ? EstimatorKind::DftCe : (estimator == 2 ? EstimatorKind::ZcpLs : EstimatorKind::Ls);
        c.detector.kind = detector ? DetectorKind::FpsSft : DetectorKind::Periodogram;
        c.detector.max_targets = std::size_t(max_targets);
        c.detector.estimate_noise = estimate_noise != 0;
        c.detector.sft_i_max = std::size_t(i_max);
        for (int32_t i = 0; i < n_extra; ++i) man.extra.emplace_back(extra_k[i], extra_v[i]);
        man.wall_ms = wall_ms;
        write_run_manifest(path, man);
        return 0;
    } catch (...) { return 2; }
}

}  // extern "C"
