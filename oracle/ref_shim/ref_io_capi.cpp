// ORACLE / TEST INFRASTRUCTURE ONLY.
// extern "C" adapters over the reference's OWN output writers (io.cpp:28-110), compiled
// where they lie by oracle/Makefile into oracle/_ref/libofdmref_io.so, so the golden
// fixtures hold the bytes the reference writes for a given map / detection list.
#include <cstdint>
#include <string>
#include <vector>

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

}  // extern "C"
