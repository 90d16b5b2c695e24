/* Seeded synthetic frame generator: parameters shared by the CPU generator
 * (paper_2209_03883_b200/csrc/gen.cpp, libofdmr_gen.so) and the GPU generator
 * (paper_2209_03883_b200/csrc/gen_kernels.cu, libofdmr_b200.so).
 *
 * The generator is the input side of the receiver hot path (SURVEY.md §8(d) "Inputs",
 * §8(f) item 1): it restates the reference's signal model
 *   make_random_frame  src/waveform.cpp:88-131
 *   apply_channel      src/channel.cpp:65-98 (model-validity check skipped)
 *   Rng / derive_seed  include/ofdmradar/rng.hpp:11-66
 * with frame_seed = derive_seed(base_seed, frame_index) and the scene stream
 * derive_seed(frame_seed, 0x7363656e). */
#ifndef OFDMR_GEN_H
#define OFDMR_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ofdmr_gen_params {
    int32_t n, m;            /* subcarriers N, OFDM symbols M */
    double df_hz, fc_hz;     /* subcarrier spacing, carrier */
    int32_t n_cp;            /* CP samples (sets Ts) */
    int32_t qam_order;       /* 4/16/64/256 */
    int32_t zc_precode;      /* 0: none; 1: direct D = N layout, sequence length N^2 */
    int64_t zc_root;
    int32_t targets_min, targets_max;
    double range_lo, range_hi;
    double vel_lo, vel_hi;
    double snr_lo_db, snr_hi_db; /* equal => fixed SNR; +inf => noiseless */
} ofdmr_gen_params;

/* GPU generator: frames [first, first + count) straight into device memory.
 *   y, x_tx   device c64 [count][N][M]
 *   sigma2    device double [count]        n_targets device int32 [count] (may be NULL)
 *   ranges, vels device double [count][max_targets] (may be NULL), snr_db device double [count] (may be NULL)
 *   status    device int32 [count]: bit 0 set when a frame hit an MT19937 rejection
 *             (probability ~2^-50 per frame); regenerate such frames with the CPU generator.
 *   stream    cudaStream_t (NULL = default stream)
 * Supports qam_order 4/16/64/256 without ZC precoding, targets_max <= 16, M <= 1024, as long
 * as the on-chip draw ring (two rows of payload bits + one MT19937 block, about
 * 16 (M - 1) log2(qam) bytes) fits the per-block shared memory: 256-QAM at M = 1024 does not.
 * Returns 0, 2 (unsupported / invalid parameters, incl. that ring limit) or 10 (CUDA error).
 * Stream-ordered: no host synchronisation or per-call allocation (ZC precoding uses
 * stream-ordered cudaMallocAsync scratch).
 * Bit-exactness: the integer streams (symbols, scene) are exact; the fp64 channel and noise
 * use the GPU's sin/cos/log/pow, so a c64 value can differ from the CPU generator's by 1 ulp
 * in rare cells (tests/test_gpu_parity.py::test_gpu_generator_matches_cpu_generator). */
int ofdmr_gen_device(const ofdmr_gen_params* p, uint64_t base_seed, int64_t first, int64_t count, void* y,
                     void* x_tx, double* sigma2, int32_t* n_targets, double* ranges, double* vels, double* snr_db,
                     int32_t max_targets, int32_t* status, void* stream);

/* run_pipeline's generator half (pipeline.cpp:65-71) for a fixed scenario, as the reference's
 * Monte-Carlo callers use it (metrics.cpp:92-143): frame i of the batch uses the run seed
 * derive_seed(seed, first + i); targets (host arrays, <= 16) and SNR are fixed.  y, x_tx,
 * sigma2, status as for ofdmr_gen_device; h_true (may be NULL): device c128 [count][N][M],
 * true_channel of the realisation (channel.cpp:100-109).  Stream-ordered on `stream`. */
int ofdmr_gen_device_explicit(const ofdmr_gen_params* p, uint64_t seed, int64_t first, int64_t count,
                              const double* target_ranges, const double* target_vels, int32_t n_targets,
                              double snr_db, void* y, void* x_tx, double* sigma2, int32_t* status, void* h_true,
                              void* stream);

/* channel_mse (estimation.cpp:41-48) per frame: out[f] = mean |h_est - h_true|^2 with h_est
 * device c64 and h_true device c128, `cells` = N*M per frame (fp64, tree-order sum). */
int ofdmr_channel_mse(const void* h_est, const void* h_true, int64_t cells, int64_t frames, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* OFDMR_GEN_H */
