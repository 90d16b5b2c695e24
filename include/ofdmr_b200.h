/*
 * ofdmr_b200.h — C-ABI drop-in boundary for the OFDM radar receiver hot path
 * (arXiv 2209.03883 reference `ofdmradar`).
 *
 * The reference exposes the receiver as C++ free functions with value semantics
 * (namespace ofdmradar).  This header replaces them with batched, stream-ordered
 * entry points on caller-owned DEVICE pointers (frames contiguous, each frame a
 * row-major N x M grid of complex64 {float re, im}; rows = subcarrier k,
 * cols = OFDM symbol l, include/ofdmradar/grid.hpp:14-18), plus one host-buffer
 * entry point (ofdmr_pipeline_host) that performs the H2D/D2H copies itself.
 * Each function names the reference interface it replaces.
 *
 * Errors: every function returns OFDMR_OK (0), OFDMR_ERR_CONFIG (2, mirrors
 * ofdmradar::ConfigError, include/ofdmradar/errors.hpp:9-12) or OFDMR_ERR_CUDA (10).
 * ofdmr_last_error() returns a thread-local message for the last failure.  A zero
 * X cell (spectral_division's ConfigError, src/estimation.cpp:17: both components exactly
 * zero; denormal or huge cells are divided in fp64, not rejected) is reported per frame
 * through the device `status` array (bit 0) — stream-ordered calls cannot throw; the
 * synchronous host entry point returns OFDMR_ERR_CONFIG for it.
 *
 * Sizes: N, M, N', M' in [2, 4096] whose prime factors are 2, 3, 5, 7, 11 or 13 (the reference
 * accepts any length through FFTW; its presets use 2048 x 560, 2048 x 200, 512 x 140 and powers of
 * two), N' >= N, M' >= M (periodogram.cpp:43, ConfigError otherwise), max_targets <= 64.
 * Powers of two in [16, 4096] with N' in {N, 2N, 4N} run the specialised power-of-two kernels
 * (and the fused ones at 1024 x 256); every other shape the mixed-radix kernels
 * (csrc/mixed_kernels.cu), the OFDM front end included; FPS-SFT limits see below.
 *
 * Threading: one context per host thread or stream (the reference functions are
 * reentrant; this context owns scratch buffers).
 */
#ifndef OFDMR_B200_H
#define OFDMR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OFDMR_OK 0
#define OFDMR_ERR_CONFIG 2
#define OFDMR_ERR_CUDA 10

#define OFDMR_WINDOW_RECT 0     /* WindowKind::Rectangular, waveform.hpp:16 */
#define OFDMR_WINDOW_HAMMING 1  /* WindowKind::Hamming */
#define OFDMR_EST_LS 0          /* EstimatorKind::Ls and ::ZcpLs (divide by the precoded x_tx), pipeline.cpp:49-53 */
#define OFDMR_EST_DFT_CE 1      /* EstimatorKind::DftCe, pipeline.cpp:54-55 */

/* Receiver configuration: the subset of WaveformConfig (waveform.hpp:20-41),
 * EstimatorSettings and DetectorSettings (config.hpp:25-37) the hot path reads. */
typedef struct ofdmr_config {
    int32_t n_subcarriers; /* N */
    int32_t n_symbols;     /* M */
    int32_t n_prime;       /* N' (delay bins) */
    int32_t m_prime;       /* M' (Doppler bins) */
    int32_t window;        /* OFDMR_WINDOW_* */
    int32_t estimator;     /* OFDMR_EST_* */
    int32_t n_cp;          /* DFT-CE truncation length L (waveform.n_cp, pipeline.cpp:55) */
    int32_t max_targets;   /* K_max (detector.max_targets) */
    double pfa;            /* waveform.pfa */
    int32_t chunk_frames;  /* frames per internal launch chunk (0 = default) */
    int32_t device;        /* CUDA device ordinal */
} ofdmr_config;

/* Fixed-size detection record (Detection, periodogram.hpp:12-18, without the
 * host-side physics fields which ofdmr_bins_to_physics computes in fp64). */
typedef struct ofdmr_context ofdmr_context;

/* --- context ------------------------------------------------------------ */
int ofdmr_create(const ofdmr_config* cfg, ofdmr_context** out);
void ofdmr_destroy(ofdmr_context* ctx);
/* Subsequent calls enqueue on this cudaStream_t (NULL = legacy default stream). */
int ofdmr_set_stream(ofdmr_context* ctx, void* cuda_stream);
const char* ofdmr_last_error(void);
/* Number of kernel launches enqueued by this context since creation. */
int64_t ofdmr_launch_count(const ofdmr_context* ctx);

/* Per-stage CUDA-event timing for profiling runs: when on, every kernel launch of the
 * pipeline / periodogram schedules is bracketed by events.  ofdmr_get_profile syncs the
 * context stream and returns (then resets) the summed milliseconds and launch counts of
 * stage 0 (column pass), 1 (row pass + detection), 2 (top-K merge). */
int ofdmr_set_profiling(ofdmr_context* ctx, int32_t on);
int ofdmr_get_profile(ofdmr_context* ctx, double* ms3, int64_t* launches3);

/* --- host-side helpers (fp64, bit-identical formulas) -------------------- */
/* make_window, periodogram.cpp:25-37 (wk: n doubles, wl: m doubles). */
int ofdmr_make_window(int32_t kind, int32_t n, int32_t m, double* wk, double* wl);
/* Window2d::power_factor, periodogram.cpp:11-16. */
double ofdmr_window_power_factor(int32_t kind, int32_t n, int32_t m);
/* detection_threshold, periodogram.cpp:77-81. */
int ofdmr_detection_threshold(double sigma2, double pfa, double power_factor, double* eta);
/* bins_to_physics, periodogram.cpp:138-144 (Ts = (1 + n_cp/N)/df, waveform.hpp:31-35). */
void ofdmr_bins_to_physics(int64_t delay_bin, int64_t doppler_bin, int32_t n_subcarriers, int32_t n_cp,
                           int32_t n_prime, int32_t m_prime, double df_hz, double fc_hz, double* range_m,
                           double* velocity_mps);

/* --- batched device entry points (stream-ordered) ----------------------- */
/* spectral_division, estimation.cpp:10-21: h = y / x; status[f] bit0 = zero X cell. */
int ofdmr_spectral_division(ofdmr_context* ctx, const void* y, const void* x, void* h, int32_t* status,
                            int64_t frames);
/* dft_ce, estimation.cpp:23-39 (L = cfg.n_cp). */
int ofdmr_dft_ce(ofdmr_context* ctx, const void* h, void* h_out, int64_t frames);
/* estimate_channel, pipeline.cpp:47-58 (LS / ZCP-LS / DFT-CE per cfg.estimator). */
int ofdmr_estimate_channel(ofdmr_context* ctx, const void* y, const void* x_tx, void* h, int32_t* status,
                           int64_t frames);
/* periodogram, periodogram.cpp:39-75: p = N' x M' fp32 per frame, Doppler fft-shifted. */
int ofdmr_periodogram(ofdmr_context* ctx, const void* h, float* p, int64_t frames);
/* detection_threshold + threshold_mask + extract_peaks, periodogram.cpp:77-136, on a
 * device map p; sigma2_h[f] is the per-frame post-division noise power.  Records are
 * [frame][max_targets]; counts[f] valid entries, ordered by (power desc, index asc).
 * k_per_frame may be NULL (= max_targets). */
int ofdmr_detect(ofdmr_context* ctx, const float* p, const double* sigma2_h, const int32_t* k_per_frame,
                 int32_t* delay_bin, int32_t* doppler_bin, float* peak_power, int32_t* counts, int64_t frames);
/* OFDM time-domain front end, waveform.cpp:133-166 (N = cfg.n_subcarriers, M = cfg.n_symbols,
 * Ncp = cfg.n_cp; requires 0 <= Ncp <= N).  stream: [frames][M][Ncp + N] c64 samples; grid:
 * [frames][N][M] c64 row-major.  ofdm_demodulate strips each symbol's cyclic prefix and takes
 * the unscaled forward FFT_N (the receiver step in front of spectral_division); ofdm_modulate
 * is its transmitter inverse (IFFT_N x 1/N, prefix = last Ncp samples). */
int ofdmr_ofdm_demodulate(ofdmr_context* ctx, const void* stream, void* grid, int64_t frames);
int ofdmr_ofdm_modulate(ofdmr_context* ctx, const void* grid, void* stream, int64_t frames);
/* write_map_pgm's pixel values (io.cpp:94-110) for a batch of device maps: out[f] holds the
 * N' x M' row-major 8-bit image (rows = delay bin, columns = fft-shifted Doppler bin) that the
 * reference writes after its "P5\n<cols> <rows>\n255\n" header.  out is device memory. */
int ofdmr_map_to_pgm(ofdmr_context* ctx, const float* p, uint8_t* out, int64_t frames);
/* estimate_noise_power, periodogram.cpp:146-152 (the detector's estimate_noise mode,
 * pipeline.cpp:86-87): sigma2_out[f] = P_f[count / 2] (nth_element order statistic of the
 * N' x M' device map) / ln 2 / window power factor.  sigma2_out is a device array; feed it to
 * ofdmr_detect as sigma2_h to run the reference's estimate-noise detection. */
int ofdmr_estimate_noise_power(ofdmr_context* ctx, const float* p, double* sigma2_out, int64_t frames);
/* threshold_mask + extract_peaks, periodogram.cpp:83-136, with the mask given by its
 * per-frame threshold eta[f] (mask = p >= eta). Same record layout as ofdmr_detect. */
int ofdmr_extract_peaks(ofdmr_context* ctx, const float* p, const double* eta, const int32_t* k_per_frame,
                        int32_t* delay_bin, int32_t* doppler_bin, float* peak_power, int32_t* counts,
                        int64_t frames);
/* Receiver half of run_pipeline, pipeline.cpp:72-96: y, x_tx -> estimate_channel ->
 * division_noise_power(sigma2) -> periodogram -> threshold -> extract_peaks.
 * Optional outputs (NULL to skip): sigma2_h_out [frames], p_out [frames][N'][M'],
 * status [frames]. */
int ofdmr_pipeline(ofdmr_context* ctx, const void* y, const void* x_tx, const double* sigma2,
                   const int32_t* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin, float* peak_power,
                   int32_t* counts, double* sigma2_h_out, float* p_out, int32_t* status, int64_t frames);
/* Status bit 1 (value 2) after ofdmr_pipeline: recompute this frame with this entry point,
 * which always takes the chunked two-pass path (exact for any candidate count, and the only
 * path that sets bit 0).  The fused fast path sets it when it kept at most 1024 strict local
 * maxima above eta per half-frame and the frame had more (only when sigma2 is mis-set far
 * below the noise floor), or when some |x|^2 fell outside the fp32 normal range (an exactly
 * zero x cell -> bit 0 on recompute, estimation.cpp:17; a denormal or huge x cell, which the
 * exact path divides in fp64 like the reference does on the upcast complex<double>). */
int ofdmr_pipeline_general(ofdmr_context* ctx, const void* y, const void* x_tx, const double* sigma2,
                           const int32_t* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin, float* peak_power,
                           int32_t* counts, double* sigma2_h_out, float* p_out, int32_t* status, int64_t frames);
/* Same on HOST buffers (pinned recommended): copies inside, double-buffered (chunk i+1's copies
 * and kernels are enqueued before chunk i's status is checked), synchronous on return; status-bit-1
 * frames are recomputed on the exact path.  Returns OFDMR_ERR_CONFIG if any frame had a zero X cell. */
int ofdmr_pipeline_host(ofdmr_context* ctx, const void* y, const void* x_tx, const double* sigma2,
                        const int32_t* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin, float* peak_power,
                        int32_t* counts, int64_t frames);

/* --- FPS-SFT (sft.cpp:185-490) ------------------------------------------ */
/* SftConfig, sft.hpp:14-33. */
typedef struct ofdmr_sft_config {
    int32_t i_max;
    double detect_threshold; /* 0 = derive from sigma2/pfa + relative floor */
    double pfa;
    int32_t decimation;
    double frac_tol;
    double amp_tol;
    int32_t max_entries;     /* entries kept per frame (<= 64) */
} ofdmr_sft_config;

/* FPS-SFT sizes: N, M in [2, 4096], Q = lcm(N, M) <= 2^20.  Power-of-two Q <= 2048 runs one CTA
 * per frame in shared memory; any other Q (e.g. table1's 2048 x 560, Q = 71680) keeps each frame's
 * work arrays in global memory and takes the slice FFTs by Bluestein in the oracle's exact
 * operation order (oracle.c fft_bluestein), so spectra and decisions stay bit-identical.
 *
 * sft_iterate (sft.cpp:185-459) over a batch of N x M c64 grids h (device).  seeds[f] =
 * SftConfig.seed, sigma2[f] = SftConfig.sigma2 (host arrays; the slope / offset draws are made on
 * the device from the seeds).  Outputs (device, [frame][max_entries]): k, l, amplitude (complex
 * double re/im interleaved), n_entries, and per-frame stats (iterations, samples_used, converged,
 * residual_energy; device, each may be NULL).  status (device, may be NULL): when given the call
 * is stream-ordered and a frame that exceeds the on-chip limits (> 128 accepted tones, or more
 * entries than max_entries) gets bit 2 (value 4); when NULL the call synchronises and returns
 * OFDMR_ERR_CONFIG for such a frame. */
int ofdmr_sft(ofdmr_context* ctx, const void* h, int32_t n, int32_t m, const ofdmr_sft_config* cfg,
              const uint64_t* seeds, const double* sigma2, int32_t* k_out, int32_t* l_out, double* amp_out,
              int32_t* n_entries, int32_t* iterations, int64_t* samples_used, int32_t* converged,
              double* residual, int32_t* status, int64_t frames);

/* detections_from_spectrum (sft.cpp:461-490) on device SFT entries ([frame][max_entries] k, l,
 * complex-double amplitudes, n_entries): power = |A|^2 N M >= eta = -sigma2[f] ln(pfa) (sigma2 on
 * the device), delay = (N - k) mod N, Doppler = (l + M/2) mod M - M/2, ordered by (power desc,
 * delay, Doppler), at most k_per_frame[f] (NULL = cfg.max_targets) records of the ofdmr_detect
 * layout.  Stream-ordered. */
int ofdmr_sft_detections(ofdmr_context* ctx, const int32_t* k, const int32_t* l, const double* amp,
                         const int32_t* n_entries, int32_t max_entries, int32_t n, int32_t m, const double* sigma2,
                         double pfa, const int32_t* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin,
                         float* peak_power, int32_t* counts, int64_t frames);

/* sft_detect (sft.cpp:492-500): sft_iterate with SftConfig{cfg, seed = seeds[f] (host),
 * sigma2 = sigma2[f] (DEVICE)} then detections_from_spectrum with the same sigma2 and cfg->pfa.
 * Stream-ordered; status (device) as in ofdmr_sft. */
int ofdmr_sft_detect(ofdmr_context* ctx, const void* h, int32_t n, int32_t m, const ofdmr_sft_config* cfg,
                     const uint64_t* seeds, const double* sigma2, const int32_t* k_per_frame, int32_t* delay_bin,
                     int32_t* doppler_bin, float* peak_power, int32_t* counts, int32_t* status, int64_t frames);

/* The FPS-SFT branch of run_pipeline (pipeline.cpp:60-113) on device frames: estimate_channel
 * (cfg.estimator: LS / ZCP-LS / DFT-CE with L = cfg.n_cp) -> sigma_h^2 = division_noise_power(
 * sigma2[f], x_tx) -> [noise_seeds != NULL: sigma2 = estimate_noise_from_slice(H, noise_seeds[f])]
 * -> sft_iterate(H, SftConfig{cfg, seed = sft_seeds[f], sigma2}) -> detections_from_spectrum(
 * sigma2, cfg->pfa, K).  sigma2 (per-frame AWGN power) on the device, seeds on the host
 * (run_pipeline: sft seed = derive_seed(seed, 0x736674), noise seed = derive_seed(seed, 0x6e6573)).
 * sigma2_used_out (device, may be NULL) = PipelineResult::sigma2_used.  status (device): bit 0
 * zero X cell, bit 2 SFT overflow.  Stream-ordered; N x M channel estimates of up to 1 GiB of
 * frames at a time live in context scratch. */
int ofdmr_pipeline_sft(ofdmr_context* ctx, const void* y, const void* x_tx, const double* sigma2,
                       const uint64_t* sft_seeds, const uint64_t* noise_seeds, const ofdmr_sft_config* cfg,
                       const int32_t* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin, float* peak_power,
                       int32_t* counts, double* sigma2_used_out, int32_t* status, int64_t frames);

/* estimate_noise_from_slice, pipeline.cpp:26-43 (run_pipeline's FPS-SFT estimate-noise mode,
 * pipeline.cpp:97-98): per frame, Rng(seeds[f]) draws the admissible slope, the slice of
 * length Q = lcm(N, M) through (0, 0) is FFT'd, sigma2_out[f] = median(|S|^2 / Q^2) * Q / ln 2.
 * seeds on the host, h and sigma2_out on the device (sizes as for ofdmr_sft). */
int ofdmr_sft_estimate_noise(ofdmr_context* ctx, const void* h, int32_t n, int32_t m, const uint64_t* seeds,
                             double* sigma2_out, int64_t frames);

/* --- multi-device ---------------------------------------- */
/* Frames are independent: a batch of F frames is split into contiguous shards
 * [r F / G, (r + 1) F / G) over G devices (ofdmr_shard_range), each processed by its own context
 * on its own host thread with no data-path exchange.  The one exchange is the gather of the
 * fixed-size detection records: into the caller's host arrays (ofdmr_multi_pipeline_host) or onto
 * the first device with cudaMemcpyPeerAsync over NVLink / NVSwitch (ofdmr_multi_pipeline).  A
 * device may be listed more than once (several contexts share it). */
typedef struct ofdmr_multi ofdmr_multi;
void ofdmr_shard_range(int64_t frames, int32_t rank, int32_t world, int64_t* lo, int64_t* hi);
int ofdmr_multi_create(const ofdmr_config* cfg, const int32_t* devices, int32_t ndev, ofdmr_multi** out);
void ofdmr_multi_destroy(ofdmr_multi* m);
int32_t ofdmr_multi_devices(const ofdmr_multi* m);
/* The single-device context of shard `rank` (owned by m). */
ofdmr_context* ofdmr_multi_context(ofdmr_multi* m, int32_t rank);
const char* ofdmr_multi_last_error(void);
/* ofdmr_pipeline_host over the devices: HOST y, x_tx, sigma2, k_per_frame (may be NULL), records
 * [frames][K] written in place per shard.  Synchronous. */
int ofdmr_multi_pipeline_host(ofdmr_multi* m, const void* y, const void* x_tx, const double* sigma2,
                              const int32_t* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin, float* peak_power,
                              int32_t* counts, int64_t frames);
/* ofdmr_pipeline over device-resident shards: y[r], x_tx[r], sigma2[r], k_per_frame[r] (the array
 * or its entries may be NULL) live on device r and hold shard r's frames; the records and status of
 * all F frames are gathered into the arrays on the FIRST device ([F][K], [F]).  Synchronous on
 * return (every shard's gather has landed). */
int ofdmr_multi_pipeline(ofdmr_multi* m, const void* const* y, const void* const* x_tx, const double* const* sigma2,
                         const int32_t* const* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin,
                         float* peak_power, int32_t* counts, int32_t* status, int64_t frames);

#ifdef __cplusplus
}
#endif
#endif /* OFDMR_B200_H */
