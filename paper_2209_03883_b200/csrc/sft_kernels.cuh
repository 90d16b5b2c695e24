// FPS-SFT (sft.cpp:185-490) on the GPU: one CTA per frame, fp64, decisions in the
// reference's order.  Host side: slope/offset draws (data-independent MT19937-64
// stream, sft.cpp:212-218) and both twiddle tables are built on the host with the
// same libm calls and uploaded.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <utility>

#include "../../include/ofdmr_b200.h"

namespace ofdmr {

struct SftScratch {
    int32_t* draws = nullptr;      // [frames][i_max][4] = v1, v2, a1, a2 (drawn on the device)
    uint64_t* seeds = nullptr;     // [frames] uploaded per call
    double* sigma2 = nullptr;      // [frames] (host sigma2 uploaded)
    int32_t* err = nullptr;        // [frames] overflow flags (synchronous API)
    int64_t cap_frames = 0;
    int64_t cap_draws = 0;
    int64_t cap_seeds = 0;
    struct Tables {
        double2* tw_ref = nullptr;  // [Q] rotation table (sft.cpp:29-44)
        double2* tw_fft = nullptr;  // [Q/2] radix-2 twiddles (power-of-two Q)
        int blu_m = 0, blu_logm = 0;  // Bluestein (other Q): FFT length m = 2^ceil(log2(2Q - 1))
        double2* chirp = nullptr;   // [Q]
        double2* bker = nullptr;    // [m] FFT_m of the conjugate-chirp kernel
        double2* twm_f = nullptr;   // [m/2] radix-2 twiddles, both signs
        double2* twm_i = nullptr;
    };
    std::map<int, Tables> tables;   // per Q, built once
    char* gbuf = nullptr;           // per-CTA global work arrays (general Q)
    int64_t cap_gbuf = 0;           // bytes
};

void sft_free(SftScratch& s);

// sft_iterate over a batch.  seeds on the host; sigma2 on the host or (sigma2_on_device) the
// device.  status != null: stream-ordered, overflow (> 128 accepted tones / 64 entries) ORs bit 2
// into status[f]; status == null: synchronous check, OFDMR_ERR_CONFIG on overflow.
int sft_run(SftScratch& s, cudaStream_t st, const float2* h, int n, int m, const ofdmr_sft_config& cfg,
            const uint64_t* seeds, const double* sigma2, bool sigma2_on_device, int32_t* k_out, int32_t* l_out,
            double* amp_out, int32_t* n_entries, int32_t* iterations, int64_t* samples_used, int32_t* converged,
            double* residual, int32_t* status, int64_t frames, int64_t* launches, std::string& err);

// pipeline.cpp:26-43 estimate_noise_from_slice for a batch of N x M c64 grids; seeds on the
// host (the Rng seed, i.e. derive_seed(run seed, 0x6e6573) in run_pipeline); output on device.
int sft_slice_noise(SftScratch& s, cudaStream_t st, const float2* h, int n, int m, const uint64_t* seeds,
                    double* sigma2_out, int64_t frames, int64_t* launches, std::string& err);

// detections_from_spectrum (sft.cpp:461-490) on device entries ([frame][max_entries]) with
// per-frame device sigma2; records [frame][kmax] like ofdmr_detect.
int sft_detections(cudaStream_t st, const int32_t* k, const int32_t* l, const double* amp, const int32_t* n_entries,
                   int max_entries, int n, int m, const double* sigma2, double pfa, const int32_t* k_per_frame, int kmax,
                   int32_t* det_delay, int32_t* det_doppler, float* det_power, int32_t* counts, int64_t frames,
                   int64_t* launches, std::string& err);

// division_noise_power (pipeline.cpp:18-23) per frame on device x_tx and sigma2.
int division_noise(cudaStream_t st, const float2* x, int64_t cells, const double* sigma2, double* out, int64_t frames,
                   int64_t* launches, std::string& err);

}  // namespace ofdmr
