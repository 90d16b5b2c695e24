// FPS-SFT (sft.cpp:185-490) on the GPU: one CTA per frame, fp64, decisions in the
// reference's order.  Host side: slope/offset draws (data-independent MT19937-64
// stream, sft.cpp:212-218) and both twiddle tables are built on the host with the
// same libm calls and uploaded.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/ofdmr_b200.h"

namespace ofdmr {

struct SftScratch {
    int32_t* draws = nullptr;      // [frames][i_max][4] = v1, v2, a1, a2
    double* sigma2 = nullptr;      // [frames]
    double2* tw_ref = nullptr;     // [Q] reference twiddle table (sft.cpp:29-44)
    double2* tw_fft = nullptr;     // [Q/2] radix-2 butterfly twiddles
    int32_t* err = nullptr;        // [frames] overflow flags
    int64_t cap_frames = 0;
    int64_t cap_draws = 0;
    int cap_q = 0;
    int tw_q = 0;                  // Q whose twiddle tables tw_ref / tw_fft currently hold (0 = none)
};

void sft_free(SftScratch& s);

int sft_run(SftScratch& s, cudaStream_t st, const float2* h, int n, int m, const ofdmr_sft_config& cfg,
            const uint64_t* seeds, const double* sigma2, int32_t* k_out, int32_t* l_out, double* amp_out,
            int32_t* n_entries, int32_t* iterations, int64_t* samples_used, int32_t* converged, double* residual,
            int64_t frames, int64_t* launches, std::string& err);

// pipeline.cpp:26-43 estimate_noise_from_slice for a batch of N x M c64 grids; seeds on the
// host (the Rng seed, i.e. derive_seed(run seed, 0x6e6573) in run_pipeline); output on device.
int sft_slice_noise(SftScratch& s, cudaStream_t st, const float2* h, int n, int m, const uint64_t* seeds,
                    double* sigma2_out, int64_t frames, int64_t* launches, std::string& err);

}  // namespace ofdmr
