// Launch arguments of the fused DFT-CE receiver kernels (fused_ce.cu, fused_ws.cu), shared
// with the host dispatcher (capi.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ofdmr {

struct FusedArgs {
    const float2* y;
    const float2* x;
    const double* sigma2;
    const int32_t* k_per_frame;
    int32_t* det_delay;
    int32_t* det_doppler;
    float* det_power;
    int32_t* counts;
    double* s2h_out;
    int32_t* status;
    const float* wk;           // null for rectangular
    const float* wl;
    const float2* tw1024_t;
    const float2* tw256_t;
    float2* dscratch;          // per cluster [2][128 * 256] compressed D (double-buffered)
    float* edges;              // per CTA [16 steps][2 edges][1024] edge-column regions + [32] counts (kFusedEdgeStride)
    unsigned long long* pend;  // per cluster [2 ranks][kFusedPend] edge candidates
    int* pend_loc;
    unsigned long long* tlist; // per CTA [kTileList] frame candidate list             // per cluster [2 ranks][kFusedPend] partner edge-column locator
    int frames;
    int L;
    int kmax;
    double log_pfa, power_factor, inv_count;
    float scale;
};

constexpr int kFusedPend = 2048;  // pending edge candidates per CTA per frame
constexpr int kFusedEdgeStride = 16 * 2 * 1024 + 32;  // floats per CTA: 32 edge-column regions + their counts

}  // namespace ofdmr

namespace ofdmr {

// Launch arguments of the warp-specialised batched periodogram (fused_pg2.cu).
struct Pg2Args {
    const float2* h;           // [frames][1024][256] channel estimates
    float* p;                  // [frames][1024][256] periodogram (Doppler fftshifted)
    const float* wk;           // subcarrier / symbol windows (Hamming only)
    const float* wl;
    const float2* tw1024_t;
    const float2* tw256_t;
    float2* gscratch;          // per group 2 x 256 x 1024 column-major G (L2 resident)
    int* counters;             // per group col / row progress counters (zeroed before each launch)
    int frames;
    float scale;               // 1 / (N M)
};

}  // namespace ofdmr
