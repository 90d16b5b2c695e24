// Microbenchmark: isolated warp_fft1024 throughput (smem-resident column, no global traffic).
#include <cstdio>
#include <vector>
#include "../../paper_2209_03883_b200/csrc/warp_fft.cuh"
using namespace ofdmr;

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) fft_loop(const float2* tw_t, float2* out, int reps) {
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* cols = sm + 1024;
    for (int i = threadIdx.x; i < 1024; i += WARPS * 32) tw[i] = tw_t[i];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float2* col = cols + w * 1057;
    float2 v[32];
    for (int i = 0; i < 32; ++i) v[i] = make_float2(lane * 0.001f + i, -i * 0.5f);
    __syncthreads();
    for (int r = 0; r < reps; ++r) {
        warp_fft1024<true, 32>(v, col, tw);
        for (int i = 0; i < 32; ++i) v[i] = cscale(v[i], 1.0f / 1024.0f);
    }
    float2 acc = make_float2(0, 0);
    for (int i = 0; i < 32; ++i) acc = cadd(acc, v[i]);
    out[blockIdx.x * WARPS * 32 + threadIdx.x] = acc;
}

template <int WARPS>
void run(int blocks_per_sm, int sms, const float2* tw, float2* out) {
    const size_t smem = (1024 + WARPS * 1057) * sizeof(float2);
    cudaFuncSetAttribute(fft_loop<WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = blocks_per_sm * sms, reps = 200;
    fft_loop<WARPS><<<grid, WARPS * 32, smem>>>(tw, out, 10);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    fft_loop<WARPS><<<grid, WARPS * 32, smem>>>(tw, out, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ffts = double(grid) * WARPS * reps;
    printf("warps/CTA %2d, CTAs/SM %d: %.3f ms, %.1f M FFT1024/s, %.0f cycles/FFT/SM(@1.965GHz), err=%s\n", WARPS,
           blocks_per_sm, ms, ffts / ms / 1e3, 1.965e9 * (ms / 1e3) * sms / ffts,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::vector<float2> t(1024);
    for (int t1 = 0; t1 < 32; ++t1)
        for (int j = 0; j < 32; ++j) {
            const double ang = -6.283185307179586 * t1 * j / 1024.0;
            t[t1 * 32 + j] = make_float2(cos(ang), sin(ang));
        }
    float2 *tw, *out;
    cudaMalloc(&tw, 1024 * sizeof(float2));
    cudaMalloc(&out, 1 << 24);
    cudaMemcpy(tw, t.data(), 1024 * sizeof(float2), cudaMemcpyHostToDevice);
    run<1>(1, sms, tw, out);
    run<2>(1, sms, tw, out);
    run<4>(1, sms, tw, out);
    run<8>(1, sms, tw, out);
    run<8>(2, sms, tw, out);
    run<4>(4, sms, tw, out);
    run<16>(1, sms, tw, out);
    return 0;
}
