// Microbenchmark: HBM streaming rate of the fused kernel's pass-A access pattern (8-symbol
// column tiles, 64-B row segments, both CTAs of a pair reading the two halves of a 128-B line)
// through a per-thread cp.async ring, with no compute.  Usage: stream_micro [frames] [ring]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kN = 1024, kM = 256;

__device__ __forceinline__ void cp16(void* s, const void* g) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int RING, int SPIN, int STAG>
__global__ void __launch_bounds__(256, 2) stream_kernel(const float2* y, const float2* x, int frames, float* out,
                                                        int* sm_count) {
    extern __shared__ float4 stg[];  // [RING][2][256]
    const int tid = threadIdx.x, rank = blockIdx.x & 1, cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    if (STAG) {
        __shared__ int order;
        if (tid == 0) {
            unsigned smid;
            asm("mov.u32 %0, %%smid;" : "=r"(smid));
            order = atomicAdd(sm_count + smid, 1);
        }
        __syncthreads();
        if (order & 1) {  // second CTA on this SM: start half a tile period later
            float z = 1.f;
#pragma unroll 1
            for (int i = 0; i < STAG; ++i) z = fmaf(z, 0.999f, 1e-7f);
            if (z == 12345.f) out[1] = z;
        }
    }
    int ifr = cid, iu = 0, ist = 0, islot = 0, cslot = 0;
    const size_t lane_off = (size_t)(tid >> 2) * kM + 8 * rank + (tid & 3) * 2;
    size_t ioff = (size_t)cid * kN * kM + lane_off;
    auto issue = [&]() {
        if (ifr < frames) {
            cp16(&stg[(islot * 2 + 0) * 256 + tid], y + ioff);
            cp16(&stg[(islot * 2 + 1) * 256 + tid], x + ioff);
        }
        commit();
        islot = islot + 1 == RING ? 0 : islot + 1;
        ioff += (size_t)64 * kM;
        if (++ist == 16) {
            ist = 0;
            if (++iu == 16) { iu = 0; ifr += ncl; }
            ioff = (size_t)ifr * kN * kM + 16 * iu + lane_off;
        }
    };
    for (int i = 0; i < RING; ++i) issue();
    float acc = 0.f;
    for (int f = cid; f < frames; f += ncl)
        for (int u = 0; u < 16; ++u) {
            for (int st = 0; st < 16; ++st) {
                waitg<RING - 1>();
                const float4 a = stg[(cslot * 2) * 256 + tid], b = stg[(cslot * 2 + 1) * 256 + tid];
                cslot = cslot + 1 == RING ? 0 : cslot + 1;
                acc += a.x * b.x + a.w * b.z;
                issue();
            }
            if (SPIN) {  // stand-in for the FFT phases: ALU work without memory traffic
                float z = acc;
#pragma unroll 1
                for (int i = 0; i < SPIN; ++i) z = fmaf(z, 0.999f, 1e-7f);
                acc = z;
            }
        }
    if (acc == 12345.f) out[0] = acc;
}

template <int RING, int SPIN, int STAG = 0>
void run(const float2* y, const float2* x, int frames, float* out, int sms) {
    const size_t smem = sizeof(float4) * RING * 2 * 256;
    cudaFuncSetAttribute(stream_kernel<RING, SPIN, STAG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = 2 * sms;
    int* cnt;
    cudaMalloc(&cnt, sizeof(int) * 1024);
    cudaMemset(cnt, 0, sizeof(int) * 1024);
    stream_kernel<RING, SPIN, STAG><<<grid, 256, smem>>>(y, x, frames, out, cnt);
    cudaMemset(cnt, 0, sizeof(int) * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    stream_kernel<RING, SPIN, STAG><<<grid, 256, smem>>>(y, x, frames, out, cnt);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(cnt);
    printf("ring %d spin %5d stagger %5d: %.3f ms  %.0f GB/s  (%.0f k frames/s)  %s\n", RING, SPIN, STAG, ms,
           frames * 4.194304e6 / (ms / 1e3) / 1e9, frames / ms, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    const int frames = argc > 1 ? atoi(argv[1]) : 4096;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float2 *y, *x;
    float* out;
    cudaMalloc(&y, sizeof(float2) * kN * kM * (size_t)frames);
    cudaMalloc(&x, sizeof(float2) * kN * kM * (size_t)frames);
    cudaMalloc(&out, 4);
    cudaMemset(y, 0, sizeof(float2) * kN * kM * (size_t)frames);
    cudaMemset(x, 0, sizeof(float2) * kN * kM * (size_t)frames);
    run<4, 0>(y, x, frames, out, sms);
    run<4, 500>(y, x, frames, out, sms);
    run<4, 500, 500>(y, x, frames, out, sms);
    run<4, 1000>(y, x, frames, out, sms);
    run<4, 1000, 1000>(y, x, frames, out, sms);
    run<4, 1000, 2000>(y, x, frames, out, sms);
    return 0;
}
