// Probe: SM <-> L2 bandwidth on L2-resident buffers (the ceiling the batched periodogram's
// exchange runs into).  Every kernel is persistent (grid = SMs x CTAs/SM) and
// streams a buffer of `bytes` (MiB, a power of two; default 32 MiB, well inside the 126 MB L2) `reps` times:
//   read   ld.global.cg 16-B loads (L1 bypassed)
//   write  st.global.cg 16-B stores
//   mix    read buffer A, write buffer B (both L2-resident): the exchange's read+write mix
// Output: TB/s per mode (bytes moved between SMs and L2 / kernel time, CUDA events).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_bw l2_bw.cu
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ float4 ldcg(const float4* p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void stcg(float4* p, float4 v) {
    asm volatile("st.global.cg.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}

template <int MODE>
__global__ void __launch_bounds__(512) l2_kernel(const float4* a, float4* b, size_t n4, int reps, float* sink) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    for (int r = 0; r < reps; ++r) {
        // rotate the start so consecutive reps do not hit the same slices in the same order
        const size_t base = ((size_t)r * 7919u * blockDim.x) & (n4 - 1);
        size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 4
        for (; i < n4; i += stride) {
            const size_t j = (i + base) & (n4 - 1);
            if (MODE == 0) {
                const float4 v = ldcg(a + j);
                acc += v.x + v.y + v.z + v.w;
            } else if (MODE == 1) {
                stcg(b + j, make_float4(acc, (float)r, 0.f, 1.f));
            } else {
                const float4 v = ldcg(a + j);
                stcg(b + j, v);
            }
        }
    }
    if (acc == 12345.f) sink[0] = acc;
}

int main(int argc, char** argv) {
    const size_t bytes = (argc > 1 ? atol(argv[1]) : 32) << 20;
    const int reps = argc > 2 ? atoi(argv[2]) : 50;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    const size_t n4 = bytes / 16;
    float4 *a, *b;
    float* sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 0, bytes);
    cudaMemset(b, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"read", "write", "mix(read A + write B)"};
    printf("SMs %d, L2 %d MiB, buffer %zu MiB, reps %d\n", sms, l2 >> 20, bytes >> 20, reps);
    for (int ctas = 1; ctas <= 4; ctas *= 2)
        for (int mode = 0; mode < 3; ++mode) {
            auto run = [&] {
                if (mode == 0) l2_kernel<0><<<sms * ctas, 512>>>(a, b, n4, reps, sink);
                if (mode == 1) l2_kernel<1><<<sms * ctas, 512>>>(a, b, n4, reps, sink);
                if (mode == 2) l2_kernel<2><<<sms * ctas, 512>>>(a, b, n4, reps, sink);
            };
            run();
            cudaDeviceSynchronize();
            float best = 1e30f;
            for (int t = 0; t < 5; ++t) {
                cudaEventRecord(e0);
                run();
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            const double moved = (double)bytes * reps * (mode == 2 ? 2 : 1);
            printf("%-22s ctas/SM %d  %8.3f ms  %6.2f TB/s\n", names[mode], ctas, best, moved / best / 1e9);
        }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
