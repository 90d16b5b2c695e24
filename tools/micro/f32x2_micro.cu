// Microbenchmark: issue/throughput of packed FP32 (FFMA2 / FADD2, sm_100a) against scalar
// FFMA / FADD.  Each thread runs 8 independent dependency chains; the kernel is timed with
// CUDA events and reports warp-instructions and FP32 lane-operations per SM per cycle.
#include <cstdio>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

template <int MODE>  // 0 FFMA, 1 FFMA2, 2 FADD, 3 FADD2, 4 mix: 1 FFMA2 + 1 FFMA
__global__ void loop(float* out, int reps, float s) {
    float a[16];
    unsigned long long p[8];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int i = 0; i < 8; ++i) p[i] = pk(a[2 * i], a[2 * i + 1]);
    const unsigned long long ps = pk(s, s), pt = pk(1e-7f, 1e-7f);
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (MODE == 0) {
#pragma unroll
                for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 1e-7f);
            } else if (MODE == 1) {
#pragma unroll
                for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(ps), "l"(pt));
            } else if (MODE == 2) {
#pragma unroll
                for (int i = 0; i < 16; ++i) a[i] = a[i] + 1e-7f;
            } else if (MODE == 3) {
#pragma unroll
                for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(pt));
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(ps), "l"(pt));
#pragma unroll
                for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 1e-7f);
            }
        }
    }
    float acc = 0;
    for (int i = 0; i < 16; ++i) acc += a[i];
    for (int i = 0; i < 8; ++i) acc += __uint_as_float((unsigned)p[i]) + __uint_as_float((unsigned)(p[i] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(const char* name, int sms, float* out, int clk_khz) {
    const int reps = 2000, threads = 512, blocks = sms * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    loop<MODE><<<blocks, threads>>>(out, 10, 1.0f);
    cudaEventRecord(e0);
    loop<MODE><<<blocks, threads>>>(out, reps, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // warp-instructions per thread-rep: 16 u x (16 scalar | 8 packed | 4 packed + 8 scalar)
    const double winst_per_rep = MODE == 0 || MODE == 2 ? 256 : MODE == 4 ? 192 : 128;
    const double lanes_per_rep = MODE == 4 ? 256 : 256;  // fp32 lane-ops per thread-rep
    const double warps = (double)blocks * threads / 32;
    const double cycles = ms * 1e-3 * clk_khz * 1e3;
    printf("%-22s %8.3f ms  warp-inst/SM/cycle %.2f  fp32 lane-ops/SM/cycle %.1f\n", name, ms,
           warps * reps * winst_per_rep / cycles / sms, warps * 32 * reps * lanes_per_rep / cycles / sms);
}

int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * sms * 4 * 512);
    printf("SMs %d, clock %d kHz\n", sms, clk);
    run<0>("FFMA", sms, out, clk);
    run<1>("FFMA2", sms, out, clk);
    run<2>("FADD", sms, out, clk);
    run<3>("FADD2", sms, out, clk);
    run<4>("FFMA2+2xFFMA mix", sms, out, clk);
    return 0;
}
