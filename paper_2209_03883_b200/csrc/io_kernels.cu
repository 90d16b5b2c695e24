// Device side of the map writers (io.cpp:94-110 write_map_pgm): quantise batched fp32
// periodogram maps to the reference's 8-bit PGM scale on the GPU, so exporting a batch only
// moves N' x M' bytes per frame to the host.  Per frame: peak = max cell (<= 0 -> 1), then
//   byte = lround(clamp((10 log10(max(v, 1e-30 peak) / peak) + 60) / 60, 0, 1) * 255)
// in fp64 with the reference's operation order.
#include <cuda_runtime.h>

#include <cstdint>

namespace ofdmr {

namespace {

__global__ void __launch_bounds__(256) map_peak_kernel(const float* __restrict__ p, int64_t count,
                                                       double* __restrict__ peak) {
    __shared__ float red[8];
    const float* v = p + (size_t)blockIdx.x * (size_t)count;
    float m = 0.f;  // maps are >= 0; an all-zero map keeps 0 -> peak 1.0
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) m = fmaxf(m, __ldcs(v + i));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
        const double pk = (double)m;
        peak[blockIdx.x] = pk <= 0.0 ? 1.0 : pk;
    }
}

__global__ void __launch_bounds__(256) map_pgm_kernel(const float* __restrict__ p, int64_t count,
                                                      const double* __restrict__ peak, uint8_t* __restrict__ out) {
    const int64_t f = blockIdx.y;
    const double pk = peak[f];
    const double floor_db = -60.0;
    const float* v = p + f * count;
    uint8_t* o = out + f * count;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = (double)__ldcs(v + i);
        const double db = 10.0 * log10(fmax(x, pk * 1e-30) / pk);
        const double t = fmin(fmax((db - floor_db) / -floor_db, 0.0), 1.0);
        o[i] = (uint8_t)llround(t * 255.0);
    }
}

}  // namespace

// scratch: frames doubles
cudaError_t launch_map_pgm(const float* p, int64_t count, uint8_t* out, int64_t frames, double* scratch,
                           cudaStream_t st, int64_t* launches) {
    for (int64_t f0 = 0; f0 < frames; f0 += 65535) {
        const int64_t nf = frames - f0 < 65535 ? frames - f0 : 65535;
        map_peak_kernel<<<(unsigned)nf, 256, 0, st>>>(p + f0 * count, count, scratch);
        const unsigned gx = (unsigned)((count + 256 * 16 - 1) / (256 * 16));
        map_pgm_kernel<<<dim3(gx, (unsigned)nf), 256, 0, st>>>(p + f0 * count, count, scratch, out + f0 * count);
        *launches += 2;
    }
    return cudaGetLastError();
}

}  // namespace ofdmr
