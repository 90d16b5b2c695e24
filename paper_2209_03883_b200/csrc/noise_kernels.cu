// estimate_noise_power (periodogram.cpp:146-152), the detector's `estimate_noise` mode
// (pipeline.cpp:86-87): per frame the order statistic vals[count / 2] of the map (what
// std::nth_element places at mid), divided by ln 2 and the window power factor.
//
// Exact radix select on the IEEE-754 bit patterns of the fp32 map: P >= 0, so the uint32
// order of the bit patterns is the value order.  Three digit passes (bits 31..21, 20..10,
// 9..0); each pass histograms, per frame, the elements whose higher digits equal the prefix
// selected so far (per-CTA shared-memory histogram, flushed to a per-frame global histogram),
// then one CTA per frame scans the histogram and narrows the prefix / residual rank.  The
// selected float is the exact element of the device map; the division happens in fp64 in the
// reference's order ((v / ln 2) / pf).
#include <algorithm>
#include <cstdint>

#include <cuda_runtime.h>

namespace ofdmr {

namespace {

constexpr int kSelBins = 2048;

__global__ void __launch_bounds__(256) sel_hist_kernel(const float* __restrict__ p, int64_t count, int shift,
                                                       int bits, uint32_t hi_mask, const uint32_t* __restrict__ prefix,
                                                       uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kSelBins];
    const int f = blockIdx.y;
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t pre = prefix[f];
    const uint32_t dmask = (1u << bits) - 1u;
    const uint4* v = reinterpret_cast<const uint4*>(p + (size_t)f * (size_t)count);
    const int64_t n4 = count / 4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 u = __ldcs(v + i);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if ((w[j] & hi_mask) == pre) atomicAdd(&h[(w[j] >> shift) & dmask], 1u);
    }
    __syncthreads();
    uint32_t* g = hist + (size_t)f * kSelBins;
    for (int i = threadIdx.x; i < (1 << bits); i += blockDim.x)
        if (h[i]) atomicAdd(g + i, h[i]);
}

// One CTA per frame: find the digit whose cumulative count passes the residual rank.
__global__ void __launch_bounds__(256) sel_pick_kernel(uint32_t* __restrict__ hist, int shift, int bits,
                                                       uint32_t* __restrict__ prefix, uint32_t* __restrict__ rank,
                                                       int last, double pf,
                                                       double* __restrict__ sigma2_out) {
    __shared__ uint32_t part[256];
    __shared__ int s_bin;
    __shared__ uint32_t s_before;
    const int f = blockIdx.x;
    uint32_t* g = hist + (size_t)f * kSelBins;
    const int nb = 1 << bits;
    const int per = nb / 256;  // bins per thread (8 or 4), contiguous
    uint32_t local = 0;
    for (int j = 0; j < per; ++j) local += g[threadIdx.x * per + j];
    part[threadIdx.x] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t r = rank[f];
        uint32_t cum = 0;
        int t = 0;
        while (t < 255 && cum + part[t] <= r) cum += part[t++];
        uint32_t c2 = cum;
        int b = t * per;
        while (b < t * per + per - 1 && c2 + g[b] <= r) c2 += g[b++];
        s_bin = b;
        s_before = c2;
    }
    __syncthreads();
    for (int j = 0; j < per; ++j) g[threadIdx.x * per + j] = 0;  // ready for the next pass
    if (threadIdx.x == 0) {
        prefix[f] |= (uint32_t)s_bin << shift;
        rank[f] -= s_before;
        if (last) {
            const double v = (double)__uint_as_float(prefix[f]);
            sigma2_out[f] = v / 0.6931471805599453 / pf;
        }
    }
}

__global__ void sel_init_kernel(uint32_t* prefix, uint32_t* rank, uint32_t mid, int64_t frames) {
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f < frames) {
        prefix[f] = 0;
        rank[f] = mid;
    }
}

}  // namespace

// scratch: hist [frames][kSelBins] (zeroed), prefix [frames], rank [frames]
size_t noise_select_scratch_bytes(int64_t frames) {
    return (size_t)frames * (kSelBins + 2) * sizeof(uint32_t);
}

cudaError_t launch_noise_select(const float* p, int64_t count, double pf, double* sigma2_out, int64_t frames,
                                void* scratch, int sms, cudaStream_t st, int64_t* launches) {
    uint32_t* hist = static_cast<uint32_t*>(scratch);
    uint32_t* prefix = hist + (size_t)frames * kSelBins;
    uint32_t* rank = prefix + frames;
    cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)frames * kSelBins * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    sel_init_kernel<<<(unsigned)((frames + 255) / 256), 256, 0, st>>>(prefix, rank, (uint32_t)(count / 2), frames);
    ++*launches;
    // enough CTAs to fill the GPU, >= 4096 elements per CTA
    int64_t chunks = (8LL * sms + frames - 1) / frames;
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, count / 4096));
    const int shifts[3] = {21, 10, 0}, bits[3] = {11, 11, 10};
    for (int pass = 0; pass < 3; ++pass) {
        const uint32_t hi_mask = pass == 0 ? 0u : (0xFFFFFFFFu << (shifts[pass] + bits[pass]));
        sel_hist_kernel<<<dim3((unsigned)chunks, (unsigned)frames), 256, 0, st>>>(p, count, shifts[pass], bits[pass],
                                                                                 hi_mask, prefix, hist);
        sel_pick_kernel<<<(unsigned)frames, 256, 0, st>>>(hist, shifts[pass], bits[pass], prefix, rank, pass == 2, pf,
                                                          sigma2_out);
        *launches += 2;
    }
    return cudaGetLastError();
}

}  // namespace ofdmr
