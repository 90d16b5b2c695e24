// OFDM time-domain front end (waveform.cpp:133-166), batched over frames:
//   ofdm_demodulate: per OFDM symbol l, strip the n_cp-sample cyclic prefix and take the
//                    unscaled forward FFT_N of the next N samples -> column l of the
//                    N x M grid (the step in front of LS division in a real receiver);
//   ofdm_modulate:   the transmitter inverse: column l -> IFFT_N x 1/N, cyclic prefix =
//                    last n_cp samples, stream layout [symbol][n_cp + N].
// One CTA per (frame, tile of C symbols): the C symbol vectors are staged in shared memory
// (coalesced stream reads/writes), transformed by the shared-memory Stockham engine
// (fft_smem.cuh), and exchanged with the row-major grid as C-symbol row segments.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "fft_smem.cuh"

namespace ofdmr {

namespace {

constexpr int kOfdmNT = 256;

template <int N> struct OfdmTile { static constexpr int C = N <= 1024 ? 8 : (N == 2048 ? 4 : 2); };

template <int N>
__global__ void __launch_bounds__(kOfdmNT) ofdm_demod_kernel(const float2* __restrict__ stream, float2* __restrict__ grid,
                                                             int m, int ncp, int ntiles, const float2* __restrict__ tw) {
    constexpr int C = OfdmTile<N>::C;
    constexpr int VS = pad_len(N);
    extern __shared__ float2 buf[];
    const int64_t frame = blockIdx.x / ntiles;
    const int l0 = (blockIdx.x % ntiles) * C;
    const int64_t ns = N + ncp;
    const float2* src = stream + frame * (int64_t)m * ns;
    for (int idx = threadIdx.x; idx < C * N; idx += kOfdmNT) {
        const int c = idx / N, i = idx % N, l = l0 + c;
        buf[c * VS + pidx(i)] = l < m ? src[(int64_t)l * ns + ncp + i] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    fft_vectors<N, false, C, kOfdmNT>(buf, VS, tw);
    float2* dst = grid + frame * (int64_t)N * m;
    for (int idx = threadIdx.x; idx < C * N; idx += kOfdmNT) {
        const int k = idx / C, c = idx % C, l = l0 + c;
        if (l < m) dst[(int64_t)k * m + l] = buf[c * VS + pidx(k)];
    }
}

template <int N>
__global__ void __launch_bounds__(kOfdmNT) ofdm_mod_kernel(const float2* __restrict__ grid, float2* __restrict__ stream,
                                                           int m, int ncp, int ntiles, const float2* __restrict__ tw) {
    constexpr int C = OfdmTile<N>::C;
    constexpr int VS = pad_len(N);
    extern __shared__ float2 buf[];
    const int64_t frame = blockIdx.x / ntiles;
    const int l0 = (blockIdx.x % ntiles) * C;
    const int64_t ns = N + ncp;
    const float2* src = grid + frame * (int64_t)N * m;
    for (int idx = threadIdx.x; idx < C * N; idx += kOfdmNT) {
        const int k = idx / C, c = idx % C, l = l0 + c;
        buf[c * VS + pidx(k)] = l < m ? src[(int64_t)k * m + l] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    fft_vectors<N, true, C, kOfdmNT>(buf, VS, tw);
    const float inv_n = 1.0f / float(N);
    float2* dst = stream + frame * (int64_t)m * ns;
    for (int idx = threadIdx.x; idx < C * (int)ns; idx += kOfdmNT) {
        const int c = idx / (int)ns, j = idx % (int)ns, l = l0 + c;
        if (l >= m) continue;
        const int i = j < ncp ? N - ncp + j : j - ncp;
        dst[(int64_t)l * ns + j] = cscale(buf[c * VS + pidx(i)], inv_n);
    }
}

template <int N>
cudaError_t launch_ofdm_n(bool inverse, const float2* in, float2* out, int m, int ncp, int64_t frames,
                          const float2* tw, cudaStream_t st) {
    constexpr int C = OfdmTile<N>::C;
    const int ntiles = (m + C - 1) / C;
    const size_t smem = sizeof(float2) * C * pad_len(N);
    auto kern = inverse ? ofdm_mod_kernel<N> : ofdm_demod_kernel<N>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    for (int64_t f0 = 0; f0 < frames;) {
        const int64_t nf = std::min<int64_t>(frames - f0, (int64_t)(0x7fffffff / ntiles));
        const int64_t in_stride = inverse ? (int64_t)N * m : (int64_t)m * (N + ncp);
        const int64_t out_stride = inverse ? (int64_t)m * (N + ncp) : (int64_t)N * m;
        kern<<<(unsigned)(nf * ntiles), kOfdmNT, smem, st>>>(in + f0 * in_stride, out + f0 * out_stride, m, ncp, ntiles,
                                                             tw);
        f0 += nf;
    }
    return cudaGetLastError();
}

}  // namespace

// n: power of two in [16, 4096]; 0 <= ncp <= n.
cudaError_t launch_ofdm(bool inverse, const float2* in, float2* out, int n, int m, int ncp, int64_t frames,
                        const float2* tw, cudaStream_t st) {
    switch (n) {
        case 16: return launch_ofdm_n<16>(inverse, in, out, m, ncp, frames, tw, st);
        case 32: return launch_ofdm_n<32>(inverse, in, out, m, ncp, frames, tw, st);
        case 64: return launch_ofdm_n<64>(inverse, in, out, m, ncp, frames, tw, st);
        case 128: return launch_ofdm_n<128>(inverse, in, out, m, ncp, frames, tw, st);
        case 256: return launch_ofdm_n<256>(inverse, in, out, m, ncp, frames, tw, st);
        case 512: return launch_ofdm_n<512>(inverse, in, out, m, ncp, frames, tw, st);
        case 1024: return launch_ofdm_n<1024>(inverse, in, out, m, ncp, frames, tw, st);
        case 2048: return launch_ofdm_n<2048>(inverse, in, out, m, ncp, frames, tw, st);
        case 4096: return launch_ofdm_n<4096>(inverse, in, out, m, ncp, frames, tw, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace ofdmr
