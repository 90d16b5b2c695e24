// Register-resident warp FFTs for the hot shapes (sm_100a, fp32).
//
//   1024 = 32 x 32 per warp: lane j holds x[j + 32 i] (i = 0..31) in registers;
//     DFT_32 over i, twiddle W_1024^{j t1}, transpose through the column's own
//     padded shared-memory buffer (pidx: t + t/32, conflict-free in both directions),
//     DFT_32 over j.  On exit lane t1 holds X[t1 + 32 t2] in v[t2].
//   256 = 16 x 16 per half-warp (two rows per warp), same scheme with DFT_16.
//
// Because the output layout of one transform (lane t1 <-> X[t1 + 32 t2]) is exactly the
// input layout of the next (lane j <-> x[j + 32 i]), the DFT-CE chain
// IFFT -> truncate -> FFT -> window -> IFFT never leaves registers between transforms;
// after truncation to L <= 128 taps only v[0..3] are non-zero, so the next DFT_32 runs
// input-pruned (dft32_in4).  Sign/scale contract of include/ofdmradar/fft.hpp:12-15.
#pragma once
#include <utility>

#include "fft_smem.cuh"

namespace ofdmr {

template <bool INV, int K>
__device__ __forceinline__ void dft32_step(float2* x, const float2* e, const float2* o) {
    bfly32<INV, K>(x[K], x[K + 16], e[K], o[K]);
}

template <bool INV, int... Ks>
__device__ __forceinline__ void dft32_combine(float2* x, const float2* e, const float2* o,
                                              std::integer_sequence<int, Ks...>) {
    (dft32_step<INV, Ks>(x, e, o), ...);
}

// Full 32-point DFT in registers, natural order in and out.
template <bool INV> __device__ __forceinline__ void dft32(float2* x) {
    float2 e[16], o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        e[i] = x[2 * i];
        o[i] = x[2 * i + 1];
    }
    dft16<INV>(e);
    dft16<INV>(o);
    dft32_combine<INV>(x, e, o, std::make_integer_sequence<int, 16>{});
}

template <bool INV, int B>
__device__ __forceinline__ void in4_step(float2* out, const float2* v) {
    float2 u[4] = {v[0], mul_w32<INV, B>(v[1]), mul_w32<INV, 2 * B>(v[2]), mul_w32<INV, 3 * B>(v[3])};
    dft4<INV>(u);
#pragma unroll
    for (int a = 0; a < 4; ++a) out[8 * a + B] = u[a];
}

template <bool INV, int... Bs>
__device__ __forceinline__ void in4_all(float2* out, const float2* v, std::integer_sequence<int, Bs...>) {
    (in4_step<INV, Bs>(out, v), ...);
}

// 32-point DFT of an input that is non-zero only at i = 0..3:
// X[8a + b] = DFT_4 over i of (v_i W_32^{ib}).
template <bool INV> __device__ __forceinline__ void dft32_in4(float2* x) {
    float2 v[4] = {x[0], x[1], x[2], x[3]};
    in4_all<INV>(x, v, std::make_integer_sequence<int, 8>{});
}

template <bool INV, int R, int K>
__device__ __forceinline__ void out4_acc(float2* acc, const float2* u) {
    const float2 t = mul_w32<INV, R * K>(u[K]);
    acc[K] = cadd(acc[K], t);
}
template <bool INV, int R>
__device__ __forceinline__ void out4_step(float2* acc, const float2* x) {
    float2 u[4] = {x[R], x[R + 8], x[R + 16], x[R + 24]};
    dft4<INV>(u);
    if constexpr (R == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = u[k];
    } else {
        out4_acc<INV, R, 0>(acc, u);
        out4_acc<INV, R, 1>(acc, u);
        out4_acc<INV, R, 2>(acc, u);
        out4_acc<INV, R, 3>(acc, u);
    }
}
template <bool INV, int... Rs>
__device__ __forceinline__ void out4_all(float2* acc, const float2* x, std::integer_sequence<int, Rs...>) {
    (out4_step<INV, Rs>(acc, x), ...);
}

// First 4 outputs of a 32-point DFT (natural order in; X[0..3] -> x[0..3]):
// X[k] = sum_r W_32^{rk} DFT_4 over m of x[8m + r], k < 4.
template <bool INV> __device__ __forceinline__ void dft32_out4(float2* x) {
    float2 acc[4];
    out4_all<INV>(acc, x, std::make_integer_sequence<int, 8>{});
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = acc[k];
}

// Warp FFT of length 1024.  On entry lane j holds v[i] = x[j + 32 i] (only v[0..NZ)
// read when NZ == 4; only v[0..4) produced when NOUT == 4).  col: this warp's padded smem vector (>= pad_len(1024) float2),
// free for use.  tw: smem table tw[t1 * 32 + j] = W_1024^{j t1} (forward).  On exit lane
// t1 holds X[t1 + 32 t2] in v[t2].
template <bool INV, int NZ, bool GTW = false, int NOUT = 32>
__device__ __forceinline__ void warp_fft1024(float2 (&v)[32], float2* col, const float2* tw) {
    const int lane = threadIdx.x & 31;
    if constexpr (NZ == 4) dft32_in4<INV>(v);
    else dft32<INV>(v);
#pragma unroll
    for (int t1 = 1; t1 < 32; ++t1) {
        float2 w = GTW ? __ldg(tw + t1 * 32 + lane) : tw[t1 * 32 + lane];  // GTW: read-only global table
        if (INV) w.y = -w.y;
        v[t1] = cmul(v[t1], w);
    }
    __syncwarp();
#pragma unroll
    for (int t1 = 0; t1 < 32; ++t1) col[t1 * 33 + lane] = v[t1];  // pidx(t1*32 + lane)
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = col[lane * 33 + j];     // pidx(lane*32 + j)
    if constexpr (NOUT == 4) dft32_out4<INV>(v);  // only X[t1 + 32 t2], t2 < 4 (v[4..] garbage)
    else dft32<INV>(v);
}

// Half-warp FFT of length 256 (lanes 0-15 one vector, 16-31 another).  On entry
// sub-lane j holds v[i] = x[j + 16 i]; buf: this half-warp's 16 x 17 padded scratch;
// tw: tw[t1 * 16 + j] = W_256^{j t1}.  On exit sub-lane t1 holds X[t1 + 16 t2] in v[t2].
template <bool INV>
__device__ __forceinline__ void halfwarp_fft256(float2 (&v)[16], float2* buf, const float2* tw) {
    const int j = threadIdx.x & 15;
    dft16<INV>(v);
#pragma unroll
    for (int t1 = 1; t1 < 16; ++t1) {
        float2 w = tw[t1 * 16 + j];
        if (INV) w.y = -w.y;
        v[t1] = cmul(v[t1], w);
    }
    __syncwarp();
#pragma unroll
    for (int t1 = 0; t1 < 16; ++t1) buf[t1 * 17 + j] = v[t1];
    __syncwarp();
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) v[jj] = buf[j * 17 + jj];
    dft16<INV>(v);
}

// Same with the sub-lane's twiddles held in registers: twr[t1] = W_256^{j t1} (forward),
// loaded once by callers that transform many rows per lane.
template <bool INV>
__device__ __forceinline__ void halfwarp_fft256_rt(float2 (&v)[16], float2* buf, const float2 (&twr)[16]) {
    const int j = threadIdx.x & 15;
    dft16<INV>(v);
#pragma unroll
    for (int t1 = 1; t1 < 16; ++t1) {
        float2 w = twr[t1];
        if (INV) w.y = -w.y;
        v[t1] = cmul(v[t1], w);
    }
    __syncwarp();
#pragma unroll
    for (int t1 = 0; t1 < 16; ++t1) buf[t1 * 17 + j] = v[t1];
    __syncwarp();
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) v[jj] = buf[j * 17 + jj];
    dft16<INV>(v);
}

}  // namespace ofdmr
