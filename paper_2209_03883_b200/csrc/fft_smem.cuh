// Shared-memory batched complex FFT engine for sm_100a (fp32).
//
// A CTA transforms NVEC contiguous vectors of length LEN that live in shared memory
// (vector v at buf + v * vs; element t at physical offset pidx(t) = t + t/32 so the
// Stockham scatter of the early passes does not pile onto one bank).  Each pass is
// a radix-R Stockham autosort step executed from registers:
//     read  x_i = in[j + i*LEN/R]               (consecutive j -> consecutive banks)
//     twiddle x_i *= W_{Ls R}^{i k}, k = j mod Ls
//     R-point DFT in registers (radix 2/4/8/16 with compile-time constants)
//     write out[(j-k)R + k + i Ls]
// in place: every thread first pulls its butterflies into registers, one barrier,
// then scatters.  Twiddles come from one 4096-entry fp32 table e^{-j2pi t/4096}
// (double-precision cos/sin rounded once, uploaded by the host) read through the
// read-only path; every LEN <= 4096 is a strided view of it.
//
// The reference performs these transforms with FFTW3 in fp64
// (src/fft.cpp:35-50 via include/ofdmradar/fft.hpp:13-29): unscaled, forward sign
// e^{-j}, inverse e^{+j}.  The same sign/scale contract is kept here.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ofdmr {

constexpr int kTwLen = 4096;  // twiddle table length (max supported FFT length)

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float cnorm(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }

__host__ __device__ constexpr int pad_len(int len) { return len + len / 32 + 1; }
__device__ __forceinline__ int pidx(int t) { return t + (t >> 5); }

template <int V> struct Log2 { static constexpr int value = 1 + Log2<V / 2>::value; };
template <> struct Log2<1> { static constexpr int value = 0; };

// multiply by W4 = e^{-j pi/2} = -j (forward) or +j (inverse)
template <bool INV> __device__ __forceinline__ float2 mul_w4(float2 a) {
    return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

template <bool INV> __device__ __forceinline__ void dft2(float2* x) {
    const float2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
}

template <bool INV> __device__ __forceinline__ void dft4(float2* x) {
    const float2 a0 = cadd(x[0], x[2]), a1 = csub(x[0], x[2]);
    const float2 a2 = cadd(x[1], x[3]), a3 = mul_w4<INV>(csub(x[1], x[3]));
    x[0] = cadd(a0, a2);
    x[2] = csub(a0, a2);
    x[1] = cadd(a1, a3);
    x[3] = csub(a1, a3);
}

template <bool INV> __device__ __forceinline__ void dft8(float2* x) {
    constexpr float c = 0.70710678118654752440f;
    float2 e[4] = {x[0], x[2], x[4], x[6]};
    float2 o[4] = {x[1], x[3], x[5], x[7]};
    dft4<INV>(e);
    dft4<INV>(o);
    // o1 *= W8, o2 *= W8^2, o3 *= W8^3  (W8 = e^{-+j pi/4})
    const float2 o1 = INV ? make_float2(c * (o[1].x - o[1].y), c * (o[1].x + o[1].y))
                          : make_float2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));
    const float2 o2 = mul_w4<INV>(o[2]);
    const float2 o3 = INV ? make_float2(-c * (o[3].x + o[3].y), c * (o[3].x - o[3].y))
                          : make_float2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));
    x[0] = cadd(e[0], o[0]);
    x[4] = csub(e[0], o[0]);
    x[1] = cadd(e[1], o1);
    x[5] = csub(e[1], o1);
    x[2] = cadd(e[2], o2);
    x[6] = csub(e[2], o2);
    x[3] = cadd(e[3], o3);
    x[7] = csub(e[3], o3);
}

template <bool INV> __device__ __forceinline__ void dft16(float2* x) {
    // cos/sin(pi k / 8), k = 0..7
    constexpr float C16[8] = {1.0f, 0.92387953251128675613f, 0.70710678118654752440f, 0.38268343236508977173f,
                              0.0f, -0.38268343236508977173f, -0.70710678118654752440f, -0.92387953251128675613f};
    constexpr float S16[8] = {0.0f, 0.38268343236508977173f, 0.70710678118654752440f, 0.92387953251128675613f,
                              1.0f, 0.92387953251128675613f, 0.70710678118654752440f, 0.38268343236508977173f};
    float2 e[8], o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        e[i] = x[2 * i];
        o[i] = x[2 * i + 1];
    }
    dft8<INV>(e);
    dft8<INV>(o);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        // W16^k = cos - (+) j sin for forward (inverse)
        const float2 w = make_float2(C16[k], INV ? S16[k] : -S16[k]);
        const float2 t = (k == 0) ? o[0] : cmul(o[k], w);
        x[k] = cadd(e[k], t);
        x[k + 8] = csub(e[k], t);
    }
}

template <int R, bool INV> __device__ __forceinline__ void dft_r(float2* x) {
    if constexpr (R == 2) dft2<INV>(x);
    else if constexpr (R == 4) dft4<INV>(x);
    else if constexpr (R == 8) dft8<INV>(x);
    else dft16<INV>(x);
}

__device__ __forceinline__ float2 twiddle(const float2* __restrict__ tw, int idx, bool inv) {
    const float2 w = __ldg(tw + idx);
    return inv ? make_float2(w.x, -w.y) : w;
}

// One Stockham pass over NVEC vectors of length LEN with radix R; Ls = product of
// radices of the passes already done.  NT threads cooperate.
template <int LEN, int R, bool INV, int NVEC, int NT>
__device__ __forceinline__ void stockham_pass(float2* buf, int vs, int Ls, const float2* __restrict__ tw) {
    constexpr int T = LEN / R;
    constexpr int TOTAL = NVEC * T;
    constexpr int BPT = (TOTAL + NT - 1) / NT;
    constexpr int LOGT = Log2<T>::value;
    float2 v[BPT][R];
    const int tstride = kTwLen / (Ls * R);
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int b = threadIdx.x + q * NT;
        if ((TOTAL % NT == 0) || b < TOTAL) {
            const int vec = b >> LOGT;
            const int j = b & (T - 1);
            const int k = j & (Ls - 1);
            const float2* base = buf + vec * vs;
#pragma unroll
            for (int i = 0; i < R; ++i) v[q][i] = base[pidx(j + i * T)];
            if (Ls > 1) {
#pragma unroll
                for (int i = 1; i < R; ++i) v[q][i] = cmul(v[q][i], twiddle(tw, i * k * tstride, INV));
            }
            dft_r<R, INV>(v[q]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int b = threadIdx.x + q * NT;
        if ((TOTAL % NT == 0) || b < TOTAL) {
            const int vec = b >> LOGT;
            const int j = b & (T - 1);
            const int k = j & (Ls - 1);
            float2* base = buf + vec * vs;
            const int o = (j - k) * R + k;
#pragma unroll
            for (int i = 0; i < R; ++i) base[pidx(o + i * Ls)] = v[q][i];
        }
    }
    __syncthreads();
}

// Full in-place FFT of NVEC vectors of length LEN (power of two, 2..4096).
// Radix plan: 16 when log2(LEN) % 3 == 1, 4 when == 2, otherwise all 8.
// Caller must __syncthreads() after filling buf; returns after a barrier.
template <int LEN, bool INV, int NVEC, int NT>
__device__ __forceinline__ void fft_vectors(float2* buf, int vs, const float2* __restrict__ tw) {
    constexpr int L2 = Log2<LEN>::value;
    constexpr int N8 = L2 / 3;
    constexpr int REM = L2 % 3;
    int Ls = 1;
    if constexpr (REM == 1) {
        if constexpr (L2 >= 4) {
            stockham_pass<LEN, 16, INV, NVEC, NT>(buf, vs, Ls, tw);
            Ls *= 16;
#pragma unroll 1
            for (int p = 0; p < N8 - 1; ++p) {
                stockham_pass<LEN, 8, INV, NVEC, NT>(buf, vs, Ls, tw);
                Ls *= 8;
            }
        } else {
            stockham_pass<LEN, 2, INV, NVEC, NT>(buf, vs, Ls, tw);
        }
    } else {
#pragma unroll 1
        for (int p = 0; p < N8; ++p) {
            stockham_pass<LEN, 8, INV, NVEC, NT>(buf, vs, Ls, tw);
            Ls *= 8;
        }
        if constexpr (REM == 2) stockham_pass<LEN, 4, INV, NVEC, NT>(buf, vs, Ls, tw);
    }
}

}  // namespace ofdmr
