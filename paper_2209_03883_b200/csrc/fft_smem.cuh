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

// Complex fp32 arithmetic on sm_100a's packed FP32x2 pipe (FADD2 / FMUL2 / FFMA2): one
// warp-instruction operates on both halves of a float2, so every complex add is ONE issue slot
// and a complex multiply TWO (FMUL2 + FFMA2 with the swapped, half-negated operand encoded as
// an operand modifier), against 2 and 4 scalar instructions.  The FP32 pipe itself is not
// faster (128 lane-ops / SM / cycle either way, tools/micro/f32x2_micro.cu) but the FFT kernels
// here are issue-bound, not FMA-pipe-bound.  Each half is the IEEE round-to-nearest operation
// of the scalar form (no contraction beyond the explicit fma).  -DOFDMR_SCALAR_FP32 restores
// the scalar code for A/B measurements.
#ifndef OFDMR_SCALAR_FP32
typedef unsigned long long f2bits;
__device__ __forceinline__ f2bits f2_pack(float a, float b) {
    f2bits r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f2bits f2_pack(float2 a) { return f2_pack(a.x, a.y); }
__device__ __forceinline__ float2 f2_unpack(f2bits r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
    f2bits r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(r);
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
    f2bits r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(r);
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
    f2bits r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(r);
}
// a * b + c, per half
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
    f2bits r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_pack(a)), "l"(f2_pack(b)), "l"(f2_pack(c)));
    return f2_unpack(r);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return f2_add(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return f2_sub(a, b); }
// a w = w.x (a.x, a.y) + w.y (-a.y, a.x): FMUL2 + FFMA2
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
    return f2_fma(make_float2(-a.y, a.x), make_float2(w.y, w.y), f2_mul(a, make_float2(w.x, w.x)));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return f2_mul(a, make_float2(s, s)); }
// e + (c + j s) o for real constants c, s: two FFMA2
__device__ __forceinline__ float2 cfma_cs(float c, float s, float2 o, float2 e) {
    return f2_fma(make_float2(-o.y, o.x), make_float2(s, s), f2_fma(o, make_float2(c, c), e));
}
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cfma_cs(float c, float s, float2 o, float2 e) {
    return make_float2(fmaf(c, o.x, fmaf(-s, o.y, e.x)), fmaf(c, o.y, fmaf(s, o.x, e.y)));
}
#endif
__device__ __forceinline__ float cnorm(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }

__host__ __device__ constexpr int pad_len(int len) { return len + len / 32 + 1; }
__device__ __forceinline__ int pidx(int t) { return t + (t >> 5); }

template <int V> struct Log2 { static constexpr int value = 1 + Log2<V / 2>::value; };
template <> struct Log2<1> { static constexpr int value = 0; };

// multiply by W4 = e^{-j pi/2} = -j (forward) or +j (inverse)
template <bool INV> __device__ __forceinline__ float2 mul_w4(float2 a) {
    return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

template <int K> struct W32c {
    // compile-time W_32^K = cos - (+) j sin (forward / inverse)
    static constexpr float c() {
        constexpr float t[32] = {
            1.0f, 0.98078528040323044913f, 0.92387953251128675613f, 0.83146961230254523708f,
            0.70710678118654752440f, 0.55557023301960222474f, 0.38268343236508977173f, 0.19509032201612826785f,
            0.0f, -0.19509032201612826785f, -0.38268343236508977173f, -0.55557023301960222474f,
            -0.70710678118654752440f, -0.83146961230254523708f, -0.92387953251128675613f, -0.98078528040323044913f,
            -1.0f, -0.98078528040323044913f, -0.92387953251128675613f, -0.83146961230254523708f,
            -0.70710678118654752440f, -0.55557023301960222474f, -0.38268343236508977173f, -0.19509032201612826785f,
            0.0f, 0.19509032201612826785f, 0.38268343236508977173f, 0.55557023301960222474f,
            0.70710678118654752440f, 0.83146961230254523708f, 0.92387953251128675613f, 0.98078528040323044913f};
        return t[K % 32];
    }
    static constexpr float s() {
        constexpr float t[32] = {
            0.0f, 0.19509032201612826785f, 0.38268343236508977173f, 0.55557023301960222474f,
            0.70710678118654752440f, 0.83146961230254523708f, 0.92387953251128675613f, 0.98078528040323044913f,
            1.0f, 0.98078528040323044913f, 0.92387953251128675613f, 0.83146961230254523708f,
            0.70710678118654752440f, 0.55557023301960222474f, 0.38268343236508977173f, 0.19509032201612826785f,
            0.0f, -0.19509032201612826785f, -0.38268343236508977173f, -0.55557023301960222474f,
            -0.70710678118654752440f, -0.83146961230254523708f, -0.92387953251128675613f, -0.98078528040323044913f,
            -1.0f, -0.98078528040323044913f, -0.92387953251128675613f, -0.83146961230254523708f,
            -0.70710678118654752440f, -0.55557023301960222474f, -0.38268343236508977173f, -0.19509032201612826785f};
        return t[K % 32];
    }
};

template <bool INV, int K> __device__ __forceinline__ float2 mul_w32(float2 a) {
    constexpr int k = K % 32;
    if constexpr (k == 0) return a;
    else if constexpr (k == 8) return mul_w4<INV>(a);
    else if constexpr (k == 16) return make_float2(-a.x, -a.y);
    else if constexpr (k == 24) return mul_w4<!INV>(a);
    else {
        constexpr float c = W32c<k>::c();
        constexpr float s = INV ? W32c<k>::s() : -W32c<k>::s();
#ifndef OFDMR_SCALAR_FP32
        return f2_fma(make_float2(-a.y, a.x), make_float2(s, s), f2_mul(a, make_float2(c, c)));
#else
        return make_float2(c * a.x - s * a.y, c * a.y + s * a.x);
#endif
    }
}


// Radix-2 butterfly with a constant twiddle w = W_32^K (forward e^{-2 pi i K/32}, inverse
// conjugate): lo = e + w o, hi = e - w o.  General K: lo with two FFMA2 and hi = 2e - lo with
// one (three packed instructions instead of a 2-instruction multiply plus two adds).
template <bool INV, int K>
__device__ __forceinline__ void bfly32(float2& lo, float2& hi, float2 e, float2 o) {
    constexpr int k = K % 32;
    if constexpr (k == 0 || k == 8 || k == 16 || k == 24) {
        const float2 t = mul_w32<INV, K>(o);
        lo = cadd(e, t);
        hi = csub(e, t);
    } else {
        constexpr float c = W32c<k>::c();
        constexpr float s = INV ? W32c<k>::s() : -W32c<k>::s();
        const float2 a = cfma_cs(c, s, o, e);
#ifndef OFDMR_SCALAR_FP32
        hi = f2_fma(e, make_float2(2.0f, 2.0f), make_float2(-a.x, -a.y));
#else
        hi = make_float2(fmaf(2.0f, e.x, -a.x), fmaf(2.0f, e.y, -a.y));
#endif
        lo = a;
    }
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
    float2 e[4] = {x[0], x[2], x[4], x[6]};
    float2 o[4] = {x[1], x[3], x[5], x[7]};
    dft4<INV>(e);
    dft4<INV>(o);
    // W_8^k = W_32^{4k}
    bfly32<INV, 0>(x[0], x[4], e[0], o[0]);
    bfly32<INV, 4>(x[1], x[5], e[1], o[1]);
    bfly32<INV, 8>(x[2], x[6], e[2], o[2]);
    bfly32<INV, 12>(x[3], x[7], e[3], o[3]);
}

template <bool INV> __device__ __forceinline__ void dft16(float2* x) {
    float2 e[8], o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        e[i] = x[2 * i];
        o[i] = x[2 * i + 1];
    }
    dft8<INV>(e);
    dft8<INV>(o);
    // W_16^k = W_32^{2k}
    bfly32<INV, 0>(x[0], x[8], e[0], o[0]);
    bfly32<INV, 2>(x[1], x[9], e[1], o[1]);
    bfly32<INV, 4>(x[2], x[10], e[2], o[2]);
    bfly32<INV, 6>(x[3], x[11], e[3], o[3]);
    bfly32<INV, 8>(x[4], x[12], e[4], o[4]);
    bfly32<INV, 10>(x[5], x[13], e[5], o[5]);
    bfly32<INV, 12>(x[6], x[14], e[6], o[6]);
    bfly32<INV, 14>(x[7], x[15], e[7], o[7]);
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
