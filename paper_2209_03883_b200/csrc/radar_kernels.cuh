// Receiver hot-path kernels (sm_100a): subcarrier-axis column pass, symbol-axis row
// pass with fused |.|^2 / fftshift / strict-3x3-local-max detection, and the per-frame
// top-K merge.  Host launch code lives in capi.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ofdmr {

constexpr int kNT = 256;      // threads per CTA for the FFT passes
constexpr int kTwLenHost = 4096;  // twiddle table length (fft_smem.cuh kTwLen)
constexpr int kMaxK = 64;     // max detections per frame (reference default max_targets, config.hpp:33)

// One LS cell h = y / x (estimation.cpp:10-21) with the reference's zero-cell semantics: only an
// exactly zero x (both components 0, `xv == cplx(0,0)`, estimation.cpp:17) flags the frame.  |x|^2
// is formed in fp32 on the fast path; when it falls outside the fp32 normal range (a denormal x,
// or |x| > 1.8e19) the cell is divided in fp64 instead, as the reference does on the upcast
// complex<double>, and its 1/|x|^2 term goes to the fp64 accumulator exactly.
__device__ __noinline__ inline float2 ls_cell_fp64(float yr, float yi, float xr, float xi, double& inv_acc,
                                                  int& zero_cell) {
    if (xr == 0.f && xi == 0.f) {
        zero_cell = 1;
        return make_float2(0.f, 0.f);
    }
    const double dr = xr, di = xi;
    const double nn = __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(di, di));
    const double iv = 1.0 / nn;
    inv_acc += iv;
    return make_float2(float((double(yr) * dr + double(yi) * di) * iv), float((double(yi) * dr - double(yr) * di) * iv));
}
__device__ __forceinline__ float2 ls_cell(float yr, float yi, float xr, float xi, double& inv_acc, int& zero_cell) {
    const float n = fmaf(xr, xr, xi * xi);
    if (__builtin_expect(n >= 1.17549435e-38f && n <= 3.40282347e38f, 1)) {
        const float i = 1.0f / n;
        inv_acc += (double)i;
        return make_float2(fmaf(yr, xr, yi * xi) * i, fmaf(yi, xr, -yr * xi) * i);
    }
    return ls_cell_fp64(yr, yi, xr, xi, inv_acc, zero_cell);
}

// Column (subcarrier / delay axis) pass over tiles of C adjacent columns of one frame.
struct ColArgs {
    const float2* y;        // LS inputs: received frame Y (N x M per frame) ...
    const float2* x;        // ... and transmitted (possibly ZC-precoded) x_tx; or null
    const float2* h;        // channel-estimate input when y == null
    float2* h_out;          // optional: H (hout_after_ce = 0) or H' after DFT-CE (= 1)
    float2* g_out;          // optional: k-pass output G (g_rows x M per frame)
    const float* wk;        // subcarrier window (N), null = rectangular
    const float* wl;        // symbol window (M), null = rectangular
    double* inv_partial;    // per (frame, tile) sum of 1/|x|^2, deterministic; or null
    int* status;            // per frame: bit0 = zero X cell (estimation.cpp:17)
    const float2* tw;       // 4096-entry twiddle table
    int m;                  // columns M
    int ce_taps;            // DFT-CE truncation L (0 = no DFT-CE)
    int hout_after_ce;
    int shortcut;           // rect window, N' = N, DFT-CE: G = IFFT_N(H) rows < L
    int g_rows;             // rows of G written per frame
    int ntiles;             // M / C
    // mixed-radix path (N or N' not a power of two, mixed_kernels.cu): runtime sizes and the
    // e^{-j 2 pi t / L} tables of the two transform lengths
    int n, np;
    const float2* tw_n;
    const float2* tw_np;
};

// Row (symbol / Doppler axis) pass over blocks of R rows of one frame (+ 1 halo row
// each side) with the detection fused in.
struct RowArgs {
    const float2* g;        // G (g_rows x m per frame), or null when p_in is given
    const float* p_in;      // P (n_prime x m_prime) for the detect-only entry point
    float* p_out;           // optional periodogram map out (n_prime x m_prime, fft-shifted)
    const double* inv_partial;  // per (frame, tile) 1/|x|^2 partials, or null
    int ntiles;
    const double* sigma2;   // per frame: noise sigma^2 (with partials) or sigma_h^2 (without)
    const double* eta_in;   // per frame threshold given directly (extract_peaks on a mask), or null
    double log_pfa;         // log(pfa) computed on the host (periodogram.cpp:80)
    double power_factor;    // window power factor (periodogram.cpp:11-16)
    double inv_count;       // 1 / (N M) for division_noise_power (pipeline.cpp:22)
    float scale;            // 1 / (N M) periodogram scale (periodogram.cpp:65)
    const float2* tw;
    int n_prime;            // rows of P
    int g_rows;             // rows of G that are non-zero (rows >= g_rows are exactly 0)
    int m;                  // input row length (M); zero-padded to m_prime
    int rows_per_block;     // R
    int kmax;               // candidates kept per block
    unsigned long long* cand;  // [frame][nblk][kmax] packed keys
    int detect;             // 0 = map only
    const float2* zp_tw;    // rowpass_zp twiddles: W_2048^{j (4 k1 + m1)} [4][32][16], then W_128^q [128]
    int mp;                 // mixed-radix path: M' (runtime) and its e^{-j 2 pi t / M'} table
    const float2* tw_mp;
};

struct MergeArgs {
    const unsigned long long* cand;
    int nblk;
    int kmax;
    const int32_t* k_per_frame;  // null -> kmax
    int m_prime;
    int32_t* det_delay;
    int32_t* det_doppler;
    float* det_power;
    int32_t* counts;
    const double* inv_partial;
    int ntiles;
    const double* sigma2;
    double log_pfa, power_factor, inv_count;
    double* s2h_out;        // optional per-frame sigma_h^2
    double* eta_out;        // optional per-frame threshold
};

// sigma_h^2 (pipeline.cpp:18-23: sigma^2 * mean(1/|x|^2)) from the per-(frame, tile) partial
// sums: lane i adds tiles i, i + 32, .. in order, then a fixed xor-shuffle tree (every lane ends
// with the same value).  Call with all 32 lanes of a warp; every kernel that thresholds or
// reports sigma_h^2 from the partials uses this one order.
__device__ __forceinline__ double sigma_h2_warp(const double* inv_partial, int ntiles, int f, double sigma2,
                                                double inv_count) {
    if (inv_partial == nullptr) return sigma2;  // caller passed sigma_h^2 directly
    if (sigma2 <= 0.0) return 0.0;
    double acc = 0.0;
    for (int t = threadIdx.x & 31; t < ntiles; t += 32) acc += inv_partial[(size_t)f * ntiles + t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    return sigma2 * acc * inv_count;
}

// Packed detection key: larger key = larger power, ties -> smaller row-major index
// (extract_peaks ordering, periodogram.cpp:98-102).  P >= 0 so the float bit pattern
// orders like the value.
__device__ __forceinline__ unsigned long long make_key(float p, uint32_t idx) {
    return (static_cast<unsigned long long>(__float_as_uint(p)) << 32) | (0xFFFFFFFFu - idx);
}

// Block-wide top-K selection over a shared-memory key list (keys unique, 0 = empty).
// Writes up to K keys in descending order to out[0..K) (zero-filled).  NT threads.
template <int NT>
__device__ __forceinline__ void block_topk(unsigned long long* list, int cnt, int K, unsigned long long* out,
                           unsigned long long* s_best, int* s_idx) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int round = 0; round < K; ++round) {
        unsigned long long best = 0;
        int bi = -1;
        for (int i = threadIdx.x; i < cnt; i += NT) {
            const unsigned long long v = list[i];
            if (v > best) { best = v; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best) { best = ob; bi = oi; }
        }
        if (lane == 0) { s_best[w] = best; s_idx[w] = bi; }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long b = 0;
            int id = -1;
            for (int i = 0; i < NT / 32; ++i)
                if (s_best[i] > b) { b = s_best[i]; id = s_idx[i]; }
            out[round] = b;
            if (id >= 0) list[id] = 0;
            s_best[0] = b;
        }
        __syncthreads();
        const bool done = s_best[0] == 0;
        __syncthreads();
        if (done) {
            for (int r = round + 1 + threadIdx.x; r < K; r += NT) out[r] = 0;
            break;
        }
    }
}

// Same selection with the list read ONCE into registers (PER entries per thread, cnt <= PER *
// NT): keys are unique (cell index in the low word), so the round's winner is retired by value
// without tracking its position; two barriers per round and no re-reads of the list.
template <int NT, int PER>
__device__ __forceinline__ void block_topk_reg(const unsigned long long* list, int cnt, int K, unsigned long long* out,
                                               unsigned long long* s_best) {
    // `out` is in shared memory: the round's winner is broadcast through out[round]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long v[PER];
#pragma unroll
    for (int p = 0; p < PER; ++p) {
        const int i = threadIdx.x + p * NT;
        v[p] = i < cnt ? list[i] : 0ull;
    }
    for (int round = 0; round < K; ++round) {
        unsigned long long best = 0;
#pragma unroll
        for (int p = 0; p < PER; ++p) best = v[p] > best ? v[p] : best;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
            best = ob > best ? ob : best;
        }
        if (lane == 0) s_best[w] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long b = 0;
            for (int i = 0; i < NT / 32; ++i) b = s_best[i] > b ? s_best[i] : b;
            out[round] = b;
        }
        __syncthreads();
        const unsigned long long b = out[round];
        if (b == 0) {
            for (int r = round + 1 + threadIdx.x; r < K; r += NT) out[r] = 0;
            break;
        }
#pragma unroll
        for (int p = 0; p < PER; ++p)
            if (v[p] == b) v[p] = 0ull;
    }
    __syncthreads();
}

__device__ __forceinline__ void block_topk_smem(unsigned long long* list, int cnt, int K, unsigned long long* out,
                                                unsigned long long* s_best, int* s_idx) {
    block_topk<256>(list, cnt, K, out, s_best, s_idx);
}
// Same over a global-memory scratch list (entries are consumed in place).
__device__ __forceinline__ void block_topk_global(unsigned long long* list, int cnt, int K, unsigned long long* out,
                                                  unsigned long long* s_best, int* s_idx) {
    block_topk<256>(list, cnt, K, out, s_best, s_idx);
}

}  // namespace ofdmr
