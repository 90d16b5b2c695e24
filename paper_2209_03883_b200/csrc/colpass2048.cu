// Column (subcarrier / delay axis) pass for N = 2048 -> N' = 4096, the cfg2 shape
// (2048 x 512 ZC-precoded frames, DFT-CE with L = 256, 4096 x 2048 map):
//     LS (estimation.cpp:10-21) -> [DFT-CE: IFFT_2048, keep L taps x 1/N, FFT_2048]
//     (estimation.cpp:23-39) -> w_k w_l, zero-pad to 4096, unscaled IFFT_4096 (the delay axis
//     of periodogram.cpp:39-75) -> G rows (the row pass, rowpass_zp.cu, does the rest).
//
// One warp per symbol column, 8 columns (64-B row segments) per tile, one 8-warp CTA per SM,
// persistent over (frame, tile) items.  Every transform is a register warp FFT_1024
// (warp_fft.cuh) and the layouts chain without data movement between them:
//   IFFT_2048 -> taps   decimation in frequency: a[k] = h[k] + h[k + 1024],
//                       b[k] = (h[k] - h[k + 1024]) W_2048^{-k}; x[2u] = IFFT_1024(a)[u],
//                       x[2u + 1] = IFFT_1024(b)[u], only u < 128 computed (output-pruned)
//   taps -> H (FFT)     E = FFT_1024(x[2u]), O = FFT_1024(x[2u + 1]) (input-pruned, 4 of 32
//                       values per lane); H[q] = E + W_2048^q O, H[q + 1024] = E - W_2048^q O
//                       land on lane q mod 32: exactly the next transform's input layout
//   H -> G (IFFT_4096)  X[4p + s] = IFFT_1024_q( W_4096^{-sq} (H'[q] + j^s H'[q + 1024]) )[p],
//                       s = 0..3, H' = H w_k w_l
// so a column costs 2 output-pruned + 2 input-pruned + 4 full warp FFT_1024s against the
// generic path's three full shared-memory Stockham transforms (2048, 2048, 4096).
//
// Inputs: Y and x_tx stream through a ring of thread-private 16-B cp.async slots (64 rows x
// 64 B per stage, no barriers); the LS divide (exact reference zero-cell semantics, ls_cell) is
// fused into the ring consumption, which writes h column-major into the tile.  The next item's
// rows are prefetched into L2 while the current one computes.  Outputs: each G row segment
// (64 B, the tile's 8 columns) is staged through shared memory and stored coalesced.
#include <cuda_runtime.h>

#include "radar_kernels.cuh"
#include "warp_fft.cuh"

namespace ofdmr {

namespace {

constexpr int kN = 2048, kNP = 4096;
constexpr int kC = 8;              // columns per tile (= warps)
constexpr int kT = 32 * kC;
constexpr int kVS = 2116;          // column pitch (float2): >= pidx(2047) + 1, = 4 mod 8 (LS stores 2-way)
constexpr int kScr = 1056;         // transpose scratch inside the column region (after the low half)
constexpr int kSP = 9;             // staging pitch per G row segment (float2): conflict-free warp writes
constexpr int kRows = 64;          // rows per ring stage (256 threads x 16 B = 64 rows x 64 B)
constexpr int kStages = kN / kRows;
constexpr int kRing = 8;           // ring depth (lives in the staging area during the LS phase)

struct __align__(16) C2Smem {
    float2 cols[kC * kVS];         // h tile, column-major; later E, H'[q] and the transpose scratch
    float2 stage[1024 * kSP];      // G staging [p][column]; the cp.async ring during the LS phase
    float2 tw[1024];               // tw[t1 * 32 + j] = W_1024^{j t1}
    double red[kC];
};
static_assert(kRing * 2 * kT * 16 <= (int)sizeof(float2) * 1024 * kSP, "ring must fit the staging area");

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// LS cell with the fused kernels' arithmetic (fused_ce.cu pass A): rcp.approx (1 ulp) instead of
// an IEEE division, 1/|x|^2 summed in fp32 over a short run; |x|^2 outside the fp32 normal range
// (zero, denormal or huge x) takes the exact fp64 cell of radar_kernels.cuh
__device__ __forceinline__ float2 ls_cell_fast(float yr, float yi, float xr, float xi, float& inv_run, double& inv_acc,
                                               int& zero_cell) {
    const float n = fmaf(xr, xr, xi * xi);
    if (__builtin_expect(n >= 1.17549435e-38f && n <= 3.40282347e38f, 1)) {
        float i;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(i) : "f"(n));
        inv_run += i;
        return make_float2(fmaf(yr, xr, yi * xi) * i, fmaf(yi, xr, -yr * xi) * i);
    }
    return ls_cell_fp64(yr, yi, xr, xi, inv_acc, zero_cell);
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kC; ++i) s += red[i];  // every thread, same order
    return s;
}

#ifdef OFDMR_PHASE_TIMING
__device__ unsigned long long g_c2_phase[8];
#define C2P_INIT() long long _ph_t = clock64();
#define C2P(i)                                                          \
    do {                                                                \
        if (tid == 0) {                                                 \
            const long long _n = clock64();                             \
            atomicAdd(&g_c2_phase[i], (unsigned long long)(_n - _ph_t)); \
            _ph_t = _n;                                                 \
        }                                                               \
    } while (0)
#else
#define C2P_INIT()
#define C2P(i)
#endif

__global__ void __launch_bounds__(kT, 1) colpass2048_kernel(ColArgs a, int frames) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C2Smem& s = *reinterpret_cast<C2Smem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int m = a.m;
    const int ntile = m / kC;
    const int items = frames * ntile;
    const int per = a.ntiles / ntile;  // partial slots per tile (the context's tiling is finer)
    const bool ls = a.y != nullptr;
    const bool ce = a.ce_taps > 0;
    const int L = a.ce_taps;
    const float2* __restrict__ tw4 = a.tw;  // e^{-j 2 pi t / 4096}

    for (int i = tid; i < 1024; i += kT) s.tw[i] = tw4[(4 * (i & 31) * (i >> 5)) & 4095];
    float4* ring = reinterpret_cast<float4*>(s.stage);  // [kRing][2][kT]
    float2* col = s.cols + w * kVS;
    float2* scr = col + kScr;
    const int q4 = tid & 3, r0 = tid >> 2;  // LS: column pair, row within a stage

    C2P_INIT();
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int f = it / ntile, tile = it - f * ntile, c0 = tile * kC;
        const size_t fbase = (size_t)f * kN * m;

        // ---- 1. LS into the column-major tile (cols[c][pidx(k)])
        const float2* src0 = (ls ? a.y : a.h) + fbase + (size_t)r0 * m + c0 + 2 * q4;
        const float2* src1 = ls ? a.x + fbase + (size_t)r0 * m + c0 + 2 * q4 : nullptr;
        auto issue = [&](int st) {
            if (st < kStages) {
                const size_t off = (size_t)st * kRows * m;
                float4* slot = ring + (st % kRing) * 2 * kT;
                cp_async16(slot + tid, src0 + off);
                if (ls) cp_async16(slot + kT + tid, src1 + off);
            }
            cp_async_commit();
        };
#pragma unroll
        for (int st = 0; st < kRing - 1; ++st) issue(st);
        double inv_acc = 0.0;
        float inv_run = 0.f;
        int zero_cell = 0;
#pragma unroll 8
        for (int st = 0; st < kStages; ++st) {
            issue(st + kRing - 1);
            cp_async_wait<kRing - 1>();
            const float4* slot = ring + (st % kRing) * 2 * kT;
            const float4 y4 = slot[tid];
            float2 h0, h1;
            if (ls) {
                const float4 x4 = slot[kT + tid];
                h0 = ls_cell_fast(y4.x, y4.y, x4.x, x4.y, inv_run, inv_acc, zero_cell);
                h1 = ls_cell_fast(y4.z, y4.w, x4.z, x4.w, inv_run, inv_acc, zero_cell);
                if ((st & 7) == 7) {  // 16 terms in fp32, then fp64
                    inv_acc += (double)inv_run;
                    inv_run = 0.f;
                }
            } else {
                h0 = make_float2(y4.x, y4.y);
                h1 = make_float2(y4.z, y4.w);
            }
            const int k = st * kRows + r0;
            const int pk = k + (k >> 5);
            s.cols[(2 * q4) * kVS + pk] = h0;
            s.cols[(2 * q4 + 1) * kVS + pk] = h1;
        }
        cp_async_wait<0>();
        if (ls) {
            if (zero_cell) atomicOr(a.status + f, 1);
            if (a.inv_partial != nullptr) {
                const double sum = block_sum(inv_acc, s.red);
                if (tid < per) a.inv_partial[(size_t)f * a.ntiles + tile * per + tid] = tid == 0 ? sum : 0.0;
            }
        }
        __syncthreads();  // tile complete; the ring (staging area) is free
        C2P(0);

        // the next item's rows into L2 while this one computes
        {
            const int nit = it + gridDim.x;
            if (nit < items) {
                const int nf = nit / ntile, nc0 = (nit - nf * ntile) * kC;
                const float2* p0 = (ls ? a.y : a.h) + (size_t)nf * kN * m + nc0;
#pragma unroll
                for (int j = 0; j < kN / kT; ++j) {
                    const size_t off = (size_t)(tid + kT * j) * m;
                    prefetch_l2(p0 + off);
                    if (ls) prefetch_l2(a.x + (size_t)nf * kN * m + nc0 + off);
                }
            }
        }

        // ---- 2./3. per column: [DFT-CE] and the window -> H'[q] parked in the own slots, H'[q + 1024] in registers
        const float wl = a.wl != nullptr ? a.wl[c0 + w] : 1.0f;
        float2 hreg[32];
        if (ce) {
            float2 v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int k = lane + 32 * i;
                const float2 lo = col[k + i];              // pidx(k)
                const float2 hi = col[k + 1056 + i];       // pidx(k + 1024)
                v[i] = cadd(lo, hi);
                float2 wv = __ldg(tw4 + 2 * k);             // W_2048^k
                wv.y = -wv.y;
                col[k + i] = cmul(csub(lo, hi), wv);       // b[k], own slot
            }
            warp_fft1024<true, 32, false, 4>(v, scr, s.tw);  // lane t1: x[2 (t1 + 32 t2)], t2 < 4
            float2 te[4];
#pragma unroll
            for (int t2 = 0; t2 < 4; ++t2) te[t2] = v[t2];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = col[lane + 33 * i];
            warp_fft1024<true, 32, false, 4>(v, scr, s.tw);  // lane t1: x[2 (t1 + 32 t2) + 1]
            constexpr float inv_n = 1.0f / (float)kN;
            float2 e[32], o[32];
#pragma unroll
            for (int t2 = 0; t2 < 4; ++t2) {
                const int u = lane + 32 * t2;
                e[t2] = 2 * u < L ? cscale(te[t2], inv_n) : make_float2(0.f, 0.f);
                o[t2] = 2 * u + 1 < L ? cscale(v[t2], inv_n) : make_float2(0.f, 0.f);
            }
            warp_fft1024<false, 4>(e, scr, s.tw);  // E[q], q = lane + 32 i
#pragma unroll
            for (int i = 0; i < 32; ++i) col[lane + 33 * i] = e[i];
            warp_fft1024<false, 4>(o, scr, s.tw);  // O[q]
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int q = lane + 32 * i;
                const float2 t = cmul(o[i], __ldg(tw4 + 2 * q));  // W_2048^q O
                const float2 eq = col[lane + 33 * i];
                float2 h0 = cadd(eq, t), h1 = csub(eq, t);
                if (a.wk != nullptr) {
                    h0 = cscale(h0, __ldg(a.wk + q) * wl);
                    h1 = cscale(h1, __ldg(a.wk + q + 1024) * wl);
                }
                col[lane + 33 * i] = h0;
                hreg[i] = h1;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int q = lane + 32 * i;
                float2 h0 = col[q + i], h1 = col[q + 1056 + i];
                if (a.wk != nullptr) {
                    h0 = cscale(h0, __ldg(a.wk + q) * wl);
                    h1 = cscale(h1, __ldg(a.wk + q + 1024) * wl);
                }
                col[q + i] = h0;
                hreg[i] = h1;
            }
        }

        C2P(1);
        // ---- 4. IFFT_4096 as four IFFT_1024 (s = 0..3) -> G rows 4p + s, staged per 64-B segment
        float2* g = a.g_out + (size_t)f * a.g_rows * m + c0;
#pragma unroll 1
        for (int sx = 0; sx < 4; ++sx) {
            float2 v[32];
            const float jc = sx == 0 ? 1.f : sx == 2 ? -1.f : 0.f, js = sx == 1 ? 1.f : sx == 3 ? -1.f : 0.f;  // j^s
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int q = lane + 32 * i;
                float2 y = cfma_cs(jc, js, hreg[i], col[lane + 33 * i]);  // H'[q] + j^s H'[q + 1024]
                if (sx) {
                    float2 wv = __ldg(tw4 + sx * q);  // W_4096^{sq}, conjugated: inverse
                    wv.y = -wv.y;
                    y = cmul(y, wv);
                }
                v[i] = y;
            }
            warp_fft1024<true, 32>(v, scr, s.tw);  // lane t1: X[4 (t1 + 32 t2) + sx]
            C2P(2);
            __syncthreads();                       // staging free (previous segment stored)
#pragma unroll
            for (int t2 = 0; t2 < 32; ++t2) s.stage[(lane + 32 * t2) * kSP + w] = v[t2];
            __syncthreads();
#pragma unroll 4
            for (int rr = 0; rr < 16; ++rr) {
                const int idx = tid + kT * rr;  // 1024 rows x 4 quarters of 16 B
                const int p = idx >> 2, qq = idx & 3;
                const float2 v0 = s.stage[p * kSP + 2 * qq], v1 = s.stage[p * kSP + 2 * qq + 1];
                *reinterpret_cast<float4*>(g + (size_t)(4 * p + sx) * m + 2 * qq) = make_float4(v0.x, v0.y, v1.x, v1.y);
            }
            C2P(3);
        }
        __syncthreads();  // staging and tile free for the next item
    }
}

}  // namespace

// cfg2's column pass: N = 2048, N' = 4096, DFT-CE with L <= 256 (or plain LS / H input), G out,
// no H output requested
}  // namespace ofdmr
extern "C" int ofdmr_debug_c2_phase_cycles(unsigned long long* out, int reset) {
#ifdef OFDMR_PHASE_TIMING
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, ofdmr::g_c2_phase, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(ofdmr::g_c2_phase, z, sizeof(z));
    }
    return 8;
#else
    (void)out;
    (void)reset;
    return 0;
#endif
}
namespace ofdmr {

bool colpass2048_applies(const ColArgs& a, int n, int np) {
    return n == kN && np == kNP && a.tw_n == nullptr && a.g_out != nullptr && a.h_out == nullptr && !a.shortcut &&
           a.ce_taps >= 0 && a.ce_taps <= 256 && a.m % kC == 0 && a.g_rows == kNP && a.m >= kC &&
           (a.y != nullptr || a.h != nullptr) && (a.y == nullptr || a.x != nullptr) &&
           (a.inv_partial == nullptr || a.ntiles % (a.m / kC) == 0) && (a.wk == nullptr) == (a.wl == nullptr);
}

cudaError_t launch_colpass2048(const ColArgs& a, int frames, cudaStream_t st) {
    const size_t smem = sizeof(C2Smem);
    cudaError_t e = cudaFuncSetAttribute(colpass2048_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int items = frames * (a.m / kC);
    const int grid = items < sms ? items : sms;
    colpass2048_kernel<<<grid, kT, smem, st>>>(a, frames);
    return cudaGetLastError();
}

}  // namespace ofdmr
