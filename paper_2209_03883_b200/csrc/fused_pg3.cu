// Batched 2-D periodogram for N = N' = 1024, M = M' = 256 (H in, P out), split-radix-32
// exchange:   P[n][(m + M/2) mod M] = |FFT_M( IFFT_N( H .* w_k w_l ) )|^2 / (N M)
// (periodogram.cpp:39-75; the map ofdmr_periodogram returns).
//
// The delay transform is factored 1024 = 32 x 32 ACROSS the exchange instead of inside one
// warp:  with k = j + 32 i and n = m + 32 q,
//     X[m + 32 q][l] = sum_j W_32^{-q j} [ W_1024^{-m j} sum_i x[j + 32 i][l] W_32^{-m i} ]
// so the column side only does the inner DFT_32 over i and the twiddle (lane j already
// holds C[j][m] for every m: no shared-memory transpose), and the row side does the outer
// DFT_32 over j together with the Doppler FFT_256 (a 32 x 256 2-D transform per m).
// Compared with fused_pg2 (whole IFFT_1024 on the column warps) this moves half of the
// column side's arithmetic and both of its transposes to the row warps, which ncu shows
// idle ~40 % of the time waiting for complete frames (profiles/r02_*).
//
//   column warps 0-3   tile = 1024 subcarriers x 4 symbols of H (one TMA box, 32-B swizzle,
//                      kHBuf tiles in flight).  Lane j: x[j + 32 i] (w_k), DFT_32 over i,
//                      times conj W_1024^{m j}; C[j][m] for symbol l goes to the group's G
//                      buffer at [m][l][j ^ (l & 31)] (256-B coalesced stores; the XOR makes
//                      the row side's per-l reads conflict-free).
//   row warps 4-11     per frame kMPerCta = 4 m-blocks per CTA; an m-block is the 64 KiB
//                      contiguous [l][j] slab of G: ONE bulk copy (cp.async.bulk) per block,
//                      double-buffered.  Lane l (256 lanes): DFT_32 over j -> X[m + 32 q][l];
//                      transpose in place to rows q; each 16-lane group then runs FFT_256 on
//                      a row (w_l, register twiddles, in-place XOR transpose) and streams
//                      |.|^2 / (N M) with the Doppler fftshift to P row n = m + 32 q.
//
// Group synchronisation is fused_pg2's: per G buffer, col_cnt counts CTAs that finished
// writing a frame, row_cnt CTAs whose row producer finished loading out of it; G is
// double-buffered per 8-CTA group (18 groups x 2 x 2 MiB = 72 MiB, L2-resident, lines
// discarded once loaded).  Cooperative launch: all CTAs co-resident.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "fused_args.cuh"
#include "radar_kernels.cuh"
#include "warp_fft.cuh"

namespace ofdmr {

namespace {

constexpr int kN = 1024, kM = 256;
#ifdef PG3_NOMATH
constexpr bool PG3_MATH_ON = false;  // diagnostic: data movement and synchronisation only (wrong maps)
#else
constexpr bool PG3_MATH_ON = true;
#endif
// PG3_TMA_STORE: the column side stages each tile's C values in the H tile buffer it just
// consumed and writes them to G with ONE TMA tensor store per tile (instead of 32 STG.64 per
// column warp); the freed LSU queue and the smem of the dropped twiddle table (column twiddles
// then come through the read-only cache) pay for a third H tile buffer.
#ifndef PG3_TMA_STORE
#define PG3_TMA_STORE 0
#endif
// P stores: 0 = 16 scalar streaming stores per row-lane, 1 = same with .cg, 2 = staged through the
// row's smem slot and written as 16-B vectors (4 per row-lane)
#ifndef PG3_PSTORE
#define PG3_PSTORE 0
#endif
#ifndef PG3_ROWPIPE
#define PG3_ROWPIPE 1  // 1: the two FFT_256 rows of a row-warp round interleaved (more ILP, fewer warp syncs)
#endif
#ifndef PG3_HBUF
#define PG3_HBUF (PG3_TMA_STORE ? 3 : 2)
#endif
// column twiddles through the read-only cache instead of a shared-memory table (frees 8 KiB:
// needed for a third H tile buffer)
#define PG3_TWG (PG3_TMA_STORE || PG3_HBUF > 2)
constexpr int kGrp = 8;                      // CTAs per frame group
constexpr int kTC = 4;                       // symbols per column tile = column warps
constexpr int kHBuf = PG3_HBUF;              // H tiles in flight
constexpr int kTpf = kM / (kTC * kGrp);      // column tiles per CTA per frame (8)
constexpr int kMPerCta = 32 / kGrp;          // m-blocks per CTA per frame (4)
constexpr int kColWarps = kTC, kRowWarps = 8;
constexpr int kThreads = 32 * (kColWarps + kRowWarps);
constexpr int kCntStride = 32;
constexpr int kGBuf = 2;                     // G buffers per group
constexpr unsigned kTileBytes = kTC * kN * 8u;       // 32 KiB
constexpr unsigned kBlockElems = 32 * kM;            // one m-block: [256 l][32 j]
constexpr unsigned kBlockBytes = kBlockElems * 8u;   // 64 KiB

struct __align__(1024) Pg3Smem {
    float2 htile[kHBuf][kN * kTC];   // [k][4 symbols], 32-B swizzle (1024-B aligned)
    float2 gbuf[2][kBlockElems];     // m-block slab [l][j ^ (l & 31)], then rows [q][l]
#if !PG3_TWG
    float2 tw[1024];                 // tw[m * 32 + j] = W_1024^{j m}
#endif
    unsigned long long mbar_h[kHBuf];
    unsigned long long mbar_g[2];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar, unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// contiguous global -> shared bulk copy (no tensor map), completion on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                          unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
#if PG3_TMA_STORE || PG3_PSTORE == 3
// shared -> global TMA tensor store of a staged tile (bulk-group completion)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<unsigned long long>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
#endif
__device__ __forceinline__ void bar_col() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kColWarps) : "memory"); }
__device__ __forceinline__ void bar_row() { asm volatile("bar.sync 2, %0;" ::"n"(32 * kRowWarps) : "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace

#ifdef OFDMR_PHASE_TIMING
__device__ unsigned long long g_pg3_phase[8];
#define P3_INIT() long long _ph_t = clock64();
#define P3(i)                                                            \
    do {                                                                 \
        if (lane == 0 && ridx == 0) {                                    \
            const long long _n = clock64();                              \
            atomicAdd(&g_pg3_phase[i], (unsigned long long)(_n - _ph_t)); \
            _ph_t = _n;                                                  \
        }                                                                \
    } while (0)
#else
#define P3_INIT()
#define P3(i)
#endif

template <bool HAMMING>
__global__ void __launch_bounds__(kThreads, 1)
    fused_pg3_kernel(Pg2Args a, const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap gmap) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-B alignment as an offset from the __shared__ symbol (keeps LDS/STS addressing)
    const unsigned s_pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    Pg3Smem& s = *reinterpret_cast<Pg3Smem*>(smem_raw + s_pad);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool is_col = warp < kColWarps;
    const int ridx = is_col ? warp : warp - kColWarps;
    const int g = blockIdx.x / kGrp, rank = blockIdx.x % kGrp, ng = gridDim.x / kGrp;
#if !PG3_TWG
    for (int i = tid; i < 1024; i += kThreads) s.tw[i] = a.tw1024_t[i];
#endif
#if !PG3_TMA_STORE
    (void)gmap;
#endif
    if (tid == 0) {
        for (int b = 0; b < kHBuf; ++b) mbar_init(&s.mbar_h[b], 1);
        mbar_init(&s.mbar_g[0], 1);
        mbar_init(&s.mbar_g[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nfr = a.frames > g ? (a.frames - g + ng - 1) / ng : 0;  // frames g, g + ng, ..
    int* col_cnt = a.counters + (size_t)g * 2 * kGBuf * kCntStride;
    int* row_cnt = col_cnt + kGBuf * kCntStride;
    P3_INIT();

    if (is_col) {
        // ------------------------------------------------------------ column warps
        const int cw = ridx;
        const bool cw0 = cw == 0 && lane == 0;
        const int ntiles = kTpf * nfr;
        auto issue_tile = [&](int tn) {
            const int b = tn % kHBuf;
            mbar_expect_tx(&s.mbar_h[b], kTileBytes);
#ifdef PG3_H_SAME  // diagnostic: every tile from frame g (H stays in L2)
            tma_load_3d(s.htile[b], &hmap, kTC * (kGrp * (tn % kTpf) + rank), 0, 4 * g, &s.mbar_h[b],
                        policy_evict_first());
#else
            tma_load_3d(s.htile[b], &hmap, kTC * (kGrp * (tn % kTpf) + rank), 0, 4 * (g + (tn / kTpf) * ng), &s.mbar_h[b],
                        policy_evict_first());
#endif
        };
        if (cw0)
            for (int tn = 0; tn < kHBuf && tn < ntiles; ++tn) issue_tile(tn);
        // 32-B swizzled tile (k = lane + 32 r, symbol cw): float2 4k + 2((cw/2) ^ ((k/4)&1)) + (cw&1)
        const int hoff = 4 * lane + 2 * ((cw >> 1) ^ ((lane >> 2) & 1)) + (cw & 1);
        float wkr[HAMMING ? 32 : 1];
#pragma unroll
        for (int r = 0; r < (HAMMING ? 32 : 1); ++r) wkr[r] = HAMMING ? a.wk[lane + 32 * r] : 1.f;
        // conj W_1024^{lane m} (the inverse transform's twiddles): registers for the rectangular
        // window, shared memory when the 32 window registers are needed
        constexpr bool kTwReg = !HAMMING;
        float2 twc[kTwReg ? 32 : 1];
        if constexpr (kTwReg) {
#pragma unroll
            for (int m = 0; m < 32; ++m) {
#if PG3_TWG
                const float2 w = __ldg(a.tw1024_t + m * 32 + lane);
#else
                const float2 w = s.tw[m * 32 + lane];
#endif
                twc[m] = make_float2(w.x, -w.y);
            }
        }
        for (int t = 0; t < ntiles; ++t) {
            const int i = t / kTpf, u = t % kTpf;
            const int c = kTC * (kGrp * u + rank) + cw;  // symbol l of this warp
            mbar_wait(&s.mbar_h[t % kHBuf], (t / kHBuf) & 1);
            P3(0);
            float2 v[32];
#pragma unroll
            for (int r = 0; r < 32; ++r) v[r] = s.htile[t % kHBuf][hoff + 32 * kTC * r];
            bar_col();  // every column is in registers: the tile buffer is free
            if (cw0) {
#if !PG3_TMA_STORE
                if (t + kHBuf < ntiles) issue_tile(t + kHBuf);
#endif
                if (t >= kTpf && u == 0) {
#if PG3_TMA_STORE
                    bulk_wait_all();  // frame i - 1's tensor stores performed
                    asm volatile("fence.proxy.async.global;" ::: "memory");
#endif
                    __threadfence();
                    atomicAdd(col_cnt + ((i - 1) % kGBuf) * kCntStride, 1);  // G of frame i - 1 complete
                }
            }
            if (HAMMING) {
#pragma unroll
                for (int r = 0; r < 32; ++r) v[r] = cscale(v[r], wkr[r]);
            }
#ifndef PG3_NOMATH
            dft32<true>(v);  // v[m] = sum_i x[lane + 32 i] W_32^{-m i}
#endif
#pragma unroll
            for (int m = 1; m < (PG3_MATH_ON ? 32 : 1); ++m) {
                float2 w;
                if constexpr (kTwReg) {
                    w = twc[m];
                } else {
#if PG3_TWG
                    w = __ldg(a.tw1024_t + m * 32 + lane);
#else
                    w = s.tw[m * 32 + lane];
#endif
                    w.y = -w.y;
                }
                v[m] = cmul(v[m], w);
            }
            P3(1);
            if (u == 0 && i >= kGBuf) {
                // G buffer i % kGBuf last held frame i - kGBuf: wait until every CTA of the group loaded it
                if (lane == 0)
                    while (ld_acquire(row_cnt + (i % kGBuf) * kCntStride) < kGrp * (i / kGBuf)) __nanosleep(32);
                __syncwarp();
            }
            P3(2);
#if PG3_TMA_STORE
            {
                // stage C[lane][m] at [m][cw][lane ^ (c & 31)] in the consumed H buffer, then one TMA
                // store of the [32 m][4 c][32 j] box to G[m][c][j] (rows verbatim: the XOR stays)
                float2* stg = s.htile[t % kHBuf];
#pragma unroll
                for (int m = 0; m < 32; ++m) stg[(m * kTC + cw) * 32 + (lane ^ (c & 31))] = v[m];
                bar_col();
                if (cw0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    tma_store_3d(&gmap, stg, 0, kTC * (kGrp * u + rank), (kGBuf * g + i % kGBuf) * 32);
                    bulk_wait_read_all();  // the staged tile has been read: the buffer takes the next H tile
                    if (t + kHBuf < ntiles) issue_tile(t + kHBuf);
                }
            }
#else
            // C[lane][m] -> G[m][c][lane ^ (c & 31)]: one 256-B line pair per m (a 16-B pair variant
            // with lane shuffles measured slower: 973 k vs 1.0 M frames/s)
            float2* gcol = a.gscratch + (size_t)(kGBuf * g + i % kGBuf) * kN * kM + (size_t)c * 32 + (lane ^ (c & 31));
#pragma unroll
            for (int m = 0; m < 32; ++m) __stcg(gcol + (size_t)m * kBlockElems, v[m]);
#endif
            P3(3);
        }
        bar_col();
        if (ntiles > 0 && cw0) {
#if PG3_TMA_STORE
            bulk_wait_all();
            asm volatile("fence.proxy.async.global;" ::: "memory");
#endif
            __threadfence();
            atomicAdd(col_cnt + ((nfr - 1) % kGBuf) * kCntStride, 1);  // last frame
        }
    } else {
        // ------------------------------------------------------------ row warps
        const int wr = ridx;
        const int l = 32 * wr + lane;  // DFT_32 stage: this lane's symbol
        // FFT_256 stage: lane -> (row h of the warp's pair, sub-lane j) as in fused_pg2
        const int h = (lane >> 3) & 1, j = (lane & 7) | ((lane >> 4) << 3);
        const int hx = 8 * h;
        const bool producer = wr == 0 && lane == 0;
        const int nrounds = kMPerCta * nfr;  // round R: frame g + (R / 4) ng, m = 4 rank + R % 4
        int issued = 0;
        auto try_issue = [&](bool block) {
            const int R = issued, i = R / kMPerCta, q = R % kMPerCta;
            if (q == 0) {
                const int* cc = col_cnt + (i % kGBuf) * kCntStride;
                const int need = kGrp * (i / kGBuf + 1);
                if (block) {
                    while (ld_acquire(cc) < need) __nanosleep(32);
                } else if (ld_acquire(cc) < need) {
                    return;
                }
                asm volatile("fence.proxy.async.global;" ::: "memory");  // peers' generic G stores -> bulk reads
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic transposes -> bulk overwrite
            mbar_expect_tx(&s.mbar_g[R & 1], kBlockBytes);
            const float2* src = a.gscratch + (size_t)(kGBuf * g + i % kGBuf) * kN * kM +
                                (size_t)(kMPerCta * rank + q) * kBlockElems;
            bulk_load(s.gbuf[R & 1], src, kBlockBytes, &s.mbar_g[R & 1], policy_evict_first());
            ++issued;
        };
        float2 twr[16];
#pragma unroll
        for (int t1 = 0; t1 < 16; ++t1) twr[t1] = a.tw256_t[t1 * 16 + j];
        float wlr[HAMMING ? 16 : 1];
#pragma unroll
        for (int r = 0; r < (HAMMING ? 16 : 1); ++r) wlr[r] = HAMMING ? a.wl[j + 16 * r] : 1.f;
        if (producer && nrounds > 0) try_issue(true);
        for (int R = 0; R < nrounds; ++R) {
            const int i = R / kMPerCta, q4 = R % kMPerCta;
            const int m = kMPerCta * rank + q4;
            if (producer && issued == R + 1 && R + 1 < nrounds) try_issue(false);  // look-ahead
            P3(4);
            mbar_wait(&s.mbar_g[R & 1], (R >> 1) & 1);
            P3(5);
            if (wr == 0) {
                // the 512 lines of this m-block are dead: drop them from L2 without write-back
                const float2* gl = a.gscratch + (size_t)(kGBuf * g + i % kGBuf) * kN * kM + (size_t)m * kBlockElems;
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(gl + 16 * (lane + 32 * k)) : "memory");
                if (q4 == kMPerCta - 1) {
                    // every m-block of frame i landed: release the G buffer (discards ordered first)
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) atomicAdd(row_cnt + (i % kGBuf) * kCntStride, 1);
                }
            }
            float2* gb = s.gbuf[R & 1];
            // DFT_32 over j for symbol l: element j of row l sits at l*32 + (j ^ lane)
            float2 v[32];
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) v[jj] = gb[l * 32 + (jj ^ lane)];
#ifndef PG3_NOMATH
            dft32<true>(v);  // v[q] = X[m + 32 q][l]
#endif
            bar_row();       // every slab element is in registers
#pragma unroll
            // rows q: [q][l ^ 8 (q & 1)] (odd rows shifted by half a bank row: the two rows a
            // warp reads below then hit disjoint banks)
            for (int q = 0; q < 32; ++q) gb[q * kM + (l ^ (8 * (q & 1)))] = v[q];
            bar_row();
            P3(6);
#if PG3_ROWPIPE
            {
                // FFT_256 over l for rows q = 2 wr + h and 16 + 2 wr + h, the two rows' chains interleaved
                float2* sl0 = gb + (2 * wr + h) * kM;
                float2* sl1 = gb + (16 + 2 * wr + h) * kM;
                float2 xa[16], xb[16];
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    xa[r] = sl0[(j ^ hx) + 16 * r];
                    xb[r] = sl1[(j ^ hx) + 16 * r];
                    if (HAMMING) {
                        xa[r] = cscale(xa[r], wlr[r]);
                        xb[r] = cscale(xb[r], wlr[r]);
                    }
                }
                dft16<false>(xa);
                dft16<false>(xb);
#pragma unroll
                for (int t1 = 1; t1 < 16; ++t1) {
                    xa[t1] = cmul(xa[t1], twr[t1]);
                    xb[t1] = cmul(xb[t1], twr[t1]);
                }
                __syncwarp();
#pragma unroll
                for (int t1 = 0; t1 < 16; ++t1) {
                    sl0[t1 * 16 + (j ^ t1 ^ hx)] = xa[t1];
                    sl1[t1 * 16 + (j ^ t1 ^ hx)] = xb[t1];
                }
                __syncwarp();
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    xa[jj] = sl0[j * 16 + (jj ^ j ^ hx)];
                    xb[jj] = sl1[j * 16 + (jj ^ j ^ hx)];
                }
                dft16<false>(xa);
                dft16<false>(xb);
                float* prow0 = a.p + ((size_t)(g + i * ng) * kN + m + 32 * (2 * wr + h)) * kM;
                float* prow1 = prow0 + (size_t)32 * 16 * kM;
#pragma unroll
                for (int t2 = 0; t2 < 16; ++t2) __stcs(prow0 + ((j + 16 * t2 + 128) & 255), cnorm(xa[t2]) * a.scale);
#pragma unroll
                for (int t2 = 0; t2 < 16; ++t2) __stcs(prow1 + ((j + 16 * t2 + 128) & 255), cnorm(xb[t2]) * a.scale);
            }
#else
            // FFT_256 over l for rows q = 16 p + 2 wr + h
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const int q = 16 * p + 2 * wr + h;
                float2* sl = gb + q * kM;
                float2 x[16];
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    x[r] = sl[(j ^ hx) + 16 * r];
                    if (HAMMING) x[r] = cscale(x[r], wlr[r]);
                }
#ifndef PG3_NOMATH
                dft16<false>(x);
#pragma unroll
                for (int t1 = 1; t1 < 16; ++t1) x[t1] = cmul(x[t1], twr[t1]);
#endif
                __syncwarp();
#pragma unroll
                for (int t1 = 0; t1 < 16; ++t1) sl[t1 * 16 + (j ^ t1 ^ hx)] = x[t1];
                __syncwarp();
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) x[jj] = sl[j * 16 + (jj ^ j ^ hx)];
#ifndef PG3_NOMATH
                dft16<false>(x);
#endif
                const int n = m + 32 * q;
#ifdef PG3_P_SAME  // diagnostic: every frame's map written over frame g's (P stays in L2)
                float* prow = a.p + ((size_t)g * kN + n) * kM;
#else
                float* prow = a.p + ((size_t)(g + i * ng) * kN + n) * kM;
#endif
#if defined(PG3_NO_P)
                if (cnorm(x[0]) == 12345.f) prow[j] = 0.f;  // diagnostic: no P traffic
#elif PG3_PSTORE == 3
                {
                    // |X|^2 / (N M), fftshifted, into this row's free slot (h = 1 rows 64 B in: the two
                    // rows of a warp on disjoint banks), then ONE bulk copy of the 1 KiB row to P by the
                    // half-warp's first lane; the copies' smem reads are waited for before the slot is
                    // refilled (end of the round)
                    float* pf = reinterpret_cast<float*>(sl) + 16 * h;
                    __syncwarp();
#pragma unroll
                    for (int t2 = 0; t2 < 16; ++t2) pf[(j + 16 * t2 + 128) & 255] = cnorm(x[t2]) * a.scale;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (j == 0) {
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1024;" ::"l"(prow),
                                     "r"(smem_u32(pf))
                                     : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                }
#elif PG3_PSTORE == 2
                {
                    // |X|^2 / (N M) with the Doppler fftshift into this row's (now free) slot as fp32
                    // (h = 1 rows XOR 16 words: the two rows of a warp on disjoint banks), then the
                    // half-warp streams the 1 KiB row as 16-B vectors: 4 STG.128 per lane
                    float* pf = reinterpret_cast<float*>(sl);
                    __syncwarp();
#pragma unroll
                    for (int t2 = 0; t2 < 16; ++t2) pf[((j + 16 * t2 + 128) & 255) ^ (16 * h)] = cnorm(x[t2]) * a.scale;
                    __syncwarp();
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int f4 = j + 16 * r;  // float4 index within the row
                        const float4 val = reinterpret_cast<const float4*>(pf)[f4 ^ (4 * h)];
                        __stcs(reinterpret_cast<float4*>(prow) + f4, val);
                    }
                }
#elif PG3_PSTORE == 1
#pragma unroll
                for (int t2 = 0; t2 < 16; ++t2) __stcg(prow + ((j + 16 * t2 + 128) & 255), cnorm(x[t2]) * a.scale);
#else
#pragma unroll
                for (int t2 = 0; t2 < 16; ++t2) __stcs(prow + ((j + 16 * t2 + 128) & 255), cnorm(x[t2]) * a.scale);
#endif
            }
#endif
#if PG3_PSTORE == 3
            if (j == 0) bulk_wait_read_all();  // this lane's P row copies have read their slots
#endif
            bar_row();  // transposes done: the buffer may be refilled
            P3(7);
            if (producer && issued == R + 1 && R + 1 < nrounds) try_issue(true);
        }
    }
}

}  // namespace ofdmr

extern "C" int ofdmr_debug_pg3_phase_cycles(unsigned long long* out, int reset) {
#ifdef OFDMR_PHASE_TIMING
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, ofdmr::g_pg3_phase, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(ofdmr::g_pg3_phase, z, sizeof(z));
    }
    return 8;
#else
    (void)out;
    (void)reset;
    return 0;
#endif
}

namespace ofdmr {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn3() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

}  // namespace

size_t fused_pg3_smem() { return sizeof(Pg3Smem) + 1024; }
size_t fused_pg3_counter_ints(int groups) { return (size_t)groups * 2 * kGBuf * kCntStride; }
size_t fused_pg3_scratch_elems(int groups) { return (size_t)groups * kGBuf * kN * kM; }

int fused_pg3_max_groups() {
    const size_t smem = fused_pg3_smem();
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!encode_fn3()) return 0;
    if (cudaFuncSetAttribute(fused_pg3_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_pg3_kernel<false>, kThreads, smem) !=
        cudaSuccess)
        return 0;
    return per_sm * sms / kGrp;
}

cudaError_t launch_fused_pg3(const Pg2Args& a, bool hamming, int groups, int scratch_groups, cudaStream_t st) {
    auto enc = encode_fn3();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap hmap, gmap;
    // G store view: [group x buffer x 32 m][256 c][32 j] f64; box = 32 j x 4 c x 32 m (32 KiB)
    {
        const cuuint64_t dims[3] = {32, 256, 32ull * kGBuf * (cuuint64_t)scratch_groups};
        const cuuint64_t strides[2] = {32 * 8, 256 * 32 * 8};
        const cuuint32_t box[3] = {32, (cuuint32_t)kTC, 32};
        const cuuint32_t es[3] = {1, 1, 1};
        if (enc(&gmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a.gscratch, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    // H: [frames][1024 k][256 l] c64 as a 3-D f64 tensor (l, k mod 256, 4 frame + k / 256);
    // box = 4 symbols x all 1024 subcarriers, 32-B swizzle
    {
        const cuuint64_t dims[3] = {256, 256, 4ull * (cuuint64_t)a.frames};
        const cuuint64_t strides[2] = {256 * 8, 256 * 256 * 8};
        const cuuint32_t box[3] = {(cuuint32_t)kTC, 256, 4};
        const cuuint32_t es[3] = {1, 1, 1};
        if (enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<float2*>(a.h), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    const size_t smem = fused_pg3_smem();
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        Pg2Args aa = a;
        void* args[] = {&aa, &hmap, &gmap};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(groups * kGrp), dim3(kThreads),
                                           args, smem, st);
    };
    return hamming ? go(fused_pg3_kernel<true>) : go(fused_pg3_kernel<false>);
}

}  // namespace ofdmr
