// Warp-specialised, TMA-fed persistent batched 2-D periodogram for N = N' = 1024,
// M = M' = 256 (H in, P out):
//   P[n][(m + M/2) mod M] = |FFT_M( IFFT_N( H .* w_k w_l ) )|^2 / (N M)
// (periodogram.cpp:39-75; the map ofdmr_periodogram returns).
//
// Design driver: at this shape the kernel is bound by FP32 issue and by the SM's L1tex/LSU
// data pipe, which serves every shared-memory wavefront AND every 128-B line a global LSU
// instruction touches.  So the bulk data movement that would gather (H tiles, the G row
// blocks) goes through the TMA engine instead, and the shared-memory exchanges are laid out
// conflict-free (profiles/r01_pg2_*.txt).
//
// One CTA per SM (16 warps); frames are handled by groups of kGrp = 8 CTAs; inside a CTA the
// two passes of the 2-D transform run CONCURRENTLY on different warps:
//
//   column warps 0-7   tile = 1024 subcarriers x 8 symbols of H, ONE TMA box (64-B swizzled
//                      rows; at step u the CTAs of a group read 8 kGrp symbols contiguous of
//                      each subcarrier row).  Each warp reads its symbol column (constant
//                      per-lane offsets thanks to the swizzle); as soon as all 8 columns are
//                      in registers the next tile's TMA is issued.  Window w_k w_l, register-
//                      resident IFFT_1024 (32 x 32; transpose through a private padded slot),
//                      then the column of G goes to the group's L2 scratch column-major, in
//                      the storage order pos = 64 b + 2 t1 + p for delay n = t1 + 32 (2b + p),
//                      so each lane stores 16-B pairs (16 x 512 B per column).
//   row warps 8-15     per frame 1024 / kGrp delay rows per CTA in rounds of 16: ONE TMA box
//                      (16 storage rows x 256 symbols, 128-B swizzled) per round, double-
//                      buffered; each 16-lane group takes one row (lane mapping chosen so each
//                      64-bit shared-memory phase hits 16 distinct bank pairs), FFT_256 with
//                      register twiddles and its 16 x 16 transpose in the round buffer itself
//                      (XOR layout), |.|^2 / (N M) with the Doppler fftshift streamed to P.
//
// Producer/consumer counters per group and G buffer replace frame barriers: the column warps
// of every CTA of the group bump col_cnt[b] after writing their part of a frame into G buffer
// b; each CTA's row producer bumps row_cnt[b] once the last G box of that frame has landed in
// shared memory.  G is double-buffered per group (18 groups x 2 x 2 MiB = 72 MiB, L2-resident;
// 3 or 4 buffers and 16-CTA groups measured slower).  All CTAs of the persistent grid are
// co-resident (1 per SM, 144 of 148 SMs).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "fused_args.cuh"
#include "radar_kernels.cuh"
#include "warp_fft.cuh"

namespace ofdmr {

namespace {

constexpr int kN = 1024, kM = 256;
#ifndef PG2_GRP
#define PG2_GRP 8
#endif
constexpr int kGrp = PG2_GRP;   // CTAs per frame group
#ifndef PG2_TC
#define PG2_TC 4  // symbols per column tile = column warps per CTA (8: 64-B swizzle, 4: 32-B swizzle)
#endif
#ifndef PG2_RW
#define PG2_RW 8  // row warps per CTA; a TMA round is 2 x PG2_RW storage rows
#endif
#ifndef PG2_CPS
#define PG2_CPS 1  // resident CTAs per SM
#endif
#ifndef PG2_HBUF
#define PG2_HBUF 1  // H tile buffers (2: the tile two ahead is in flight while one is consumed)
#endif
constexpr int kTC = PG2_TC;
constexpr int kHBuf = PG2_HBUF;
constexpr int kTpf = 256 / (kTC * kGrp);  // column tiles per CTA per frame
constexpr int kRowsPerCta = kN / kGrp;
constexpr int kVS = 1058;       // padded column-FFT scratch stride (float2)
constexpr int kColWarps = kTC, kRowWarps = PG2_RW;
constexpr int kThreads = 32 * (kColWarps + kRowWarps);
constexpr int kCntStride = 32;  // ints between counters (own 128-B line)
#ifndef PG2_GBUF
#define PG2_GBUF 2
#endif
constexpr int kGBuf = PG2_GBUF;  // G buffers per group (frames in flight between the passes)
#ifndef PG2_RPG
#define PG2_RPG 2  // rows per 16-lane group per round (2: a round is two 16-row halves, 3-D TMA box)
#endif
constexpr int kHalves = PG2_RPG;
static_assert(kHalves == 1 || kRowWarps == 8, "two rows per group needs 8 row warps");
constexpr int kRoundRows = 2 * kRowWarps * kHalves;  // G storage rows per TMA round (8, 16 or 32)
constexpr int kRounds = kN / kGrp / kRoundRows;         // rounds per frame per CTA (4)
constexpr unsigned kTileBytes = kTC * kN * 8u;         // 64 / 32 KiB
constexpr unsigned kRoundBytes = kRoundRows * kM * 8u;  // 32 KiB

struct __align__(1024) Pg2Smem {
    float2 htile[kHBuf][kN * kTC];        // [k][kTC symbols], 64/32-B swizzle   (1024-B aligned)
    float2 gbuf[2][kM * kRoundRows];      // [l][round rows], 128/64-B swizzle   (1024-B aligned)
    float2 cs[kColWarps][kVS];            // column-FFT transpose slots
    float2 tw[1024];                      // tw[t1*32 + j] = W_1024^{j t1}
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
// L2 policy for the TMA loads: H and G are read exactly once (evict first)
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
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar, unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bar_col() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kColWarps) : "memory"); }
__device__ __forceinline__ void bar_row() { asm volatile("bar.sync 2, %0;" ::"n"(32 * kRowWarps) : "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace

#ifdef OFDMR_PHASE_TIMING
__device__ unsigned long long g_pg2_phase[8];
#define P2_INIT() long long _ph_t = clock64();
#define P2(i)                                                            \
    do {                                                                 \
        if (lane == 0 && ridx == 0) {                                    \
            const long long _n = clock64();                              \
            atomicAdd(&g_pg2_phase[i], (unsigned long long)(_n - _ph_t)); \
            _ph_t = _n;                                                  \
        }                                                                \
    } while (0)
#else
#define P2_INIT()
#define P2(i)
#endif

template <bool HAMMING>
__global__ void __launch_bounds__(kThreads, PG2_CPS)
    fused_pg2_kernel(Pg2Args a, const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap gmap) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-B alignment (TMA swizzle atoms) as an offset from the __shared__ symbol: the pointer
    // stays in the shared window, so every access below compiles to LDS/STS (a round trip
    // through uintptr_t would make them 64-bit generic LD.E/ST.E on the LSU's global queue)
    const unsigned s_pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    Pg2Smem& s = *reinterpret_cast<Pg2Smem*>(smem_raw + s_pad);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool is_col = warp < kColWarps;  // (interleaving the roles across schedulers measured slower)
    const int ridx = is_col ? warp : warp - kColWarps;
    const int g = blockIdx.x / kGrp, rank = blockIdx.x % kGrp, ng = gridDim.x / kGrp;
    for (int i = tid; i < 1024; i += kThreads) {
        s.tw[i] = a.tw1024_t[i];
    }
    if (tid == 0) {
        for (int b = 0; b < kHBuf; ++b) mbar_init(&s.mbar_h[b], 1);
        mbar_init(&s.mbar_g[0], 1);
        mbar_init(&s.mbar_g[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nfr = a.frames > g ? (a.frames - g + ng - 1) / ng : 0;  // frames g, g + ng, ..
    // per G buffer b: col_cnt[b] counts CTAs that finished writing a frame into b, row_cnt[b] CTAs
    // whose row producer finished loading one out of it (per-buffer, not cumulative: a CTA
    // running a frame ahead cannot stand in for a slower one)
    int* col_cnt = a.counters + (size_t)g * 2 * kGBuf * kCntStride;
    int* row_cnt = col_cnt + kGBuf * kCntStride;
    P2_INIT();

    // diagnostics: PG2_ROW_ONLY / PG2_COL_ONLY run one role alone (wrong results, rates only)
#ifdef PG2_ROW_ONLY
    if (is_col) return;
#endif
#ifdef PG2_COL_ONLY
    if (!is_col) return;
#endif
    if (is_col) {
        // ------------------------------------------------------------ column warps
        const int cw = ridx;
        const bool cw0 = cw == 0 && lane == 0;
        const int ntiles = kTpf * nfr;  // tile t: frame g + (t / kTpf) ng, symbols kTC (kGrp (t % kTpf) + rank) ..
        auto issue_tile = [&](int tn) {
            const int b = tn % kHBuf;
            mbar_expect_tx(&s.mbar_h[b], kTileBytes);
            tma_load_3d(s.htile[b], &hmap, kTC * (kGrp * (tn % kTpf) + rank), 0, 4 * (g + (tn / kTpf) * ng), &s.mbar_h[b],
                        policy_evict_first());
        };
        if (cw0)
            for (int tn = 0; tn < kHBuf && tn < ntiles; ++tn) issue_tile(tn);
        // swizzled (k = lane + 32 r, symbol `warp`): float2 8k + 2((warp/2) ^ ((k/2)&3)) + (warp&1)
        // kTC = 4 (32-B rows, SW32): 4k + 2((cw/2) ^ ((k/4)&1)) + (cw&1)
        const int hoff = kTC == 8 ? 8 * lane + 2 * ((cw >> 1) ^ ((lane >> 1) & 3)) + (cw & 1)
                                  : 4 * lane + 2 * ((cw >> 1) ^ ((lane >> 2) & 1)) + (cw & 1);
        float2* col = s.cs[cw];
        // registers of the column warps: w_k[lane + 32 r] with the Hamming window; without it the
        // inverse transform's twiddles conj W_1024^{lane t1} instead (31 fewer shared-memory loads
        // per column: +4 %; holding both costs more than it saves, measured)
        constexpr bool kTwReg = !HAMMING;
        float wkr[HAMMING ? 32 : 1];
        float2 twc[kTwReg ? 32 : 1];
#pragma unroll
        for (int r = 0; r < (HAMMING ? 32 : 1); ++r) wkr[r] = HAMMING ? a.wk[lane + 32 * r] : 1.f;
        if constexpr (kTwReg) {
#pragma unroll
            for (int t1 = 0; t1 < 32; ++t1) twc[t1] = make_float2(s.tw[t1 * 32 + lane].x, -s.tw[t1 * 32 + lane].y);
        }
        for (int t = 0; t < ntiles; ++t) {
            const int i = t / kTpf, u = t % kTpf;
            const int c = kTC * (kGrp * u + rank) + cw;
            mbar_wait(&s.mbar_h[t % kHBuf], (t / kHBuf) & 1);
            P2(0);
            float2 v[32];
#pragma unroll
            for (int r = 0; r < 32; ++r) v[r] = s.htile[t % kHBuf][hoff + 32 * kTC * r];
            bar_col();  // every column is in registers: the tile buffer is free
            if (cw0) {
                if (t + kHBuf < ntiles) issue_tile(t + kHBuf);  // into the buffer just read
                if (t >= kTpf && u == 0) {
                    __threadfence();
                    atomicAdd(col_cnt + ((i - 1) % kGBuf) * kCntStride, 1);  // G of frame i - 1 complete
                }
            }
            if constexpr (kTwReg) {  // warp_fft1024 with the twiddles from registers
                dft32<true>(v);
#pragma unroll
                for (int t1 = 1; t1 < 32; ++t1) v[t1] = cmul(v[t1], twc[t1]);
                __syncwarp();
#pragma unroll
                for (int t1 = 0; t1 < 32; ++t1) col[t1 * 33 + lane] = v[t1];
                __syncwarp();
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) v[jj] = col[lane * 33 + jj];
                dft32<true>(v);  // lane t1: G[t1 + 32 t2] in v[t2]
            } else {
                if (HAMMING) {  // w_k here (register copy), w_l on the row side
#pragma unroll
                    for (int r = 0; r < 32; ++r) v[r] = cscale(v[r], wkr[r]);
                }
                warp_fft1024<true, 32>(v, col, s.tw);  // lane t1: G[t1 + 32 t2] in v[t2]
            }
            P2(1);
#ifdef PG2_COL_ONLY
            if (false) {
#else
            if (u == 0 && i >= kGBuf) {
#endif
                // G buffer i % kGBuf last held frame i - kGBuf: wait until every CTA of the group loaded it
                if (lane == 0)
                    while (ld_acquire(row_cnt + (i % kGBuf) * kCntStride) < kGrp * (i / kGBuf)) __nanosleep(32);
                __syncwarp();
            }
            P2(2);
            // G column storage order: position 64 b + 2 t1 + p holds delay n = t1 + 32 (2 b + p), so lane
            // t1 stores its pair (t2 = 2b, 2b + 1) as one 16-B vector (16 stores of 512 B per column)
            float2* gcol = a.gscratch + ((size_t)(kGBuf * g + i % kGBuf) * kM + c) * kN;
#pragma unroll
            for (int b = 0; b < 16; ++b)
                __stcg(reinterpret_cast<float4*>(gcol + 64 * b) + lane,
                       make_float4(v[2 * b].x, v[2 * b].y, v[2 * b + 1].x, v[2 * b + 1].y));
            P2(3);
        }
        bar_col();
        if (ntiles > 0 && cw0) {
            __threadfence();
            atomicAdd(col_cnt + ((nfr - 1) % kGBuf) * kCntStride, 1);  // last frame
        }
    } else {
        // ------------------------------------------------------------ row warps
        // lane -> (row h of the warp's pair, sub-lane j): the 16-lane phases of 64-bit shared
        // accesses then hold 8 lanes of each row, so every phase hits 16 distinct bank pairs
        const int wr = ridx, h = (lane >> 3) & 1, j = (lane & 7) | ((lane >> 4) << 3);
        const int hx = 8 * h;  // XOR of the transpose layout of row h (disjoint bank halves)
        const bool producer = wr == 0 && lane == 0;
        const int nrounds = kRounds * nfr;
        // round R: frame g + (R / kRounds) ng, rows 64 rank + 16 (R % kRounds) .. +15, buffer R & 1
        int issued = 0;  // rounds whose TMA has been issued (producer only)
        auto try_issue = [&](bool block) {
            const int R = issued, i = R / kRounds, q = R % kRounds;
            if (q == 0) {
                const int* cc = col_cnt + (i % kGBuf) * kCntStride;
#ifdef PG2_ROW_ONLY
                const int need = 0;
#else
                const int need = kGrp * (i / kGBuf + 1);
#endif
                if (block) {
                    while (ld_acquire(cc) < need) __nanosleep(32);
                } else if (ld_acquire(cc) < need) {
                    return;
                }
                asm volatile("fence.proxy.async.global;" ::: "memory");  // peers' generic G stores -> TMA reads
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic transposes -> TMA overwrite
            mbar_expect_tx(&s.mbar_g[R & 1], kRoundBytes);
            if (kHalves == 2)
                tma_load_3d(s.gbuf[R & 1], &gmap, 0, (kGBuf * g + i % kGBuf) * kM, (kRowsPerCta * rank + kRoundRows * q) / 16,
                            &s.mbar_g[R & 1], policy_evict_first());
            else
                tma_load_2d(s.gbuf[R & 1], &gmap, kRowsPerCta * rank + kRoundRows * q, (kGBuf * g + i % kGBuf) * kM,
                            &s.mbar_g[R & 1], policy_evict_first());
            ++issued;
        };
        float2 twr[16];
#pragma unroll
        for (int t1 = 0; t1 < 16; ++t1) twr[t1] = a.tw256_t[t1 * 16 + j];
        float wlr[HAMMING ? 16 : 1];  // w_l[j + 16 r]: the symbol window, applied to the rows' inputs
#pragma unroll
        for (int r = 0; r < (HAMMING ? 16 : 1); ++r) wlr[r] = HAMMING ? a.wl[j + 16 * r] : 1.f;
        // swizzled (l = j + 16 r, row 2 wr + h): float2 16 l + 2 (wr ^ (l & 7)) + h
        // kRoundRows = 8 (64-B rows, SW64): 8 l + 2 (wr ^ ((l/2)&3)) + h
        const int goff = kRoundRows >= 16 ? 16 * j + 2 * (wr ^ (j & 7)) + h : 8 * j + 2 * (wr ^ ((j >> 1) & 3)) + h;
        if (producer && nrounds > 0) try_issue(true);
        for (int R = 0; R < nrounds; ++R) {
            const int i = R / kRounds, q = R % kRounds;
            if (producer && issued == R + 1 && R + 1 < nrounds) try_issue(false);  // look-ahead when G is ready
            P2(5);
            mbar_wait(&s.mbar_g[R & 1], (R >> 1) & 1);
#ifndef PG2_NO_DISCARD
            if (wr == 0 && (kRoundRows >= 16 || (q & 1))) {
                // the 256 lines of G (one 128-B line = 16 storage rows per symbol) read so far are dead:
                // drop them from L2 without write-back (G otherwise costs a DRAM write on eviction);
                // with 8-row rounds a line is complete after every second round
                const float2* gl = a.gscratch + (size_t)(kGBuf * g + i % kGBuf) * kM * kN + kRowsPerCta * rank +
                                   16 * (kRoundRows * q / 16);
#pragma unroll
                for (int hh = 0; hh < kHalves; ++hh)
#pragma unroll
                    for (int k = 0; k < kM / 32; ++k)
                        asm volatile("discard.global.L2 [%0], 128;" ::"l"(gl + 16 * hh + (size_t)(lane + 32 * k) * kN)
                                     : "memory");
            }
#endif
            if (wr == 0 && q == kRounds - 1) {
                // every G box of frame i landed: the buffer is reusable.  Every lane fences first, so
                // all of this warp's discards of frame i's lines are ordered before the release (a late
                // discard would otherwise drop a line of frame i + kGBuf already written into it)
                __threadfence();
                __syncwarp();
                if (lane == 0) atomicAdd(row_cnt + (i % kGBuf) * kCntStride, 1);
            }
            float2* gb = s.gbuf[R & 1];
            constexpr int kHalfElems = kHalves == 2 ? 16 * kM : 0;  // [half][l][16 rows] with 2 halves
            constexpr int kLStride = kHalves == 2 ? 16 : kRoundRows;
            float2 v[kHalves][16];
#pragma unroll
            for (int hh = 0; hh < kHalves; ++hh)
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    v[hh][r] = gb[hh * kHalfElems + goff + 16 * kLStride * r];
                    if (HAMMING) v[hh][r] = cscale(v[hh][r], wlr[r]);
                }
            bar_row();  // the round buffer is now transpose scratch
            // 16-lane FFT_256 of each of the group's rows; 16 x 16 transposes in own 2 KiB slots, XOR layout
#pragma unroll
            for (int hh = 0; hh < kHalves; ++hh) {
                dft16<false>(v[hh]);
#pragma unroll
                for (int t1 = 1; t1 < 16; ++t1) v[hh][t1] = cmul(v[hh][t1], twr[t1]);
                float2* sl = gb + (hh * 16 + 2 * wr + h) * 256;
#pragma unroll
                for (int t1 = 0; t1 < 16; ++t1) sl[t1 * 16 + (j ^ t1 ^ hx)] = v[hh][t1];
            }
            __syncwarp();
#pragma unroll
            for (int hh = 0; hh < kHalves; ++hh) {
                float2* sl = gb + (hh * 16 + 2 * wr + h) * 256;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) v[hh][jj] = sl[j * 16 + (jj ^ j ^ hx)];
                dft16<false>(v[hh]);
            }
#pragma unroll
            for (int hh = 0; hh < kHalves; ++hh) {
                // storage position -> delay row n (see the column store): pos = 64 b + 2 t1 + p, n = t1 + 32 (2b + p)
                const int pos = kRowsPerCta * rank + kRoundRows * q + 16 * hh + 2 * wr + h;
                const int n = ((pos & 63) >> 1) + 64 * (pos >> 6) + 32 * (pos & 1);
                float* prow = a.p + ((size_t)(g + i * ng) * kN + n) * kM;
#pragma unroll
                for (int t2 = 0; t2 < 16; ++t2)
                    __stcs(prow + ((j + 16 * t2 + 128) & 255), cnorm(v[hh][t2]) * a.scale);
            }
            P2(6);
            bar_row();  // transposes done: the buffer may be refilled
            if (producer && issued == R + 1 && R + 1 < nrounds) try_issue(true);
        }
    }
}

}  // namespace ofdmr

extern "C" int ofdmr_debug_pg2_phase_cycles(unsigned long long* out, int reset) {
#ifdef OFDMR_PHASE_TIMING
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, ofdmr::g_pg2_phase, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(ofdmr::g_pg2_phase, z, sizeof(z));
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

size_t fused_pg2_smem() { return sizeof(Pg2Smem) + 1024; }
int fused_pg2_group() { return kGrp; }
size_t fused_pg2_counter_ints(int groups) { return (size_t)groups * 2 * kGBuf * kCntStride; }
size_t fused_pg2_scratch_elems(int groups) { return (size_t)groups * kGBuf * kN * kM; }

// Frame groups of the persistent grid: one CTA per SM, kGrp CTAs per group.
int fused_pg2_max_groups() {
    const size_t smem = fused_pg2_smem();
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!encode_fn()) return 0;
    if (cudaFuncSetAttribute(fused_pg2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_pg2_kernel<false>, kThreads, smem) !=
        cudaSuccess)
        return 0;
    return per_sm * sms / kGrp;
}

cudaError_t launch_fused_pg2(const Pg2Args& a, bool hamming, int groups, int scratch_groups, cudaStream_t st) {
    auto enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap hmap, gmap;
    // H: [frames][1024 k][256 l] c64 as a 3-D f64 tensor (l, k mod 256, 4 frame + k / 256);
    // box = 8 symbols x all 1024 subcarriers, 64-B swizzle
    {
        const cuuint64_t dims[3] = {256, 256, 4ull * (cuuint64_t)a.frames};
        const cuuint64_t strides[2] = {256 * 8, 256 * 256 * 8};
        const cuuint32_t box[3] = {(cuuint32_t)kTC, 256, 4};
        const cuuint32_t es[3] = {1, 1, 1};
        if (enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<float2*>(a.h), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, kTC == 8 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    // G scratch: per group kGBuf x [256 l][1024 n] c64 (column-major); box = round rows x 256 symbols
    // (two rows per group: 3-D view (16 rows, l, 16-row block) with a [2][256][16] box)
    if (kHalves == 2) {
        const cuuint64_t dims[3] = {16, 256ull * kGBuf * (cuuint64_t)scratch_groups, 1024 / 16};
        const cuuint64_t strides[2] = {1024 * 8, 16 * 8};
        const cuuint32_t box[3] = {16, 256, 2};
        const cuuint32_t es[3] = {1, 1, 1};
        if (enc(&gmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a.gscratch, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    } else {
        const cuuint64_t dims[2] = {1024, 256ull * kGBuf * (cuuint64_t)scratch_groups};
        const cuuint64_t strides[1] = {1024 * 8};
        const cuuint32_t box[2] = {kRoundRows, 256};
        const cuuint32_t es[2] = {1, 1};
        if (enc(&gmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a.gscratch, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, kRoundRows == 16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    const size_t smem = fused_pg2_smem();
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        // cooperative launch: the frame groups spin on each other's counters, so every CTA of
        // the persistent grid must be co-resident (guaranteed, or the launch fails loudly)
        Pg2Args aa = a;
        void* args[] = {&aa, &hmap, &gmap};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(groups * kGrp), dim3(kThreads),
                                           args, smem, st);
    };
    return hamming ? go(fused_pg2_kernel<true>) : go(fused_pg2_kernel<false>);
}

}  // namespace ofdmr
