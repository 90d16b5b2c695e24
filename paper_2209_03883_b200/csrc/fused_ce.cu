// Persistent fused receiver kernel for the DFT-CE pipeline at N = N' = 1024, M = M' = 256,
// L <= 128 (cfg1 / cfg4): one CTA owns one frame at a time, all three passes in-CTA, no
// cross-CTA synchronisation, one launch per batch.
//
//   pass A  (32 column tiles of 8 symbols, one warp per column): tile load fuses LS
//           division (estimation.cpp:10-21), the zero-cell check and sum 1/|x|^2
//           (pipeline.cpp:18-23); warp IFFT_1024; keep the first L taps x 1/N (DFT-CE,
//           estimation.cpp:23-39) -> D (L x M c64, per-CTA scratch, L2-resident).
//   pass B  row FFT_256 of the L tap rows with the symbol window w_l (periodogram.cpp:52-57)
//           -> D' in place.  Linear k-axis and l-axis operators commute, so doing the
//           l-axis transform on the L-row compressed form is exact and 8x cheaper than on
//           all N' rows.
//   pass C  per column tile: input-pruned FFT_1024 of the L taps (back to subcarriers),
//           x w_k, delay IFFT_1024 (periodogram.cpp:60), |.|^2/(NM) (:63-73) into a rolling
//           window of P columns in shared memory; strict wrapped 3x3 local maxima >= eta
//           (:77-136) over columns whose neighbours are resident; running per-frame top-K.
//           With a rectangular window the k-chain is the identity up to N (exact shortcut).
//
// Memory per frame: 4 MiB of HBM reads (Y, x_tx), 1 MiB of L2 traffic (D, D'), ~100 B out.
#include <cooperative_groups.h>

#include "radar_kernels.cuh"
#include "warp_fft.cuh"
#include "fused_args.cuh"

namespace ofdmr {

#ifndef PF_AHEAD
#define PF_AHEAD 0  // L2 prefetch distance of pass-A tiles
#endif
#ifndef TW_GLOBAL
#define TW_GLOBAL 0  // 1: FFT1024 twiddles read through L1 from global (frees 8 KB of smem)
#endif
#ifndef RING
#define RING 4
#endif
constexpr int kRing = RING;  // pass-A cp.async staging ring depth (stages of 64 rows x 8 symbols)

#ifdef OFDMR_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[16];
#define PH_INIT() long long _ph_t = clock64();
#define PH(i)                                                              \
    do {                                                                   \
        if (threadIdx.x == 0) {                                            \
            const long long _n = clock64();                                \
            atomicAdd(&g_phase_cycles[i], (unsigned long long)(_n - _ph_t)); \
            _ph_t = _n;                                                    \
        }                                                                  \
    } while (0)
#else
#define PH_INIT()
#define PH(i)
#endif



namespace {

constexpr int kM = 256;
constexpr int kN = 1024;
constexpr int kVS = 1058;         // padded column buffer (>= pad_len(1024); 2 mod 8 -> conflict-free tile writes)
constexpr int kTileList = 1024;   // per-CTA frame candidate list (exact fallback beyond)

struct FusedSmem {
#if !TW_GLOBAL
    float2 tw[1024];
#endif
    float2 tw256[256];
    float2 cols[8 * kVS];         // per-warp column buffers / pass-A,C tiles / pass-B scratch
    float4 stg[kRing][2][256];    // pass-A staging ring: thread-private 16-B slots of Y and x_tx
    unsigned long long prun[kMaxK];    // partner CTA's top-K (rank 0 merge)
    unsigned long long run[kMaxK];     // per-CTA top-K (descending, 0-padded)
    unsigned long long cand2[kMaxK];
    unsigned long long sbest[8];
    int sidx[8];
    unsigned short clist[8][64];       // per-column candidate rows of the current step
    int ccnt[8];
    double red[8];
    int tcnt;
    int pcnt;                          // pending edge candidates of the frame (global scratch)
    int zc_part;
    int overflow;
    int zcs[2];
    double part;
    double etas[2];
    double s2hs[2];
};

// Strict wrapped 3x3 maximum test on P columns a, b, c (b tested) at row r.

// Warp 0: merge the tile list (cnt keys) into the running top-K (K keys, sorted desc).
__device__ void warp_merge_topk(unsigned long long* run, unsigned long long* tl, int cnt, int K,
                                unsigned long long* tmp) {
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < K; ++r) {
        unsigned long long best = 0;
        int where = -1;  // >= 0: tl index; < 0: -(run index) - 2
        for (int i = lane; i < cnt; i += 32)
            if (tl[i] > best) { best = tl[i]; where = i; }
        for (int i = lane; i < K; i += 32)
            if (run[i] > best) { best = run[i]; where = -i - 2; }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int ow = __shfl_xor_sync(0xffffffffu, where, o);
            if (ob > best) { best = ob; where = ow; }
        }
        if (lane == 0) {
            tmp[r] = best;
            if (best != 0) {
                if (where >= 0) tl[where] = 0;
                else run[-where - 2] = 0;
            }
        }
        __syncwarp();
    }
    for (int i = lane; i < K; i += 32) run[i] = tmp[i];
    __syncwarp();
}

}  // namespace

// Pull the 128-B lines of one 8-column tile (1024 rows of Y and x_tx) into L2 so the next
// tile's loads hit L2 while this tile computes (the pair covers both 64-B halves of a line).
#ifndef CE_EVICT_FIRST
#define CE_EVICT_FIRST 1  // 1: the streamed Y / x_tx lines are marked evict-first in L2 (the D / D' scratch stays)
#endif
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16_pol(void* smem, const void* gmem, unsigned long long pol) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "l"(pol) : "memory");
}
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void prefetch_tile(const float2* y, const float2* x, size_t fbase, int c0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const size_t off = fbase + (size_t)(threadIdx.x + 256 * j) * kM + c0;
#ifdef CE_PF_NORMAL
        asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(y + off));
        asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(x + off));
#else
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(y + off));
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(x + off));
#endif
    }
}

// Smallest float t with (double)v >= eta  <=>  v >= t for every float v (exact fp32 test).
__device__ __forceinline__ float eta_float(double eta) {
    float e = (float)eta;
    if ((double)e < eta) e = nextafterf(e, INFINITY);
    return e;
}

template <bool HAMMING>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2) fused_ce1024_kernel(FusedArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FusedSmem& s = *reinterpret_cast<FusedSmem*>(smem_raw);
    const int rank = (int)cluster.block_rank();             // 0 or 1: which 8-column half of each 16
    FusedSmem& p = *cluster.map_shared_rank(&s, rank ^ 1);  // partner CTA's shared memory (DSMEM)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int L = a.L;
    const int K = a.kmax;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const float* pbase = reinterpret_cast<const float*>(s.cols);
    auto lcol = [&](int c) -> const float* { return pbase + c * (2 * kVS); };
    auto dbuf = [&](int parity) { return a.dscratch + ((size_t)cid * 2 + parity) * 128 * kM; };

#if TW_GLOBAL
    const float2* twp = a.tw1024_t;
#else
    for (int i = tid; i < 1024; i += 256) s.tw[i] = a.tw1024_t[i];
    const float2* twp = s.tw;
#endif
    s.tw256[tid] = a.tw256_t[tid];
    if (tid == 0) s.overflow = 0;
    __syncthreads();
    PH_INIT();

    // pass-A input stream: cp.async ring over this CTA's linear sequence of tiles
    // (frame cid tiles 0..15, frame cid + ncl tiles 0..15, ...); stage = 64 rows x 8 symbols
    // of Y and x_tx; one commit group per stage; each thread only reads its own slots
    int ifr = cid, iu = 0, ist = 0, islot = 0, cslot = 0;
    const size_t lane_off = (size_t)(tid >> 2) * kM + 8 * rank + (tid & 3) * 2;
    size_t ioff = (size_t)cid * kN * kM + lane_off;
#if CE_EVICT_FIRST
    unsigned long long pol_stream;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
#endif
    auto a_issue = [&]() {
        if (ifr < a.frames) {
#if CE_EVICT_FIRST
            cp_async16_pol(&s.stg[islot][0][tid], a.y + ioff, pol_stream);
            cp_async16_pol(&s.stg[islot][1][tid], a.x + ioff, pol_stream);
#else
            cp_async16(&s.stg[islot][0][tid], a.y + ioff);
            cp_async16(&s.stg[islot][1][tid], a.x + ioff);
#endif
        }
        cp_async_commit();
        islot = islot + 1 == kRing ? 0 : islot + 1;
        ioff += (size_t)64 * kM;
        if (++ist == 16) {
            ist = 0;
            if (++iu == 16) {
                iu = 0;
                ifr += ncl;
            }
            ioff = (size_t)ifr * kN * kM + 16 * iu + lane_off;
        }
    };
    for (int st = 0; st < kRing; ++st) a_issue();

    // ---------------------------------------------------------------- pass A, one tile
    // column tile u (8 symbols) of frame f: LS divide -> IFFT_N -> L taps x 1/N -> D
    // dC: pass-C D' of the step's C tile, loaded into dpre right after the FFT so the
    // L2 latency overlaps the tap store
    auto A_tile = [&](int f, int u, float2* dsc, double& inv_acc, int& zero_cell, const float2* dC, float4 (&dpre)[2]) {
        const int c0 = 16 * u + 8 * rank;
        float inv_tile = 0.f, nmax = 0.f;
#pragma unroll 4
        for (int st = 0; st < 16; ++st) {
            // stage st of this tile landed in ring slot (this thread's own 16-B slots)
            cp_async_wait<kRing - 1>();
            const float4 y4 = s.stg[cslot][0][tid];
            const float4 x4 = s.stg[cslot][1][tid];
            cslot = cslot + 1 == kRing ? 0 : cslot + 1;
            const int idx = tid + st * 256;
            const int k = idx >> 2, c = (idx & 3) * 2;
            const float n0 = fmaf(x4.x, x4.x, x4.y * x4.y);
            const float n1 = fmaf(x4.z, x4.z, x4.w * x4.w);
            // a zero / denormal (flushed) |x|^2 gives rcp = +inf and an overflowing one +inf in
            // nmax: caught once per tile below
            const float i0 = rcp_approx(n0);
            const float i1 = rcp_approx(n1);
            inv_tile += i0 + i1;
            nmax = fmaxf(nmax, fmaxf(n0, n1));
            const int pk = k + (k >> 5);
            const float2 r0 = make_float2(fmaf(y4.x, x4.x, y4.y * x4.y) * i0, fmaf(y4.y, x4.x, -y4.x * x4.y) * i0);
            const float2 r1 = make_float2(fmaf(y4.z, x4.z, y4.w * x4.w) * i1, fmaf(y4.w, x4.z, -y4.z * x4.w) * i1);
            s.cols[c * kVS + pk] = r0;
            s.cols[(c + 1) * kVS + pk] = r1;
            // refill the slot (its values were consumed above) with the stage kRing ahead
            a_issue();
        }
        // |x|^2 outside the fp32 normal range somewhere in the tile (an exactly zero x cell,
        // estimation.cpp:17, or a denormal / huge one the reference divides in fp64): the frame is
        // flagged for the exact general path (status bit 1), which decides the zero-cell error
        zero_cell |= !(inv_tile <= 3.40282347e38f) || !(nmax <= 3.40282347e38f);
        inv_acc += (double)inv_tile;  // fp32 within a tile (32 terms), fp64 across tiles
        __syncthreads();
        PH(0);
        // stream the next tile into L2 while this one computes (one step ahead)
        // stream tile PF_AHEAD steps ahead into L2 while this one computes
        if (PF_AHEAD > 0) {
            int pu = u + PF_AHEAD, pf = f;
            if (pu >= 16) {
                pu -= 16;
                pf += ncl;
            }
            if (pf < a.frames) prefetch_tile(a.y, a.x, (size_t)pf * kN * kM, 16 * pu + 8 * rank);
        }
        {
            float2* col = s.cols + w * kVS;
            float2 v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = col[lane + 33 * i];
            warp_fft1024<true, 32, TW_GLOBAL, 4>(v, col, twp);  // lane t1: taps t1 + 32 t2, t2 < 4
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int idx = tid + j * 256;
                const int k = idx >> 2;
                dpre[j] = dC && k < L ? __ldcg(reinterpret_cast<const float4*>(dC + (size_t)k * kM + c0 + (idx & 3) * 2))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            __syncwarp();
            constexpr float inv_n = 1.0f / 1024.0f;
#pragma unroll
            for (int t2 = 0; t2 < 4; ++t2) {
                const int tap = lane + 32 * t2;
                col[lane + 33 * t2] = tap < L ? cscale(v[t2], inv_n) : make_float2(0.f, 0.f);
            }
        }
        __syncthreads();
        PH(1);
        for (int idx = tid; idx < L * 4; idx += 256) {
            const int k = idx >> 2, c = (idx & 3) * 2;
            const int pk = k + (k >> 5);
            const float2 v0 = s.cols[c * kVS + pk];
            const float2 v1 = s.cols[(c + 1) * kVS + pk];
            __stcg(reinterpret_cast<float4*>(dsc + (size_t)k * kM + c0 + c), make_float4(v0.x, v0.y, v1.x, v1.y));
        }
        __syncthreads();
        PH(2);
    };

    // ---------------------------------------------------------------- end of pass A
    // combine the pair's sum 1/|x|^2 -> sigma_h^2, eta (slot = frame parity); D complete
    auto A_finish = [&](int f, int slot, double inv_acc, int zero_cell) {
        double v = inv_acc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const int zc = __any_sync(0xffffffffu, zero_cell);
        if (lane == 0) s.red[w] = v;
        if (tid == 0) s.zc_part = 0;
        __syncthreads();
        if (lane == 0 && zc) atomicOr(&s.zc_part, 1);
        if (tid == 0) {
            double acc = 0.0;
            for (int i = 0; i < 8; ++i) acc += s.red[i];
            s.part = acc;
        }
        __threadfence();
        cluster.sync();  // D complete in global (both halves); partials visible
        if (tid == 0) {
            const double p0 = rank == 0 ? s.part : p.part;
            const double p1 = rank == 0 ? p.part : s.part;
            const double acc = p0 + p1;  // same order in both CTAs
            const double sg = a.sigma2[f];
            const double s2h = sg <= 0.0 ? 0.0 : sg * acc * a.inv_count;
            s.zcs[slot] = s.zc_part | p.zc_part;
            s.etas[slot] = -s2h * a.log_pfa * a.power_factor;
            s.s2hs[slot] = s2h;
        }
        // (no second barrier: the partner's part / zc_part are next written in the next
        // frame's A_finish, behind the B-pass and C_finish cluster barriers)
        PH(3);
    };

    // ---------------------------------------------------------------- pass B
    auto B_pass = [&](float2* dsc) {
        const int hw = tid >> 4, j = tid & 15;
        float2* tb = s.cols + hw * (16 * 17);
        const int rlo = rank * (L / 2), rhi = rank == 0 ? L / 2 : L;
        for (int r0 = rlo; r0 < rhi; r0 += 16) {
            const int r = r0 + hw;
            const bool valid = r < rhi;
            float2 v[16];
            const float2* src = dsc + (size_t)(valid ? r : rlo) * kM;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                float2 uu = valid ? __ldcg(src + j + 16 * i) : make_float2(0.f, 0.f);
                if (HAMMING) uu = cscale(uu, __ldg(a.wl + j + 16 * i));
                v[i] = uu;
            }
            halfwarp_fft256<false>(v, tb, s.tw256);
            if (valid) {
                float2* dst = dsc + (size_t)r * kM;
#pragma unroll
                for (int t2 = 0; t2 < 16; ++t2) __stcg(dst + j + 16 * t2, v[t2]);
            }
        }
        __syncthreads();
        __threadfence();
        cluster.sync();  // D' complete
        PH(4);
    };

    // ---------------------------------------------------------------- pass C, one step
    // Pass C, one step.  Columns 1..6 of the tile are tested locally; the tile's edge
    // columns 0 and 7 are pre-tested against their own side here and finished at the end of
    // the frame against the partner's stored edge columns, so no cluster barrier is needed
    // inside the step loop.
    // per CTA: 16 steps x 2 edge columns; a column's region holds either a sparse list of its
    // cells >= eta ((row << 32) | value bits, at most 64) or, when there are more, the whole column
    // (1024 floats); the per-column counts follow the regions
    float* my_edges = a.edges + ((size_t)cid * 2 + rank) * kFusedEdgeStride;
    const float* partner_edges = a.edges + ((size_t)cid * 2 + (rank ^ 1)) * kFusedEdgeStride;
    int* my_ecnt = reinterpret_cast<int*>(my_edges + 16 * 2 * kN);
    const int* partner_ecnt = reinterpret_cast<const int*>(partner_edges + 16 * 2 * kN);
    unsigned long long* my_pend = a.pend + ((size_t)cid * 2 + rank) * kFusedPend;
    int* my_ploc = a.pend_loc + ((size_t)cid * 2 + rank) * kFusedPend;
    unsigned long long* tl = a.tlist + (size_t)blockIdx.x * kTileList;  // frame candidates (L2)
    auto C_tile = [&](int u, const float2* dsc, float ef, bool pre, const float4 (&dpre)[2]) {
        const int c0 = 16 * u + 8 * rank;
        if (tid < 8) s.ccnt[tid] = 0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int idx = tid + j * 256;
            const int k = idx >> 2, c = (idx & 3) * 2;
            float4 v4 = dpre[j];
            if (!pre)
                v4 = k < L ? __ldcg(reinterpret_cast<const float4*>(dsc + (size_t)k * kM + c0 + c))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            const int pk = k + (k >> 5);
            s.cols[c * kVS + pk] = make_float2(v4.x, v4.y);
            s.cols[(c + 1) * kVS + pk] = make_float2(v4.z, v4.w);
        }
        __syncthreads();
        PH(5);
        {
            float2* col = s.cols + w * kVS;
            float* pcol = reinterpret_cast<float*>(col);
            float2 v[32];
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = col[lane + 33 * i];
            if constexpr (HAMMING) {
                warp_fft1024<false, 4, TW_GLOBAL>(v, col, twp);
#pragma unroll
                for (int t2 = 0; t2 < 32; ++t2) v[t2] = cscale(v[t2], __ldg(a.wk + lane + 32 * t2));
                warp_fft1024<true, 32, TW_GLOBAL>(v, col, twp);
                __syncwarp();
#pragma unroll
                for (int t2 = 0; t2 < 32; ++t2) {
                    const float pv = cnorm(v[t2]);  // a.wk carries sqrt(scale)
                    pcol[lane + 32 * t2] = pv;
                    if (pv >= ef) {  // rare: ~1 % of cells
                        const int pos = atomicAdd(&s.ccnt[w], 1);
                        if (pos < 64) s.clist[w][pos] = (unsigned short)(lane + 32 * t2);
                    }
                }
            } else {
                __syncwarp();
#pragma unroll
                for (int t2 = 0; t2 < 32; ++t2) {
                    float pv = 0.f;
                    if (t2 < 4) pv = cnorm(cscale(v[t2], 2.0f));  // |1024 v|^2 * 2^-18, exact
                    pcol[lane + 32 * t2] = pv;
                    if (pv >= ef) {
                        const int pos = atomicAdd(&s.ccnt[w], 1);
                        if (pos < 64) s.clist[w][pos] = (unsigned short)(lane + 32 * t2);
                    }
                }
            }
        }
        __syncthreads();
        PH(6);
        {
            // warp w tests tile column w: interior columns completely, edge columns (0, 7)
            // against their own-side neighbours only (-> pending, finished at frame end)
            const float* pb = reinterpret_cast<const float*>(s.cols);
            const int jdx = w;
            const float* B = pb + jdx * (2 * kVS);
            const float* A = jdx > 0 ? pb + (jdx - 1) * (2 * kVS) : nullptr;
            const float* Cc = jdx < 7 ? pb + (jdx + 1) * (2 * kVS) : nullptr;
            const int sn = c0 + jdx;
            const int sc = (sn + kM / 2) & (kM - 1);
            const int cnt = s.ccnt[jdx];
            const int lim = cnt > 64 ? kN : cnt;  // overflowed list: scan every row
            for (int i = lane; i < lim; i += 32) {
                const int r = cnt > 64 ? i : (int)s.clist[jdx][i];
                const float vv = B[r];
                if (!(vv >= ef)) continue;
                const int ru = (r - 1) & (kN - 1), rd = (r + 1) & (kN - 1);
                if (B[ru] >= vv || B[rd] >= vv) continue;
                if (A && (A[ru] >= vv || A[r] >= vv || A[rd] >= vv)) continue;
                if (Cc && (Cc[ru] >= vv || Cc[r] >= vv || Cc[rd] >= vv)) continue;
                const unsigned long long key = make_key(vv, (uint32_t)(r * kM + sc));
                if (A && Cc) {
                    const int slot = atomicAdd(&s.tcnt, 1);
                    if (slot < kTileList) tl[slot] = key;
                } else {
                    // partner edge column holding the missing neighbour: (partner step, edge)
                    int pu, pe;
                    if (rank == 0) {
                        if (jdx == 0) { pu = (u + 15) & 15; pe = 1; }   // 16u-1: partner step u-1, col 7
                        else { pu = u; pe = 0; }                        // 16u+8: partner step u, col 0
                    } else {
                        if (jdx == 0) { pu = u; pe = 1; }               // 16u+7: partner step u, col 7
                        else { pu = (u + 1) & 15; pe = 0; }             // 16u+16: partner step u+1, col 0
                    }
                    const int slot = atomicAdd(&s.pcnt, 1);
                    if (slot < kFusedPend) {
                        my_pend[slot] = key;
                        my_ploc[slot] = pu * 2 + pe;
                    }
                }
            }
        }
        // this step's edge columns for the partner's end-of-frame tests: only cells >= eta can
        // beat a pending candidate, so the column goes out as its (short) candidate list
        if (w == 0 || w == 7) {
            const int e = w == 7;
            const float* B = reinterpret_cast<const float*>(s.cols) + w * (2 * kVS);
            const int cnt = s.ccnt[w];
            float* reg = my_edges + ((size_t)u * 2 + e) * kN;
            if (cnt <= 64) {
                for (int i = lane; i < cnt; i += 32) {
                    const unsigned r = s.clist[w][i];
                    __stcg(reinterpret_cast<unsigned long long*>(reg) + i,
                           ((unsigned long long)r << 32) | (unsigned long long)__float_as_uint(B[r]));
                }
            } else {
                for (int i = lane; i < kN / 4; i += 32)
                    __stcg(reinterpret_cast<float4*>(reg) + i, *reinterpret_cast<const float4*>(B + 4 * i));
            }
            if (lane == 0) __stcg(my_ecnt + u * 2 + e, cnt);
        }
        __syncthreads();
        PH(8);
    };

    // ---------------------------------------------------------------- end of pass C
    auto C_finish = [&](int f, int slot, float ef) {
        (void)ef;
        __threadfence();
        cluster.sync();  // both CTAs' edge columns and pending lists are in global memory
        PH(9);
        const int np = min(s.pcnt, kFusedPend);
        for (int i = tid; i < np; i += 256) {
            const unsigned long long key = __ldcg(my_pend + i);
            const int loc = __ldcg(my_ploc + i);
            const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
            const int r = (int)(idx >> 8);
            const float vv = __uint_as_float((uint32_t)(key >> 32));
            const float* col = partner_edges + (size_t)loc * kN;
            const int ru = (r - 1) & (kN - 1), rd = (r + 1) & (kN - 1);
            const int pc = __ldcg(partner_ecnt + loc);
            if (pc <= 64) {
                bool beaten = false;
                const unsigned long long* pl = reinterpret_cast<const unsigned long long*>(col);
                for (int q = 0; q < pc; ++q) {
                    const unsigned long long e = __ldcg(pl + q);
                    const int pr = (int)(e >> 32);
                    beaten |= (pr == ru || pr == r || pr == rd) && __uint_as_float((uint32_t)e) >= vv;
                }
                if (beaten) continue;
            } else {
                const float n0 = __ldcg(col + ru), n1 = __ldcg(col + r), n2 = __ldcg(col + rd);
                if (n0 >= vv || n1 >= vv || n2 >= vv) continue;
            }
            const int sl = atomicAdd(&s.tcnt, 1);
            if (sl < kTileList) tl[sl] = key;
        }
        __syncthreads();
        // per-CTA top-K of the frame's candidates (> kTileList / kFusedPend candidates in one
        // half-frame sets status bit 1 so the host recomputes the frame on the general path)
        if (tid == 0 && (s.tcnt > kTileList || s.pcnt > kFusedPend)) s.overflow = 1;
        block_topk_reg<256, kTileList / 256>(tl, min(s.tcnt, kTileList), K, s.run, s.sbest);
        __syncthreads();
        cluster.sync();  // both per-CTA lists final
        if (rank == 0) {
            if (w == 0) {
                for (int i = lane; i < K; i += 32) s.prun[i] = p.run[i];
                __syncwarp();
                warp_merge_topk(s.run, s.prun, K, K, s.cand2);
            }
            __syncthreads();
            const int kf = a.k_per_frame ? min(a.k_per_frame[f], K) : K;
            if (tid < K) {
                const unsigned long long key = tid < kf ? s.run[tid] : 0ull;
                const size_t o = (size_t)f * K + tid;
                if (key == 0) {
                    a.det_delay[o] = 0;
                    a.det_doppler[o] = 0;
                    a.det_power[o] = 0.f;
                } else {
                    const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
                    a.det_delay[o] = (int32_t)(idx >> 8);
                    a.det_doppler[o] = (int32_t)(idx & 255) - 128;
                    a.det_power[o] = __uint_as_float((uint32_t)(key >> 32));
                }
            }
            if (tid == 0) {
                int n = 0;
                for (int i = 0; i < kf; ++i) n += s.run[i] != 0;
                a.counts[f] = n;
                if (a.s2h_out) a.s2h_out[f] = s.s2hs[slot];
                if (a.status && s.zcs[slot]) atomicOr(a.status + f, 2);  // abnormal |x|^2: exact recompute
                if (a.status && (s.overflow || p.overflow)) atomicOr(a.status + f, 2);
            }
        }
        // (no barrier here: rank 1's run / overflow are next modified at the next round
        // start, behind the next A_finish cluster barrier; the kernel ends with one)
        PH(10);
    };

    // ---------------------------------------------------------------- schedule
    // prologue: pass A + B of the first frame; then each round interleaves pass A of frame
    // i+1 (HBM streaming) with pass C of frame i (issue-bound) tile by tile.
    if (cid < a.frames) {
        double inv_acc = 0.0;
        int zc = 0;
        float4 dpre[2];
        for (int u = 0; u < 16; ++u) A_tile(cid, u, dbuf(0), inv_acc, zc, nullptr, dpre);
        A_finish(cid, 0, inv_acc, zc);
        B_pass(dbuf(0));
    }
    int it = 0;
    for (int fC = cid; fC < a.frames; fC += ncl, ++it) {
        const int fN = fC + ncl;
        const bool hasN = fN < a.frames;
        const int sc = it & 1, sn = sc ^ 1;
        if (tid == 0) {
            s.tcnt = 0;
            s.pcnt = 0;
            s.overflow = 0;
        }
        for (int i = tid; i < K; i += 256) s.run[i] = 0ull;
        const float ef = eta_float(s.etas[sc]);
        __syncthreads();
        double inv_acc = 0.0;
        int zc = 0;
        for (int u = 0; u < 16; ++u) {
            float4 dpre[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
            if (hasN) A_tile(fN, u, dbuf(sn), inv_acc, zc, dbuf(sc), dpre);
            C_tile(u, dbuf(sc), ef, hasN, dpre);
        }
        C_finish(fC, sc, ef);
        if (hasN) {
            A_finish(fN, sn, inv_acc, zc);
            B_pass(dbuf(sn));
        }
    }
    cluster.sync();  // no CTA leaves while its partner may still read its shared memory
}

size_t fused_ce_smem() { return sizeof(FusedSmem); }

}  // namespace ofdmr

extern "C" int ofdmr_debug_phase_cycles(unsigned long long* out, int reset) {
#ifdef OFDMR_PHASE_TIMING
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, ofdmr::g_phase_cycles, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(ofdmr::g_phase_cycles, z, sizeof(z));
    }
    return 16;
#else
    (void)out;
    (void)reset;
    return 0;
#endif
}

namespace ofdmr {

cudaError_t launch_fused_ce(const FusedArgs& a, bool hamming, int grid, cudaStream_t st) {
    const size_t smem = sizeof(FusedSmem);
    grid &= ~1;  // whole clusters
    if (grid < 2) grid = 2;
    if (hamming) {
        cudaError_t e = cudaFuncSetAttribute(fused_ce1024_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        fused_ce1024_kernel<true><<<grid, 256, smem, st>>>(a);
    } else {
        cudaError_t e = cudaFuncSetAttribute(fused_ce1024_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        fused_ce1024_kernel<false><<<grid, 256, smem, st>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace ofdmr
