// Warp-specialised persistent fused receiver for the DFT-CE pipeline at N = N' = 1024,
// M = M' = 256, L <= 128 (cfg1 / cfg4).  Same math, outputs and pass structure as
// fused_ce.cu (see its header for the reference citations):
//   pass A  LS divide + IFFT_N + keep L taps x 1/N          -> D  (L x M, per-cluster scratch)
//   pass B  w_l + FFT_M on the L tap rows                  -> D'
//   pass C  pruned FFT_N, x w_k, IFFT_N, |.|^2/(NM), strict 3x3 maxima >= eta, top-K
// Execution model (one 2-CTA cluster per frame, one 384-thread CTA per SM):
//   * warps 0-7  (consumers): one OFDM-symbol column each; FFT chains in registers.
//   * warps 8-11 (producers): stream the NEXT pass-A column tile of Y and x_tx from HBM,
//     divide (LS) and write H into the other half of a double-buffered tile, while the
//     consumers transform the current one.  Loads are L2-prefetched one tile ahead.
//   * rounds are software-pipelined: step u of a round does pass A tile u of frame i+1 and
//     pass C tile u of frame i, so every step both streams HBM and computes.
//   * the two CTAs of a cluster take the two 64-B halves of each 128-B row segment; pass C
//     detection exchanges edge P columns through DSMEM.  Producers join the two mid-step
//     cluster barriers with split arrive/wait so their loads overlap the exchange.
#include <cooperative_groups.h>

#include "radar_kernels.cuh"
#include "warp_fft.cuh"
#include "fused_args.cuh"

namespace ofdmr {



namespace {

constexpr int kM = 256;
constexpr int kN = 1024;
constexpr int kVS = 1057;
constexpr int kList = 1024;
constexpr int kCons = 256;   // consumer threads (8 warps)
constexpr int kProd = 128;   // producer threads (4 warps)
constexpr int kThreads = kCons + kProd;

struct WsSmem {
    float2 buf[2][8 * kVS];   // double-buffered column tiles (H in, taps, D' tile, P columns)
    float2 tw[1024];
    float2 tw256[256];
    float keep[2][kN];        // rank 1: previous step's columns 6, 7; rank 0: frame columns 0, 1
    float ext[2][kN];         // partner edge columns staged for detection
    unsigned long long tl[kList];
    unsigned long long run[kMaxK];
    unsigned long long cand2[kMaxK];
    unsigned long long sbest[8];
    int sidx[8];
    double red[4];
    double part;
    double etas[2];
    double s2hs[2];
    int zcs[2];
    int zc_part;
    int tcnt;
    int overflow;
};

__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__device__ __forceinline__ bool strict_max3(const float* a, const float* b, const float* c, int r, float v) {
    const int ru = (r - 1) & (kN - 1), rd = (r + 1) & (kN - 1);
    return !(a[ru] >= v || a[r] >= v || a[rd] >= v || b[ru] >= v || b[rd] >= v || c[ru] >= v || c[r] >= v ||
             c[rd] >= v);
}

__device__ __forceinline__ float eta_float(double eta) {
    float e = (float)eta;
    if ((double)e < eta) e = nextafterf(e, INFINITY);
    return e;
}

__device__ __forceinline__ void prefetch_rows(const float2* y, const float2* x, size_t fbase, int c0, int t) {
    // producer thread t (0..127) prefetches rows t + 128 j of the tile's 128-B segments
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const size_t off = fbase + (size_t)(t + 128 * j) * kM + c0;
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(y + off));
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(x + off));
    }
}

// Consumer-warp merge of cnt keys into the sorted top-K list run (warp-cooperative).
__device__ void warp_merge(unsigned long long* run, unsigned long long* tl, int cnt, int K, unsigned long long* tmp) {
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < K; ++r) {
        unsigned long long best = 0;
        int where = -1;
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

// Consumer-only block top-K (256 threads, named barrier 1).
__device__ void cons_topk(unsigned long long* list, int cnt, int K, unsigned long long* out, unsigned long long* sb,
                          int* si) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int round = 0; round < K; ++round) {
        unsigned long long best = 0;
        int bi = -1;
        for (int i = threadIdx.x; i < cnt; i += kCons)
            if (list[i] > best) { best = list[i]; bi = i; }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best) { best = ob; bi = oi; }
        }
        if (lane == 0) { sb[w] = best; si[w] = bi; }
        cons_sync();
        if (threadIdx.x == 0) {
            unsigned long long b = 0;
            int id = -1;
            for (int i = 0; i < 8; ++i)
                if (sb[i] > b) { b = sb[i]; id = si[i]; }
            out[round] = b;
            if (id >= 0) list[id] = 0;
        }
        cons_sync();
    }
}

}  // namespace

template <bool HAMMING>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) fused_ws_kernel(FusedArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WsSmem& s = *reinterpret_cast<WsSmem*>(smem_raw);
    const int rank = (int)cluster.block_rank();
    WsSmem& p = *cluster.map_shared_rank(&s, rank ^ 1);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const bool producer = w >= 8;
    const int ptid = tid - kCons;  // producer thread index 0..127
    const int L = a.L;
    const int K = a.kmax;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    auto dbuf = [&](int parity) { return a.dscratch + ((size_t)cid * 2 + parity) * 128 * kM; };

    for (int i = tid; i < 1024; i += kThreads) s.tw[i] = a.tw1024_t[i];
    for (int i = tid; i < 256; i += kThreads) s.tw256[i] = a.tw256_t[i];
    if (tid == 0) s.overflow = 0;
    __syncthreads();

    // ------------------------------------------------------------ producer: one A tile
    // Y, x_tx column tile (8 symbols x 1024 subcarriers) -> LS divide -> H into buf[b]
    // producer-private sums of 1/|x|^2 per in-flight frame (parity of the frame's ordinal)
    double p_inv0 = 0.0, p_inv1 = 0.0;
    int p_zero0 = 0, p_zero1 = 0;
    auto produce = [&](int f, int u, int b) {
        const size_t fbase = (size_t)f * kN * kM;
        const int c0 = 16 * u + 8 * rank;
        float2* tile = s.buf[b];
        float inv_tile = 0.f;
        int zt = 0;
#pragma unroll 1
        for (int half = 0; half < 4; ++half) {
            float4 yv[8], xv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = ptid + (half * 8 + q) * kProd;
                const size_t off = fbase + (size_t)(idx >> 2) * kM + c0 + (idx & 3) * 2;
                yv[q] = __ldcs(reinterpret_cast<const float4*>(a.y + off));
                xv[q] = __ldcs(reinterpret_cast<const float4*>(a.x + off));
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = ptid + (half * 8 + q) * kProd;
                const int k = idx >> 2, c = (idx & 3) * 2;
                const float4 y4 = yv[q], x4 = xv[q];
                const float n0 = fmaf(x4.x, x4.x, x4.y * x4.y);
                const float n1 = fmaf(x4.z, x4.z, x4.w * x4.w);
                zt |= (n0 == 0.f) | (n1 == 0.f);
                const float i0 = n0 == 0.f ? 0.f : __frcp_rn(n0);
                const float i1 = n1 == 0.f ? 0.f : __frcp_rn(n1);
                inv_tile += i0 + i1;
                const int pk = k + (k >> 5);
                tile[c * kVS + pk] =
                    make_float2(fmaf(y4.x, x4.x, y4.y * x4.y) * i0, fmaf(y4.y, x4.x, -y4.x * x4.y) * i0);
                tile[(c + 1) * kVS + pk] =
                    make_float2(fmaf(y4.z, x4.z, y4.w * x4.w) * i1, fmaf(y4.w, x4.z, -y4.z * x4.w) * i1);
            }
        }
        if (((f - cid) / ncl) & 1) {
            p_inv1 += (double)inv_tile;
            p_zero1 |= zt;
        } else {
            p_inv0 += (double)inv_tile;
            p_zero0 |= zt;
        }
        // prefetch the tile after this one (next step's load) into L2
        if (u < 15) prefetch_rows(a.y, a.x, fbase, c0 + 16, ptid);
        else if (f + ncl < a.frames) prefetch_rows(a.y, a.x, (size_t)(f + ncl) * kN * kM, 8 * rank, ptid);
    };

    // ------------------------------------------------------------ consumer: A FFT
    // buf[b] holds H of A tile u (written by the producers last step) -> taps -> D
    auto consume_A = [&](int u, int b, float2* dsc) {
        const int c0 = 16 * u + 8 * rank;
        float2* tile = s.buf[b];
        {
            float2* col = tile + w * kVS;
            float2 v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = col[lane + 33 * i];
            warp_fft1024<true, 32>(v, col, s.tw);
            __syncwarp();
            constexpr float inv_n = 1.0f / 1024.0f;
#pragma unroll
            for (int t2 = 0; t2 < 4; ++t2) {
                const int tap = lane + 32 * t2;
                col[lane + 33 * t2] = tap < L ? cscale(v[t2], inv_n) : make_float2(0.f, 0.f);
            }
        }
        cons_sync();
        for (int idx = tid; idx < L * 4; idx += kCons) {
            const int k = idx >> 2, c = (idx & 3) * 2;
            const int pk = k + (k >> 5);
            const float2 v0 = tile[c * kVS + pk];
            const float2 v1 = tile[(c + 1) * kVS + pk];
            __stcg(reinterpret_cast<float4*>(dsc + (size_t)k * kM + c0 + c), make_float4(v0.x, v0.y, v1.x, v1.y));
        }
        cons_sync();
    };

    // ------------------------------------------------------------ consumer: C FFT chain
    auto consume_C_fft = [&](int u, int b, const float2* dsc) {
        const int c0 = 16 * u + 8 * rank;
        float2* tile = s.buf[b];
        for (int idx = tid; idx < 128 * 4; idx += kCons) {
            const int k = idx >> 2, c = (idx & 3) * 2;
            float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k < L) v4 = __ldcg(reinterpret_cast<const float4*>(dsc + (size_t)k * kM + c0 + c));
            const int pk = k + (k >> 5);
            tile[c * kVS + pk] = make_float2(v4.x, v4.y);
            tile[(c + 1) * kVS + pk] = make_float2(v4.z, v4.w);
        }
        cons_sync();
        float2* col = tile + w * kVS;
        float* pcol = reinterpret_cast<float*>(col);
        float2 v[32];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = col[lane + 33 * i];
        if constexpr (HAMMING) {
            warp_fft1024<false, 4>(v, col, s.tw);
#pragma unroll
            for (int t2 = 0; t2 < 32; ++t2) v[t2] = cscale(v[t2], __ldg(a.wk + lane + 32 * t2));
            warp_fft1024<true, 32>(v, col, s.tw);
            __syncwarp();
#pragma unroll
            for (int t2 = 0; t2 < 32; ++t2) pcol[lane + 32 * t2] = cnorm(v[t2]) * a.scale;
        } else {
            __syncwarp();
#pragma unroll
            for (int t2 = 0; t2 < 32; ++t2) {
                float pv = 0.f;
                if (t2 < 4) pv = cnorm(cscale(v[t2], 1024.0f)) * a.scale;
                pcol[lane + 32 * t2] = pv;
            }
        }
    };

    // ------------------------------------------------------------ consumer: C detection
    // called between the two cluster phases: partner P columns are final
    auto consume_C_detect = [&](int u, int b, float ef) {
        const int c0 = 16 * u + 8 * rank;
        const float* lb = reinterpret_cast<const float*>(s.buf[b]);
        const float* pb = reinterpret_cast<const float*>(p.buf[b]);
        auto lcol = [&](int c) -> const float* { return lb + c * (2 * kVS); };
        for (int r = tid; r < kN; r += kCons) {
            if (rank == 0) {
                s.ext[0][r] = p.keep[1][r];           // 16u-1: partner's previous last column
                s.ext[1][r] = pb[r];                  // 16u+8: partner's first column
            } else {
                s.ext[0][r] = pb[7 * (2 * kVS) + r];  // 16u+7: partner's last column
                s.ext[1][r] = pb[r];                  // 16u:   partner's first column
            }
        }
        cons_sync();
        // rank 0 tests 16u..16u+7 (16u at the wrap when u == 0); rank 1 tests 16u+8..16u+14
        // and its deferred 16u-1; each consumer warp takes one column, lanes stride rows
        for (int jdx = w; jdx < 9; jdx += 8) {
            const float *A, *B, *Cc;
            int sn;
            bool active = true;
            if (jdx == 8) {
                active = rank == 1 && u > 0;
                A = s.keep[0];
                B = s.keep[1];
                Cc = s.ext[1];
                sn = c0 - 9;
            } else if (rank == 0) {
                active = !(u == 0 && jdx == 0);
                B = lcol(jdx);
                A = jdx == 0 ? s.ext[0] : lcol(jdx - 1);
                Cc = jdx == 7 ? s.ext[1] : lcol(jdx + 1);
                sn = c0 + jdx;
            } else {
                active = jdx != 7;
                B = lcol(jdx);
                A = jdx == 0 ? s.ext[0] : lcol(jdx - 1);
                Cc = lcol(jdx + 1);
                sn = c0 + jdx;
            }
            if (!active) continue;
            const int sc = (sn + kM / 2) & (kM - 1);
#pragma unroll 4
            for (int r = lane; r < kN; r += 32) {
                const float vv = B[r];
                if (vv >= ef && strict_max3(A, B, Cc, r, vv)) {
                    const int slot = atomicAdd(&s.tcnt, 1);
                    if (slot < kList) s.tl[slot] = make_key(vv, (uint32_t)(r * kM + sc));
                }
            }
        }
    };
    // after the partner has read our kept columns (second cluster phase of the step)
    auto consume_C_keep = [&](int u, int b) {
        const float* lb = reinterpret_cast<const float*>(s.buf[b]);
        for (int r = tid; r < kN; r += kCons) {
            if (rank == 1) {
                s.keep[0][r] = lb[6 * (2 * kVS) + r];
                s.keep[1][r] = lb[7 * (2 * kVS) + r];
            } else if (u == 0) {
                s.keep[0][r] = lb[r];
                s.keep[1][r] = lb[2 * kVS + r];
            }
        }
    };

    // ------------------------------------------------------------ frame bookkeeping
    // sigma_h^2 / eta of the frame whose pass A just finished (all threads participate)
    auto finish_A = [&](int f, int slot) {
        const bool odd = ((f - cid) / ncl) & 1;
        if (producer) {
            double v = odd ? p_inv1 : p_inv0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            const int zc = __any_sync(0xffffffffu, odd ? p_zero1 : p_zero0);
            if (lane == 0) s.red[w - 8] = v;
            if (lane == 0 && zc) atomicOr(&s.zc_part, 1);
        }
        __syncthreads();
        if (tid == 0) s.part = s.red[0] + s.red[1] + s.red[2] + s.red[3];
        __threadfence();
        cluster.sync();  // D complete (both halves); partials visible
        if (tid == 0) {
            const double p0 = rank == 0 ? s.part : p.part;
            const double p1 = rank == 0 ? p.part : s.part;
            const double acc = p0 + p1;
            const double sg = a.sigma2[f];
            const double s2h = sg <= 0.0 ? 0.0 : sg * acc * a.inv_count;
            s.zcs[slot] = s.zc_part | p.zc_part;
            s.etas[slot] = -s2h * a.log_pfa * a.power_factor;
            s.s2hs[slot] = s2h;
        }
        cluster.sync();
        if (tid == 0) s.zc_part = 0;
        if (odd) {
            p_inv1 = 0.0;
            p_zero1 = 0;
        } else {
            p_inv0 = 0.0;
            p_zero0 = 0;
        }
    };

    // pass B on the L tap rows (consumers; rows split between the pair)
    auto pass_B = [&](float2* dsc, int b) {
        if (!producer) {
            const int hw = tid >> 4, j = tid & 15;
            float2* tb = s.buf[b] + hw * (16 * 17);
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
        }
        __syncthreads();
        __threadfence();
        cluster.sync();  // D' complete
    };

    // wrap columns, per-CTA top-K, cross-CTA merge, outputs (consumers + cluster syncs)
    auto finish_C = [&](int f, int slot, float ef, int b) {
        cluster.sync();
        if (!producer)
            for (int r = tid; r < kN; r += kCons) s.ext[0][r] = rank == 0 ? p.keep[1][r] : p.keep[0][r];
        cluster.sync();
        if (!producer) {
            for (int r = tid; r < kN; r += kCons) {
                const float *A, *B, *Cc;
                int sn;
                if (rank == 0) {
                    A = s.ext[0];
                    B = s.keep[0];
                    Cc = s.keep[1];
                    sn = 0;
                } else {
                    A = s.keep[0];
                    B = s.keep[1];
                    Cc = s.ext[0];
                    sn = 255;
                }
                const float vv = B[r];
                if (!(vv >= ef) || !strict_max3(A, B, Cc, r, vv)) continue;
                const int sc = (sn + kM / 2) & (kM - 1);
                const int sl = atomicAdd(&s.tcnt, 1);
                if (sl < kList) s.tl[sl] = make_key(vv, (uint32_t)(r * kM + sc));
            }
            cons_sync();
            if (tid == 0 && s.tcnt > kList) s.overflow = 1;
            cons_topk(s.tl, min(s.tcnt, kList), K, s.run, s.sbest, s.sidx);
        }
        __syncthreads();
        cluster.sync();  // both per-CTA lists final
        if (rank == 0 && !producer) {
            if (w == 0) {
                for (int i = lane; i < K; i += 32) s.tl[i] = p.run[i];
                __syncwarp();
                warp_merge(s.run, s.tl, K, K, s.cand2);
            }
            cons_sync();
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
                if (a.status && s.zcs[slot]) atomicOr(a.status + f, 1);
                if (a.status && (s.overflow || p.overflow)) atomicOr(a.status + f, 2);
            }
        }
        cluster.sync();  // partner's list consumed
        if (tid == 0) {
            s.overflow = 0;
            s.tcnt = 0;
        }
        for (int i = tid; i < K; i += kThreads) s.run[i] = 0ull;
        __syncthreads();
        (void)b;
    };

    // ------------------------------------------------------------ schedule
    // g = global step counter; consumers use buf[g & 1], producers fill buf[(g + 1) & 1].
    if (cid >= a.frames) return;  // whole clusters exit together (cid is per cluster)
    if (tid == 0) s.tcnt = 0;
    for (int i = tid; i < K; i += kThreads) s.run[i] = 0ull;
    if (tid == 0) s.zc_part = 0;
    if (producer) produce(cid, 0, 0);
    __syncthreads();
    int g = 0;
    // prologue: pass A of the first frame, then pass B
    for (int u = 0; u < 16; ++u, ++g) {
        if (producer) {
            if (u < 15) produce(cid, u + 1, (g + 1) & 1);
            else if (cid + ncl < a.frames) produce(cid + ncl, 0, (g + 1) & 1);
        } else {
            consume_A(u, g & 1, dbuf(0));
        }
        __syncthreads();
    }
    int it = 0;
    for (int fC = cid; fC < a.frames; fC += ncl, ++it) {
        const int fN = fC + ncl;
        const bool hasN = fN < a.frames;
        const int sc = it & 1, sn = sc ^ 1;
        if (it == 0) {
            finish_A(fC, sc);
            pass_B(dbuf(sc), (g + 1) & 1);  // buf[g & 1] holds the pending next A tile
        }
        const float ef = eta_float(s.etas[sc]);
        for (int u = 0; u < 16; ++u, ++g) {
            const int b = g & 1;
            if (producer) {
                // next step's A tile: tile u + 1 of fN, or tile 0 of the frame after it
                cl_arrive();
                if (hasN) {
                    if (u < 15) produce(fN, u + 1, b ^ 1);
                    else if (fN + ncl < a.frames) produce(fN + ncl, 0, b ^ 1);
                }
                cl_wait();
                cl_arrive();
                cl_wait();
            } else {
                if (hasN) consume_A(u, b, dbuf(sn));
                consume_C_fft(u, b, dbuf(sc));
                cons_sync();
                cl_arrive();
                cl_wait();  // partner's P columns final
                consume_C_detect(u, b, ef);
                cl_arrive();
                cl_wait();  // partner finished reading ours
                consume_C_keep(u, b);
            }
            __syncthreads();
        }
        finish_C(fC, sc, ef, g & 1);
        if (hasN) {
            finish_A(fN, sn);
            pass_B(dbuf(sn), (g + 1) & 1);
        }
    }
}

size_t fused_ws_smem() { return sizeof(WsSmem); }

cudaError_t launch_fused_ws(const FusedArgs& a, bool hamming, int grid, cudaStream_t st) {
    const size_t smem = sizeof(WsSmem);
    grid &= ~1;
    if (grid < 2) grid = 2;
    if (hamming) {
        cudaError_t e = cudaFuncSetAttribute(fused_ws_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        fused_ws_kernel<true><<<grid, kThreads, smem, st>>>(a);
    } else {
        cudaError_t e = cudaFuncSetAttribute(fused_ws_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        fused_ws_kernel<false><<<grid, kThreads, smem, st>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace ofdmr
