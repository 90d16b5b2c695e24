// Fast path for the hot shapes N = N' = 1024, M = M' = 256 (cfg0 / cfg1 / cfg4 and the
// batched 2-D periodogram).  Same math and outputs as the generic kernels in
// radar_kernels.cu; see DESIGN.md "Kernels" for the roofline analysis.
//
//   colpass1024_fast<MODE>: CTA = 8 adjacent columns (OFDM symbols) x 1024 subcarriers
//     of one frame; one warp per column with the column in registers (warp_fft.cuh).
//     LS divide + sum 1/|x|^2 (estimation.cpp:10-21, pipeline.cpp:18-23) on the tile
//     load; DFT-CE (estimation.cpp:23-39) as IFFT -> truncate -> input-pruned FFT; the
//     separable window (periodogram.cpp:52-56); the delay IFFT (periodogram.cpp:60).
//     With a rectangular window and N' = N the DFT-CE + delay IFFT collapse exactly to
//     the first L rows of IFFT_N(H) (MODE & kShortcut).
//   rowpass256_fast: CTA = 30 rows of P (+1 halo row each side); half-warp FFT_256 per
//     row (periodogram.cpp:57), |.|^2/(NM) + fftshift (:63-73), optional map store,
//     strict wrapped 3x3 local maxima >= eta (:77-136), per-block top-K, and the per-frame
//     top-K merge done by the last block of each frame (no separate merge launch).
#include "radar_kernels.cuh"
#include "warp_fft.cuh"

namespace ofdmr {

constexpr int kFastC = 8;            // columns per colpass CTA (one warp each)
constexpr int kColVS = 1057;         // pad_len(1024)
constexpr int kRowR = 30;            // P rows per rowpass CTA (+2 halo = 32 = 2 rounds of 16)
constexpr int kListCap = 512;        // candidate list in smem; exact fallback scan beyond it

enum : int { kLS = 1, kCE = 2, kPrune = 4, kWin = 8, kShortcut = 16 };

// One column tile (8 symbols x 1024 subcarriers) of input frame f; G / partials are
// addressed by frame slot fslot (== f for the per-chunk launches, a ring slot for the
// persistent schedule).  tw must already hold the 1024-entry table (synced by the caller
// or by the first barrier below).
template <int MODE>
__device__ __forceinline__ void col_item(const ColArgs& a, const float2* tw, float2* tile, double* red, int f,
                                         int tile_idx, int fslot) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int c0 = tile_idx * kFastC;
    const int m = a.m;
    const size_t fbase = (size_t)f * 1024 * m;

    // Tile load: 16 float4 per thread per array, issued in two batches of 8 so that
    // 8 (H) or 16 (Y and X) independent 16-B loads per thread are in flight.
    double inv_acc = 0.0;
    int zero_cell = 0;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        float4 yv[8], xv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int idx = tid + (half * 8 + q) * 256;
            const size_t off = fbase + (size_t)(idx >> 2) * m + c0 + (idx & 3) * 2;
            if constexpr (MODE & kLS) {
                yv[q] = __ldcs(reinterpret_cast<const float4*>(a.y + off));
                xv[q] = __ldcs(reinterpret_cast<const float4*>(a.x + off));
            } else {
                yv[q] = __ldcs(reinterpret_cast<const float4*>(a.h + off));
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int idx = tid + (half * 8 + q) * 256;
            const int k = idx >> 2;
            const int c = (idx & 3) * 2;
            float2 h0, h1;
            if constexpr (MODE & kLS) {
                const float4 y4 = yv[q], x4 = xv[q];
                h0 = ls_cell(y4.x, y4.y, x4.x, x4.y, inv_acc, zero_cell);
                h1 = ls_cell(y4.z, y4.w, x4.z, x4.w, inv_acc, zero_cell);
            } else {
                h0 = make_float2(yv[q].x, yv[q].y);
                h1 = make_float2(yv[q].z, yv[q].w);
            }
            const int p = k + (k >> 5);
            tile[c * kColVS + p] = h0;
            tile[(c + 1) * kColVS + p] = h1;
        }
    }
    if constexpr (MODE & kLS) {
        if (zero_cell) atomicOr(a.status + f, 1);
        if (a.inv_partial != nullptr) {
            double v = inv_acc;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) red[w] = v;
        }
    }
    __syncthreads();
    if constexpr (MODE & kLS) {
        if (a.inv_partial != nullptr && tid == 0) {
            double s = 0.0;
            for (int i = 0; i < 8; ++i) s += red[i];
            a.inv_partial[(size_t)fslot * a.ntiles + tile_idx] = s;
        }
    }

    // ---- per-warp column chain, registers only between transforms
    float2* col = tile + w * kColVS;
    float2 v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = col[lane + 33 * i];
    const float wl = (MODE & kWin) ? a.wl[c0 + w] : 1.0f;
    int out_rows = 1024;
    if constexpr (MODE & kCE) {
        warp_fft1024<true, 32>(v, col, tw);  // IFFT_N: lane t1 holds taps t1 + 32 t2
        const int L = a.ce_taps;
        if constexpr (MODE & kShortcut) {
#pragma unroll
            for (int t2 = 0; t2 < 32; ++t2)
                if (lane + 32 * t2 < L) col[lane + 33 * t2] = v[t2];
            out_rows = L;
        } else {
            constexpr float inv_n = 1.0f / 1024.0f;
#pragma unroll
            for (int t2 = 0; t2 < 32; ++t2) v[t2] = (lane + 32 * t2 < L) ? cscale(v[t2], inv_n) : make_float2(0.f, 0.f);
            if constexpr (MODE & kPrune) warp_fft1024<false, 4>(v, col, tw);   // L <= 128: taps in v[0..3]
            else warp_fft1024<false, 32>(v, col, tw);
            if constexpr (MODE & kWin) {
#pragma unroll
                for (int t2 = 0; t2 < 32; ++t2) v[t2] = cscale(v[t2], __ldg(a.wk + lane + 32 * t2) * wl);
            }
            warp_fft1024<true, 32>(v, col, tw);  // delay IFFT_N'
#pragma unroll
            for (int t2 = 0; t2 < 32; ++t2) col[lane + 33 * t2] = v[t2];
        }
    } else {
        if constexpr (MODE & kWin) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = cscale(v[i], __ldg(a.wk + lane + 32 * i) * wl);
        }
        warp_fft1024<true, 32>(v, col, tw);
#pragma unroll
        for (int t2 = 0; t2 < 32; ++t2) col[lane + 33 * t2] = v[t2];
    }
    __syncthreads();

    // ---- coalesced row-segment store of G (out_rows x 8 columns); G stays in L2
    float2* g = a.g_out + (size_t)fslot * a.g_rows * m;
#pragma unroll 4
    for (int idx = tid; idx < out_rows * (kFastC / 2); idx += 256) {
        const int k = idx >> 2;
        const int c = (idx & 3) * 2;
        const int p = k + (k >> 5);
        const float2 v0 = tile[c * kColVS + p];
        const float2 v1 = tile[(c + 1) * kColVS + p];
        *reinterpret_cast<float4*>(g + (size_t)k * m + c0 + c) = make_float4(v0.x, v0.y, v1.x, v1.y);
    }
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) colpass1024_fast(ColArgs a, const float2* __restrict__ tw_t) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* tw = reinterpret_cast<float2*>(smem_raw);   // 1024: tw[t1*32 + j] = W^{j t1}
    float2* tile = tw + 1024;                            // 8 x kColVS
    __shared__ double red[8];
    for (int i = threadIdx.x; i < 1024; i += 256) tw[i] = tw_t[i];
    col_item<MODE>(a, tw, tile, red, blockIdx.y, blockIdx.x, blockIdx.y);
}

struct FastRowArgs {
    RowArgs r;
    const float2* tw256_t;      // tw[t1*16 + j] = W_256^{j t1}
    // fused merge (per frame, by the last row block to finish)
    int* frame_done;            // per-frame block counters (zeroed; reset by the merging block)
    const int32_t* k_per_frame;
    int32_t* det_delay;
    int32_t* det_doppler;
    float* det_power;
    int32_t* counts;
    double* s2h_out;
};

// Strict wrapped 3x3 local max >= eta at tile row tr (1..nrows), column c; key or 0.
__device__ __forceinline__ unsigned long long qualify256(const float* pt, int tr, int c, double eta, int r0) {
    const float v = pt[tr * 256 + c];
    if (!((double)v >= eta)) return 0ull;
    const int cl = (c - 1) & 255, cr = (c + 1) & 255;
    const float* up = pt + (tr - 1) * 256;
    const float* mid = pt + tr * 256;
    const float* dn = pt + (tr + 1) * 256;
    if (up[cl] >= v || up[c] >= v || up[cr] >= v || mid[cl] >= v || mid[cr] >= v || dn[cl] >= v || dn[c] >= v ||
        dn[cr] >= v)
        return 0ull;
    return make_key(v, (uint32_t)((r0 + tr - 1) * 256 + c));
}



// Row-pass region: (R + 2) x 256 fp32 P tile, 16 half-warp transpose buffers, list.
constexpr size_t kRowRegion = sizeof(float) * (kRowR + 2) * 256 + sizeof(float2) * (16 * 16 * 17) +
                              sizeof(unsigned long long) * kListCap;

// One block of kRowR rows of P for input frame f (outputs by f; G, partials, candidates and
// the merge counter by frame slot fslot); nblk blocks per frame.
__device__ void row_item(const FastRowArgs& e, unsigned char* region, const float2* tw, int f, int fslot, int rb,
                         int nblk) {
    const RowArgs& a = e.r;
    float* ptile = reinterpret_cast<float*>(region);                                   // (R + 2) x 256
    float2* tbufs = reinterpret_cast<float2*>(ptile + (kRowR + 2) * 256);             // 16 x (16 x 17)
    unsigned long long* list = reinterpret_cast<unsigned long long*>(tbufs + 16 * 16 * 17);
    __shared__ unsigned long long s_top[kMaxK];
    __shared__ unsigned long long s_best[8];
    __shared__ int s_idx[8];
    __shared__ int s_cnt, s_last;

    const int tid = threadIdx.x;
    const int np = 1024, m = 256;
    const int r0 = rb * kRowR;
    const int nrows = min(kRowR, np - r0);
    const int TR = nrows + 2;
    const int hw = tid >> 4, j = tid & 15;

    const float2* gf = a.g + (size_t)fslot * a.g_rows * m;
    for (int t0 = 0; t0 < TR; t0 += 16) {
        // a warp's two half-warps must stay converged (the half-warp FFT uses __syncwarp):
        // rows past the tile or at/after g_rows (exactly zero) load zeros, stores are predicated
        const int tr = t0 + hw;
        const bool in_tile = tr < TR;
        const int gr = (r0 - 1 + tr + np) & (np - 1);
        const bool nonzero = in_tile && gr < a.g_rows;
        const int wtr = t0 + (hw & ~1);                      // first tile row of this warp
        const bool warp_active = wtr < TR;
        const bool warp_any = warp_active && ((((r0 - 1 + wtr + np) & (np - 1)) < a.g_rows) ||
                                              (wtr + 1 < TR && ((r0 + wtr + np) & (np - 1)) < a.g_rows));
        float* prow = ptile + tr * 256;
        if (warp_any) {
            float2 v[16];
            const float2* src = gf + (size_t)(nonzero ? gr : 0) * m;
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = nonzero ? __ldcg(src + j + 16 * i) : make_float2(0.f, 0.f);
            halfwarp_fft256<false>(v, tbufs + hw * 16 * 17, tw);
            if (in_tile) {
#pragma unroll
                for (int t2 = 0; t2 < 16; ++t2) prow[(j + 16 * t2 + 128) & 255] = cnorm(v[t2]) * a.scale;
            }
        } else if (in_tile) {
#pragma unroll
            for (int t2 = 0; t2 < 16; ++t2) prow[j + 16 * t2] = 0.f;
        }
    }
    __syncthreads();

    if (a.p_out != nullptr) {
        float* po = a.p_out + (size_t)f * np * 256 + (size_t)r0 * 256;
        for (int idx = tid; idx < nrows * 64; idx += 256) {
            const int r = idx >> 6, q = idx & 63;
            __stcs(reinterpret_cast<float4*>(po + (size_t)r * 256) + q,
                   reinterpret_cast<const float4*>(ptile + (r + 1) * 256)[q]);
        }
    }
    if (!a.detect) return;

    double eta;
    if (a.eta_in != nullptr) {
        eta = a.eta_in[f];
    } else {
        double s2h = a.sigma2[f];
        if (a.inv_partial != nullptr) {
            if (s2h <= 0.0) {
                s2h = 0.0;
            } else {
                double acc = 0.0;
                for (int t = 0; t < a.ntiles; ++t) acc += a.inv_partial[(size_t)fslot * a.ntiles + t];
                s2h = s2h * acc * a.inv_count;
            }
        }
        eta = -s2h * a.log_pfa * a.power_factor;
    }
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (int idx = tid; idx < nrows * 256; idx += 256) {
        const unsigned long long key = qualify256(ptile, (idx >> 8) + 1, idx & 255, eta, r0);
        if (key) {
            const int slot = atomicAdd(&s_cnt, 1);
            if (slot < kListCap) list[slot] = key;
        }
    }
    __syncthreads();
    const int cnt = s_cnt;
    const int K = a.kmax;
    if (cnt <= kListCap) {
        block_topk_smem(list, cnt, K, s_top, s_best, s_idx);
    } else {
        // exact fallback: K rounds of "largest qualifying key below the previous one"
        unsigned long long prev = ~0ull;
        for (int round = 0; round < K; ++round) {
            unsigned long long best = 0;
            for (int idx = tid; idx < nrows * 256; idx += 256) {
                const unsigned long long key = qualify256(ptile, (idx >> 8) + 1, idx & 255, eta, r0);
                if (key < prev && key > best) best = key;
            }
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
                best = ob > best ? ob : best;
            }
            if ((tid & 31) == 0) s_best[tid >> 5] = best;
            __syncthreads();
            if (tid == 0) {
                unsigned long long b = 0;
                for (int i = 0; i < 8; ++i) b = s_best[i] > b ? s_best[i] : b;
                s_top[round] = b;
            }
            __syncthreads();
            prev = s_top[round];
            __syncthreads();
            if (prev == 0) {
                for (int r = round + 1 + tid; r < K; r += 256) s_top[r] = 0;
                break;
            }
        }
    }
    __syncthreads();
    unsigned long long* out = a.cand + ((size_t)fslot * nblk + rb) * K;
    for (int i = tid; i < K; i += 256) out[i] = s_top[i];

    // ---- last block of this frame merges all blocks' candidates
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const int prev = atomicAdd(e.frame_done + fslot, 1);
        s_last = prev == nblk - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    unsigned long long* all = a.cand + (size_t)fslot * nblk * K;
    const int total = nblk * K;
    const int kf = e.k_per_frame ? min(e.k_per_frame[f], K) : K;
    block_topk_global(all, total, kf, s_top, s_best, s_idx);
    __syncthreads();
    if (tid < K) {
        const unsigned long long key = tid < kf ? s_top[tid] : 0ull;
        const size_t o = (size_t)f * K + tid;
        if (key == 0) {
            e.det_delay[o] = 0;
            e.det_doppler[o] = 0;
            e.det_power[o] = 0.f;
        } else {
            const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
            e.det_delay[o] = (int32_t)(idx >> 8);
            e.det_doppler[o] = (int32_t)(idx & 255) - 128;
            e.det_power[o] = __uint_as_float((uint32_t)(key >> 32));
        }
    }
    if (tid == 0) {
        int n = 0;
        for (int i = 0; i < kf; ++i) n += s_top[i] != 0;
        e.counts[f] = n;
        e.frame_done[fslot] = 0;  // ready for the next use of this slot
        if (e.s2h_out != nullptr) {
            double s2h = a.sigma2[f];
            if (a.inv_partial != nullptr) {
                if (s2h <= 0.0) {
                    s2h = 0.0;
                } else {
                    double acc = 0.0;
                    for (int t = 0; t < a.ntiles; ++t) acc += a.inv_partial[(size_t)fslot * a.ntiles + t];
                    s2h = s2h * acc * a.inv_count;
                }
            }
            e.s2h_out[f] = s2h;
        }
    }
}

__global__ void __launch_bounds__(256) rowpass256_fast(FastRowArgs e) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* tw = reinterpret_cast<float2*>(smem_raw);
    tw[threadIdx.x] = e.tw256_t[threadIdx.x];
    __syncthreads();
    row_item(e, smem_raw + 256 * sizeof(float2), tw, blockIdx.y, blockIdx.y, blockIdx.x, gridDim.x);
}

// ------------------------------------------------------------------ persistent ------
// One launch for a whole batch: CTAs pull ordered tickets; ticket space per step s is
// [column items of chunk s | row items of chunk s - 1].  Row items of frame f wait on
// done_cols[f] == 32; column items of chunk c wait until the row items of chunk c - ring
// (previous user of the same intermediate slot) are done.  Every waited-on item has a
// smaller ticket and waits only on smaller tickets, and all CTAs are resident, so the
// spins always terminate.
struct PersistArgs {
    ColArgs col;
    FastRowArgs row;
    const float2* tw1024_t;
    int frames, cf, ring, nchunks, nblk;
    int* ticket;
    int* done_cols;   // [frames]
    int* done_rows;   // [nchunks]
};

__device__ __forceinline__ void spin_until(const int* p, int target) {
    if (threadIdx.x == 0) {
        while (atomicAdd(const_cast<int*>(p), 0) < target) __nanosleep(64);
        __threadfence();
    }
    __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) pgram_persist(PersistArgs pa) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* tw = reinterpret_cast<float2*>(smem_raw);   // 1024
    float2* tw256 = tw + 1024;                           // 256
    unsigned char* region = reinterpret_cast<unsigned char*>(tw256 + 256);
    __shared__ double red[8];
    __shared__ int s_ticket;
    for (int i = threadIdx.x; i < 1024; i += 256) tw[i] = pa.tw1024_t[i];
    tw256[threadIdx.x] = pa.row.tw256_t[threadIdx.x];
    __syncthreads();
    const int Lc = pa.cf * 32, Lr = pa.cf * pa.nblk;
    const long long total = (long long)(pa.nchunks + 1) * (Lc + Lr);
    for (;;) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(pa.ticket, 1);
        __syncthreads();
        const long long t = s_ticket;
        __syncthreads();
        if (t >= total) break;
        const int s = (int)(t / (Lc + Lr));
        const int r = (int)(t % (Lc + Lr));
        if (r < Lc) {
            const int c = s;
            if (c >= pa.nchunks) continue;
            const int f = c * pa.cf + r / 32, tile = r % 32;
            if (f >= pa.frames) continue;
            if (c >= pa.ring) spin_until(pa.done_rows + (c - pa.ring), Lr);
            const int fslot = (c % pa.ring) * pa.cf + (f - c * pa.cf);
            col_item<MODE>(pa.col, tw, reinterpret_cast<float2*>(region), red, f, tile, fslot);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(pa.done_cols + f, 1);
            }
        } else {
            const int c = s - 1;
            if (c < 0) continue;
            const int rr = r - Lc;
            const int f = c * pa.cf + rr / pa.nblk, rb = rr % pa.nblk;
            if (f < pa.frames) {
                spin_until(pa.done_cols + f, 32);
                const int fslot = (c % pa.ring) * pa.cf + (f - c * pa.cf);
                row_item(pa.row, region, tw256, f, fslot, rb, pa.nblk);
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(pa.done_rows + c, 1);  // counts every row ticket of the chunk
            }
        }
    }
}

constexpr size_t kPersistSmem = sizeof(float2) * (1024 + 256) +
                                (kRowRegion > sizeof(float2) * kFastC * kColVS ? kRowRegion
                                                                                : sizeof(float2) * kFastC * kColVS);

cudaError_t launch_pgram_persist(const PersistArgs& pa, bool ls, bool win, int grid, cudaStream_t st) {
    auto go = [&](auto kern) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPersistSmem);
        if (e != cudaSuccess) return e;
        kern<<<grid, 256, kPersistSmem, st>>>(pa);
        return cudaGetLastError();
    };
    if (ls) return win ? go(pgram_persist<kLS | kWin>) : go(pgram_persist<kLS>);
    return win ? go(pgram_persist<kWin>) : go(pgram_persist<0>);
}

// ------------------------------------------------------------------ launch ------

template <int MODE>
cudaError_t launch_col_fast_t(const ColArgs& a, const float2* tw_t, int frames, cudaStream_t st) {
    const size_t smem = (1024 + kFastC * kColVS) * sizeof(float2);
    auto kern = colpass1024_fast<MODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(a.m / kFastC, frames);
    kern<<<grid, 256, smem, st>>>(a, tw_t);
    return cudaGetLastError();
}

cudaError_t launch_colpass_fast(const ColArgs& a, bool ls, bool win, const float2* tw_t, int frames,
                                cudaStream_t st) {
    const bool ce = a.ce_taps > 0;
    const bool prune = ce && a.ce_taps <= 128;
    if (!ce) {
        if (ls) return win ? launch_col_fast_t<kLS | kWin>(a, tw_t, frames, st) : launch_col_fast_t<kLS>(a, tw_t, frames, st);
        return win ? launch_col_fast_t<kWin>(a, tw_t, frames, st) : launch_col_fast_t<0>(a, tw_t, frames, st);
    }
    if (!ls) return cudaErrorInvalidValue;  // pipeline CE always starts from (Y, X)
    if (a.shortcut) return launch_col_fast_t<kLS | kCE | kShortcut>(a, tw_t, frames, st);
    if (win) {
        return prune ? launch_col_fast_t<kLS | kCE | kPrune | kWin>(a, tw_t, frames, st)
                     : launch_col_fast_t<kLS | kCE | kWin>(a, tw_t, frames, st);
    }
    return prune ? launch_col_fast_t<kLS | kCE | kPrune>(a, tw_t, frames, st)
                 : launch_col_fast_t<kLS | kCE>(a, tw_t, frames, st);
}

cudaError_t launch_rowpass_fast(const FastRowArgs& a, int frames, cudaStream_t st) {
    constexpr size_t kRowSmem = sizeof(float2) * 256 + kRowRegion;
    cudaError_t err = cudaFuncSetAttribute(rowpass256_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRowSmem);
    if (err != cudaSuccess) return err;
    dim3 grid((1024 + kRowR - 1) / kRowR, frames);
    rowpass256_fast<<<grid, 256, kRowSmem, st>>>(a);
    return cudaGetLastError();
}

int fast_rows_per_block() { return kRowR; }

}  // namespace ofdmr
