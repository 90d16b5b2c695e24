// Receiver hot-path kernels for sm_100a.  See DESIGN.md "Kernels".
//
//   colpass<N, NP, C>: one CTA = C adjacent columns (OFDM symbols) of one frame, all
//     N subcarriers.  Fuses LS spectral division (estimation.cpp:10-21) with the
//     zero-cell check, the sum of 1/|x|^2 for division_noise_power (pipeline.cpp:18-23),
//     DFT-CE (IFFT_N, keep L taps x 1/N, FFT_N; estimation.cpp:23-39), the separable
//     window (periodogram.cpp:52-56) and the zero-padded delay IFFT_N'
//     (periodogram.cpp:60).  Output: G = k-axis transform (N' x M), kept L2-resident by
//     the chunked launch schedule.
//   rowpass<MP>: one CTA = R rows of P (+1 halo row each side).  Zero-pad to M',
//     forward FFT_M' (periodogram.cpp:57), |.|^2/(NM) + fftshift (:63-73), optional map
//     store, threshold (:77-87) and strict wrapped 3x3 local maxima with a per-block
//     top-K (extract_peaks, :89-136 — equivalent to the greedy claim loop because two
//     strict local maxima are never 8-adjacent; SURVEY.md §7 hard part 1).
//   merge: per-frame top-K over the block candidates -> detection records.
#include "fft_smem.cuh"
#include <cstdlib>

#include "radar_kernels.cuh"

namespace ofdmr {

// ---------------------------------------------------------------- helpers --

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum (fixed shuffle tree, then warps in order by thread 0).
template <int NT>
__device__ double block_sum_d(double v, double* scratch) {
    v = warp_sum_d(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NT / 32; ++i) s += scratch[i];
        scratch[0] = s;
    }
    __syncthreads();
    s = scratch[0];
    __syncthreads();
    return s;
}

// ---------------------------------------------------------------- colpass --

template <int N, int NP, int C>
__global__ void __launch_bounds__(kNT) colpass_kernel(ColArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* buf = reinterpret_cast<float2*>(smem_raw);
    constexpr int VS = pad_len(NP);
    __shared__ double red[kNT / 32];

    const int f = blockIdx.y;
    const int tile = blockIdx.x;
    const int c0 = tile * C;
    const int m = a.m;
    const size_t fbase = (size_t)f * N * m;
    constexpr int PAIRS = C / 2;

    // ---- 1. load the N x C tile (float4 = two adjacent columns), LS divide
    double inv_acc = 0.0;
    int zero_cell = 0;
    for (int idx = threadIdx.x; idx < N * PAIRS; idx += kNT) {
        const int k = idx / PAIRS;
        const int c = (idx % PAIRS) * 2;
        const size_t off = fbase + (size_t)k * m + c0 + c;
        float2 h0, h1;
        if (a.y != nullptr) {
            const float4 yv = __ldcs(reinterpret_cast<const float4*>(a.y + off));
            const float4 xv = __ldcs(reinterpret_cast<const float4*>(a.x + off));
            // y / x = y * conj(x) / |x|^2 (exact zero-cell semantics, radar_kernels.cuh ls_cell)
            h0 = ls_cell(yv.x, yv.y, xv.x, xv.y, inv_acc, zero_cell);
            h1 = ls_cell(yv.z, yv.w, xv.z, xv.w, inv_acc, zero_cell);
        } else {
            const float4 hv = __ldcs(reinterpret_cast<const float4*>(a.h + off));
            h0 = make_float2(hv.x, hv.y);
            h1 = make_float2(hv.z, hv.w);
        }
        buf[c * VS + pidx(k)] = h0;
        buf[(c + 1) * VS + pidx(k)] = h1;
        if (a.h_out != nullptr && !a.hout_after_ce)
            *reinterpret_cast<float4*>(a.h_out + off) = make_float4(h0.x, h0.y, h1.x, h1.y);
    }
    if (a.y != nullptr) {
        if (zero_cell) atomicOr(a.status + f, 1);
        if (a.inv_partial != nullptr) {
            const double s = block_sum_d<kNT>(inv_acc, red);
            if (threadIdx.x == 0) a.inv_partial[(size_t)f * a.ntiles + tile] = s;
        }
    }
    __syncthreads();

    // ---- 2. DFT-CE: IFFT_N, keep L taps (x 1/N), FFT_N
    if (a.ce_taps > 0) {
        fft_vectors<N, true, C, kNT>(buf, VS, a.tw);
        const int L = a.ce_taps;
        if (a.shortcut) {
            // rect window and N' == N: IFFT_N(FFT_N(trunc(g)/N)) = trunc(g): the delay
            // rows of the periodogram are IFFT_N(H) rows < L and exactly zero beyond.
            for (int idx = threadIdx.x; idx < L * PAIRS; idx += kNT) {
                const int k = idx / PAIRS;
                const int c = (idx % PAIRS) * 2;
                const float2 v0 = buf[c * VS + pidx(k)];
                const float2 v1 = buf[(c + 1) * VS + pidx(k)];
                *reinterpret_cast<float4*>(a.g_out + (size_t)f * a.g_rows * m + (size_t)k * m + c0 + c) =
                    make_float4(v0.x, v0.y, v1.x, v1.y);
            }
            return;
        }
        const float inv_n = 1.0f / (float)N;
        for (int idx = threadIdx.x; idx < C * N; idx += kNT) {
            const int c = idx / N, k = idx % N;
            float2& v = buf[c * VS + pidx(k)];
            v = (k < L) ? cscale(v, inv_n) : make_float2(0.f, 0.f);
        }
        __syncthreads();
        fft_vectors<N, false, C, kNT>(buf, VS, a.tw);
        if (a.h_out != nullptr && a.hout_after_ce) {
            for (int idx = threadIdx.x; idx < N * PAIRS; idx += kNT) {
                const int k = idx / PAIRS;
                const int c = (idx % PAIRS) * 2;
                const float2 v0 = buf[c * VS + pidx(k)];
                const float2 v1 = buf[(c + 1) * VS + pidx(k)];
                *reinterpret_cast<float4*>(a.h_out + fbase + (size_t)k * m + c0 + c) =
                    make_float4(v0.x, v0.y, v1.x, v1.y);
            }
        }
    }
    if (a.g_out == nullptr) return;

    // ---- 3. window (w_k w_l) + zero-pad to N' + unscaled IFFT_N' (delay axis)
    for (int idx = threadIdx.x; idx < C * NP; idx += kNT) {
        const int c = idx / NP, k = idx % NP;
        float2& v = buf[c * VS + pidx(k)];
        if (k >= N) {
            v = make_float2(0.f, 0.f);
        } else if (a.wk != nullptr) {
            const float w = a.wk[k] * a.wl[c0 + c];
            v = cscale(v, w);
        }
    }
    __syncthreads();
    fft_vectors<NP, true, C, kNT>(buf, VS, a.tw);
    float2* g = a.g_out + (size_t)f * a.g_rows * m;
    for (int idx = threadIdx.x; idx < NP * PAIRS; idx += kNT) {
        const int k = idx / PAIRS;
        const int c = (idx % PAIRS) * 2;
        const float2 v0 = buf[c * VS + pidx(k)];
        const float2 v1 = buf[(c + 1) * VS + pidx(k)];
        *reinterpret_cast<float4*>(g + (size_t)k * m + c0 + c) = make_float4(v0.x, v0.y, v1.x, v1.y);
    }
}

// ---------------------------------------------------------------- rowpass --

template <int MP, int RB>
__global__ void __launch_bounds__(kNT) rowpass_kernel(RowArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int VS = pad_len(MP);
    const int R = a.rows_per_block;
    float2* cbuf = reinterpret_cast<float2*>(smem_raw);                   // RB x VS complex
    float* ptile = reinterpret_cast<float*>(cbuf + ((RB * VS + 1) & ~1));  // (R + 2) x MP, 16-B aligned
    unsigned long long* list = reinterpret_cast<unsigned long long*>(ptile + (size_t)(R + 2) * MP);
    __shared__ int s_cnt;
    __shared__ unsigned long long s_best[kNT / 32];
    __shared__ int s_idx[kNT / 32];
    __shared__ unsigned long long s_top[kMaxK];

    const int f = blockIdx.y;
    const int rb = blockIdx.x;
    const int np = a.n_prime;
    const int r0 = rb * R;
    const int nrows = min(R, np - r0);            // last block may be partial
    const int m = a.m;
    const int half = MP / 2;
    const int TR = nrows + 2;                     // tile rows incl. halo

    // ---- 1. P tile rows (global row (r0 - 1 + tr) mod N')
    if (a.p_in != nullptr) {
        const float* pf = a.p_in + (size_t)f * np * MP;
        for (int idx = threadIdx.x; idx < TR * (MP / 4); idx += kNT) {
            const int tr = idx / (MP / 4), q = idx % (MP / 4);
            const int gr = (r0 - 1 + tr + np) % np;
            reinterpret_cast<float4*>(ptile + (size_t)tr * MP)[q] =
                __ldcs(reinterpret_cast<const float4*>(pf + (size_t)gr * MP) + q);
        }
        __syncthreads();
    } else {
        const float2* gf = a.g + (size_t)f * a.g_rows * m;
        for (int t0 = 0; t0 < TR; t0 += RB) {
            // any non-zero rows in this chunk?
            bool any = false;
            for (int j = 0; j < RB && t0 + j < TR; ++j) {
                const int gr = (r0 - 1 + t0 + j + np) % np;
                any |= gr < a.g_rows;
            }
            if (!any) {
                for (int idx = threadIdx.x; idx < RB * MP; idx += kNT) {
                    const int j = idx / MP, s = idx % MP;
                    if (t0 + j < TR) ptile[(size_t)(t0 + j) * MP + s] = 0.f;
                }
                continue;  // uniform across the block
            }
            for (int idx = threadIdx.x; idx < RB * (MP / 2); idx += kNT) {
                const int j = idx / (MP / 2), s = (idx % (MP / 2)) * 2;
                const int gr = (r0 - 1 + t0 + j + np) % np;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (t0 + j < TR && gr < a.g_rows && s < m)
                    v = __ldcs(reinterpret_cast<const float4*>(gf + (size_t)gr * m + s));
                cbuf[j * VS + pidx(s)] = make_float2(v.x, v.y);
                cbuf[j * VS + pidx(s + 1)] = make_float2(v.z, v.w);
            }
            __syncthreads();
            fft_vectors<MP, false, RB, kNT>(cbuf, VS, a.tw);
            for (int idx = threadIdx.x; idx < RB * MP; idx += kNT) {
                const int j = idx / MP, s = idx % MP;
                if (t0 + j < TR)
                    ptile[(size_t)(t0 + j) * MP + ((s + half) & (MP - 1))] = cnorm(cbuf[j * VS + pidx(s)]) * a.scale;
            }
            __syncthreads();
        }
        __syncthreads();  // the last chunk may have been a zero-fill without a barrier
    }

    // ---- 2. map store (interior rows)
    if (a.p_out != nullptr) {
        float* po = a.p_out + (size_t)f * np * MP + (size_t)r0 * MP;
        for (int idx = threadIdx.x; idx < nrows * (MP / 4); idx += kNT) {
            const int r = idx / (MP / 4), q = idx % (MP / 4);
            __stcs(reinterpret_cast<float4*>(po + (size_t)r * MP) + q,
                   reinterpret_cast<const float4*>(ptile + (size_t)(r + 1) * MP)[q]);
        }
    }
    if (!a.detect) return;

    // ---- 3. threshold + strict wrapped 3x3 local maxima
    double eta;
    if (a.eta_in != nullptr) {
        eta = a.eta_in[f];
    } else {
        const double s2h = sigma_h2_warp(a.inv_partial, a.ntiles, f, a.sigma2[f], a.inv_count);
        eta = -s2h * a.log_pfa * a.power_factor;  // periodogram.cpp:80
    }
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int idx = threadIdx.x; idx < nrows * MP; idx += kNT) {
        const int tr = idx / MP + 1, c = idx % MP;
        const float v = ptile[(size_t)tr * MP + c];
        if (!((double)v >= eta)) continue;
        const int cl = (c - 1) & (MP - 1), cr = (c + 1) & (MP - 1);
        const float* up = ptile + (size_t)(tr - 1) * MP;
        const float* mid = ptile + (size_t)tr * MP;
        const float* dn = ptile + (size_t)(tr + 1) * MP;
        if (up[cl] >= v || up[c] >= v || up[cr] >= v || mid[cl] >= v || mid[cr] >= v || dn[cl] >= v ||
            dn[c] >= v || dn[cr] >= v)
            continue;
        const int slot = atomicAdd(&s_cnt, 1);
        list[slot] = make_key(v, (uint32_t)((r0 + tr - 1) * MP + c));
    }
    __syncthreads();
    const int cnt = s_cnt;
    block_topk<kNT>(list, cnt, a.kmax, s_top, s_best, s_idx);
    __syncthreads();
    unsigned long long* out = a.cand + ((size_t)f * gridDim.x + rb) * a.kmax;
    for (int i = threadIdx.x; i < a.kmax; i += kNT) out[i] = s_top[i];
}

// ------------------------------------------------------------------ merge --

__global__ void __launch_bounds__(kNT) merge_kernel(MergeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* list = reinterpret_cast<unsigned long long*>(smem_raw);
    __shared__ unsigned long long s_best[kNT / 32];
    __shared__ int s_idx[kNT / 32];
    __shared__ unsigned long long s_top[kMaxK];
    const int f = blockIdx.x;
    const int total = a.nblk * a.kmax;
    const unsigned long long* src = a.cand + (size_t)f * total;
    for (int i = threadIdx.x; i < total; i += kNT) list[i] = src[i];
    __syncthreads();
    const int kf = a.k_per_frame ? min(a.k_per_frame[f], a.kmax) : a.kmax;
    block_topk<kNT>(list, total, kf, s_top, s_best, s_idx);
    __syncthreads();
    const double s2h = (a.s2h_out != nullptr || a.eta_out != nullptr)
                           ? sigma_h2_warp(a.inv_partial, a.ntiles, f, a.sigma2[f], a.inv_count)
                           : 0.0;
    if (threadIdx.x == 0) {
        int n = 0;
        for (int i = 0; i < a.kmax; ++i) {
            const unsigned long long key = i < kf ? s_top[i] : 0ull;
            const size_t o = (size_t)f * a.kmax + i;
            if (key == 0) {  // unused slots are cleared so outputs are fully defined
                a.det_delay[o] = 0;
                a.det_doppler[o] = 0;
                a.det_power[o] = 0.f;
                continue;
            }
            const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
            a.det_delay[o] = (int32_t)(idx / a.m_prime);
            a.det_doppler[o] = (int32_t)(idx % a.m_prime) - a.m_prime / 2;
            a.det_power[o] = __uint_as_float((uint32_t)(key >> 32));
            ++n;
        }
        a.counts[f] = n;
        if (a.s2h_out != nullptr || a.eta_out != nullptr) {
            if (a.s2h_out) a.s2h_out[f] = s2h;
            if (a.eta_out) a.eta_out[f] = -s2h * a.log_pfa * a.power_factor;
        }
    }
}

// ------------------------------------------------------ launch dispatchers --

template <int NP> constexpr int col_tile() {
    return NP >= 4096 ? 2 : NP >= 2048 ? 4 : NP >= 1024 ? 8 : 16;
}

template <int N, int NP>
cudaError_t launch_colpass_t(const ColArgs& a, int frames, cudaStream_t st) {
    constexpr int C = col_tile<NP>();
    const size_t smem = (size_t)C * pad_len(NP) * sizeof(float2);
    auto kern = colpass_kernel<N, NP, C>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(a.m / C, frames);
    kern<<<grid, kNT, smem, st>>>(a);
    return cudaGetLastError();
}

int colpass_tile_cols(int np) {
    return np >= 4096 ? 2 : np >= 2048 ? 4 : np >= 1024 ? 8 : 16;
}

template <int N>
cudaError_t launch_colpass_n(const ColArgs& a, int np, int frames, cudaStream_t st) {
    if (np == N) return launch_colpass_t<N, N>(a, frames, st);
    if constexpr (2 * N <= kTwLen) if (np == 2 * N) return launch_colpass_t<N, 2 * N>(a, frames, st);
    if constexpr (4 * N <= kTwLen) if (np == 4 * N) return launch_colpass_t<N, 4 * N>(a, frames, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_colpass_mixed(const ColArgs& a, int frames, cudaStream_t st);
cudaError_t launch_rowpass_mixed(const RowArgs& a, int frames, cudaStream_t st);

bool colpass2048_applies(const ColArgs& a, int n, int np);
cudaError_t launch_colpass2048(const ColArgs& a, int frames, cudaStream_t st);

cudaError_t launch_colpass(const ColArgs& a, int n, int np, int frames, cudaStream_t st) {
    if (a.tw_n != nullptr) return launch_colpass_mixed(a, frames, st);  // sizes not powers of two
    // cfg2's 2048 -> 4096 column pass on register warp FFTs (colpass2048.cu); OFDMR_COL2048=0 keeps
    // the generic Stockham kernel (cross-check)
    const char* e2048 = getenv("OFDMR_COL2048");
    if (!(e2048 && e2048[0] == '0') && colpass2048_applies(a, n, np)) return launch_colpass2048(a, frames, st);
    switch (n) {
        case 16: return launch_colpass_n<16>(a, np, frames, st);
        case 32: return launch_colpass_n<32>(a, np, frames, st);
        case 64: return launch_colpass_n<64>(a, np, frames, st);
        case 128: return launch_colpass_n<128>(a, np, frames, st);
        case 256: return launch_colpass_n<256>(a, np, frames, st);
        case 512: return launch_colpass_n<512>(a, np, frames, st);
        case 1024: return launch_colpass_n<1024>(a, np, frames, st);
        case 2048: return launch_colpass_n<2048>(a, np, frames, st);
        case 4096: return launch_colpass_n<4096>(a, np, frames, st);
        default: return cudaErrorInvalidValue;
    }
}

template <int MP> constexpr int row_chunk() { return MP >= 4096 ? 1 : MP >= 2048 ? 2 : MP >= 1024 ? 4 : 8; }

bool rowpass_zp_applies(const RowArgs& a, int mp);
int rowpass_zp_rows();
cudaError_t launch_rowpass_zp(const RowArgs& a, int frames, cudaStream_t st);

int rowpass_rows(int mp, int np, int m) {
    // M = 512 -> M' = 2048 (cfg2): rows per block of the zero-padded row pass (rowpass_zp.cu)
    if (mp == 2048 && m == 512 && np >= rowpass_zp_rows()) return rowpass_zp_rows();
    int r = mp >= 4096 ? 4 : mp >= 2048 ? 6 : mp >= 1024 ? 14 : 30;  // R + 2 a multiple of the chunk
    if (r > np) r = np;
    return r;
}

size_t rowpass_smem(int mp, int rows) {
    const int rb = mp >= 4096 ? 1 : mp >= 2048 ? 2 : mp >= 1024 ? 4 : 8;
    // strict 3x3 maxima are never 8-adjacent: at most ceil(R/2) * (M'/2) per block
    const size_t cap = (size_t)((rows + 1) / 2) * (size_t)(mp / 2) + 16;
    return (size_t)((rb * pad_len(mp) + 1) & ~1) * sizeof(float2) + (size_t)(rows + 2) * mp * sizeof(float) +
           cap * sizeof(unsigned long long);
}

template <int MP>
cudaError_t launch_rowpass_t(const RowArgs& a, int frames, cudaStream_t st) {
    constexpr int RB = row_chunk<MP>();
    const size_t smem = rowpass_smem(MP, a.rows_per_block);
    auto kern = rowpass_kernel<MP, RB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((a.n_prime + a.rows_per_block - 1) / a.rows_per_block, frames);
    kern<<<grid, kNT, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_rowpass(const RowArgs& a, int mp, int frames, cudaStream_t st) {
    if (a.tw_mp != nullptr) return launch_rowpass_mixed(a, frames, st);  // M' not a power of two
    if (rowpass_zp_applies(a, mp)) return launch_rowpass_zp(a, frames, st);
    switch (mp) {
        case 16: return launch_rowpass_t<16>(a, frames, st);
        case 32: return launch_rowpass_t<32>(a, frames, st);
        case 64: return launch_rowpass_t<64>(a, frames, st);
        case 128: return launch_rowpass_t<128>(a, frames, st);
        case 256: return launch_rowpass_t<256>(a, frames, st);
        case 512: return launch_rowpass_t<512>(a, frames, st);
        case 1024: return launch_rowpass_t<1024>(a, frames, st);
        case 2048: return launch_rowpass_t<2048>(a, frames, st);
        case 4096: return launch_rowpass_t<4096>(a, frames, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_merge(const MergeArgs& a, int frames, cudaStream_t st) {
    const size_t smem = (size_t)a.nblk * a.kmax * sizeof(unsigned long long);
    cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    merge_kernel<<<frames, kNT, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace ofdmr
