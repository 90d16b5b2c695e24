// Receiver kernels for grids whose sizes are NOT powers of two (the reference's default
// table1 2048 x 560, fig6's M = 200, the desk numerology 512 x 140, ...: FFTW accepts any
// length, src/fft.cpp:35-40).  Same dataflow as radar_kernels.cu (colpass: LS / DFT-CE /
// window / zero-padded delay IFFT_N' per tile of symbol columns; rowpass: zero-padded
// FFT_M', |.|^2 / (NM) with the floor(M'/2) fftshift, strict wrapped 3 x 3 maxima and a
// per-block top-K; the merge kernel is shared), with the transforms done by a runtime
// mixed-radix Stockham engine in shared memory: radices 8, 4, 2, 3, 5, 7, 11, 13 (each pass a
// compile-time radix picked by a switch), twiddles from a per-length fp32 table
// e^{-j 2 pi t / L} built in fp64 on the host.  Lengths must factor into those primes.
#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "fft_smem.cuh"
#include "radar_kernels.cuh"

namespace ofdmr {

namespace {

constexpr int kMrNT = 256;
constexpr int kMrMaxPasses = 24;

struct MrPlan {
    int len;
    int npass;
    int radix[kMrMaxPasses];
};

// W_R^t = e^{-j 2 pi t / R} for the odd radices, fp32-rounded fp64 values
template <int R> struct OddW;
#define ODDW(R, ...)                                                     \
    template <> struct OddW<R> {                                         \
        static __device__ __forceinline__ float2 w(int t) {              \
            constexpr float c[2 * R] = {__VA_ARGS__};                    \
            return make_float2(c[2 * t], c[2 * t + 1]);                  \
        }                                                                \
    };
ODDW(3, 1.0f, 0.0f, -0.5f, -0.86602540378443865f, -0.5f, 0.86602540378443865f)
ODDW(5, 1.0f, 0.0f, 0.30901699437494742f, -0.95105651629515357f, -0.80901699437494742f, -0.58778525229247313f,
     -0.80901699437494742f, 0.58778525229247313f, 0.30901699437494742f, 0.95105651629515357f)
ODDW(7, 1.0f, 0.0f, 0.62348980185873353f, -0.78183148246802981f, -0.22252093395631440f, -0.97492791218182361f,
     -0.90096886790241913f, -0.43388373911755812f, -0.90096886790241913f, 0.43388373911755812f,
     -0.22252093395631440f, 0.97492791218182361f, 0.62348980185873353f, 0.78183148246802981f)
ODDW(11, 1.0f, 0.0f, 0.84125353283118117f, -0.54064081745559758f, 0.41541501300188643f, -0.90963199535451837f,
     -0.14231483827328514f, -0.98982144188093273f, -0.65486073394528506f, -0.75574957435425828f,
     -0.95949297361449739f, -0.28173255684142970f, -0.95949297361449739f, 0.28173255684142970f,
     -0.65486073394528506f, 0.75574957435425828f, -0.14231483827328514f, 0.98982144188093273f,
     0.41541501300188643f, 0.90963199535451837f, 0.84125353283118117f, 0.54064081745559758f)
ODDW(13, 1.0f, 0.0f, 0.88545602565320989f, -0.46472317204376854f, 0.56806474673115581f, -0.82298386589365639f,
     0.12053668025532305f, -0.99270887409805399f, -0.35460488704253562f, -0.93501624268541483f,
     -0.74851074817110109f, -0.66312265824079520f, -0.97094181742605203f, -0.23931566428755777f,
     -0.97094181742605203f, 0.23931566428755777f, -0.74851074817110109f, 0.66312265824079520f,
     -0.35460488704253562f, 0.93501624268541483f, 0.12053668025532305f, 0.99270887409805399f,
     0.56806474673115581f, 0.82298386589365639f, 0.88545602565320989f, 0.46472317204376854f)
#undef ODDW

template <int R, bool INV>
__device__ __forceinline__ void dft_small(float2 (&x)[R]) {
    if constexpr (R == 2) {
        dft2<INV>(x);
    } else if constexpr (R == 4) {
        dft4<INV>(x);
    } else if constexpr (R == 8) {
        dft8<INV>(x);
    } else {  // odd prime radix: direct O(R^2) sum with constant W_R^{tk}
        float2 y[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            float2 acc = x[0];
#pragma unroll
            for (int t = 1; t < R; ++t) {
                float2 w = OddW<R>::w((t * k) % R);
                if (INV) w.y = -w.y;
                acc = cadd(acc, cmul(x[t], w));
            }
            y[k] = acc;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = y[k];
    }
}

// One Stockham pass (radix R, Ls = product of the earlier radices) over nv vectors of length L
// at stride vs: src -> dst.  W_{Ls R}^{i k} = tw[i k L / (Ls R)].
template <int R, bool INV>
__device__ void mr_pass(const float2* src, float2* dst, int vs, int nv, int L, int Ls, const float2* __restrict__ tw) {
    const int T = L / R;
    const int total = nv * T;
    const int tscale = L / (Ls * R);
    for (int b = threadIdx.x; b < total; b += blockDim.x) {
        const int vec = b / T, j = b - vec * T, k = j % Ls;
        float2 x[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            float2 v = src[vec * vs + j + i * T];
            if (i > 0 && k > 0) {
                float2 w = __ldg(tw + (i * k * tscale) % L);
                if (INV) w.y = -w.y;
                v = cmul(v, w);
            }
            x[i] = v;
        }
        dft_small<R, INV>(x);
#pragma unroll
        for (int i = 0; i < R; ++i) dst[vec * vs + (j - k) * R + k + i * Ls] = x[i];
    }
}

// Unscaled FFT (forward e^{-j}, INV e^{+j}) of nv vectors in a (stride vs); b is scratch of the
// same size.  Returns the buffer holding the result.  Ends with a barrier.
template <bool INV>
__device__ float2* mr_fft(float2* a, float2* b, int vs, int nv, const MrPlan& p, const float2* __restrict__ tw) {
    int Ls = 1;
    for (int s = 0; s < p.npass; ++s) {
        const int R = p.radix[s];
        switch (R) {
            case 2: mr_pass<2, INV>(a, b, vs, nv, p.len, Ls, tw); break;
            case 3: mr_pass<3, INV>(a, b, vs, nv, p.len, Ls, tw); break;
            case 4: mr_pass<4, INV>(a, b, vs, nv, p.len, Ls, tw); break;
            case 5: mr_pass<5, INV>(a, b, vs, nv, p.len, Ls, tw); break;
            case 7: mr_pass<7, INV>(a, b, vs, nv, p.len, Ls, tw); break;
            case 8: mr_pass<8, INV>(a, b, vs, nv, p.len, Ls, tw); break;
            case 11: mr_pass<11, INV>(a, b, vs, nv, p.len, Ls, tw); break;
            default: mr_pass<13, INV>(a, b, vs, nv, p.len, Ls, tw); break;
        }
        Ls *= R;
        __syncthreads();
        float2* t = a;
        a = b;
        b = t;
    }
    return a;
}

__device__ double block_sum_mr(double v, double* scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kMrNT / 32; ++i) s += scratch[i];
        scratch[0] = s;
    }
    __syncthreads();
    s = scratch[0];
    __syncthreads();
    return s;
}

// colpass for runtime N, N' (see radar_kernels.cu colpass_kernel for the dataflow)
__global__ void __launch_bounds__(kMrNT) mr_colpass_kernel(ColArgs a, MrPlan pn, MrPlan pnp, int C, int VS) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* bufA = reinterpret_cast<float2*>(smem_raw);
    float2* bufB = bufA + (size_t)C * VS;
    __shared__ double red[kMrNT / 32];
    const int N = a.n, NP = a.np, m = a.m;
    const int f = blockIdx.y, tile = blockIdx.x, c0 = tile * C;
    const size_t fbase = (size_t)f * N * m;
    double inv_acc = 0.0;
    int zero_cell = 0;
    for (int idx = threadIdx.x; idx < N * C; idx += kMrNT) {
        const int k = idx / C, c = idx - k * C;
        const size_t off = fbase + (size_t)k * m + c0 + c;
        float2 h;
        if (a.y != nullptr) {
            const float2 yv = __ldcs(a.y + off), xv = __ldcs(a.x + off);
            h = ls_cell(yv.x, yv.y, xv.x, xv.y, inv_acc, zero_cell);
        } else {
            h = __ldcs(a.h + off);
        }
        bufA[c * VS + k] = h;
        if (a.h_out != nullptr && !a.hout_after_ce) a.h_out[off] = h;
    }
    if (a.y != nullptr) {
        if (zero_cell) atomicOr(a.status + f, 1);
        if (a.inv_partial != nullptr) {
            const double s = block_sum_mr(inv_acc, red);
            if (threadIdx.x == 0) a.inv_partial[(size_t)f * a.ntiles + tile] = s;
        }
    }
    __syncthreads();
    float2* cur = bufA;
    float2* oth = bufB;
    if (a.ce_taps > 0) {
        // dft_ce (estimation.cpp:23-39): IFFT_N, taps < L x 1/N, zero the rest, FFT_N
        cur = mr_fft<true>(cur, oth, VS, C, pn, a.tw_n);
        oth = cur == bufA ? bufB : bufA;
        const float inv_n = 1.0f / (float)N;
        for (int idx = threadIdx.x; idx < C * N; idx += kMrNT) {
            const int c = idx / N, k = idx - c * N;
            float2& v = cur[c * VS + k];
            v = k < a.ce_taps ? cscale(v, inv_n) : make_float2(0.f, 0.f);
        }
        __syncthreads();
        cur = mr_fft<false>(cur, oth, VS, C, pn, a.tw_n);
        oth = cur == bufA ? bufB : bufA;
        if (a.h_out != nullptr && a.hout_after_ce) {
            for (int idx = threadIdx.x; idx < N * C; idx += kMrNT) {
                const int k = idx / C, c = idx - k * C;
                a.h_out[fbase + (size_t)k * m + c0 + c] = cur[c * VS + k];
            }
        }
    }
    if (a.g_out == nullptr) return;
    // window w_k w_l, zero-pad to N', unscaled IFFT_N' (periodogram.cpp:52-60)
    for (int idx = threadIdx.x; idx < C * NP; idx += kMrNT) {
        const int c = idx / NP, k = idx - c * NP;
        float2& v = cur[c * VS + k];
        if (k >= N) v = make_float2(0.f, 0.f);
        else if (a.wk != nullptr) v = cscale(v, a.wk[k] * a.wl[c0 + c]);
    }
    __syncthreads();
    cur = mr_fft<true>(cur, oth, VS, C, pnp, a.tw_np);
    float2* g = a.g_out + (size_t)f * NP * m;
    for (int idx = threadIdx.x; idx < NP * C; idx += kMrNT) {
        const int k = idx / C, c = idx - k * C;
        g[(size_t)k * m + c0 + c] = cur[c * VS + k];
    }
}

constexpr int kMrRowChunk = 2;  // rows transformed together

// rowpass for runtime M' (see radar_kernels.cu rowpass_kernel for the dataflow)
__global__ void __launch_bounds__(kMrNT) mr_rowpass_kernel(RowArgs a, MrPlan pmp, int VS) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int MP = a.mp, R = a.rows_per_block;
    float2* cbA = reinterpret_cast<float2*>(smem_raw);
    float2* cbB = cbA + (size_t)kMrRowChunk * VS;
    float* ptile = reinterpret_cast<float*>(cbB + (size_t)kMrRowChunk * VS);
    unsigned long long* list =
        reinterpret_cast<unsigned long long*>(ptile + (((size_t)(R + 2) * MP + 1) & ~size_t(1)));
    __shared__ int s_cnt;
    __shared__ unsigned long long s_best[kMrNT / 32];
    __shared__ int s_idx[kMrNT / 32];
    __shared__ unsigned long long s_top[kMaxK];
    const int f = blockIdx.y, rb = blockIdx.x, np = a.n_prime;
    const int r0 = rb * R, nrows = min(R, np - r0), TR = nrows + 2, m = a.m;
    const int half = MP / 2;
    if (a.p_in != nullptr) {
        const float* pf = a.p_in + (size_t)f * np * MP;
        for (int idx = threadIdx.x; idx < TR * MP; idx += kMrNT) {
            const int tr = idx / MP, c = idx - tr * MP;
            const int gr = (r0 - 1 + tr + np) % np;
            ptile[(size_t)tr * MP + c] = __ldcs(pf + (size_t)gr * MP + c);
        }
        __syncthreads();
    } else {
        const float2* gf = a.g + (size_t)f * a.g_rows * m;
        for (int t0 = 0; t0 < TR; t0 += kMrRowChunk) {
            for (int idx = threadIdx.x; idx < kMrRowChunk * MP; idx += kMrNT) {
                const int j = idx / MP, s = idx - j * MP;
                const int gr = (r0 - 1 + t0 + j + np) % np;
                float2 v = make_float2(0.f, 0.f);
                if (t0 + j < TR && gr < a.g_rows && s < m) v = __ldcs(gf + (size_t)gr * m + s);
                cbA[j * VS + s] = v;
            }
            __syncthreads();
            const float2* res = mr_fft<false>(cbA, cbB, VS, kMrRowChunk, pmp, a.tw_mp);
            for (int idx = threadIdx.x; idx < kMrRowChunk * MP; idx += kMrNT) {
                const int j = idx / MP, s = idx - j * MP;
                if (t0 + j < TR) {
                    int col = s + half;
                    if (col >= MP) col -= MP;
                    ptile[(size_t)(t0 + j) * MP + col] = cnorm(res[j * VS + s]) * a.scale;
                }
            }
            __syncthreads();
        }
    }
    if (a.p_out != nullptr) {
        float* po = a.p_out + (size_t)f * np * MP + (size_t)r0 * MP;
        for (int idx = threadIdx.x; idx < nrows * MP; idx += kMrNT) {
            const int r = idx / MP, c = idx - r * MP;
            __stcs(po + (size_t)r * MP + c, ptile[(size_t)(r + 1) * MP + c]);
        }
    }
    if (!a.detect) return;
    double eta;
    if (a.eta_in != nullptr) {
        eta = a.eta_in[f];
    } else {
        const double s2h = sigma_h2_warp(a.inv_partial, a.ntiles, f, a.sigma2[f], a.inv_count);
        eta = -s2h * a.log_pfa * a.power_factor;  // periodogram.cpp:80
    }
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int idx = threadIdx.x; idx < nrows * MP; idx += kMrNT) {
        const int tr = idx / MP + 1, c = idx - (tr - 1) * MP;
        const float v = ptile[(size_t)tr * MP + c];
        if (!((double)v >= eta)) continue;
        const int cl = c == 0 ? MP - 1 : c - 1, cr = c == MP - 1 ? 0 : c + 1;
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
    block_topk<kMrNT>(list, s_cnt, a.kmax, s_top, s_best, s_idx);
    __syncthreads();
    unsigned long long* out = a.cand + ((size_t)f * gridDim.x + rb) * a.kmax;
    for (int i = threadIdx.x; i < a.kmax; i += kMrNT) out[i] = s_top[i];
}

// OFDM front end (waveform.cpp:133-166) for a non-power-of-two N: one CTA per (frame, tile of
// C symbols), demodulate = strip the cyclic prefix + unscaled FFT_N, modulate = IFFT_N x 1/N with
// the last n_cp samples as prefix (see ofdm_kernels.cu for the power-of-two version)
__global__ void __launch_bounds__(kMrNT) mr_ofdm_kernel(bool inverse, const float2* __restrict__ in,
                                                        float2* __restrict__ out, int n, int m, int ncp, int ntiles,
                                                        int C, MrPlan pn, const float2* __restrict__ tw) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int VS = n + 1;
    float2* bufA = reinterpret_cast<float2*>(smem_raw);
    float2* bufB = bufA + (size_t)C * VS;
    const int64_t frame = blockIdx.x / ntiles;
    const int l0 = (int)(blockIdx.x % ntiles) * C;
    const int64_t ns = n + ncp;
    if (!inverse) {
        const float2* src = in + frame * (int64_t)m * ns;
        for (int idx = threadIdx.x; idx < C * n; idx += kMrNT) {
            const int c = idx / n, i = idx - c * n, l = l0 + c;
            bufA[c * VS + i] = l < m ? src[(int64_t)l * ns + ncp + i] : make_float2(0.f, 0.f);
        }
        __syncthreads();
        const float2* res = mr_fft<false>(bufA, bufB, VS, C, pn, tw);
        float2* dst = out + frame * (int64_t)n * m;
        for (int idx = threadIdx.x; idx < C * n; idx += kMrNT) {
            const int k = idx / C, c = idx - k * C, l = l0 + c;
            if (l < m) dst[(int64_t)k * m + l] = res[c * VS + k];
        }
    } else {
        const float2* src = in + frame * (int64_t)n * m;
        for (int idx = threadIdx.x; idx < C * n; idx += kMrNT) {
            const int k = idx / C, c = idx - k * C, l = l0 + c;
            bufA[c * VS + k] = l < m ? src[(int64_t)k * m + l] : make_float2(0.f, 0.f);
        }
        __syncthreads();
        const float2* res = mr_fft<true>(bufA, bufB, VS, C, pn, tw);
        const float inv_n = 1.0f / float(n);
        float2* dst = out + frame * (int64_t)m * ns;
        for (int idx = threadIdx.x; idx < C * (int)ns; idx += kMrNT) {
            const int c = idx / (int)ns, j = idx - c * (int)ns, l = l0 + c;
            if (l >= m) continue;
            const int i = j < ncp ? n - ncp + j : j - ncp;
            dst[(int64_t)l * ns + j] = cscale(res[c * VS + i], inv_n);
        }
    }
}

bool mr_factor(int len, MrPlan& p) {
    p.len = len;
    p.npass = 0;
    int r = len;
    while (r % 8 == 0 && p.npass < kMrMaxPasses) { p.radix[p.npass++] = 8; r /= 8; }
    while (r % 4 == 0 && p.npass < kMrMaxPasses) { p.radix[p.npass++] = 4; r /= 4; }
    while (r % 2 == 0 && p.npass < kMrMaxPasses) { p.radix[p.npass++] = 2; r /= 2; }
    for (int q : {3, 5, 7, 11, 13})
        while (r % q == 0 && p.npass < kMrMaxPasses) { p.radix[p.npass++] = q; r /= q; }
    return r == 1;
}

}  // namespace

bool mixed_size_supported(int len) {
    MrPlan p;
    return len >= 2 && len <= 4096 && mr_factor(len, p);
}

int mixed_col_tile(int np, int m) {
    // columns per CTA: two ping-pong buffers of C x (N' + 1) complex within ~100 KiB
    for (int c : {8, 4, 2})
        if (m % c == 0 && size_t(2) * c * (np + 1) * sizeof(float2) <= 100 * 1024) return c;
    return 1;
}

size_t mixed_rowpass_smem(int mp, int rows) {
    const int vs = mp + 1;
    const size_t cap = (size_t)((rows + 1) / 2) * (size_t)((mp + 1) / 2) + 16;
    return size_t(2) * kMrRowChunk * vs * sizeof(float2) + (((size_t)(rows + 2) * mp + 1) & ~size_t(1)) * sizeof(float) +
           cap * sizeof(unsigned long long);
}

cudaError_t launch_colpass_mixed(const ColArgs& a, int frames, cudaStream_t st) {
    MrPlan pn, pnp;
    if (!mr_factor(a.n, pn) || !mr_factor(a.np, pnp) || !a.tw_n || !a.tw_np) return cudaErrorInvalidValue;
    const int C = mixed_col_tile(a.np, a.m);
    const int VS = (a.np > a.n ? a.np : a.n) + 1;
    const size_t smem = size_t(2) * C * VS * sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(mr_colpass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    mr_colpass_kernel<<<dim3(a.m / C, frames), kMrNT, smem, st>>>(a, pn, pnp, C, VS);
    return cudaGetLastError();
}

cudaError_t launch_rowpass_mixed(const RowArgs& a, int frames, cudaStream_t st) {
    MrPlan p;
    if (!mr_factor(a.mp, p) || !a.tw_mp) return cudaErrorInvalidValue;
    const size_t smem = mixed_rowpass_smem(a.mp, a.rows_per_block);
    cudaError_t e = cudaFuncSetAttribute(mr_rowpass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    mr_rowpass_kernel<<<dim3((a.n_prime + a.rows_per_block - 1) / a.rows_per_block, frames), kMrNT, smem, st>>>(
        a, p, a.mp + 1);
    return cudaGetLastError();
}

cudaError_t launch_ofdm_mixed(bool inverse, const float2* in, float2* out, int n, int m, int ncp, int64_t frames,
                              const float2* tw_n, cudaStream_t st) {
    MrPlan pn;
    if (!mr_factor(n, pn) || !tw_n) return cudaErrorInvalidValue;
    int C = 1;
    for (int c : {8, 4, 2})
        if (size_t(2) * c * (n + 1) * sizeof(float2) <= 100 * 1024) {
            C = c;
            break;
        }
    const int ntiles = (m + C - 1) / C;
    const size_t smem = size_t(2) * C * (n + 1) * sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(mr_ofdm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    for (int64_t f0 = 0; f0 < frames;) {
        const int64_t nf = std::min<int64_t>(frames - f0, (int64_t)(0x7fffffff / ntiles));
        const int64_t in_stride = inverse ? (int64_t)n * m : (int64_t)m * (n + ncp);
        const int64_t out_stride = inverse ? (int64_t)m * (n + ncp) : (int64_t)n * m;
        mr_ofdm_kernel<<<(unsigned)(nf * ntiles), kMrNT, smem, st>>>(inverse, in + f0 * in_stride, out + f0 * out_stride,
                                                                    n, m, ncp, ntiles, C, pn, tw_n);
        f0 += nf;
    }
    return cudaGetLastError();
}

}  // namespace ofdmr
