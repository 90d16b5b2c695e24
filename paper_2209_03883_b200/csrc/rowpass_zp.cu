// Symbol-axis (Doppler) row pass for M = 512 symbols zero-padded to M' = 2048 (BASELINE cfg2:
// 2048 x 512 frames -> 4096 x 2048 periodogram), with |.|^2 / (N M), the fftshift, the optional
// map store and the strict wrapped 3x3 local-maximum detection fused in
// (periodogram.cpp:39-75 rows + :77-136).  Replaces the shared-memory Stockham rowpass_kernel
// (radar_kernels.cu) at this shape; same RowArgs contract, same per-block candidate output.
//
// Zero padding: only the first M = M'/4 inputs of a row are non-zero, so
//     X[m1 + 4 k] = FFT_512( x[l] W_2048^{l m1} )[k],   m1 = 0..3,  l, k < 512
// i.e. four 512-point FFTs of modulated copies of the row instead of one 2048-point FFT
// whose first two radix-2 stages would only see zeros.  Each FFT_512 runs on one half-warp
// (16 lanes x 32 values in registers): lane j holds y[j + 16 n]; DFT_32 over n; twiddle
// W_512^{j k1} (the per-lane modulation factor W_2048^{j m1} folded into the same table); one
// transpose through the half-warp's own XOR-swizzled 16 x 16 shared-memory slot in two steps
// (k1 < 16, then k1 >= 16: conflict-free both ways, 2 KiB per half-warp), each followed by one
// DFT_16 over j per lane.  A warp-unit is (row, pass): its half-warps take m1 = 2 pass and
// 2 pass + 1, so one |.|^2 store of the warp covers adjacent Doppler bins.  16 warps per CTA
// (128 registers per thread), 32 units per tile: two balanced rounds.
//
// A CTA produces R = 14 output rows and computes R + 2 rows (one halo row each side, the 3x3
// test needs them) into a shared-memory P tile.  Detection: while a row's |.|^2 values are
// still in registers, the (rare, ~P_fa) cells >= eta of the interior rows are appended to a
// shared-memory list; after the tile is complete only those cells take the strict wrapped 3x3
// test, and the surviving maxima are ranked against each other directly (keys are unique, the
// rank is the count of larger keys) -- no scan of the tile and no block-wide argmax rounds.
// A tile with more than kZCand cells above the threshold (eta at or below the noise floor)
// falls back to the full scan with per-thread top-8 lists and the block-wide top-K.
// 1/(N M) is folded into the post twiddles when its square root is a power of two (exact).
#include "fft_smem.cuh"
#include "radar_kernels.cuh"
#include "warp_fft.cuh"

#include <math.h>

namespace ofdmr {

namespace {

#ifndef ZP_WARPS
#define ZP_WARPS 16
#endif
constexpr int kZM = 512, kZMP = 2048, kZR = 14, kZTR = kZR + 2, kZW = ZP_WARPS, kZK = 8;
constexpr int kZThreads = 32 * kZW;
constexpr int kZCand = 2048;       // cells >= eta per tile kept for the 3x3 test (more: full scan)
constexpr int kZSurv = kZThreads;  // strict local maxima per tile ranked directly (more: full scan)

struct ZpSmem {
    float ptile[kZTR * kZMP];     // P rows r0 - 1 .. r0 + R (mod N'), fft-shifted
    float2 sc[2 * kZW][16 * 16];  // per half-warp 16 x 16 transpose slot [kk][j ^ kk]; full-scan path: the key list
    float2 post[4][32 * 16];      // post[m1][k1 * 16 + j] = W_2048^{j (4 k1 + m1)} (x sqrt(scale) when exact)
    float2 pre[128];              // W_128^q
    unsigned cand[kZCand];        // (tile row << 11) | physical column of the cells >= eta
    unsigned long long surv[kZSurv];
    unsigned long long best[kZW];
    int idx[kZW];
    unsigned long long top[kMaxK];
    unsigned cnt[2][2];           // [item parity][candidates, survivors]
    float eta_f;  // smallest float >= eta: (double)v >= eta  <=>  v >= eta_f (exact)
};
static_assert(2 * kZW * 16 * 16 * sizeof(float2) >= kZThreads * kZK * sizeof(unsigned long long), "key list");

// P tile column swizzle: flips bit 1 when bit 5 is set, so the 32 lanes of one |.|^2 store
// (m = m1 + 4 j + .., m1 in {a, a + 1}) hit 32 distinct banks; an aligned float4 of the tile
// holds logical columns c0 + (u ^ 2 * bit5(c0)).  An involution: logical = zp_phys(physical).
__device__ __forceinline__ int zp_phys(int m) { return m ^ (((m >> 5) & 1) << 1); }

// strict wrapped 3x3 local-maximum test of tile cell (tr, physical column pc) holding v
__device__ __forceinline__ bool zp_is_peak(const float* ptile, int tr, int pc, float v) {
    const int c = zp_phys(pc);
    const int pl = zp_phys((c - 1) & (kZMP - 1)), pr = zp_phys((c + 1) & (kZMP - 1));
    const float* mid = ptile + tr * kZMP;
    const float* up = mid - kZMP;
    const float* dn = mid + kZMP;
    return !(up[pl] >= v || up[pc] >= v || up[pr] >= v || mid[pl] >= v || mid[pr] >= v || dn[pl] >= v ||
             dn[pc] >= v || dn[pr] >= v);
}

}  // namespace

// PRES: the 1/(N M) scale is an even power of two and folded into the post twiddles (exact)
template <bool PRES>
__global__ void __launch_bounds__(kZThreads, 1) rowpass_zp_kernel(RowArgs a, int frames) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ZpSmem& s = *reinterpret_cast<ZpSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int hw = tid >> 4, j = tid & 15, hsel = (tid >> 4) & 1;
    const int np = a.n_prime;
    const int nblk = (np + kZR - 1) / kZR;
    const float fin = PRES ? 1.f : a.scale;

    // twiddle tables (host-built, zp_tw layout: post[4][512] then pre[128]), once per CTA
    {
        const float rs = PRES ? sqrtf(a.scale) : 1.f;
        const float4* src = reinterpret_cast<const float4*>(a.zp_tw);
        float4* dst = reinterpret_cast<float4*>(&s.post[0][0]);
        for (int i = tid; i < (4 * 512 + 128) / 2; i += kZThreads) {
            float4 v = __ldg(src + i);
            if (PRES && i < 4 * 512 / 2) v = make_float4(v.x * rs, v.y * rs, v.z * rs, v.w * rs);
            dst[i] = v;
        }
    }
    // persistent over (frame, row block) items; consecutive items of a CTA are usually of one frame
    int cur_f = -1, par = 0;
    for (int it = blockIdx.x; it < frames * nblk; it += gridDim.x, par ^= 1) {
    const int f = it / nblk, rb = it - f * nblk, r0 = rb * kZR;
    const int nrows = min(kZR, np - r0), TR = nrows + 2;
    if (tid == 0) {  // this parity's counters were last read two items ago
        s.cnt[par][0] = 0;
        s.cnt[par][1] = 0;
    }
    if (f != cur_f && warp == 0 && a.detect) {
        // threshold once per frame (sigma_h^2 in the order the merge kernel reports it)
        double eta;
        if (a.eta_in != nullptr) {
            eta = a.eta_in[f];
        } else {
            const double s2h = sigma_h2_warp(a.inv_partial, a.ntiles, f, a.sigma2[f], a.inv_count);
            eta = -s2h * a.log_pfa * a.power_factor;  // periodogram.cpp:80
        }
        float e = (float)eta;
        if ((double)e < eta) e = nextafterf(e, INFINITY);
        if (lane == 0) s.eta_f = e;
    }
    cur_f = f;
    __syncthreads();  // tables / eta / counters visible; the previous item's tile, slots and lists are free
    const float eta_f = a.detect ? s.eta_f : INFINITY;

    // ---- 1. P tile: rows (r0 - 1 + t) mod N', t < TR; a warp-unit is (row, pass): m1 = hsel + 2 pass
    const float2* gf = a.g + (size_t)f * a.g_rows * kZM;
    float2* sc = s.sc[hw];
    for (int u = warp; u < 2 * TR; u += kZW) {
        const int t = u >> 1, pass = u & 1;
        const int gr = (r0 - 1 + t + np) % np;
        float* prow = s.ptile + t * kZMP;
        if (gr >= a.g_rows) {  // DFT-CE shortcut rows: exactly zero
            for (int c = lane; c < kZMP / 2; c += 32) prow[pass * (kZMP / 2) + c] = 0.f;
            continue;
        }
        const bool interior = t >= 1 && t <= nrows;
        const float2* grow = gf + (size_t)gr * kZM;
        const int m1 = hsel + 2 * pass;
        float2 v[32];
#pragma unroll
        for (int n = 0; n < 32; ++n) v[n] = __ldg(grow + j + 16 * n);
        // m1 = 0 multiplies by pre[0] = 1 exactly: no divergent branch between the half-warps
#pragma unroll
        for (int n = 1; n < 32; ++n) v[n] = cmul(v[n], s.pre[(m1 * n) & 127]);
        dft32<false>(v);
        const float2* pw = s.post[m1] + j;
#pragma unroll
        for (int k1 = 0; k1 < 32; ++k1) v[k1] = cmul(v[k1], pw[k1 * 16]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            __syncwarp();  // the slot's previous readers are done
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) sc[kk * 16 + (j ^ kk)] = v[16 * h + kk];
            __syncwarp();
            float2 w[16];
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) w[jj] = sc[j * 16 + (jj ^ j)];
            dft16<false>(w);
            // X[m1 + 4 (k1 + 32 k2)], k1 = j + 16 h, fft-shifted by M'/2
            // zp_phys only flips bit 1 from bit 5, which the 128 k2 steps leave unchanged
            const int base = zp_phys(m1 + 4 * (j + 16 * h) + kZMP / 2);
            float val[16], vmax = 0.f;
#pragma unroll
            for (int k2 = 0; k2 < 16; ++k2) {
                val[k2] = cnorm(w[k2]) * fin;
                prow[(base + 128 * k2) & (kZMP - 1)] = val[k2];
                vmax = fmaxf(vmax, val[k2]);
            }
            if (interior && vmax >= eta_f) {  // rare: ~P_fa of the cells
#pragma unroll
                for (int k2 = 0; k2 < 16; ++k2)
                    if (val[k2] >= eta_f) {
                        const unsigned i = atomicAdd(&s.cnt[par][0], 1u);
                        if (i < (unsigned)kZCand) s.cand[i] = ((unsigned)t << 11) | (unsigned)((base + 128 * k2) & (kZMP - 1));
                    }
            }
        }
    }
    __syncthreads();

    // the next item's G rows (16 x 4 KiB) into L2 while this one stores / detects
    {
        const int nit = it + gridDim.x;
        if (nit < frames * nblk) {
            const int nf = nit / nblk, nr0 = (nit - nf * nblk) * kZR;
            const char* gb = reinterpret_cast<const char*>(a.g + (size_t)nf * a.g_rows * kZM);
            for (int i = tid; i < kZTR * 32; i += kZThreads) {  // 32 lines of 128 B per row
                const int gr = (nr0 - 1 + i / 32 + np) % np;
                if (gr < a.g_rows) asm volatile("prefetch.global.L2 [%0];" ::"l"(gb + (size_t)gr * kZM * 8 + (i % 32) * 128));
            }
        }
    }

    // ---- 2. map store (interior rows)
    if (a.p_out != nullptr) {
        float* po = a.p_out + (size_t)f * np * kZMP + (size_t)r0 * kZMP;
        for (int i = tid; i < nrows * (kZMP / 4); i += kZThreads) {
            const int r = i / (kZMP / 4), q = i % (kZMP / 4);
            float4 v = reinterpret_cast<const float4*>(s.ptile + (r + 1) * kZMP)[q];
            if ((q >> 3) & 1) v = make_float4(v.z, v.w, v.x, v.y);  // undo zp_phys
            __stcs(reinterpret_cast<float4*>(po + (size_t)r * kZMP) + q, v);
        }
    }
    if (!a.detect) continue;

    // ---- 3. strict wrapped 3x3 local maxima among the cells >= eta, top-K (periodogram.cpp:77-136)
    unsigned long long* out = a.cand + ((size_t)f * nblk + rb) * a.kmax;
    const unsigned nc = s.cnt[par][0];
    bool full_scan = nc > (unsigned)kZCand;
    if (!full_scan) {
        for (unsigned i = tid; i < nc; i += kZThreads) {
            const unsigned e = s.cand[i];
            const int tr = (int)(e >> 11), pc = (int)(e & (kZMP - 1));
            const float v = s.ptile[tr * kZMP + pc];
            if (zp_is_peak(s.ptile, tr, pc, v)) {
                const unsigned k = atomicAdd(&s.cnt[par][1], 1u);
                if (k < (unsigned)kZSurv) s.surv[k] = make_key(v, (uint32_t)((r0 + tr - 1) * kZMP + zp_phys(pc)));
            }
        }
        __syncthreads();
        const unsigned ns = s.cnt[par][1];
        if (ns > (unsigned)kZSurv) {
            full_scan = true;
        } else {
            // keys are unique: a survivor's rank is the number of larger keys
            if ((unsigned)tid < ns) {
                const unsigned long long key = s.surv[tid];
                int rank = 0;
                for (unsigned q = 0; q < ns; ++q) rank += s.surv[q] > key ? 1 : 0;
                if (rank < a.kmax) out[rank] = key;
            } else if (tid < a.kmax) {
                out[tid] = 0ull;
            }
        }
    }
    if (!full_scan) continue;

    // ---- 3b. full scan of the tile (threshold at or below the noise floor: rare), per-thread top-8
    unsigned long long top[kZK];
#pragma unroll
    for (int i = 0; i < kZK; ++i) top[i] = 0ull;
    for (int i = tid; i < nrows * (kZMP / 4); i += kZThreads) {
        const int tr = i / (kZMP / 4) + 1, c0 = 4 * (i % (kZMP / 4));
        const float4 q4 = *reinterpret_cast<const float4*>(s.ptile + tr * kZMP + c0);
        if (!(q4.x >= eta_f || q4.y >= eta_f || q4.z >= eta_f || q4.w >= eta_f)) continue;
        const float qv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float v = qv[u];
            if (!(v >= eta_f)) continue;
            if (!zp_is_peak(s.ptile, tr, c0 + u, v)) continue;
            unsigned long long key = make_key(v, (uint32_t)((r0 + tr - 1) * kZMP + zp_phys(c0 + u)));
#pragma unroll
            for (int q = 0; q < kZK; ++q) {  // sorted insert (descending), keys unique
                const unsigned long long t = top[q];
                top[q] = key > t ? key : t;
                key = key > t ? t : key;
            }
        }
    }
    unsigned long long* list = reinterpret_cast<unsigned long long*>(&s.sc[0][0]);  // slots are free
#pragma unroll
    for (int q = 0; q < kZK; ++q) list[q * kZThreads + tid] = top[q];
    __syncthreads();
    block_topk<kZThreads>(list, kZThreads * kZK, a.kmax, s.top, s.best, s.idx);
    __syncthreads();
    for (int i = tid; i < a.kmax; i += kZThreads) out[i] = s.top[i];
    }
}

bool rowpass_zp_applies(const RowArgs& a, int mp) {
    return a.g != nullptr && a.p_in == nullptr && mp == kZMP && a.m == kZM && a.kmax <= kZK &&
           a.rows_per_block == kZR;
}

int rowpass_zp_rows() { return kZR; }

cudaError_t launch_rowpass_zp(const RowArgs& a, int frames, cudaStream_t st) {
    const size_t smem = sizeof(ZpSmem);
    // 1/(N M) = 4^-k: sqrt(scale) is a power of two and goes into the twiddles without rounding
    const float rs = sqrtf(a.scale);
    int ex = 0;
    const bool pres = a.scale > 0.f && rs * rs == a.scale && frexpf(rs, &ex) == 0.5f && a.scale > 1e-30f;
    auto kern = pres ? rowpass_zp_kernel<true> : rowpass_zp_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int items = frames * ((a.n_prime + kZR - 1) / kZR);
    kern<<<items < sms ? items : sms, kZThreads, smem, st>>>(a, frames);
    return cudaGetLastError();
}

}  // namespace ofdmr
