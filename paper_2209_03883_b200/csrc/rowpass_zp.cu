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
// transpose through the half-warp's own XOR-swizzled shared-memory slot (conflict-free both
// ways); two DFT_16 over j per lane.  A warp handles one row: its half-warps take m1 = 0, 2
// and 1, 3.
//
// A CTA produces R = 14 output rows and computes R + 2 rows (one halo row each side, the 3x3
// test needs them) into a shared-memory P tile; the detection keeps a per-thread top-8 of the
// strict local maxima >= eta in registers (keys are unique), then one block-wide top-K.
#include "fft_smem.cuh"
#include "radar_kernels.cuh"
#include "warp_fft.cuh"

#include <math.h>

namespace ofdmr {

namespace {

constexpr int kZM = 512, kZMP = 2048, kZR = 14, kZTR = kZR + 2, kZW = 8, kZK = 8;
constexpr int kZThreads = 32 * kZW;

struct ZpSmem {
    float ptile[kZTR * kZMP];     // P rows r0 - 1 .. r0 + R (mod N'), fft-shifted
    float2 sc[2 * kZW][32 * 16];  // per half-warp transpose slot [k1][j ^ (k1 & 15)]; later the key list
    float2 post[4][32 * 16];      // post[m1][k1 * 16 + j] = W_2048^{j (4 k1 + m1)}
    float2 pre[128];              // W_128^q
    unsigned long long best[kZW];
    int idx[kZW];
    unsigned long long top[kMaxK];
    float eta_f;  // smallest float >= eta: (double)v >= eta  <=>  v >= eta_f (exact)
};
static_assert(2 * kZW * 32 * 16 * sizeof(float2) >= kZThreads * kZK * sizeof(unsigned long long), "key list");

// P tile column swizzle: flips bit 1 when bit 5 is set, so the 32 lanes of one |.|^2 store
// (m = m1 + 4 j + .., m1 in {a, a + 1}) hit 32 distinct banks; an aligned float4 of the tile
// holds logical columns c0 + (u ^ 2 * bit5(c0))
__device__ __forceinline__ int zp_phys(int m) { return m ^ (((m >> 5) & 1) << 1); }

}  // namespace

__global__ void __launch_bounds__(kZThreads, 1) rowpass_zp_kernel(RowArgs a, int frames) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ZpSmem& s = *reinterpret_cast<ZpSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int hw = tid >> 4, j = tid & 15, hsel = (tid >> 4) & 1;
    const int np = a.n_prime;
    const int nblk = (np + kZR - 1) / kZR;

    // twiddle tables (host-built, zp_tw layout: post[4][512] then pre[128]), once per CTA
    {
        const float4* src = reinterpret_cast<const float4*>(a.zp_tw);
        float4* dst = reinterpret_cast<float4*>(&s.post[0][0]);
        for (int i = tid; i < (4 * 512 + 128) / 2; i += kZThreads) dst[i] = __ldg(src + i);
    }
    // persistent over (frame, row block) items; consecutive items of a CTA are usually of one frame
    int cur_f = -1;
    for (int it = blockIdx.x; it < frames * nblk; it += gridDim.x) {
    const int f = it / nblk, rb = it - f * nblk, r0 = rb * kZR;
    const int nrows = min(kZR, np - r0), TR = nrows + 2;
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
    __syncthreads();  // tables / eta visible; the previous item's tile, slots and key list are free

    // ---- 1. P tile: rows (r0 - 1 + t) mod N', t < TR
    const float2* gf = a.g + (size_t)f * a.g_rows * kZM;
    float2* sc = s.sc[hw];
    for (int t = warp; t < TR; t += kZW) {
        const int gr = (r0 - 1 + t + np) % np;
        float* prow = s.ptile + t * kZMP;
        if (gr >= a.g_rows) {  // DFT-CE shortcut rows: exactly zero
            for (int c = lane; c < kZMP; c += 32) prow[c] = 0.f;
            continue;
        }
        const float2* grow = gf + (size_t)gr * kZM;
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
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
            __syncwarp();
#pragma unroll
            for (int k1 = 0; k1 < 32; ++k1) sc[k1 * 16 + (j ^ (k1 & 15))] = v[k1];
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int k1 = j + 16 * h;
                float2 w[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) w[jj] = sc[k1 * 16 + (jj ^ j)];
                dft16<false>(w);
                // X[m1 + 4 (k1 + 32 k2)], fft-shifted by M'/2
                // zp_phys only flips bit 1 from bit 5, which the 128 k2 steps leave unchanged
                const int base = zp_phys(m1 + 4 * k1 + kZMP / 2);
#pragma unroll
                for (int k2 = 0; k2 < 16; ++k2) prow[(base + 128 * k2) & (kZMP - 1)] = cnorm(w[k2]) * a.scale;
            }
            __syncwarp();  // the slot is rewritten by the next pass
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

    // ---- 3. threshold + strict wrapped 3x3 local maxima, per-thread top-8 (periodogram.cpp:77-136)
    const float eta_f = s.eta_f;
    unsigned long long top[kZK];
#pragma unroll
    for (int i = 0; i < kZK; ++i) top[i] = 0ull;
    for (int i = tid; i < nrows * (kZMP / 4); i += kZThreads) {
        const int tr = i / (kZMP / 4) + 1, c0 = 4 * (i % (kZMP / 4));
        const float* mid = s.ptile + tr * kZMP;
        const float4 q4 = *reinterpret_cast<const float4*>(mid + c0);
        if (!(q4.x >= eta_f || q4.y >= eta_f || q4.z >= eta_f || q4.w >= eta_f)) continue;
        const float qv[4] = {q4.x, q4.y, q4.z, q4.w};
        const int sw = ((c0 >> 5) & 1) << 1;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float v = qv[u];
            if (!(v >= eta_f)) continue;
            const int c = c0 + (u ^ sw);  // logical column; physical c0 + u
            const int pc = c0 + u, pl = zp_phys((c - 1) & (kZMP - 1)), pr = zp_phys((c + 1) & (kZMP - 1));
            const float* up = mid - kZMP;
            const float* dn = mid + kZMP;
            if (up[pl] >= v || up[pc] >= v || up[pr] >= v || mid[pl] >= v || mid[pr] >= v || dn[pl] >= v ||
                dn[pc] >= v || dn[pr] >= v)
                continue;
            unsigned long long key = make_key(v, (uint32_t)((r0 + tr - 1) * kZMP + c));
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
    unsigned long long* out = a.cand + ((size_t)f * nblk + rb) * a.kmax;
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
    cudaError_t e = cudaFuncSetAttribute(rowpass_zp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int items = frames * ((a.n_prime + kZR - 1) / kZR);
    rowpass_zp_kernel<<<items < sms ? items : sms, kZThreads, smem, st>>>(a, frames);
    return cudaGetLastError();
}

}  // namespace ofdmr
