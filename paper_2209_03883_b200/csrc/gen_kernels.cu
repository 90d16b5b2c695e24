// GPU frame generator: the CPU generator (csrc/gen.cpp, itself a
// restatement of the reference's make_random_frame / apply_channel / Rng, see the header of
// include/ofdmr_gen.h) executed on the device, one CTA (256 threads) per frame, so 8192-frame
// runs need no PCIe traffic.
//
// Every random stream is the reference's std::mt19937_64 stream:
//   scene   Rng(derive_seed(fs, 0x7363656e))   thread 0, sequential
//   phases  Rng(derive_seed(fs, 0x70686173))   thread 0, sequential  (channel.cpp:74-83)
//   pilots  Rng(derive_seed(fx, 0))            warp 0, parallel twist (waveform.cpp:92-96)
//   payload Rng(derive_seed(fx, 1))            warp 0, parallel twist (waveform.cpp:97-108)
//   noise   Rng(derive_seed(fs, 0x6e6f6973))   warp 0, parallel twist (channel.cpp:90-95)
// with fs = derive_seed(base_seed, frame), fx = derive_seed(fs, 0x667261).  The twist is
// parallelised across the warp in its two data-independent halves; draws are consumed in the
// reference's order: one pilot per subcarrier row, bps payload bits per payload cell
// (MSB first), one Box-Muller pair per cell with the imaginary part taking the first normal
// (GCC evaluates `cplx(sd*normal(), sd*normal())` right to left, checked in
// tests/test_gpu_parity.py against the CPU generator).  Rejection draws (uniform_int at
// v >= limit, Box-Muller at u1 == 0; probability ~2^-50 per frame) set status bit 0 and the
// host regenerates that frame on the CPU.
//
// Arithmetic is fp64 in the CPU code's operation order (compiled with -fmad=false, IEEE
// div/sqrt); sin/cos/log/pow are the GPU's (<= 2 ulp), so rare c64 cells differ by 1 ulp.
// mean_power(x) is summed sequentially in cell order by one thread, as the CPU does.
// Pass 1 writes x_tx (and the running |x|^2 sum); pass 2 re-reads x_tx (exact decode of the
// c64 value back to its fp64 constellation point), applies the channel and adds the noise.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include <cuda_runtime.h>

#include "../../include/ofdmr_gen.h"
#include "mt64.cuh"

namespace ofdmr {
namespace {

constexpr double kTwoPiG = 6.283185307179586476925286766559;
constexpr double kCG = 3.0e8;
constexpr int kMaxT = 16;
constexpr int kMaxM = 1024;
// 8 consumer warps (one cell per thread and row) + warp 8, which draws row k + 1's MT19937-64
// outputs while the consumers process row k (the draws' order and values are unchanged)
constexpr int kGenThreads = 288;
constexpr int kProducerWarp = 8;
using namespace mt64;

struct GenArgs {
    ofdmr_gen_params p;
    uint64_t base_seed;
    int64_t first;
    int count;
    float2* y;
    float2* x;
    double* sigma2;
    int32_t* n_targets;
    double* ranges;
    double* vels;
    double* snr_db;
    int max_targets;
    int32_t* status;
    int bps;
    int levels;             // per-axis constellation levels
    double lev_d[16];       // axis level values (fp64, gen.cpp's li * scale), by Gray-decoded index
    float lev_f[16];        // the same rounded to fp32 (decode of the stored c64 x)
    int lev_of_gray[16];    // Gray code -> level index
    double inv_sqrt2;
    uint32_t ring_mask;     // ring size - 1 (power of two >= bits per row + 312)
    double2* h_true;        // optional: true_channel (channel.cpp:100-109) as c128 [count][N][M]
    int explicit_scene;     // 1: fixed targets / SNR below instead of the scene stream
    int exp_count;
    double exp_range[kMaxT], exp_vel[kMaxT];
    double exp_snr;
    // ZC-precoded frames (zadoffchu.cpp:58-87,133-136) run as three launches:
    //   mode 1: scene + pilots + payload -> fp64 x in xd (no channel),
    //   (precode_kernel: x_tx = Z x per column, fp64),
    //   mode 2: scene again (same streams), mean_power of the fp64 x_tx, channel + noise.
    int fph_rows;           // target rows of the fph table in shared memory (max targets of the launch)
    int uniform_power;      // 1: every cell has the same |x|^2 (QPSK): mean_power's sequential sum is
    double uniform_mp;      //    frame-independent, summed once on the host in the same order
    int mode;               // 0: unprecoded single pass
    double2* xd;            // mode 1: fp64 x out; mode 2: fp64 x_tx in ([count][N][M])
};

struct GenShared {
    uint64_t mt[kMtN];
    int ntar;
    int rej;
    double snr_db;
    double b_re[kMaxT], b_im[kMaxT], delay[kMaxT], dopp[kMaxT];
    double d_re2[2][kMaxT], d_im2[2][kMaxT];  // delay phasors of rows k (k & 1) and k + 1
    double mp;                        // running sequential sum of |x|^2
    double sd;
};

// dynamic smem after GenShared: fph[kMaxT][M] double2, nrm[2][M] double, pilot codes [N] bytes,
// draw ring [ring] u64
__global__ void __launch_bounds__(kGenThreads) gen_frame_kernel(GenArgs a) {
    extern __shared__ __align__(16) unsigned char gsm[];
    GenShared& s = *reinterpret_cast<GenShared*>(gsm);
    const ofdmr_gen_params& p = a.p;
    const int n = p.n, m = p.m, tid = threadIdx.x, w = tid >> 5;
    double2* fph = reinterpret_cast<double2*>(gsm + ((sizeof(GenShared) + 15) & ~size_t(15)));
    double* nrm = reinterpret_cast<double*>(fph + (size_t)a.fph_rows * m);
    uint64_t* ring = reinterpret_cast<uint64_t*>(nrm + 2 * m);
    unsigned char* pil = reinterpret_cast<unsigned char*>(ring + a.ring_mask + 1);

    const int f = blockIdx.x;
    const int64_t fidx = a.first + f;
    const uint64_t fs = splitmix(a.base_seed, (uint64_t)fidx);
    const uint64_t fx = splitmix(fs, 0x667261ull);
    float2* xo = a.x + (size_t)f * n * m;
    float2* yo = a.y + (size_t)f * n * m;

    // ---- scene + per-target constants (thread 0, sequential streams)
    if (tid == 0) {
        int rej = 0;
        int cnt;
        double rg[kMaxT], vl[kMaxT];
        double snr;
        if (a.explicit_scene) {  // run_pipeline with the scenario's targets (pipeline.cpp:65-71)
            cnt = a.exp_count;
            for (int t = 0; t < cnt; ++t) {
                rg[t] = a.exp_range[t];
                vl[t] = a.exp_vel[t];
            }
            snr = a.exp_snr;
        } else {
            MtScalar r{s.mt, kMtN};
            mt_seed(s.mt, splitmix(fs, 0x7363656eull));
            cnt = p.targets_min;
            if (p.targets_max > p.targets_min)
                cnt += (int)r.uniform_int((uint64_t)(p.targets_max - p.targets_min + 1), rej);
            for (int t = 0; t < cnt; ++t) {
                rg[t] = r.uniform(p.range_lo, p.range_hi);
                vl[t] = r.uniform(p.vel_lo, p.vel_hi);
            }
            snr = p.snr_lo_db;
            if (p.snr_hi_db != p.snr_lo_db && isfinite(p.snr_lo_db)) snr = r.uniform(p.snr_lo_db, p.snr_hi_db);
        }
        // phases (channel.cpp:74-83)
        MtScalar ph{s.mt, kMtN};
        mt_seed(s.mt, splitmix(fs, 0x70686173ull));
        for (int t = 0; t < cnt; ++t) {
            const double phase = ph.uniform(0.0, kTwoPiG);
            const double gain = 1.0;
            s.delay[t] = 2.0 * rg[t] / kCG;
            s.dopp[t] = 2.0 * vl[t] * p.fc_hz / kCG;
            double sn, cs;
            sincos(phase, &sn, &cs);
            s.b_re[t] = gain * cs;
            s.b_im[t] = gain * sn;
        }
        s.ntar = cnt;
        s.rej = rej;
        s.snr_db = snr;
        s.mp = a.uniform_power ? a.uniform_mp : 0.0;
        if (a.n_targets) a.n_targets[f] = cnt;
        if (a.snr_db) a.snr_db[f] = snr;
        for (int t = 0; t < cnt && t < a.max_targets; ++t) {
            if (a.ranges) a.ranges[(size_t)f * a.max_targets + t] = rg[t];
            if (a.vels) a.vels[(size_t)f * a.max_targets + t] = vl[t];
        }
    }
    __syncthreads();
    const int T = s.ntar;
    const double t_useful = 1.0 / p.df_hz;
    const double ts = t_useful + (double)p.n_cp * (t_useful / (double)n);
    for (int i = tid; tid < 256 && i < T * m; i += 256) {
        const int t = i / m, l = i % m;
        double sn, cs;
        sincos(kTwoPiG * (double)l * ts * s.dopp[t], &sn, &cs);
        fph[(size_t)t * m + l] = make_double2(1.0 * cs, 1.0 * sn);
    }

    // ---- pilots: n draws of uniform_int(4) (warp 0)
    const uint32_t mask = a.ring_mask;
    double2* xdf = a.xd ? a.xd + (size_t)f * n * m : nullptr;
    if (a.mode != 2) {
    if (w == 0) {
        if (tid == 0) mt_seed(s.mt, splitmix(fx, 0ull));
        __syncwarp();
        int rej = 0;
        for (int k0 = 0; k0 < n; k0 += kMtN) {
            mt_block(s.mt, ring, 0, mask);
            for (int i = tid; i < kMtN && k0 + i < n; i += 32) {
                const uint64_t v = ring[i];
                if (v >= 0xFFFFFFFFFFFFFFFCull) rej = 1;
                pil[k0 + i] = (unsigned char)(v % 4);
            }
            __syncwarp();
        }
        if (__any_sync(0xffffffffu, rej) && tid == 0) s.rej = 1;
        if (tid == 0) mt_seed(s.mt, splitmix(fx, 1ull));  // payload stream
    }
    __syncthreads();

    // ---- pass 1: x_tx row by row; mean_power summed sequentially (warp 1, lane 0)
    const int bps = a.bps, half = bps / 2;
    const uint32_t need = (uint32_t)(m - 1) * bps;  // payload draws per row
    uint32_t produced = 0, consumed = 0;             // produced: producer warp only
    if (w == kProducerWarp)
        while (produced < need) {  // row 0
            mt_block(s.mt, ring, produced, mask);
            produced += kMtN;
        }
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        double* nr = nrm + (k & 1) * m;
        if (w == kProducerWarp) {
            // row k + 1's draws land behind row k's window (ring >= 2 rows + one block)
            if (k + 1 < n)
                while (produced < consumed + 2 * need) {
                    mt_block(s.mt, ring, produced, mask);
                    produced += kMtN;
                }
        } else {
            for (int l = tid; l < m; l += 256) {
                double xr, xi;
                if (l == 0) {
                    const unsigned b = pil[k];
                    xr = (b & 1) ? -a.inv_sqrt2 : a.inv_sqrt2;
                    xi = (b & 2) ? -a.inv_sqrt2 : a.inv_sqrt2;
                } else {
                    unsigned wd = 0;
                    const uint32_t base = consumed + (uint32_t)(l - 1) * bps;
                    for (int b = 0; b < bps; ++b) {
                        const uint64_t v = ring[(base + b) & mask];
                        if (v >= 0xFFFFFFFFFFFFFFFEull) atomicOr(&s.rej, 1);
                        wd = (wd << 1) | (unsigned)(v & 1ull);
                    }
                    const unsigned gi = wd >> half, gq = wd & ((1u << half) - 1u);
                    xr = a.lev_d[a.lev_of_gray[gi]];
                    xi = a.lev_d[a.lev_of_gray[gq]];
                }
                if (a.mode == 1) {
                    xdf[(size_t)k * m + l] = make_double2(xr, xi);
                } else {
                    xo[(size_t)k * m + l] = make_float2((float)xr, (float)xi);
                    nr[l] = xr * xr + xi * xi;
                }
            }
        }
        consumed += need;
        __syncthreads();
        if (tid == 32 && a.mode == 0 && !a.uniform_power) {  // sequential sum of this row (gen.cpp mean_power order)
            double acc = s.mp;
            for (int l = 0; l < m; ++l) acc += nr[l];
            s.mp = acc;
        }
    }
    __syncthreads();
    if (a.mode == 1) {
        if (tid == 0) a.status[f] = s.rej ? 1 : 0;
        return;
    }
    } else {
        // mode 2: mean_power of the precoded fp64 x_tx, sequentially in cell order (gen.cpp)
        if (tid == 32) {
            double acc = 0.0;
            for (size_t i = 0; i < (size_t)n * m; ++i) {
                const double2 v = xdf[i];
                acc += v.x * v.x + v.y * v.y;
            }
            s.mp = acc;
        }
        __syncthreads();
    }

    // ---- sigma2 (channel.cpp:86-89) and the noise stream
    const bool noisy = isfinite(s.snr_db);
    if (tid == 0) {
        double sigma2 = 0.0;
        if (noisy) {
            const double snr_lin = pow(10.0, s.snr_db / 10.0);
            double tg = 0.0;
            for (int t = 0; t < T; ++t) tg += 1.0 * 1.0;
            const double ref_gain2 = T == 0 ? 1.0 : tg;
            const double mp = s.mp / (double)((size_t)n * m);
            sigma2 = ref_gain2 * mp / snr_lin;
        }
        s.sd = sqrt(sigma2 / 2.0);
        a.sigma2[f] = sigma2;
        mt_seed(s.mt, splitmix(fs, 0x6e6f6973ull));
    }
    __syncthreads();

    // ---- pass 2: channel + noise, row by row (the producer warp draws row k + 1's noise and
    // computes its delay phasors while the consumers process row k)
    uint32_t produced = 0, consumed = 0;
    const uint32_t need2 = noisy ? 2u * (uint32_t)m : 0u;
    const double sd = s.sd;
    auto phasors = [&](int k, int lane_t) {
        double sn, cs;
        sincos(-kTwoPiG * (double)k * p.df_hz * s.delay[lane_t], &sn, &cs);
        s.d_re2[k & 1][lane_t] = 1.0 * cs;
        s.d_im2[k & 1][lane_t] = 1.0 * sn;
    };
    if (w == kProducerWarp) {
        while (produced < need2) {  // row 0
            mt_block(s.mt, ring, produced, mask);
            produced += kMtN;
        }
        if ((tid & 31) < T) phasors(0, tid & 31);
    }
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        if (w == kProducerWarp) {
            if (k + 1 < n) {
                while (produced < consumed + 2 * need2) {
                    mt_block(s.mt, ring, produced, mask);
                    produced += kMtN;
                }
                if ((tid & 31) < T) phasors(k + 1, tid & 31);
            }
        } else {
        const double* d_re = s.d_re2[k & 1];
        const double* d_im = s.d_im2[k & 1];
        for (int l = tid; l < m; l += 256) {
            // exact fp64 x from the stored c64 value (or the precoded fp64 x_tx in mode 2)
            double xr, xi;
            if (a.mode == 2) {
                const double2 xv = xdf[(size_t)k * m + l];
                xr = xv.x;
                xi = xv.y;
                xo[(size_t)k * m + l] = make_float2((float)xr, (float)xi);
            } else if (const float2 xf = xo[(size_t)k * m + l]; l == 0) {
                xr = xf.x < 0.f ? -a.inv_sqrt2 : a.inv_sqrt2;
                xi = xf.y < 0.f ? -a.inv_sqrt2 : a.inv_sqrt2;
            } else {
                int ir = 0, iq = 0;
                for (int q = 0; q < a.levels; ++q) {
                    if (a.lev_f[q] == xf.x) ir = q;
                    if (a.lev_f[q] == xf.y) iq = q;
                }
                xr = a.lev_d[ir];
                xi = a.lev_d[iq];
            }
            double yr = 0.0, yi = 0.0, hr = 0.0, hi = 0.0;
            for (int t = 0; t < T; ++t) {
                // row = b * dph[k]; y += row * fph[l] * x  (std::complex products, left to right)
                const double rr = s.b_re[t] * d_re[t] - s.b_im[t] * d_im[t];
                const double ri = s.b_re[t] * d_im[t] + s.b_im[t] * d_re[t];
                const double2 fp = fph[(size_t)t * m + l];
                const double t1r = rr * fp.x - ri * fp.y;
                const double t1i = rr * fp.y + ri * fp.x;
                const double t2r = t1r * xr - t1i * xi;
                const double t2i = t1r * xi + t1i * xr;
                yr = yr + t2r;
                yi = yi + t2i;
                hr = hr + t1r;  // true_channel: the same target term with x = 1 (exact)
                hi = hi + t1i;
            }
            if (a.h_true) a.h_true[((size_t)f * n + k) * m + l] = make_double2(hr, hi);
            if (noisy) {
                const uint64_t v1 = ring[(consumed + 2u * l) & mask];
                const uint64_t v2 = ring[(consumed + 2u * l + 1u) & mask];
                const double u1 = (double)(v1 >> 11) * 0x1.0p-53;
                const double u2 = (double)(v2 >> 11) * 0x1.0p-53;
                if (u1 <= 0.0) atomicOr(&s.rej, 1);
                const double r = sqrt(-2.0 * log(u1));
                const double ang = kTwoPiG * u2;
                double sn, cs;
                sincos(ang, &sn, &cs);
                // imaginary part takes the first normal (r cos), real part the cached r sin
                yr = yr + sd * (r * sn);
                yi = yi + sd * (r * cs);
            }
            yo[(size_t)k * m + l] = make_float2((float)yr, (float)yi);
        }
        }
        consumed += need2;
        __syncthreads();
    }
    if (tid == 0) a.status[f] = a.mode == 2 ? (a.status[f] | (s.rej ? 1 : 0)) : (s.rej ? 1 : 0);
}

// zadoffchu.cpp:98-119 sequence of length D^2 (D = N), reshaped row-major into the D x D
// matrix (gen.cpp zc_matrix): the same fp64 expressions, GPU sincos.
__global__ void zc_matrix_kernel(int n, long long root, double2* z) {
    const long long l = (long long)n * (long long)n;
    const double rl = double(root) / double(l);
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < l; k += (long long)gridDim.x * blockDim.x) {
        const double kk = double(k);
        double cycles;
        if (l % 2 == 0) cycles = rl * (kk * kk / 2.0 + 0.0 * kk);
        else cycles = rl * (kk * (kk + 1.0) / 2.0 + 0.0 * kk);
        cycles -= floor(cycles);
        double sn, cs;
        sincos(kTwoPiG * cycles, &sn, &cs);
        z[k] = make_double2(1.0 * cs, 1.0 * sn);
    }
}

// x_tx[:, l] = Z x[:, l] (gen.cpp precode_direct / zadoffchu.cpp apply_matrix, d == n): every
// output is the sequential sum over mm = 0..n-1 of std::complex products (re = ac - bd,
// im = ad + bc, no FMA: this unit is built with -fmad=false).  64 x 64 output tiles, 4 x 4
// per thread, K chunks of 16 through shared memory.
__global__ void __launch_bounds__(256) zc_precode_kernel(const double2* __restrict__ z, const double2* __restrict__ x,
                                                         double2* __restrict__ out, int n, int m) {
    __shared__ double2 zs[64][17];
    __shared__ double2 xs[16][65];
    const int tiles_l = (m + 63) / 64;
    const int i0 = (blockIdx.x / tiles_l) * 64, l0 = (blockIdx.x % tiles_l) * 64;
    const size_t fo = (size_t)blockIdx.y * n * m;
    const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;  // outputs i0 + ty + 16 a, l0 + tx + 16 b
    double ar[4][4], ai[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) ar[u][v] = ai[u][v] = 0.0;
    for (int k0 = 0; k0 < n; k0 += 16) {
        for (int idx = threadIdx.x; idx < 64 * 16; idx += 256) {
            const int r = idx / 16, c = idx % 16;
            zs[r][c] = (i0 + r < n) ? z[(size_t)(i0 + r) * n + k0 + c] : make_double2(0.0, 0.0);
            const int r2 = idx / 64, c2 = idx % 64;
            xs[r2][c2] = (l0 + c2 < m) ? x[fo + (size_t)(k0 + r2) * m + l0 + c2] : make_double2(0.0, 0.0);
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < 16; ++kk) {
            double2 zv[4], xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) zv[u] = zs[ty + 16 * u][kk];
#pragma unroll
            for (int v = 0; v < 4; ++v) xv[v] = xs[kk][tx + 16 * v];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const double pr = zv[u].x * xv[v].x - zv[u].y * xv[v].y;
                    const double pi = zv[u].x * xv[v].y + zv[u].y * xv[v].x;
                    ar[u][v] = ar[u][v] + pr;
                    ai[u][v] = ai[u][v] + pi;
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int i = i0 + ty + 16 * u, l = l0 + tx + 16 * v;
            if (i < n && l < m) out[fo + (size_t)i * m + l] = make_double2(ar[u][v], ai[u][v]);
        }
}

int gray_decode_h(unsigned g) {
    unsigned b = 0;
    for (; g; g >>= 1) b ^= g;
    return (int)b;
}

}  // namespace
}  // namespace ofdmr

namespace {
// Device ZC matrices, built once per (device, N, root) and kept for the process.
double2* zc_device_matrix(int n, long long root, cudaStream_t st) {
    static std::mutex mtx;
    static std::map<std::tuple<int, int, long long>, double2*> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mtx);
    const auto key = std::make_tuple(dev, n, root);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    double2* z = nullptr;
    if (cudaMalloc(&z, sizeof(double2) * (size_t)n * n) != cudaSuccess) return nullptr;
    ofdmr::zc_matrix_kernel<<<1184, 256, 0, st>>>(n, root, z);
    if (cudaGetLastError() != cudaSuccess) return nullptr;
    cache.emplace(key, z);
    return z;
}

int gen_launch(const ofdmr_gen_params* p, uint64_t base_seed, int64_t first, int64_t count, void* y, void* x_tx,
               double* sigma2, int32_t* n_targets, double* ranges, double* vels, double* snr_db, int32_t max_targets,
               int32_t* status, void* stream, const double* exp_ranges, const double* exp_vels, int32_t exp_count,
               double exp_snr, void* h_true = nullptr) {
    using namespace ofdmr;
    if (!p || !y || !x_tx || !sigma2 || !status || count < 0) return 2;  // n_targets may be null
    if (count == 0) return 0;
    int bps = 0;
    switch (p->qam_order) {
        case 4: bps = 2; break;
        case 16: bps = 4; break;
        case 64: bps = 6; break;
        case 256: bps = 8; break;
        default: return 2;
    }
    if (p->n <= 0 || p->m < 2 || p->m > kMaxM || p->targets_max > kMaxT || p->targets_min < 0 ||
        p->targets_max < p->targets_min || count > (int64_t)1 << 30 || (p->zc_precode && p->n > 4096))
        return 2;
    GenArgs a{};
    a.p = *p;
    a.base_seed = base_seed;
    a.first = first;
    a.count = (int)count;
    a.y = static_cast<float2*>(y);
    a.x = static_cast<float2*>(x_tx);
    a.sigma2 = sigma2;
    a.n_targets = n_targets;
    a.ranges = ranges;
    a.vels = vels;
    a.snr_db = snr_db;
    a.max_targets = max_targets;
    a.status = status;
    a.h_true = static_cast<double2*>(h_true);
    a.bps = bps;
    // constellation axis levels exactly as gen.cpp constellation(): li = (L-1) - 2*gray_decode(g)
    const int half = bps / 2, levels = 1 << half;
    const double scale = 1.0 / std::sqrt(2.0 * (double(levels) * levels - 1.0) / 3.0);
    a.levels = levels;
    for (int g = 0; g < levels; ++g) {
        const int q = gray_decode_h((unsigned)g);
        a.lev_of_gray[g] = q;
        const double li = double(levels - 1) - 2.0 * q;
        a.lev_d[q] = li * scale;
        a.lev_f[q] = (float)a.lev_d[q];
    }
    a.inv_sqrt2 = 1.0 / std::sqrt(2.0);
    if (bps == 2 && !p->zc_precode) {
        // QPSK pilots and payload: |x|^2 = xr xr + xi xi is the same double in every cell, so the
        // kernel's sequential mean_power sum (cell order, gen.cpp mean_power) is a constant of the
        // grid size: summed here once, in the same order (the per-row chain leaves the critical path)
        const double v = a.inv_sqrt2 * a.inv_sqrt2 + a.inv_sqrt2 * a.inv_sqrt2;
        static thread_local int64_t cached_cells = -1;
        static thread_local double cached_sum = 0.0;
        const int64_t cells = (int64_t)p->n * p->m;
        if (cached_cells != cells) {
            double acc = 0.0;
            for (int64_t i = 0; i < cells; ++i) acc += v;
            cached_cells = cells;
            cached_sum = acc;
        }
        a.uniform_power = 1;
        a.uniform_mp = cached_sum;
    }
    if (exp_ranges) {
        if (exp_count < 0 || exp_count > kMaxT || (exp_count > 0 && !exp_vels)) return 2;
        a.explicit_scene = 1;
        a.exp_count = exp_count;
        for (int t = 0; t < exp_count; ++t) {
            a.exp_range[t] = exp_ranges[t];
            a.exp_vel[t] = exp_vels[t];
        }
        a.exp_snr = exp_snr;
    }
    uint32_t ring = 1;
    const uint32_t need = 2u * (uint32_t)std::max((p->m - 1) * bps, 2 * p->m) + kMtN;  // rows k, k + 1 + a block
    while (ring < need) ring <<= 1;
    if (ring < 512) ring = 512;
    a.ring_mask = ring - 1;
    // fph holds one row per target of the launch (not kMaxT): 32 KiB less shared memory per CTA at
    // cfg4's 8 targets, 4 instead of 2 resident CTAs per SM to overlap one CTA's MT19937 production
    // with another's consumption
    a.fph_rows = std::max(1, a.explicit_scene ? a.exp_count : p->targets_max);
    const size_t smem = ((sizeof(GenShared) + 15) & ~size_t(15)) + sizeof(double2) * a.fph_rows * p->m +
                        sizeof(double) * 2 * p->m + sizeof(uint64_t) * ring + (size_t)p->n;
    {
        // the draw ring holds two rows of payload bits plus one MT19937 block: high QAM orders at large
        // M exceed the per-block shared memory (e.g. 256-QAM at M = 1024 needs 256 KiB): config error
        int dev = 0, max_smem = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (smem > (size_t)max_smem) return 2;
    }
    cudaError_t e = cudaFuncSetAttribute(gen_frame_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return 10;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!p->zc_precode) {
        gen_frame_kernel<<<(unsigned)count, kGenThreads, smem, st>>>(a);
        return cudaGetLastError() == cudaSuccess ? 0 : 10;
    }
    // ZC precode (D = N): x (fp64) -> Z x per column -> channel, in chunks of frames
    const size_t cells = (size_t)p->n * p->m;
    double2* z = zc_device_matrix(p->n, p->zc_root, st);
    if (!z) return 10;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(count, ((int64_t)512 << 20) / (int64_t)(cells * 16)));
    double2 *xb = nullptr, *tb = nullptr;
    if (cudaMallocAsync(&xb, sizeof(double2) * cells * chunk, st) != cudaSuccess ||
        cudaMallocAsync(&tb, sizeof(double2) * cells * chunk, st) != cudaSuccess)
        return 10;
    const int tiles = ((p->n + 63) / 64) * ((p->m + 63) / 64);
    for (int64_t c0 = 0; c0 < count; c0 += chunk) {
        const int64_t nc = std::min<int64_t>(chunk, count - c0);
        GenArgs b = a;
        b.first = first + c0;
        b.count = (int)nc;
        b.y = a.y + c0 * cells;
        b.x = a.x + c0 * cells;
        b.sigma2 = a.sigma2 + c0;
        b.n_targets = a.n_targets ? a.n_targets + c0 : nullptr;
        b.status = a.status + c0;
        if (a.ranges) b.ranges = a.ranges + c0 * a.max_targets;
        if (a.vels) b.vels = a.vels + c0 * a.max_targets;
        if (a.snr_db) b.snr_db = a.snr_db + c0;
        if (a.h_true) b.h_true = a.h_true + c0 * cells;
        b.mode = 1;
        b.xd = xb;
        gen_frame_kernel<<<(unsigned)nc, kGenThreads, smem, st>>>(b);
        zc_precode_kernel<<<dim3((unsigned)tiles, (unsigned)nc), 256, 0, st>>>(z, xb, tb, p->n, p->m);
        b.mode = 2;
        b.xd = tb;
        gen_frame_kernel<<<(unsigned)nc, kGenThreads, smem, st>>>(b);
    }
    cudaFreeAsync(xb, st);
    cudaFreeAsync(tb, st);
    return cudaGetLastError() == cudaSuccess ? 0 : 10;
}
}  // namespace

extern "C" int ofdmr_gen_device(const ofdmr_gen_params* p, uint64_t base_seed, int64_t first, int64_t count, void* y,
                                void* x_tx, double* sigma2, int32_t* n_targets, double* ranges, double* vels,
                                double* snr_db, int32_t max_targets, int32_t* status, void* stream) {
    return gen_launch(p, base_seed, first, count, y, x_tx, sigma2, n_targets, ranges, vels, snr_db, max_targets, status,
                      stream, nullptr, nullptr, 0, 0.0);
}

extern "C" int ofdmr_gen_device_explicit(const ofdmr_gen_params* p, uint64_t seed, int64_t first, int64_t count,
                                         const double* target_ranges, const double* target_vels, int32_t n_targets,
                                         double snr_db, void* y, void* x_tx, double* sigma2, int32_t* status,
                                         void* h_true, void* stream) {
    static const double kNone = 0.0;
    if (!p || n_targets < 0 || n_targets > 16) return 2;
    // stream-ordered: no per-call scratch (the per-frame target count is the fixed scene's)
    return gen_launch(p, seed, first, count, y, x_tx, sigma2, nullptr, nullptr, nullptr, nullptr, 0, status, stream,
                      n_targets > 0 ? target_ranges : &kNone, n_targets > 0 ? target_vels : &kNone, n_targets, snr_db,
                      h_true);
}

namespace {
// channel_mse (estimation.cpp:41-48) per frame: mean |h_est - h_true|^2, h_est c64, h_true c128;
// one CTA per frame, fp64 accumulation (tree order, not the CPU's sequential order).
__global__ void __launch_bounds__(256) channel_mse_kernel(const float2* h, const double2* ht, int64_t cells,
                                                          double* out) {
    const size_t base = (size_t)blockIdx.x * cells;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < cells; i += 256) {
        const float2 e = h[base + i];
        const double2 t = ht[base + i];
        const double dr = (double)e.x - t.x, di = (double)e.y - t.y;
        acc += dr * dr + di * di;
    }
    __shared__ double red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = red[0] / (double)cells;
}
}  // namespace

extern "C" int ofdmr_channel_mse(const void* h_est, const void* h_true, int64_t cells, int64_t frames, double* out,
                                 void* stream) {
    if (!h_est || !h_true || !out || cells <= 0 || frames < 0 || frames > (int64_t)1 << 30) return 2;
    if (frames == 0) return 0;
    channel_mse_kernel<<<(unsigned)frames, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const float2*>(h_est), static_cast<const double2*>(h_true), cells, out);
    return cudaGetLastError() == cudaSuccess ? 0 : 10;
}
