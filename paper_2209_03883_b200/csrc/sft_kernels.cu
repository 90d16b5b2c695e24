// FPS-SFT on sm_100a: one CTA per frame, fp64.  Compiled with -fmad=false so every
// complex product / sum rounds exactly like the reference's std::complex<double>
// arithmetic on x86-64 (no FMA contraction), and the slice FFT is the same radix-2
// decimation-in-time schedule with the same host-built twiddles as the oracle's FFT,
// so slice spectra, candidate sets, thresholds and the decimation back-off are
// bit-identical to the CPU oracle on identical c64 inputs.  Transcendentals inside
// the per-candidate decode (atan2 / cos / sin / hypot) are CUDA's fp64 functions
// (<= 1-2 ulp), which only matter at decision near-ties.
//
// Reference: src/sft.cpp:185-459 (sft_iterate), :29-44 (twiddle_table), :46-63
// (slope_admissible / sample_slice), :71-156 (tone_bin, egcd, wrap_dist,
// lattice_decode).
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "sft_kernels.cuh"
#include "mt64.cuh"

namespace ofdmr {
namespace {

constexpr int kSftNT = 256;
constexpr int kMaxCand = 256;   // sft.cpp:263
constexpr int kMaxComp = 128;   // accepted tones per frame held on chip
constexpr double kTwoPiD = 6.283185307179586476925286766559;

struct SftArgs {
    const float2* h;
    int n, m, q, logq;
    int i_max;
    double detect_threshold, pfa, frac_tol, amp_tol;
    int decimation;
    int max_entries;
    const int32_t* draws;
    const double* sigma2;
    const double2* tw_ref;
    const double2* tw_fft;
    int32_t *k_out, *l_out;
    double* amp_out;
    int32_t* n_entries;
    int32_t* iterations;
    int64_t* samples_used;
    int32_t* converged;
    double* residual;
    int32_t* err;     // per-frame overflow flag (synchronous API), or null
    int32_t* status;  // per-frame status, bit 2 = overflow (stream-ordered API), or null
    // general sizes (Q not a power of two <= 2048): per-CTA work arrays in global memory
    // (gbuf + blockIdx.x * gstride bytes) and the slice FFT by Bluestein exactly as oracle.c
    // fft_bluestein: chirp[q], FFT_m of the kernel bker[m], radix-2 twiddles of m for both signs
    char* gbuf;
    size_t gstride;
    int blu_m, blu_logm;
    const double2* chirp;
    const double2* bker;
    const double2* twm_f;
    const double2* twm_i;
};

__device__ __forceinline__ double2 dmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 dadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 dsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double dnorm(double2 a) { return a.x * a.x + a.y * a.y; }
// libgcc __divdc3 (Smith's method) for finite, normal operands.
__device__ __forceinline__ double2 ddiv(double2 a, double2 b) {
    double x, y;
    if (fabs(b.x) < fabs(b.y)) {
        const double ratio = b.x / b.y;
        const double denom = (b.x * ratio) + b.y;
        x = ((a.x * ratio) + a.y) / denom;
        y = ((a.y * ratio) - a.x) / denom;
    } else {
        const double ratio = b.y / b.x;
        const double denom = (b.y * ratio) + b.x;
        x = ((a.y * ratio) + a.x) / denom;
        y = (a.y - (a.x * ratio)) / denom;
    }
    return make_double2(x, y);
}
__device__ __forceinline__ double2 polar1(double th) { return make_double2(cos(th), sin(th)); }

__device__ __forceinline__ long long pmod(long long a, long long m) {
    const long long r = a % m;
    return r < 0 ? r + m : r;
}

__device__ __forceinline__ int tone_bin(long long k, long long l, long long v1, long long v2, int n, int m, int q) {
    // sft.cpp:71-81: (v1 k Q/N + v2 l Q/M) mod Q in unsigned 64-bit (k < N, l < M, v < 4096, Q < 2^21:
    // no overflow); v1 k (Q/N) = (Q/N)((v1 k) mod N) mod Q, so the reduced form is the same value
    if ((q & (q - 1)) == 0 && q <= 2048) {  // powers of two (N, M | Q): 32-bit masks, same value
        const unsigned qn = (unsigned)(q / n), qm = (unsigned)(q / m);
        return (int)((qn * (((unsigned)v1 * (unsigned)k) & (unsigned)(n - 1)) +
                      qm * (((unsigned)v2 * (unsigned)l) & (unsigned)(m - 1))) &
                     (unsigned)(q - 1));
    }
    const unsigned long long qn = (unsigned long long)(q / n), qm = (unsigned long long)(q / m);
    const unsigned long long f = ((unsigned long long)v1 * (unsigned long long)k * qn +
                                  (unsigned long long)v2 * (unsigned long long)l * qm) %
                                 (unsigned long long)q;
    return (int)f;
}

__device__ long long egcd(long long a, long long b, long long* x, long long* y) {
    // iterative form of sft.cpp:85-96 (same Bezout coefficients), 64-bit
    long long aa = a, bb = b, x0 = 1, y0 = 0, x1 = 0, y1 = 1;
    while (bb != 0) {
        const long long qt = aa / bb;
        long long t = aa - qt * bb; aa = bb; bb = t;
        t = x0 - qt * x1; x0 = x1; x1 = t;
        t = y0 - qt * y1; y0 = y1; y1 = t;
    }
    *x = x0;
    *y = y0;
    return aa;
}

__device__ double wrap_dist(double a, long long b, int period) {
    double d = a - (double)b;
    if (fabs(d) >= (double)period) d = fmod(d, (double)period);  // fmod is the identity below the period
    if (d > (double)period / 2) d -= (double)period;
    if (d < -(double)period / 2) d += (double)period;
    return fabs(d);
}

__device__ bool lattice_decode(double kap, double lam, int f, long long v1, long long v2, int n, int m, int q,
                               double tol, long long* out_k, long long* out_l) {
    const long long a = (long long)(((unsigned long long)v2 * (unsigned long long)(q / m)) % (unsigned long long)q);
    long long x, y;
    const long long d = egcd(a == 0 ? q : a, q, &x, &y);
    double best = tol;
    bool found = false;
    const long long kc = llround(kap);
    for (long long dk = -2; dk <= 2; ++dk) {
        const long long k = pmod(kc + dk, n);
        const double kd = wrap_dist(kap, k, n);
        if (kd >= best) continue;
        const long long fk = tone_bin(k, 0, v1, v2, n, m, q);
        const long long rhs = pmod((long long)f - fk, q);
        if (a == 0) {
            if (rhs != 0) continue;
            const long long l = pmod(llround(lam), m);
            const double dist = hypot(kd, wrap_dist(lam, l, m));
            if (dist < best) { best = dist; *out_k = k; *out_l = l; found = true; }
            continue;
        }
        if (rhs % d != 0) continue;
        const long long qd = q / d;
        long long inv, tmp;
        egcd(pmod(a / d, qd), qd, &inv, &tmp);
        inv = pmod(inv, qd);
        const long long l0 = pmod(((rhs / d) * inv) % qd, qd);
        const long long start = l0 % m, cnt = start < m ? (m - 1 - start) / qd + 1 : 0;
        if (cnt <= 8) {
            for (long long l = start; l < m; l += qd) {
                if (l < 0) continue;
                if (tone_bin(k, l, v1, v2, n, m, q) != f) continue;
                const double dist = hypot(kd, wrap_dist(lam, l, m));
                if (dist < best) { best = dist; *out_k = k; *out_l = l; found = true; }
            }
        } else {
            // the reference scans all cnt solutions l = start + j qd in increasing order with a
            // strict "<" (sft.cpp:141-155); wrap_dist only grows away from lam (circularly), so the
            // minimum -- and every l tying with it -- lies among the progression elements that
            // bracket lam and the two at each end (wrap-around): evaluate just those, in increasing
            // l, with the same arithmetic (identical result, O(1) instead of O(cnt))
            const long long jb = (long long)floor((lam - (double)start) / (double)qd);
            long long js[8] = {jb - 1, jb, jb + 1, jb + 2, 0, 1, cnt - 2, cnt - 1};
            for (int x = 1; x < 8; ++x)  // insertion sort (8 entries)
                for (int y = x; y > 0 && js[y - 1] > js[y]; --y) {
                    const long long t = js[y];
                    js[y] = js[y - 1];
                    js[y - 1] = t;
                }
            long long prev = -1;
            for (int x = 0; x < 8; ++x) {
                const long long jj = js[x];
                if (jj < 0 || jj >= cnt || jj == prev) continue;
                prev = jj;
                const long long l = start + jj * qd;
                if (tone_bin(k, l, v1, v2, n, m, q) != f) continue;
                const double dist = hypot(kd, wrap_dist(lam, l, m));
                if (dist < best) { best = dist; *out_k = k; *out_l = l; found = true; }
            }
        }
    }
    return found;
}

// In-place radix-2 DIT FFT (forward, unscaled) on q points in shared memory; same
// bit-reversal + butterfly schedule and twiddles as oracle.c fft_pow2.
__device__ void fft_r2(double2* a, int q, int logq, const double2* __restrict__ tw) {
    for (int i = threadIdx.x; i < q; i += kSftNT) {
        const int j = (int)(__brev((unsigned)i) >> (32 - logq));
        if (i < j) {
            const double2 t = a[i];
            a[i] = a[j];
            a[j] = t;
        }
    }
    __syncthreads();
    // stages ls and ls + 1 fused per thread: the 4 points {i, i + h, i + 2h, i + 3h} (h = 2^(ls-1))
    // are closed under both stages' butterflies, which run in registers in the oracle's order with
    // its twiddles (bit-identical), one barrier per pair of stages
    auto bfly = [](double2& u, double2& v, const double2 w) {
        const double vr = v.x * w.x - v.y * w.y;
        const double vi = v.x * w.y + v.y * w.x;
        v = make_double2(u.x - vr, u.y - vi);
        u = make_double2(u.x + vr, u.y + vi);
    };
    int ls = 1;
    for (; ls + 1 <= logq; ls += 2) {
        const int half = 1 << (ls - 1), len = 2 * half;
        for (int b = threadIdx.x; b < q / 4; b += kSftNT) {
            const int grp = b >> (ls - 1), k = b & (half - 1);
            const int i = grp * 2 * len + k;
            double2 x0 = a[i], x1 = a[i + half], x2 = a[i + len], x3 = a[i + len + half];
            const double2 w1 = tw[k * (q >> ls)];  // stage ls: pairs (i, i + h), (i + 2h, i + 3h)
            bfly(x0, x1, w1);
            bfly(x2, x3, w1);
            bfly(x0, x2, tw[k * (q >> (ls + 1))]);  // stage ls + 1: pairs (i, i + 2h), (i + h, i + 3h)
            bfly(x1, x3, tw[(k + half) * (q >> (ls + 1))]);
            a[i] = x0;
            a[i + half] = x1;
            a[i + len] = x2;
            a[i + len + half] = x3;
        }
        __syncthreads();
    }
    if (ls == logq) {  // odd log2(q): one radix-2 stage left
        const int len = 1 << ls, half = len >> 1, step = q >> ls;
        for (int b = threadIdx.x; b < q / 2; b += kSftNT) {
            const int grp = b >> (ls - 1), k = b & (half - 1);
            const int i = grp * len + k;
            double2 u = a[i], v = a[i + half];
            bfly(u, v, tw[k * step]);
            a[i] = u;
            a[i + half] = v;
        }
        __syncthreads();
    }
}

// sft.cpp:333-348 targeted DFT with incremental rotation and a resync every 256.
__device__ double2 targeted(const double2* smp, int cnt, int stride, int f, int q, const double2* __restrict__ tw) {
    double2 acc = make_double2(0.0, 0.0);
    const int step = (int)(((long long)stride * f) % q);
    const double2 rot = tw[step];
    double2 cur = make_double2(1.0, 0.0);
    int idx = 0;
    for (int t = 0; t < cnt; ++t) {
        if ((t & 255) == 0) cur = tw[idx];
        acc = dadd(acc, dmul(smp[t], cur));
        cur = dmul(cur, rot);
        idx += step;
        if (idx >= q) idx -= q;
    }
    return make_double2(acc.x / (double)cnt, acc.y / (double)cnt);
}

// The forward slice FFT (fft.hpp forward, unscaled) of q points: the oracle's radix-2 schedule
// for powers of two, otherwise Bluestein in oracle.c fft_bluestein's operation order (chirp
// multiply, radix-2 FFT_m, kernel multiply, inverse radix-2 FFT_m, 1/m, chirp) on the CTA's
// global work array: bit-identical spectra for every Q.
__device__ void sft_fft(double2* x, double2* work, const SftArgs& a) {
    const int q = a.q;
    if (a.blu_m == 0) {
        fft_r2(x, q, a.logq, a.tw_fft);
        return;
    }
    const int mm = a.blu_m;
    for (int k = threadIdx.x; k < mm; k += kSftNT) work[k] = k < q ? dmul(x[k], a.chirp[k]) : make_double2(0.0, 0.0);
    __syncthreads();
    fft_r2(work, mm, a.blu_logm, a.twm_f);
    for (int k = threadIdx.x; k < mm; k += kSftNT) work[k] = dmul(work[k], a.bker[k]);
    __syncthreads();
    fft_r2(work, mm, a.blu_logm, a.twm_i);
    const double inv_m = 1.0 / (double)mm;
    for (int k = threadIdx.x; k < q; k += kSftNT) {
        const double2 c = make_double2(work[k].x * inv_m, work[k].y * inv_m);
        x[k] = dmul(c, a.chirp[k]);
    }
    __syncthreads();
}

// GMEM: work arrays in this CTA's global slice (general Q) instead of shared memory (power-of-two
// Q <= 2048); a compile-time choice so the shared-memory build keeps LDS/STS addressing
template <bool GMEM>
__global__ void __launch_bounds__(kSftNT) sft_kernel(SftArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int q = a.q, n = a.n, m = a.m;
    unsigned char* wbase = GMEM ? reinterpret_cast<unsigned char*>(a.gbuf) + (size_t)blockIdx.x * a.gstride : smem_raw;
    double2* spec = reinterpret_cast<double2*>(wbase);       // [q]
    double2* sp1 = spec + q;                                  // [q] offset spectrum / full slice
    double2* sp2 = sp1 + q;                                   // [q]
    double2* s1d = sp2 + q;                                   // [q/2]
    double2* s2d = s1d + q / 2;                               // [q/2]
    double* pw = reinterpret_cast<double*>(s2d + q / 2);      // [q]
    int* clist = reinterpret_cast<int*>(pw + q);              // [q]
    int* alias = clist + q;                                   // [q]
    double2* bwork = reinterpret_cast<double2*>(alias + q + (q & 1));  // [blu_m] Bluestein work (global mode)
    const bool p2 = ((n & (n - 1)) == 0) && ((m & (m - 1)) == 0);
    __shared__ int s_cand[kMaxCand];
    __shared__ double2 s_c1[kMaxCand], s_c2[kMaxCand];
    __shared__ int s_dkl[kMaxCand];  // decoded (k << 12) | l per candidate, -1 = rejected
    __shared__ int s_ck[kMaxComp], s_cl[kMaxComp];
    __shared__ double2 s_camp[kMaxComp];
    __shared__ double s_red[kSftNT / 32];
    __shared__ int s_ncomp, s_nall, s_ncand, s_g, s_qd, s_full, s_stop, s_conv, s_iters, s_err;
    __shared__ long long s_samples;
    __shared__ double s_threshold, s_rel_floor, s_residual, s_total;

    const int fr = blockIdx.x;
    const float2* h = a.h + (size_t)fr * n * m;
    const double sigma2 = a.sigma2[fr];
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_ncomp = 0;
        s_samples = 0;
        s_threshold = a.detect_threshold;
        s_rel_floor = 0.0;
        s_residual = 0.0;
        s_conv = 0;
        s_iters = 0;
        s_stop = 0;
        s_err = 0;
    }
    __syncthreads();
    const bool threshold_fixed = a.detect_threshold > 0.0;
    const double inv_q = 1.0 / (double)q;

    for (int it = 0; it < a.i_max; ++it) {
        const int32_t* dr = a.draws + ((size_t)fr * a.i_max + it) * 4;
        const long long v1 = dr[0], v2 = dr[1], a1 = dr[2], a2 = dr[3];
        const int rs = (int)(v1 % n), cs = (int)(v2 % m);
        if (tid == 0) s_iters = it + 1;

        // (2) reference slice s0[q] = H[(a1 + v1 q) mod N, (a2 + v2 q) mod M], FFT, 1/Q
        for (int t = tid; t < q; t += kSftNT) {
            const long long rr = a1 + (long long)rs * t, cc = a2 + (long long)cs * t;
            const int r = (int)(p2 ? (rr & (n - 1)) : rr % n), c = (int)(p2 ? (cc & (m - 1)) : cc % m);
            const float2 v = h[(size_t)r * m + c];
            spec[t] = make_double2((double)v.x, (double)v.y);
        }
        __syncthreads();
        sft_fft(spec, bwork, a);
        for (int t = tid; t < q; t += kSftNT) spec[t] = make_double2(spec[t].x * inv_q, spec[t].y * inv_q);
        // (3) accepted tones' bins and phasors in parallel (s_dkl / s_c1 are free here) ...
        for (int i = tid; i < s_ncomp; i += kSftNT) {
            s_dkl[i] = tone_bin(s_ck[i], s_cl[i], v1, v2, n, m, q);
            const double th = kTwoPiD * ((double)(a1 * s_ck[i]) / (double)n + (double)(a2 * s_cl[i]) / (double)m);
            s_c1[i] = dmul(s_camp[i], polar1(th));
        }
        __syncthreads();
        if (tid == 0) {
            s_samples += q;
            // ... subtracted from their bins in list order (sft.cpp:232-236)
            for (int i = 0; i < s_ncomp; ++i) spec[s_dkl[i]] = dsub(spec[s_dkl[i]], s_c1[i]);
        }
        __syncthreads();
        // (4) threshold on the first iteration (sft.cpp:238-249)
        if (it == 0) {
            double pk = 0.0;
            for (int t = tid; t < q; t += kSftNT) pk = fmax(pk, dnorm(spec[t]));
            for (int o = 16; o > 0; o >>= 1) pk = fmax(pk, __shfl_xor_sync(0xffffffffu, pk, o));
            if ((tid & 31) == 0) s_red[tid >> 5] = pk;
            __syncthreads();
            if (tid == 0) {
                double peak = 0.0;
                for (int i = 0; i < kSftNT / 32; ++i) peak = fmax(peak, s_red[i]);
                s_rel_floor = 1e-9 * peak;
                if (!threshold_fixed) {
                    const double noise_part =
                        sigma2 > 0.0 ? 4.0 * sigma2 / (double)q * log((double)q / a.pfa) : 0.0;
                    s_threshold = fmax(noise_part, s_rel_floor);
                }
            }
            __syncthreads();
        }
        // (5) candidates >= threshold, ordered by (power desc, bin asc), cap 256
        const double threshold = s_threshold;
        if (tid == 0) s_nall = 0;
        __syncthreads();
        for (int t = tid; t < q; t += kSftNT) {
            const double p = dnorm(spec[t]);
            pw[t] = p;
            if (p >= threshold && p > 0.0) clist[atomicAdd(&s_nall, 1)] = t;
        }
        __syncthreads();
        const int nall = s_nall;
        for (int i = tid; i < nall; i += kSftNT) {
            const int fi = clist[i];
            const double pi = pw[fi];
            int rank = 0;
            for (int j = 0; j < nall; ++j) {
                const int fj = clist[j];
                const double pj = pw[fj];
                rank += (pj > pi) || (pj == pi && fj < fi);
            }
            if (rank < kMaxCand) s_cand[rank] = fi;
        }
        if (tid == 0) {
            double tp = 0.0;
            for (int t = 0; t < q; ++t) tp += pw[t];  // sequential, as the reference sums
            s_total = tp;
            s_ncand = nall < kMaxCand ? nall : kMaxCand;
            if (nall == 0) {
                s_residual = tp;
                s_conv = 1;
                s_stop = 1;
            }
        }
        __syncthreads();
        if (s_stop) break;
        const int ncand = s_ncand;

        // (7) decimation back-off (sft.cpp:274-289)
        if (tid == 0) {
            double weakest = pw[s_cand[0]];
            for (int i = 0; i < ncand; ++i) weakest = fmin(weakest, pw[s_cand[i]]);
            int g = a.decimation > 1 ? a.decimation : 1;
            const double dim = (double)(n > m ? n : m);
            while (g > 1) {
                const bool divides = q % g == 0 && q / g >= 16;
                bool quiet = true;
                if (sigma2 > 0.0) {
                    const double angle_var = sigma2 * (1.0 + (double)g) / (2.0 * (double)q * weakest);
                    quiet = dim / kTwoPiD * sqrt(angle_var) <= 0.3;
                }
                if (divides && quiet) break;
                --g;
            }
            s_g = g;
            s_qd = q / g;
        }
        __syncthreads();
        const int g = s_g, qd = s_qd;
        for (int t = tid; t < qd; t += kSftNT) alias[t] = 0;
        __syncthreads();
        if (tid == 0) {
            for (int i = 0; i < ncand; ++i) alias[s_cand[i] % qd]++;
            for (int i = 0; i < s_ncomp; ++i) alias[tone_bin(s_ck[i], s_cl[i], v1, v2, n, m, q) % qd]++;
            int full = 0;
            if (g > 1)
                for (int i = 0; i < ncand; ++i) full |= alias[s_cand[i] % qd] > 1;
            s_full = full;
        }
        __syncthreads();
        // (9) offset slices at (r+1, c) and (r, c+1)
        if (g == 1 || s_full) {
            for (int t = tid; t < q; t += kSftNT) {
                const long long rr = a1 + (long long)rs * t, cc = a2 + (long long)cs * t;
                const int r = (int)(p2 ? (rr & (n - 1)) : rr % n), c = (int)(p2 ? (cc & (m - 1)) : cc % m);
                const int r1 = r + 1 == n ? 0 : r + 1, c1 = c + 1 == m ? 0 : c + 1;
                const float2 u = h[(size_t)r1 * m + c], w = h[(size_t)r * m + c1];
                sp1[t] = make_double2((double)u.x, (double)u.y);
                sp2[t] = make_double2((double)w.x, (double)w.y);
            }
        }
        if (g > 1) {
            const int rsd = (int)((v1 * g) % n), csd = (int)((v2 * g) % m);
            for (int t = tid; t < qd; t += kSftNT) {
                const long long rr = a1 + (long long)rsd * t, cc = a2 + (long long)csd * t;
                const int r = (int)(p2 ? (rr & (n - 1)) : rr % n), c = (int)(p2 ? (cc & (m - 1)) : cc % m);
                const int r1 = r + 1 == n ? 0 : r + 1, c1 = c + 1 == m ? 0 : c + 1;
                const float2 u = h[(size_t)r1 * m + c], w = h[(size_t)r * m + c1];
                s1d[t] = make_double2((double)u.x, (double)u.y);
                s2d[t] = make_double2((double)w.x, (double)w.y);
            }
        }
        __syncthreads();
        if (g == 1) {
            sft_fft(sp1, bwork, a);
            sft_fft(sp2, bwork, a);
            for (int t = tid; t < q; t += kSftNT) {
                sp1[t] = make_double2(sp1[t].x * inv_q, sp1[t].y * inv_q);
                sp2[t] = make_double2(sp2[t].x * inv_q, sp2[t].y * inv_q);
            }
            __syncthreads();
        }
        if (tid == 0) s_samples += g == 1 ? 2LL * q : 2LL * qd + (s_full ? 2LL * (q - qd) : 0LL);
        // raw offset-slice readings per candidate, in parallel
        for (int i = tid; i < ncand; i += kSftNT) {
            const int f = s_cand[i];
            if (g == 1) {
                s_c1[i] = sp1[f];
                s_c2[i] = sp2[f];
            } else if (alias[f % qd] > 1) {
                s_c1[i] = targeted(sp1, q, 1, f, q, a.tw_ref);
                s_c2[i] = targeted(sp2, q, 1, f, q, a.tw_ref);
            } else {
                s_c1[i] = targeted(s1d, qd, g, f, q, a.tw_ref);
                s_c2[i] = targeted(s2d, qd, g, f, q, a.tw_ref);
            }
        }
        __syncthreads();
        // (11)-(15) per candidate, in parallel: a candidate's subtraction, decode, gate and amplitude
        // only involve components whose tone bin is its own bin (or its residue mod Q/g when it is
        // not aliased), and no other candidate of this iteration adds, merges or erases one of
        // those (distinct bins; an aliased residue forces full slices) -- so the order-dependent
        // part is only (16)-(17), applied below by one thread in candidate order
        for (int i = tid; i < ncand; i += kSftNT) {
            s_dkl[i] = -1;
            {
                const int f = s_cand[i];
                const double2 c0 = spec[f];
                if (dnorm(c0) < threshold) continue;
                if (dnorm(c0) == 0.0) continue;
                double2 c1 = s_c1[i], c2 = s_c2[i];
                const bool full_bin = g == 1 || alias[f % qd] > 1;
                for (int j = 0; j < s_ncomp; ++j) {
                    const int fc = tone_bin(s_ck[j], s_cl[j], v1, v2, n, m, q);
                    if (full_bin ? (fc != f) : (fc % qd != f % qd)) continue;
                    const double2 psi = dmul(
                        s_camp[j],
                        polar1(kTwoPiD * ((double)(a1 * s_ck[j]) / (double)n + (double)(a2 * s_cl[j]) / (double)m)));
                    c1 = dsub(c1, dmul(psi, polar1(kTwoPiD * (double)s_ck[j] / (double)n)));
                    c2 = dsub(c2, dmul(psi, polar1(kTwoPiD * (double)s_cl[j] / (double)m)));
                }
                const double2 r1 = ddiv(c1, c0), r2 = ddiv(c2, c0);
                double kap = atan2(r1.y, r1.x) / kTwoPiD * (double)n;
                if (kap < 0) kap += (double)n;
                double lam = atan2(r2.y, r2.x) / kTwoPiD * (double)m;
                if (lam < 0) lam += (double)m;
                long long k = 0, l = 0;
                if (!lattice_decode(kap, lam, f, v1, v2, n, m, q, a.frac_tol * 5.0, &k, &l)) continue;
                const double m0 = hypot(c0.x, c0.y), m1 = hypot(c1.x, c1.y), m2 = hypot(c2.x, c2.y);
                const double mean_mag = (m0 + m1 + m2) / 3.0;
                if (fmax(m0, fmax(m1, m2)) - fmin(m0, fmin(m1, m2)) > a.amp_tol * mean_mag) continue;
                const double2 psi0 = polar1(kTwoPiD * ((double)(a1 * k) / (double)n + (double)(a2 * l) / (double)m));
                const double2 psi1 = dmul(psi0, polar1(kTwoPiD * (double)k / (double)n));
                const double2 psi2 = dmul(psi0, polar1(kTwoPiD * (double)l / (double)m));
                const double2 sum = dadd(dadd(ddiv(c0, psi0), ddiv(c1, psi1)), ddiv(c2, psi2));
                s_c1[i] = make_double2(sum.x / 3.0, sum.y / 3.0);  // amp
                s_c2[i].x = dnorm(c0);
                s_dkl[i] = (int)((k << 12) | l);
            }
        }
        __syncthreads();
        // (16)-(18) merge / erase / consume in candidate order
        if (tid == 0) {
            double total_power = s_total;
            for (int i = 0; i < ncand; ++i) {
                if (s_dkl[i] < 0) continue;
                const int f = s_cand[i];
                const long long k = s_dkl[i] >> 12, l = s_dkl[i] & 4095;
                const double2 amp = s_c1[i];
                int found = -1;
                for (int j = 0; j < s_ncomp; ++j)
                    if (s_ck[j] == k && s_cl[j] == l) { found = j; break; }
                if (found >= 0) {
                    s_camp[found] = dadd(s_camp[found], amp);
                    if (dnorm(s_camp[found]) < threshold) {
                        for (int j = found; j + 1 < s_ncomp; ++j) {
                            s_ck[j] = s_ck[j + 1];
                            s_cl[j] = s_cl[j + 1];
                            s_camp[j] = s_camp[j + 1];
                        }
                        --s_ncomp;
                    }
                } else if (s_ncomp < kMaxComp) {
                    s_ck[s_ncomp] = (int)k;
                    s_cl[s_ncomp] = (int)l;
                    s_camp[s_ncomp] = amp;
                    ++s_ncomp;
                } else {
                    s_err = 1;
                }
                total_power -= s_c2[i].x;
                spec[f] = make_double2(0.0, 0.0);
            }
            const double residual = total_power > 0.0 ? total_power : 0.0;
            s_residual = residual;
            const double conv_floor = sigma2 * (1.0 + 6.0 / sqrt((double)q)) + s_rel_floor * (double)q;
            if (residual <= conv_floor) {
                s_conv = 1;
                s_stop = 1;
            }
        }
        __syncthreads();
        if (s_stop) break;
    }

    if (tid == 0) {
        // sft.cpp:448-458 order: |A|^2 desc, then k, then l
        const int nc = s_ncomp;
        for (int i = 1; i < nc; ++i) {
            const int kk = s_ck[i], ll = s_cl[i];
            const double2 av = s_camp[i];
            int j = i;
            while (j > 0) {
                const double pa = dnorm(av), pb = dnorm(s_camp[j - 1]);
                const bool before = (pa != pb) ? (pa > pb) : (kk != s_ck[j - 1] ? kk < s_ck[j - 1] : ll < s_cl[j - 1]);
                if (!before) break;
                s_ck[j] = s_ck[j - 1];
                s_cl[j] = s_cl[j - 1];
                s_camp[j] = s_camp[j - 1];
                --j;
            }
            s_ck[j] = kk;
            s_cl[j] = ll;
            s_camp[j] = av;
        }
        for (int i = 0; i < nc && i < a.max_entries; ++i) {
            const size_t o = (size_t)fr * a.max_entries + i;
            a.k_out[o] = s_ck[i];
            a.l_out[o] = s_cl[i];
            a.amp_out[2 * o] = s_camp[i].x;
            a.amp_out[2 * o + 1] = s_camp[i].y;
        }
        a.n_entries[fr] = nc;
        if (a.iterations) a.iterations[fr] = s_iters;
        if (a.samples_used) a.samples_used[fr] = s_samples;
        if (a.converged) a.converged[fr] = s_conv;
        if (a.residual) a.residual[fr] = s_residual;
        if (a.err) a.err[fr] = s_err;
        if (a.status && s_err) atomicOr(a.status + fr, 4);
    }
}

long long gcd_ll(long long a, long long b) {
    while (b) { const long long t = a % b; a = b; b = t; }
    return a < 0 ? -a : a;
}
long long lcm_ll(long long a, long long b) { return a / gcd_ll(a, b) * b; }

__device__ long long gcd_d(long long a, long long b) {
    while (b) {
        const long long t = a % b;
        a = b;
        b = t;
    }
    return a < 0 ? -a : a;
}
// sft.cpp:46-51 slope_admissible: lcm(N / gcd(v1 mod N, N), M / gcd(v2 mod M, M)) == lcm(N, M)
__device__ bool slope_admissible_d(long long v1, long long v2, long long n, long long m) {
    const long long q = n / gcd_d(n, m) * m;
    const long long r1 = ((v1 % n) + n) % n, r2 = ((v2 % m) + m) % m;
    const long long a = n / gcd_d(r1, n), b = m / gcd_d(r2, m);
    return a / gcd_d(a, b) * b == q;
}

// The data-independent random draws, on the device (one thread per frame walks the frame's
// MT19937-64 stream, bit-identical to std::mt19937_64 + Rng::uniform_int):
//   mode 0, FPS-SFT (sft.cpp:191, 212-218): Rng(derive_seed(seed, 0x73667421)); per iteration an
//           admissible slope (v1, v2), then offsets a1 < N, a2 < M -> draws[f][it] = {v1, v2, a1, a2}
//   mode 1, estimate_noise_from_slice (pipeline.cpp:31-35): Rng(seed); one admissible slope
//           -> draws[f] = {v1, v2}
__global__ void __launch_bounds__(64) sft_draws_kernel(const uint64_t* __restrict__ seeds, int frames, int n, int m,
                                                       int iters, int mode, int32_t* __restrict__ draws) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= frames) return;
    uint64_t mt[mt64::kMtN];
    mt64::mt_seed(mt, mode == 0 ? mt64::splitmix(seeds[f], 0x73667421ull) : seeds[f]);
    mt64::MtScalar r{mt, mt64::kMtN};
    for (int it = 0; it < iters; ++it) {
        long long v1, v2;
        do {
            v1 = (long long)(1 + r.uniform_int(n > 1 ? (uint64_t)(n - 1) : 1ull));
            v2 = (long long)(1 + r.uniform_int(m > 1 ? (uint64_t)(m - 1) : 1ull));
        } while (!slope_admissible_d(v1, v2, n, m));
        if (mode == 0) {
            const long long a1 = (long long)r.uniform_int((uint64_t)n), a2 = (long long)r.uniform_int((uint64_t)m);
            int32_t* d = draws + ((size_t)f * iters + it) * 4;
            d[0] = (int32_t)v1;
            d[1] = (int32_t)v2;
            d[2] = (int32_t)a1;
            d[3] = (int32_t)a2;
        } else {
            draws[2 * (size_t)f] = (int32_t)v1;
            draws[2 * (size_t)f + 1] = (int32_t)v2;
        }
    }
}

// detections_from_spectrum (sft.cpp:461-490), one warp per frame: power = |A|^2 N M (fp64, no
// FMA: this unit is compiled -fmad=false), kept when !(power < eta) with eta = -sigma2 ln(pfa)
// (detection_threshold with power factor 1, ln(pfa) from the host's libm), delay (N - k) mod N,
// Doppler (l + M/2) mod M - M/2, ordered by (power desc, delay asc, Doppler asc), cut at K.
struct SftDetArgs {
    const int32_t* k;
    const int32_t* l;
    const double* amp;
    const int32_t* n_entries;
    int max_entries;
    int n, m;
    const double* sigma2;
    double log_pfa;
    const int32_t* k_per_frame;
    int kmax;
    int32_t* det_delay;
    int32_t* det_doppler;
    float* det_power;
    int32_t* counts;
    int frames;
};
__global__ void __launch_bounds__(128) sft_detect_kernel(SftDetArgs a) {
    const int lane = threadIdx.x & 31;
    const int f = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (f >= a.frames) return;
    const int ne = min(a.n_entries[f], a.max_entries);
    const double eta = -a.sigma2[f] * a.log_pfa * 1.0;
    const double nm = (double)a.n * (double)a.m;
    const long long half = a.m / 2;
    double pw[2];
    long long dl[2], dp[2];
    bool keep[2];
    for (int t = 0; t < 2; ++t) {
        const int i = lane + 32 * t;
        keep[t] = false;
        pw[t] = 0.0;
        dl[t] = dp[t] = 0;
        if (i < ne) {
            const size_t o = (size_t)f * a.max_entries + i;
            const double re = a.amp[2 * o], im = a.amp[2 * o + 1];
            pw[t] = (re * re + im * im) * nm;
            keep[t] = !(pw[t] < eta);
            dl[t] = ((long long)a.n - a.k[o]) % (long long)a.n;
            dp[t] = ((long long)a.l[o] + half) % (long long)a.m - half;
        }
    }
    const int kf = a.k_per_frame ? min(a.k_per_frame[f], a.kmax) : a.kmax;
    int kept = __popc(__ballot_sync(0xffffffffu, keep[0])) + __popc(__ballot_sync(0xffffffffu, keep[1]));
    for (int t = 0; t < 2; ++t) {
        int rank = 0;
        for (int src = 0; src < 64; ++src) {  // entry src = lane' + 32 t'
            const int sl = src & 31, st = src >> 5;
            const double pj = __shfl_sync(0xffffffffu, st ? pw[1] : pw[0], sl);
            const long long dj = __shfl_sync(0xffffffffu, st ? dl[1] : dl[0], sl);
            const long long vj = __shfl_sync(0xffffffffu, st ? dp[1] : dp[0], sl);
            const bool kj = __shfl_sync(0xffffffffu, st ? keep[1] : keep[0], sl);
            if (kj && keep[t] && src != lane + 32 * t &&
                (pj != pw[t] ? pj > pw[t] : (dj != dl[t] ? dj < dl[t] : vj < dp[t])))
                ++rank;
        }
        if (keep[t] && rank < kf) {
            const size_t o = (size_t)f * a.kmax + rank;
            a.det_delay[o] = (int32_t)dl[t];
            a.det_doppler[o] = (int32_t)dp[t];
            a.det_power[o] = (float)pw[t];
        }
    }
    const int cnt = min(kept, kf);
    for (int i = cnt + lane; i < a.kmax; i += 32) {
        const size_t o = (size_t)f * a.kmax + i;
        a.det_delay[o] = 0;
        a.det_doppler[o] = 0;
        a.det_power[o] = 0.f;
    }
    if (lane == 0) a.counts[f] = cnt;
}

// division_noise_power (pipeline.cpp:18-23): sigma2 * mean(1 / |x|^2) per frame, one CTA per frame,
// each term 1 / (re^2 + im^2) in fp64 on the upcast c64 cell (as std::norm of complex<double>),
// summed in a fixed tree order (deterministic; the reference's sequential order is not
// reproduced, so sigma_h^2 agrees to ~1e-15 relative, not bit for bit).
__global__ void __launch_bounds__(256) division_noise_kernel(const float2* __restrict__ x, long long cells,
                                                             const double* __restrict__ sigma2, double* __restrict__ out) {
    __shared__ double red[256];
    const int f = blockIdx.x;
    const float2* xf = x + (size_t)f * cells;
    double acc = 0.0;
    for (long long i = threadIdx.x; i < cells; i += 256) {
        const float2 v = __ldcs(xf + i);
        const double re = v.x, im = v.y;
        acc += 1.0 / (re * re + im * im);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double sg = sigma2[f];
        out[f] = sg <= 0.0 ? 0.0 : sg * red[0] / (double)cells;
    }
}

// pipeline.cpp:26-43 estimate_noise_from_slice: one CTA per frame; the slice through (0, 0)
// along the device-drawn slope, the slice FFT with the oracle's schedule (sft_fft: radix-2 or
// Bluestein, bit-identical spectrum), p = |s|^2 / Q^2, bitonic sort (padded with +inf to a power
// of two), p[Q/2] * Q / ln 2.  Work arrays in shared memory for power-of-two Q <= 2048, else in
// this CTA's slice of a.gbuf.
template <bool GMEM>
__global__ void __launch_bounds__(kSftNT) slice_noise_kernel(SftArgs a, const int32_t* __restrict__ slopes,
                                                             double* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int q = a.q, n = a.n, m = a.m;
    int qp = 1;
    while (qp < q) qp <<= 1;
    unsigned char* wbase = GMEM ? reinterpret_cast<unsigned char*>(a.gbuf) + (size_t)blockIdx.x * a.gstride : smem_raw;
    double2* sp = reinterpret_cast<double2*>(wbase);  // [q]
    double* pw = reinterpret_cast<double*>(sp + q);   // [qp]
    double2* bwork = reinterpret_cast<double2*>(pw + qp + (qp & 1));
    const int fr = blockIdx.x;
    const float2* h = a.h + (size_t)fr * n * m;
    const long long v1 = slopes[2 * fr], v2 = slopes[2 * fr + 1];
    for (int t = threadIdx.x; t < q; t += kSftNT) {
        const int r = (int)((v1 * t) % n), c = (int)((v2 * t) % m);
        const float2 v = h[(size_t)r * m + c];
        sp[t] = make_double2((double)v.x, (double)v.y);
    }
    __syncthreads();
    sft_fft(sp, bwork, a);
    const double qq = (double)q * (double)q;
    for (int t = threadIdx.x; t < qp; t += kSftNT) pw[t] = t < q ? dnorm(sp[t]) / qq : __longlong_as_double(0x7ff0000000000000LL);
    __syncthreads();
    for (int k = 2; k <= qp; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < qp; i += kSftNT) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const double a0 = pw[i], a1 = pw[ixj];
                    const bool up = (i & k) == 0;
                    if (up ? (a0 > a1) : (a0 < a1)) {
                        pw[i] = a1;
                        pw[ixj] = a0;
                    }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x == 0) out[fr] = pw[q / 2] * (double)q / 0.6931471805599453;
}

template <typename T>
cudaError_t ensure(T** p, int64_t& cap, int64_t need) {
    if (*p && cap >= need) return cudaSuccess;
    cudaFree(*p);
    *p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(p, sizeof(T) * size_t(need));
    if (e == cudaSuccess) cap = need;
    return e;
}

}  // namespace

void sft_free(SftScratch& s) {
    cudaFree(s.draws);
    cudaFree(s.seeds);
    cudaFree(s.sigma2);
    cudaFree(s.err);
    cudaFree(s.gbuf);
    for (auto& t : s.tables) {
        cudaFree(t.second.tw_ref);
        cudaFree(t.second.tw_fft);
        cudaFree(t.second.chirp);
        cudaFree(t.second.bker);
        cudaFree(t.second.twm_f);
        cudaFree(t.second.twm_i);
    }
    s = SftScratch{};
}

namespace {

// radix-2 twiddles of an n-point transform, oracle.c pow2_twiddles: (cos, sin)(sign 2 pi k / n)
std::vector<double2> r2_twiddles(int n, int sign) {
    std::vector<double2> t(n / 2 > 0 ? n / 2 : 1);
    for (int k = 0; k < n / 2; ++k) {
        const double ang = (double)sign * kTwoPiD * (double)k / (double)n;
        t[k] = make_double2(std::cos(ang), std::sin(ang));
    }
    return t;
}

// In-place radix-2 FFT with the oracle's schedule (oracle.c fft_pow2: bit reversal, then levels
// with the top-level twiddles at stride n / len), on the host: the Bluestein kernel transform
// is built once per Q exactly as the oracle builds it.
void host_fft_pow2(std::vector<double2>& a, int sign) {
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; i++) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    const std::vector<double2> tw = r2_twiddles(int(n), sign);
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len / 2, step = n / len;
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < half; k++) {
                const double wr = tw[k * step].x, wi = tw[k * step].y;
                double2& u = a[i + k];
                double2& v = a[i + k + half];
                const double vr = v.x * wr - v.y * wi;
                const double vi = v.x * wi + v.y * wr;
                v = make_double2(u.x - vr, u.y - vi);
                u = make_double2(u.x + vr, u.y + vi);
            }
    }
}

template <typename T>
cudaError_t upload(T** d, const std::vector<T>& h) {
    cudaError_t e = cudaMalloc(d, sizeof(T) * (h.empty() ? 1 : h.size()));
    if (e == cudaSuccess && !h.empty()) e = cudaMemcpy(*d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice);
    return e;
}

// Tables of one Q, built once on the host with the reference's / oracle's libm calls and kept for
// the life of the context (never rewritten, so stream-ordered launches may use them).
int sft_tables(SftScratch& s, int q, const SftScratch::Tables** out, std::string& err) {
    auto it = s.tables.find(q);
    if (it == s.tables.end()) {
        SftScratch::Tables t;
        std::vector<double2> twr(q);
        const double sa = -kTwoPiD / double(q);
        double cr = 1.0, ci = 0.0;
        const double sr = std::cos(sa), si = std::sin(sa);
        for (int j = 0; j < q; ++j) {
            if ((j & 255) == 0) {
                const double th = -kTwoPiD * double(j) / double(q);
                cr = std::cos(th);
                ci = std::sin(th);
            }
            twr[j] = make_double2(cr, ci);
            const double nr = cr * sr - ci * si, ni = cr * si + ci * sr;
            cr = nr;
            ci = ni;
        }
        cudaError_t e = upload(&t.tw_ref, twr);
        if ((q & (q - 1)) == 0) {
            if (e == cudaSuccess) e = upload(&t.tw_fft, r2_twiddles(q, -1));
        } else {
            // oracle.c fft_bluestein: m, chirp e^{-j pi (k^2 mod 2Q) / Q}, kernel conj(chirp) at k and m - k
            int mm = 1, lg = 0;
            while (mm < 2 * q - 1) {
                mm <<= 1;
                ++lg;
            }
            t.blu_m = mm;
            t.blu_logm = lg;
            std::vector<double2> w(q), b(mm, make_double2(0.0, 0.0));
            for (int k = 0; k < q; k++) {
                const unsigned long long k2 = ((unsigned long long)k * k) % (2ULL * q);
                const double ang = (double)(-1) * kTwoPiD * 0.5 * (double)k2 / (double)q;
                w[k] = make_double2(std::cos(ang), std::sin(ang));
            }
            b[0] = make_double2(w[0].x, -w[0].y);
            for (int k = 1; k < q; k++) b[k] = b[mm - k] = make_double2(w[k].x, -w[k].y);
            host_fft_pow2(b, -1);
            if (e == cudaSuccess) e = upload(&t.chirp, w);
            if (e == cudaSuccess) e = upload(&t.bker, b);
            if (e == cudaSuccess) e = upload(&t.twm_f, r2_twiddles(mm, -1));
            if (e == cudaSuccess) e = upload(&t.twm_i, r2_twiddles(mm, +1));
        }
        if (e != cudaSuccess) {
            cudaFree(t.tw_ref);
            cudaFree(t.tw_fft);
            cudaFree(t.chirp);
            cudaFree(t.bker);
            cudaFree(t.twm_f);
            cudaFree(t.twm_i);
            err = std::string("sft: twiddle tables: ") + cudaGetErrorString(e);
            return OFDMR_ERR_CUDA;
        }
        it = s.tables.emplace(q, t).first;
    }
    *out = &it->second;
    return OFDMR_OK;
}

// Q handled in shared memory (power of two <= 2048, one CTA per frame); otherwise the CTA's work
// arrays live in global memory and frames are launched in chunks of kGlobalChunk CTAs
bool sft_smem_q(int q) { return (q & (q - 1)) == 0 && q <= 2048; }
constexpr int64_t kGlobalChunk = 296;

size_t sft_gstride(int q, int blu_m) {
    const size_t bytes = sizeof(double2) * (3 * size_t(q) + size_t(q)) + sizeof(double) * q + sizeof(int) * 2 * q +
                         8 + sizeof(double2) * size_t(blu_m);
    return (bytes + 255) & ~size_t(255);
}
size_t noise_gstride(int q, int blu_m) {
    size_t qp = 1;
    while (qp < size_t(q)) qp <<= 1;
    const size_t bytes = sizeof(double2) * q + sizeof(double) * qp + 8 + sizeof(double2) * size_t(blu_m);
    return (bytes + 255) & ~size_t(255);
}

int ensure_gbuf(SftScratch& s, size_t bytes, std::string& err) {
    if (s.gbuf && s.cap_gbuf >= int64_t(bytes)) return OFDMR_OK;
    cudaFree(s.gbuf);
    s.gbuf = nullptr;
    s.cap_gbuf = 0;
    const cudaError_t e = cudaMalloc(&s.gbuf, bytes);
    if (e != cudaSuccess) {
        err = std::string("sft: work arrays: ") + cudaGetErrorString(e);
        return OFDMR_ERR_CUDA;
    }
    s.cap_gbuf = int64_t(bytes);
    return OFDMR_OK;
}

int upload_seeds(SftScratch& s, cudaStream_t st, const uint64_t* seeds, int64_t frames, std::string& err) {
    cudaError_t e = ensure(&s.seeds, s.cap_seeds, frames);
    // pageable source: the copy is staged before cudaMemcpyAsync returns (the host array may go)
    if (e == cudaSuccess) e = cudaMemcpyAsync(s.seeds, seeds, sizeof(uint64_t) * frames, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
        err = std::string("sft: seeds: ") + cudaGetErrorString(e);
        return OFDMR_ERR_CUDA;
    }
    return OFDMR_OK;
}

}  // namespace

namespace {
int sft_size_check(int n, int m, int q, const char* what, std::string& err) {
    if (n < 2 || m < 2 || n > 4096 || m > 4096) {
        err = std::string(what) + ": N and M must lie in [2, 4096] on the GPU path";
        return OFDMR_ERR_CONFIG;
    }
    if (q < 16 || q > (1 << 20)) {
        err = std::string(what) + ": Q = lcm(N, M) must lie in [16, 2^20] on the GPU path";
        return OFDMR_ERR_CONFIG;
    }
    return OFDMR_OK;
}
}  // namespace

int sft_run(SftScratch& s, cudaStream_t st, const float2* h, int n, int m, const ofdmr_sft_config& cfg,
            const uint64_t* seeds, const double* sigma2, bool sigma2_on_device, int32_t* k_out, int32_t* l_out,
            double* amp_out, int32_t* n_entries, int32_t* iterations, int64_t* samples_used, int32_t* converged,
            double* residual, int32_t* status, int64_t frames, int64_t* launches, std::string& err) {
    const long long ql = lcm_ll(n, m);
    const int q = ql > (1 << 21) ? (1 << 21) : int(ql);
    int rc = sft_size_check(n, m, q, "sft", err);
    if (rc) return rc;
    if (cfg.i_max < 0 || cfg.max_entries < 1 || cfg.max_entries > 64 || frames > 65535 * 32) {
        err = "sft: bad i_max / max_entries";
        return OFDMR_ERR_CONFIG;
    }
    const int i_max = cfg.i_max;
    const int iters = i_max > 0 ? i_max : 1;
    rc = upload_seeds(s, st, seeds, frames, err);
    if (rc) return rc;
    cudaError_t e = ensure(&s.draws, s.cap_draws, frames * iters * 4);
    int64_t cap_s2 = s.cap_frames, cap_err = s.cap_frames;
    if (e == cudaSuccess && !sigma2_on_device) e = ensure(&s.sigma2, cap_s2, frames);
    if (e == cudaSuccess && !status) e = ensure(&s.err, cap_err, frames);
    if (e != cudaSuccess) { err = std::string("sft: allocation: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    s.cap_frames = std::min(sigma2_on_device ? cap_err : cap_s2, status ? cap_s2 : cap_err);
    if (i_max > 0) {
        sft_draws_kernel<<<unsigned((frames + 63) / 64), 64, 0, st>>>(s.seeds, int(frames), n, m, i_max, 0, s.draws);
        e = cudaGetLastError();
        if (e != cudaSuccess) { err = std::string("sft: draws: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
        if (launches) ++*launches;
    }
    const double* s2 = sigma2;
    if (!sigma2_on_device) {
        e = cudaMemcpyAsync(s.sigma2, sigma2, sizeof(double) * frames, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) { err = std::string("sft: upload: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
        s2 = s.sigma2;
    }
    const SftScratch::Tables* tb = nullptr;
    rc = sft_tables(s, q, &tb, err);
    if (rc) return rc;

    SftArgs a{};
    a.n = n;
    a.m = m;
    a.q = q;
    a.logq = 0;
    while ((1 << a.logq) < q) ++a.logq;
    a.i_max = i_max;
    a.detect_threshold = cfg.detect_threshold;
    a.pfa = cfg.pfa;
    a.frac_tol = cfg.frac_tol;
    a.amp_tol = cfg.amp_tol;
    a.decimation = cfg.decimation;
    a.max_entries = cfg.max_entries;
    a.tw_ref = tb->tw_ref;
    a.tw_fft = tb->tw_fft;
    a.blu_m = tb->blu_m;
    a.blu_logm = tb->blu_logm;
    a.chirp = tb->chirp;
    a.bker = tb->bker;
    a.twm_f = tb->twm_f;
    a.twm_i = tb->twm_i;
    const bool smem_mode = sft_smem_q(q);
    size_t smem = 0;
    int64_t chunk = frames;
    if (smem_mode) {
        smem = sizeof(double2) * (3 * size_t(q) + size_t(q)) + sizeof(double) * q + sizeof(int) * 2 * q;
    } else {
        a.gstride = sft_gstride(q, tb->blu_m);
        chunk = std::min<int64_t>(frames, kGlobalChunk);
        rc = ensure_gbuf(s, a.gstride * size_t(chunk), err);
        if (rc) return rc;
        a.gbuf = s.gbuf;
    }
    auto kern = smem_mode ? sft_kernel<false> : sft_kernel<true>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) { err = std::string("sft: smem attr: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    const int me = cfg.max_entries;
    for (int64_t f0 = 0; f0 < frames; f0 += chunk) {
        const int64_t nf = std::min<int64_t>(chunk, frames - f0);
        SftArgs b = a;
        b.h = h + f0 * int64_t(n) * m;
        b.draws = s.draws + f0 * iters * 4;
        b.sigma2 = s2 + f0;
        b.k_out = k_out + f0 * me;
        b.l_out = l_out + f0 * me;
        b.amp_out = amp_out + 2 * f0 * me;
        b.n_entries = n_entries + f0;
        b.iterations = iterations ? iterations + f0 : nullptr;
        b.samples_used = samples_used ? samples_used + f0 : nullptr;
        b.converged = converged ? converged + f0 : nullptr;
        b.residual = residual ? residual + f0 : nullptr;
        b.err = status ? nullptr : s.err + f0;
        b.status = status ? status + f0 : nullptr;
        kern<<<unsigned(nf), kSftNT, smem, st>>>(b);
        e = cudaGetLastError();
        if (e != cudaSuccess) { err = std::string("sft: launch: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
        if (launches) ++*launches;
    }
    if (status) return OFDMR_OK;  // stream-ordered: overflow reported in status bit 2
    // no status array: the reference's exception needs the flags now (synchronous)
    std::vector<int32_t> ef(frames);
    e = cudaMemcpyAsync(ef.data(), s.err, sizeof(int32_t) * frames, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { err = std::string("sft: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    for (int64_t f = 0; f < frames; ++f)
        if (ef[f]) { err = "sft: more than 128 accepted tones or 64 entries in a frame"; return OFDMR_ERR_CONFIG; }
    return OFDMR_OK;
}

int sft_slice_noise(SftScratch& s, cudaStream_t st, const float2* h, int n, int m, const uint64_t* seeds,
                    double* sigma2_out, int64_t frames, int64_t* launches, std::string& err) {
    const long long ql = lcm_ll(n, m);
    const int q = ql > (1 << 21) ? (1 << 21) : int(ql);
    int rc = sft_size_check(n, m, q, "estimate_noise_from_slice", err);
    if (rc) return rc;
    if (frames > 0x7fffffff) { err = "estimate_noise_from_slice: too many frames"; return OFDMR_ERR_CONFIG; }
    rc = upload_seeds(s, st, seeds, frames, err);
    if (rc) return rc;
    cudaError_t e = ensure(&s.draws, s.cap_draws, frames * 4);
    if (e != cudaSuccess) { err = std::string("estimate_noise_from_slice: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    const SftScratch::Tables* tb = nullptr;
    rc = sft_tables(s, q, &tb, err);
    if (rc) return rc;
    sft_draws_kernel<<<unsigned((frames + 63) / 64), 64, 0, st>>>(s.seeds, int(frames), n, m, 1, 1, s.draws);
    SftArgs a{};
    a.n = n;
    a.m = m;
    a.q = q;
    while ((1 << a.logq) < q) ++a.logq;
    a.tw_fft = tb->tw_fft;
    a.blu_m = tb->blu_m;
    a.blu_logm = tb->blu_logm;
    a.chirp = tb->chirp;
    a.bker = tb->bker;
    a.twm_f = tb->twm_f;
    a.twm_i = tb->twm_i;
    size_t smem = 0;
    int64_t chunk = frames;
    const bool smem_mode = sft_smem_q(q);
    auto kern = smem_mode ? slice_noise_kernel<false> : slice_noise_kernel<true>;
    if (smem_mode) {
        smem = sizeof(double2) * q + sizeof(double) * q;
    } else {
        a.gstride = noise_gstride(q, tb->blu_m);
        chunk = std::min<int64_t>(frames, kGlobalChunk);
        rc = ensure_gbuf(s, a.gstride * size_t(chunk), err);
        if (rc) return rc;
        a.gbuf = s.gbuf;
    }
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int64_t f0 = 0; f0 < frames && e == cudaSuccess; f0 += chunk) {
        const int64_t nf = std::min<int64_t>(chunk, frames - f0);
        SftArgs b = a;
        b.h = h + f0 * int64_t(n) * m;
        kern<<<unsigned(nf), kSftNT, smem, st>>>(b, s.draws + 2 * f0, sigma2_out + f0);
        e = cudaGetLastError();
        if (launches) ++*launches;
    }
    if (e != cudaSuccess) { err = std::string("estimate_noise_from_slice: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    if (launches) ++*launches;
    return OFDMR_OK;
}

int sft_detections(cudaStream_t st, const int32_t* k, const int32_t* l, const double* amp, const int32_t* n_entries,
                   int max_entries, int n, int m, const double* sigma2, double pfa, const int32_t* k_per_frame, int kmax,
                   int32_t* det_delay, int32_t* det_doppler, float* det_power, int32_t* counts, int64_t frames,
                   int64_t* launches, std::string& err) {
    if (!(pfa > 0.0 && pfa <= 1.0)) { err = "threshold: pfa must lie in (0,1]"; return OFDMR_ERR_CONFIG; }
    if (max_entries < 1 || max_entries > 64 || kmax < 1 || kmax > 64) {
        err = "detections_from_spectrum: max_entries and max_targets must lie in [1, 64] on the GPU path";
        return OFDMR_ERR_CONFIG;
    }
    for (int64_t f0 = 0; f0 < frames; f0 += 4 * 65535) {
        const int64_t nf = std::min<int64_t>(4 * 65535, frames - f0);
        SftDetArgs a{};
        a.k = k + f0 * max_entries;
        a.l = l + f0 * max_entries;
        a.amp = amp + 2 * f0 * max_entries;
        a.n_entries = n_entries + f0;
        a.max_entries = max_entries;
        a.n = n;
        a.m = m;
        a.sigma2 = sigma2 + f0;
        a.log_pfa = std::log(pfa);
        a.k_per_frame = k_per_frame ? k_per_frame + f0 : nullptr;
        a.kmax = kmax;
        a.det_delay = det_delay + f0 * kmax;
        a.det_doppler = det_doppler + f0 * kmax;
        a.det_power = det_power + f0 * kmax;
        a.counts = counts + f0;
        a.frames = int(nf);
        sft_detect_kernel<<<unsigned((nf + 3) / 4), 128, 0, st>>>(a);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { err = std::string("detections_from_spectrum: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
        if (launches) ++*launches;
    }
    return OFDMR_OK;
}

int division_noise(cudaStream_t st, const float2* x, int64_t cells, const double* sigma2, double* out, int64_t frames,
                   int64_t* launches, std::string& err) {
    for (int64_t f0 = 0; f0 < frames; f0 += 65535) {
        const int64_t nf = std::min<int64_t>(65535, frames - f0);
        division_noise_kernel<<<unsigned(nf), 256, 0, st>>>(x + f0 * cells, cells, sigma2 + f0, out + f0);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { err = std::string("division_noise_power: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
        if (launches) ++*launches;
    }
    return OFDMR_OK;
}

}  // namespace ofdmr
