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
    int32_t* err;
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
    // (v1 k Q/N + v2 l Q/M) mod Q with N, M, Q powers of two (the GPU path's precondition):
    // v1 k (Q/N) mod Q = (Q/N) ((v1 k) mod N), and k < N, v1 < N <= 2048 keep v1 k in 32 bits
    const unsigned qn = (unsigned)(q / n), qm = (unsigned)(q / m);
    const unsigned f = (qn * (((unsigned)v1 * (unsigned)k) & (unsigned)(n - 1)) +
                        qm * (((unsigned)v2 * (unsigned)l) & (unsigned)(m - 1))) &
                       (unsigned)(q - 1);
    return (int)f;
}

__device__ long long egcd(long long a, long long b, long long* x, long long* y) {
    // iterative form of sft.cpp:85-96 (same Bezout coefficients); the operands here are < Q <= 2048,
    // so the quotients and the coefficients (|x|, |y| <= Q) are exact in 32-bit arithmetic
    int aa = (int)a, bb = (int)b, x0 = 1, y0 = 0, x1 = 0, y1 = 1;
    while (bb != 0) {
        const int qt = aa / bb;
        int t = aa - qt * bb; aa = bb; bb = t;
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

__global__ void __launch_bounds__(kSftNT) sft_kernel(SftArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int q = a.q, n = a.n, m = a.m;
    double2* spec = reinterpret_cast<double2*>(smem_raw);   // [q]
    double2* sp1 = spec + q;                                  // [q] offset spectrum / full slice
    double2* sp2 = sp1 + q;                                   // [q]
    double2* s1d = sp2 + q;                                   // [q/2]
    double2* s2d = s1d + q / 2;                               // [q/2]
    double* pw = reinterpret_cast<double*>(s2d + q / 2);      // [q]
    int* clist = reinterpret_cast<int*>(pw + q);              // [q]
    int* alias = clist + q;                                   // [q]
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
            const int r = (int)((a1 + (long long)rs * t) & (n - 1)), c = (int)((a2 + (long long)cs * t) & (m - 1));
            const float2 v = h[(size_t)r * m + c];
            spec[t] = make_double2((double)v.x, (double)v.y);
        }
        __syncthreads();
        fft_r2(spec, q, a.logq, a.tw_fft);
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
                const int r = (int)((a1 + (long long)rs * t) & (n - 1)), c = (int)((a2 + (long long)cs * t) & (m - 1));
                const int r1 = r + 1 == n ? 0 : r + 1, c1 = c + 1 == m ? 0 : c + 1;
                const float2 u = h[(size_t)r1 * m + c], w = h[(size_t)r * m + c1];
                sp1[t] = make_double2((double)u.x, (double)u.y);
                sp2[t] = make_double2((double)w.x, (double)w.y);
            }
        }
        if (g > 1) {
            const int rsd = (int)((v1 * g) % n), csd = (int)((v2 * g) % m);
            for (int t = tid; t < qd; t += kSftNT) {
                const int r = (int)((a1 + (long long)rsd * t) & (n - 1)), c = (int)((a2 + (long long)csd * t) & (m - 1));
                const int r1 = r + 1 == n ? 0 : r + 1, c1 = c + 1 == m ? 0 : c + 1;
                const float2 u = h[(size_t)r1 * m + c], w = h[(size_t)r * m + c1];
                s1d[t] = make_double2((double)u.x, (double)u.y);
                s2d[t] = make_double2((double)w.x, (double)w.y);
            }
        }
        __syncthreads();
        if (g == 1) {
            fft_r2(sp1, q, a.logq, a.tw_fft);
            fft_r2(sp2, q, a.logq, a.tw_fft);
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
        a.err[fr] = s_err;
    }
}

long long gcd_ll(long long a, long long b) {
    while (b) { const long long t = a % b; a = b; b = t; }
    return a < 0 ? -a : a;
}
long long lcm_ll(long long a, long long b) { return a / gcd_ll(a, b) * b; }
long long pmod_h(long long a, long long m) {
    const long long r = a % m;
    return r < 0 ? r + m : r;
}
bool slope_admissible(long long v1, long long v2, long long n, long long m) {
    const long long q = lcm_ll(n, m);
    const long long g1 = gcd_ll(pmod_h(v1, n), n), g2 = gcd_ll(pmod_h(v2, m), m);
    return lcm_ll(n / g1, m / g2) == q;
}
uint64_t derive_seed(uint64_t base, uint64_t stream) {
    uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t uniform_int(std::mt19937_64& e, uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t v;
    do { v = e(); } while (v >= limit);
    return v % n;
}

// pipeline.cpp:26-43 estimate_noise_from_slice: one CTA per frame; the slice through (0, 0)
// along the host-drawn slope, the oracle's radix-2 fp64 FFT (bit-identical spectrum),
// p = |s|^2 / Q^2, bitonic sort, p[Q/2] * Q / ln 2.
__global__ void __launch_bounds__(kSftNT) slice_noise_kernel(const float2* __restrict__ hall, int n, int m, int q,
                                                             int logq, const int32_t* __restrict__ slopes,
                                                             const double2* __restrict__ tw, double* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* sp = reinterpret_cast<double2*>(smem_raw);  // [q]
    double* pw = reinterpret_cast<double*>(sp + q);       // [q]
    const int fr = blockIdx.x;
    const float2* h = hall + (size_t)fr * n * m;
    const long long v1 = slopes[2 * fr], v2 = slopes[2 * fr + 1];
    for (int t = threadIdx.x; t < q; t += kSftNT) {
        const int r = (int)((v1 * t) % n), c = (int)((v2 * t) % m);
        const float2 v = h[(size_t)r * m + c];
        sp[t] = make_double2((double)v.x, (double)v.y);
    }
    __syncthreads();
    fft_r2(sp, q, logq, tw);
    const double qq = (double)q * (double)q;
    for (int t = threadIdx.x; t < q; t += kSftNT) pw[t] = dnorm(sp[t]) / qq;
    __syncthreads();
    for (int k = 2; k <= q; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < q; i += kSftNT) {
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

int sft_slice_noise(SftScratch& s, cudaStream_t st, const float2* h, int n, int m, const uint64_t* seeds,
                    double* sigma2_out, int64_t frames, int64_t* launches, std::string& err) {
    auto pow2 = [](int v) { return v >= 2 && (v & (v - 1)) == 0; };
    if (!pow2(n) || !pow2(m)) { err = "estimate_noise_from_slice: N and M must be powers of two on the GPU path"; return OFDMR_ERR_CONFIG; }
    const int q = int(lcm_ll(n, m));
    if (q > 2048 || q < 16) { err = "estimate_noise_from_slice: Q = lcm(N, M) must lie in [16, 2048]"; return OFDMR_ERR_CONFIG; }
    if (frames > 0x7fffffff) { err = "estimate_noise_from_slice: too many frames"; return OFDMR_ERR_CONFIG; }
    std::vector<int32_t> slopes(size_t(frames) * 2);
    for (int64_t f = 0; f < frames; ++f) {  // Rng(seed), pipeline.cpp:31-35
        std::mt19937_64 e(seeds[f]);
        long long v1, v2;
        do {
            v1 = (long long)(1 + uniform_int(e, n > 1 ? n - 1 : 1));
            v2 = (long long)(1 + uniform_int(e, m > 1 ? m - 1 : 1));
        } while (!slope_admissible(v1, v2, n, m));
        slopes[2 * f] = int32_t(v1);
        slopes[2 * f + 1] = int32_t(v2);
    }
    std::vector<double2> twf(q / 2);
    for (int k = 0; k < q / 2; ++k) {
        const double ang = (double)(-1) * kTwoPiD * (double)k / (double)q;
        twf[k] = make_double2(std::cos(ang), std::sin(ang));
    }
    int64_t cap_q = s.cap_q;
    cudaError_t e = ensure(&s.draws, s.cap_draws, int64_t(slopes.size()));
    if (e == cudaSuccess) e = ensure(&s.tw_fft, cap_q, q);
    if (e != cudaSuccess) { err = std::string("estimate_noise_from_slice: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    s.cap_q = int(std::min<int64_t>(cap_q, s.cap_q ? s.cap_q : cap_q));
    e = cudaMemcpyAsync(s.draws, slopes.data(), sizeof(int32_t) * slopes.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(s.tw_fft, twf.data(), sizeof(double2) * (q / 2), cudaMemcpyHostToDevice, st);
    s.tw_q = 0;  // tw_fft rewritten here: sft_run rebuilds its tables on its next call
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // host vectors go out of scope
    if (e != cudaSuccess) { err = std::string("estimate_noise_from_slice: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    int logq = 0;
    while ((1 << logq) < q) ++logq;
    const size_t smem = sizeof(double2) * q + sizeof(double) * q;
    slice_noise_kernel<<<unsigned(frames), kSftNT, smem, st>>>(h, n, m, q, logq, s.draws, s.tw_fft, sigma2_out);
    e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("estimate_noise_from_slice: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    if (launches) ++*launches;
    return OFDMR_OK;
}

void sft_free(SftScratch& s) {
    cudaFree(s.draws);
    cudaFree(s.sigma2);
    cudaFree(s.tw_ref);
    cudaFree(s.tw_fft);
    cudaFree(s.err);
    s = SftScratch{};
}

namespace {

// Persistent host worker pool for the per-frame draws: run(nt, fn) calls fn(t, nt) for t < nt,
// t = 0 on the caller, and returns when all are done.  One run at a time (contexts on several host
// threads queue); the pool lives for the process (never destroyed: no joins at exit).
class HostPool {
   public:
    static HostPool& get() {
        static HostPool* pool = new HostPool;
        return *pool;
    }
    int size() const { return (int)workers_.size() + 1; }
    void run(int nt, const std::function<void(int, int)>& fn) {
        std::lock_guard<std::mutex> run_lock(run_mu_);
        nt = std::max(1, std::min(nt, size()));
        if (nt == 1) {
            fn(0, 1);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            active_ = nt - 1;
            pending_ = nt - 1;
            nt_ = nt;
            ++gen_;
        }
        cv_.notify_all();
        fn(0, nt);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

   private:
    HostPool() {
        const int n = (int)std::max(1u, std::thread::hardware_concurrency()) - 1;
        for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
        for (auto& w : workers_) w.detach();
    }
    void loop(int id) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int, int)>* f;
            int nt;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (id > active_) continue;
                f = fn_;
                nt = nt_;
            }
            (*f)(id, nt);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> workers_;
    const std::function<void(int, int)>* fn_ = nullptr;
    int active_ = 0, pending_ = 0, nt_ = 1;
    uint64_t gen_ = 0;
};

}  // namespace

int sft_run(SftScratch& s, cudaStream_t st, const float2* h, int n, int m, const ofdmr_sft_config& cfg,
            const uint64_t* seeds, const double* sigma2, int32_t* k_out, int32_t* l_out, double* amp_out,
            int32_t* n_entries, int32_t* iterations, int64_t* samples_used, int32_t* converged, double* residual,
            int64_t frames, int64_t* launches, std::string& err) {
    auto pow2 = [](int v) { return v >= 2 && (v & (v - 1)) == 0; };
    if (!pow2(n) || !pow2(m)) { err = "sft: N and M must be powers of two on the GPU path"; return OFDMR_ERR_CONFIG; }
    const int q = int(lcm_ll(n, m));
    if (q > 2048 || q < 16) { err = "sft: Q = lcm(N, M) must lie in [16, 2048] on the GPU path"; return OFDMR_ERR_CONFIG; }
    if (cfg.i_max < 0 || cfg.max_entries < 1 || cfg.max_entries > 64 || frames > 65535 * 32) {
        err = "sft: bad i_max / max_entries";
        return OFDMR_ERR_CONFIG;
    }
    const int i_max = cfg.i_max;
    // host-side data-independent draws (sft.cpp:191, 212-218)
    std::vector<int32_t> draws(size_t(frames) * size_t(i_max > 0 ? i_max : 1) * 4);
    auto draw_frames = [&](int64_t f0, int64_t f1) {
        for (int64_t f = f0; f < f1; ++f) {
            std::mt19937_64 e(derive_seed(seeds[f], 0x73667421));
            for (int it = 0; it < i_max; ++it) {
                long long v1, v2;
                do {
                    v1 = (long long)(1 + uniform_int(e, n > 1 ? n - 1 : 1));
                    v2 = (long long)(1 + uniform_int(e, m > 1 ? m - 1 : 1));
                } while (!slope_admissible(v1, v2, n, m));
                const long long a1 = (long long)uniform_int(e, n), a2 = (long long)uniform_int(e, m);
                int32_t* d = &draws[(size_t(f) * i_max + it) * 4];
                d[0] = int32_t(v1);
                d[1] = int32_t(v2);
                d[2] = int32_t(a1);
                d[3] = int32_t(a2);
            }
        }
    };
    // one engine per frame (seeding + first twist dominate): frames split over a persistent pool of
    // host threads (spawning threads per call cost more than the draws); every frame's draws are
    // independent of the split
    {
        const int nt = (int)std::min<int64_t>(HostPool::get().size(), frames / 64 + 1);
        HostPool::get().run(nt, [&](int t, int nt_run) {
            draw_frames(frames * t / nt_run, frames * (t + 1) / nt_run);
        });
    }
    const double2* old_ref = s.tw_ref;
    const double2* old_fft = s.tw_fft;
    int64_t cap_s2 = s.cap_frames, cap_err = s.cap_frames, cap_q = s.cap_q, cap_q2 = s.cap_q;
    cudaError_t e = ensure(&s.draws, s.cap_draws, int64_t(draws.size()));
    if (e == cudaSuccess) e = ensure(&s.sigma2, cap_s2, frames);
    if (e == cudaSuccess) e = ensure(&s.err, cap_err, frames);
    if (e == cudaSuccess) e = ensure(&s.tw_ref, cap_q, q);
    if (e == cudaSuccess) e = ensure(&s.tw_fft, cap_q2, q);
    if (e != cudaSuccess) { err = std::string("sft: allocation: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    s.cap_frames = std::min(cap_s2, cap_err);
    s.cap_q = int(std::min(cap_q, cap_q2));
    e = cudaMemcpyAsync(s.draws, draws.data(), sizeof(int32_t) * draws.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(s.sigma2, sigma2, sizeof(double) * frames, cudaMemcpyHostToDevice, st);
    // twiddle tables: reference rotation table (sft.cpp:29-44) and radix-2 table (oracle.c),
    // built and uploaded only when Q changed or the buffers were reallocated
    if (e == cudaSuccess && (s.tw_q != q || s.tw_ref != old_ref || s.tw_fft != old_fft)) {
        std::vector<double2> twr(q), twf(q / 2);
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
        for (int k = 0; k < q / 2; ++k) {
            const double ang = (double)(-1) * kTwoPiD * (double)k / (double)q;
            twf[k] = make_double2(std::cos(ang), std::sin(ang));
        }
        e = cudaMemcpyAsync(s.tw_ref, twr.data(), sizeof(double2) * q, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(s.tw_fft, twf.data(), sizeof(double2) * (q / 2), cudaMemcpyHostToDevice, st);
        s.tw_q = e == cudaSuccess ? q : 0;
    }
    if (e != cudaSuccess) { err = std::string("sft: upload: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }

    SftArgs a{};
    a.h = h;
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
    a.draws = s.draws;
    a.sigma2 = s.sigma2;
    a.tw_ref = s.tw_ref;
    a.tw_fft = s.tw_fft;
    a.k_out = k_out;
    a.l_out = l_out;
    a.amp_out = amp_out;
    a.n_entries = n_entries;
    a.iterations = iterations;
    a.samples_used = samples_used;
    a.converged = converged;
    a.residual = residual;
    a.err = s.err;
    const size_t smem = sizeof(double2) * (3 * size_t(q) + size_t(q)) + sizeof(double) * q + sizeof(int) * 2 * q;
    e = cudaFuncSetAttribute(sft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) { err = std::string("sft: smem attr: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    sft_kernel<<<unsigned(frames), kSftNT, smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) { err = std::string("sft: launch: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    if (launches) ++*launches;
    // overflow flags (comps > kMaxComp) — stream-ordered check requires a sync
    std::vector<int32_t> ef(frames);
    e = cudaMemcpyAsync(ef.data(), s.err, sizeof(int32_t) * frames, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { err = std::string("sft: ") + cudaGetErrorString(e); return OFDMR_ERR_CUDA; }
    for (int64_t f = 0; f < frames; ++f)
        if (ef[f]) { err = "sft: more than 128 accepted tones in a frame"; return OFDMR_ERR_CONFIG; }
    return OFDMR_OK;
}

}  // namespace ofdmr
