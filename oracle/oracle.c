/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  CPU restatement (plain C, fp64) of the
 * reference receiver hot path (arXiv 2209.03883 `ofdmradar`).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this library, and only as the checker or the timed CPU
 * baseline — never as the product path.
 *
 * Parity pinning: this restatement is checked (tests/test_oracle_*.py) against
 *   (1) the known-answer values of the reference tests, and
 *   (2) golden vectors produced by the reference's OWN sources compiled with a
 *       substitute FFT (oracle/_ref, recipe oracle/Makefile; fixtures committed
 *       under tests/golden/ with the generating script tests/golden/make_golden.py).
 *
 * Each function cites the reference file:line it restates.  FFTW3 (unpinned,
 * FFTW_ESTIMATE, proj/CMakeLists.txt:12-13) is not present; its contract
 * (unscaled, forward e^{-j}, inverse e^{+j}; include/ofdmradar/fft.hpp:12-15) is
 * restated by orc_fft below (radix-2 for powers of two, Bluestein otherwise).
 */
#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cd;
static const double kTwoPi = 6.283185307179586476925286766559;

/* ------------------------------------------------------------------ FFT -- */

static int is_pow2(size_t n) { return n && !(n & (n - 1)); }

/* Per-(n, sign) twiddle tables, computed once with the same expression as before and cached
 * for the life of the process (the reference caches its FFTW plans the same way, fft.cpp:17-43),
 * so a transform no longer pays malloc + n/2 cos/sin per call.  Values and butterfly order are
 * unchanged: every output is bit-identical to the uncached version. */
#define ORC_TW_MAX_LOG2 40
static double* g_tw_cache[2][ORC_TW_MAX_LOG2];
static pthread_mutex_t g_tw_mu = PTHREAD_MUTEX_INITIALIZER;

static const double* pow2_twiddles(size_t n, int sign) {
    int lg = 0;
    while (((size_t)1 << lg) < n) lg++;
    const int si = sign > 0;
    double* tw = __atomic_load_n(&g_tw_cache[si][lg], __ATOMIC_ACQUIRE);
    if (tw) return tw;
    pthread_mutex_lock(&g_tw_mu);
    tw = g_tw_cache[si][lg];
    if (!tw) {
        tw = (double*)malloc(sizeof(double) * (n > 1 ? n : 2)); /* n/2 complex twiddles of the top level */
        for (size_t k = 0; k < n / 2; k++) {
            const double ang = (double)sign * kTwoPi * (double)k / (double)n;
            tw[2 * k] = cos(ang);
            tw[2 * k + 1] = sin(ang);
        }
        __atomic_store_n(&g_tw_cache[si][lg], tw, __ATOMIC_RELEASE);
    }
    pthread_mutex_unlock(&g_tw_mu);
    return tw;
}

/* In-place iterative radix-2 on interleaved doubles. sign = -1 forward, +1 inverse. */
static void fft_pow2(double* a, size_t n, int sign) {
    if (n <= 1) return;
    for (size_t i = 1, j = 0; i < n; i++) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double t0 = a[2 * i], t1 = a[2 * i + 1];
            a[2 * i] = a[2 * j];
            a[2 * i + 1] = a[2 * j + 1];
            a[2 * j] = t0;
            a[2 * j + 1] = t1;
        }
    }
    const double* tw = pow2_twiddles(n, sign);
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len / 2, step = n / len;
        for (size_t i = 0; i < n; i += len) {
            for (size_t k = 0; k < half; k++) {
                const double wr = tw[2 * k * step], wi = tw[2 * k * step + 1];
                double* u = a + 2 * (i + k);
                double* v = a + 2 * (i + k + half);
                const double vr = v[0] * wr - v[1] * wi;
                const double vi = v[0] * wi + v[1] * wr;
                v[0] = u[0] - vr;
                v[1] = u[1] - vi;
                u[0] += vr;
                u[1] += vi;
            }
        }
    }
}

/* Bluestein chirp-z for arbitrary n (reference tests use 48, 70, 560, lcm sizes).  The chirp w
 * and the transformed kernel FFT(B) depend only on (n, sign): cached like the radix-2 twiddles
 * (same expressions, same transform: bit-identical results). */
typedef struct blu_plan {
    size_t n, m;
    int sign;
    double* w;   /* 2n: chirp e^{sign j pi k^2 / n} */
    double* fb;  /* 2m: FFT_m of the conjugate chirp kernel */
    struct blu_plan* next;
} blu_plan;
static blu_plan* g_blu_plans;
static pthread_mutex_t g_blu_mu = PTHREAD_MUTEX_INITIALIZER;

static const blu_plan* bluestein_plan(size_t n, int sign) {
    pthread_mutex_lock(&g_blu_mu);
    for (blu_plan* p = g_blu_plans; p; p = p->next)
        if (p->n == n && p->sign == sign) {
            pthread_mutex_unlock(&g_blu_mu);
            return p;
        }
    size_t m = 1;
    while (m < 2 * n - 1) m <<= 1;
    blu_plan* p = (blu_plan*)malloc(sizeof(blu_plan));
    p->n = n;
    p->m = m;
    p->sign = sign;
    p->w = (double*)malloc(sizeof(double) * 2 * n);
    p->fb = (double*)calloc(2 * m, sizeof(double));
    for (size_t k = 0; k < n; k++) {
        const unsigned long long k2 = ((unsigned long long)k * k) % (2ULL * n);
        const double ang = (double)sign * kTwoPi * 0.5 * (double)k2 / (double)n;
        p->w[2 * k] = cos(ang);
        p->w[2 * k + 1] = sin(ang);
    }
    double* B = p->fb;
    B[0] = p->w[0];
    B[1] = -p->w[1];
    for (size_t k = 1; k < n; k++) {
        B[2 * k] = B[2 * (m - k)] = p->w[2 * k];
        B[2 * k + 1] = B[2 * (m - k) + 1] = -p->w[2 * k + 1];
    }
    pthread_mutex_unlock(&g_blu_mu);
    fft_pow2(B, m, -1);
    pthread_mutex_lock(&g_blu_mu);
    p->next = g_blu_plans;
    g_blu_plans = p;
    pthread_mutex_unlock(&g_blu_mu);
    return p;
}

static void fft_bluestein(double* a, size_t n, int sign) {
    const blu_plan* pl = bluestein_plan(n, sign);
    const size_t m = pl->m;
    const double* w = pl->w;
    const double* B = pl->fb;
    double* A = (double*)calloc(2 * m, sizeof(double));
    for (size_t k = 0; k < n; k++) {
        A[2 * k] = a[2 * k] * w[2 * k] - a[2 * k + 1] * w[2 * k + 1];
        A[2 * k + 1] = a[2 * k] * w[2 * k + 1] + a[2 * k + 1] * w[2 * k];
    }
    fft_pow2(A, m, -1);
    for (size_t k = 0; k < m; k++) {
        const double r = A[2 * k] * B[2 * k] - A[2 * k + 1] * B[2 * k + 1];
        const double i = A[2 * k] * B[2 * k + 1] + A[2 * k + 1] * B[2 * k];
        A[2 * k] = r;
        A[2 * k + 1] = i;
    }
    fft_pow2(A, m, +1);
    const double inv_m = 1.0 / (double)m;
    for (size_t k = 0; k < n; k++) {
        const double cr = A[2 * k] * inv_m, ci = A[2 * k + 1] * inv_m;
        a[2 * k] = cr * w[2 * k] - ci * w[2 * k + 1];
        a[2 * k + 1] = cr * w[2 * k + 1] + ci * w[2 * k];
    }
    free(A);
}

/* fft.hpp:12-15 contract: unscaled; sign -1 = forward e^{-j}, +1 = inverse e^{+j}. */
void orc_fft(double* data, size_t n, int sign) {
    if (n <= 1) return;
    if (is_pow2(n)) fft_pow2(data, n, sign);
    else fft_bluestein(data, n, sign);
}

/* Strided batch helper: transform `count` vectors of length n at (stride, dist). */
static void fft_strided(cd* data, size_t n, size_t count, size_t stride, size_t dist, int sign) {
    double* buf = (double*)malloc(sizeof(double) * 2 * n);
    for (size_t c = 0; c < count; c++) {
        cd* base = data + c * dist;
        for (size_t i = 0; i < n; i++) {
            buf[2 * i] = creal(base[i * stride]);
            buf[2 * i + 1] = cimag(base[i * stride]);
        }
        orc_fft(buf, n, sign);
        for (size_t i = 0; i < n; i++) base[i * stride] = CMPLX(buf[2 * i], buf[2 * i + 1]);
    }
    free(buf);
}

/* ------------------------------------------------------ OFDM front end -- */

/* waveform.cpp:133-149 ofdm_modulate: per symbol l, unscaled inverse FFT_N of column l
 * times 1/N; stream[l][0..ncp) = sym[n - ncp + i], stream[l][ncp..) = sym. */
int orc_ofdm_modulate(const cd* x, size_t n, size_t m, size_t ncp, cd* stream) {
    if (ncp > n) return 2;
    const size_t ns = n + ncp;
    const double inv_n = 1.0 / (double)n;
    double* sym = (double*)malloc(sizeof(double) * 2 * n);
    for (size_t l = 0; l < m; l++) {
        for (size_t k = 0; k < n; k++) {
            sym[2 * k] = creal(x[k * m + l]);
            sym[2 * k + 1] = cimag(x[k * m + l]);
        }
        orc_fft(sym, n, +1);
        cd* dst = stream + l * ns;
        for (size_t i = 0; i < ncp; i++) dst[i] = CMPLX(sym[2 * (n - ncp + i)] * inv_n, sym[2 * (n - ncp + i) + 1] * inv_n);
        for (size_t i = 0; i < n; i++) dst[ncp + i] = CMPLX(sym[2 * i] * inv_n, sym[2 * i + 1] * inv_n);
    }
    free(sym);
    return 0;
}

/* waveform.cpp:152-166 ofdm_demodulate: strip the cyclic prefix of symbol l and take the
 * unscaled forward FFT_N of the next N samples -> column l of the N x M grid. */
int orc_ofdm_demodulate(const cd* stream, size_t n, size_t m, size_t ncp, cd* x) {
    const size_t ns = n + ncp;
    double* sym = (double*)malloc(sizeof(double) * 2 * n);
    for (size_t l = 0; l < m; l++) {
        const cd* src = stream + l * ns + ncp;
        for (size_t i = 0; i < n; i++) {
            sym[2 * i] = creal(src[i]);
            sym[2 * i + 1] = cimag(src[i]);
        }
        orc_fft(sym, n, -1);
        for (size_t k = 0; k < n; k++) x[k * m + l] = CMPLX(sym[2 * k], sym[2 * k + 1]);
    }
    free(sym);
    return 0;
}

/* --------------------------------------------------------- estimation -- */

/* estimation.cpp:10-21 spectral_division: H = Y / X, error 2 on a zero X cell. */
int orc_spectral_division(const cd* y, const cd* x, cd* h, size_t n, size_t m) {
    const size_t total = n * m;
    for (size_t i = 0; i < total; i++) {
        const cd xv = x[i];
        if (creal(xv) == 0.0 && cimag(xv) == 0.0) return 2;
        h[i] = y[i] / xv;
    }
    return 0;
}

/* estimation.cpp:23-39 dft_ce: per column IFFT_N, taps < L scaled 1/N, taps >= L zeroed, FFT_N. */
int orc_dft_ce(const cd* h, cd* out, size_t n, size_t m, size_t n_cp) {
    if (n_cp > n) return 2;
    double* col = (double*)malloc(sizeof(double) * 2 * n);
    const double inv_n = 1.0 / (double)n;
    for (size_t l = 0; l < m; l++) {
        for (size_t k = 0; k < n; k++) {
            col[2 * k] = creal(h[k * m + l]);
            col[2 * k + 1] = cimag(h[k * m + l]);
        }
        orc_fft(col, n, +1);
        for (size_t k = 0; k < n_cp; k++) {
            col[2 * k] *= inv_n;
            col[2 * k + 1] *= inv_n;
        }
        for (size_t k = n_cp; k < n; k++) col[2 * k] = col[2 * k + 1] = 0.0;
        orc_fft(col, n, -1);
        for (size_t k = 0; k < n; k++) out[k * m + l] = CMPLX(col[2 * k], col[2 * k + 1]);
    }
    free(col);
    return 0;
}

/* pipeline.cpp:18-23 division_noise_power: sigma2 * mean(1/|x|^2). */
double orc_division_noise_power(double sigma2, const cd* x, size_t count) {
    if (sigma2 <= 0.0) return 0.0;
    double inv_acc = 0.0;
    for (size_t i = 0; i < count; i++) {
        const double re = creal(x[i]), im = cimag(x[i]);
        inv_acc += 1.0 / (re * re + im * im);
    }
    return sigma2 * inv_acc / (double)count;
}

/* -------------------------------------------------------- periodogram -- */

/* periodogram.cpp:25-37 make_window (0 = rectangular, 1 = Hamming, symmetric n-1). */
void orc_make_window(int kind, size_t n, size_t m, double* wk, double* wl) {
    for (size_t k = 0; k < n; k++) wk[k] = 1.0;
    for (size_t l = 0; l < m; l++) wl[l] = 1.0;
    if (kind == 1) {
        for (size_t k = 0; k < n; k++) wk[k] = 0.54 - 0.46 * cos(kTwoPi * (double)k / (double)(n - 1));
        for (size_t l = 0; l < m; l++) wl[l] = 0.54 - 0.46 * cos(kTwoPi * (double)l / (double)(m - 1));
    }
}

/* periodogram.cpp:11-16 Window2d::power_factor. */
double orc_power_factor(const double* wk, size_t n, const double* wl, size_t m) {
    double sk = 0.0, sl = 0.0;
    for (size_t k = 0; k < n; k++) sk += wk[k] * wk[k];
    for (size_t l = 0; l < m; l++) sl += wl[l] * wl[l];
    return sk * sl / ((double)n * (double)m);
}

/* periodogram.cpp:39-75: window, zero-pad M', forward FFT along symbols, zero-pad N',
 * inverse FFT along subcarriers, |.|^2/(NM), fftshift of the Doppler axis. */
int orc_periodogram(const cd* h, size_t n, size_t m, const double* wk, const double* wl, size_t np,
                    size_t mp, double* p) {
    if (np < n || mp < m) return 2;
    cd* full = (cd*)calloc(np * mp, sizeof(cd));
    for (size_t k = 0; k < n; k++) {
        const double w = wk[k];
        for (size_t l = 0; l < m; l++) full[k * mp + l] = h[k * m + l] * (w * wl[l]);
    }
    fft_strided(full, mp, n, 1, mp, -1);  /* forward_rows over the first N rows */
    fft_strided(full, np, mp, mp, 1, +1); /* inverse_cols over N' rows */
    const double scale = 1.0 / ((double)n * (double)m);
    const size_t half = mp / 2;
    for (size_t r = 0; r < np; r++) {
        for (size_t s = 0; s < mp; s++) {
            const cd v = full[r * mp + s];
            const double re = creal(v), im = cimag(v);
            p[r * mp + (s + half) % mp] = (re * re + im * im) * scale;
        }
    }
    free(full);
    return 0;
}

/* periodogram.cpp:77-81 detection_threshold. Returns 2 on bad arguments. */
int orc_detection_threshold(double sigma2, double pfa, double pf, double* eta) {
    if (sigma2 < 0.0) return 2;
    if (!(pfa > 0.0 && pfa <= 1.0)) return 2;
    *eta = -sigma2 * log(pfa) * pf;
    return 0;
}

/* Stable merge sort of cell indices by (p desc, index asc); reentrant (no global comparator state). */
static void sort_cells(size_t* cells, size_t count, const double* p) {
    if (count < 2) return;
    size_t* tmp = (size_t*)malloc(sizeof(size_t) * count);
    for (size_t width = 1; width < count; width *= 2) {
        for (size_t lo = 0; lo < count; lo += 2 * width) {
            size_t mid = lo + width < count ? lo + width : count;
            size_t hi = lo + 2 * width < count ? lo + 2 * width : count;
            size_t i = lo, j = mid, o = lo;
            while (i < mid && j < hi) {
                const double pi = p[cells[i]], pj = p[cells[j]];
                int take_i = (pi != pj) ? (pi > pj) : (cells[i] < cells[j]);
                tmp[o++] = take_i ? cells[i++] : cells[j++];
            }
            while (i < mid) tmp[o++] = cells[i++];
            while (j < hi) tmp[o++] = cells[j++];
        }
        memcpy(cells, tmp, sizeof(size_t) * count);
    }
    free(tmp);
}

/* periodogram.cpp:89-136 extract_peaks: cells with mask set, sorted by (P desc, index asc);
 * greedy strict 3x3 (wrapped) local maxima, neighbourhood claiming, cap max_targets.
 * Outputs delay bin, signed Doppler bin (periodogram.hpp:43-45), power. Returns count. */
long orc_extract_peaks(const double* p, size_t rows, size_t cols, const uint8_t* mask,
                       size_t max_targets, long* delay, long* doppler, double* power) {
    const size_t total = rows * cols;
    size_t* cells = (size_t*)malloc(sizeof(size_t) * (total ? total : 1));
    size_t nc = 0;
    for (size_t i = 0; i < total; i++)
        if (mask[i]) cells[nc++] = i;
    sort_cells(cells, nc, p);
    uint8_t* claimed = (uint8_t*)calloc(total ? total : 1, 1);
    long out = 0;
    for (size_t ci = 0; ci < nc; ci++) {
        if ((size_t)out >= max_targets) break;
        const size_t idx = cells[ci];
        if (claimed[idx]) continue;
        const size_t r = idx / cols, c = idx % cols;
        const double v = p[idx];
        int is_max = 1;
        for (int dr = -1; dr <= 1 && is_max; ++dr) {
            if (dr != 0 && rows == 1) continue;
            for (int dc = -1; dc <= 1; ++dc) {
                if (dc != 0 && cols == 1) continue;
                if (dr == 0 && dc == 0) continue;
                const size_t rr = (size_t)(((long)r + dr + (long)rows) % (long)rows);
                const size_t cc = (size_t)(((long)c + dc + (long)cols) % (long)cols);
                if (p[rr * cols + cc] >= v) { is_max = 0; break; }
            }
        }
        if (!is_max) continue;
        for (int dr = -1; dr <= 1; ++dr)
            for (int dc = -1; dc <= 1; ++dc) {
                const size_t rr = (size_t)(((long)r + dr + (long)rows) % (long)rows);
                const size_t cc = (size_t)(((long)c + dc + (long)cols) % (long)cols);
                claimed[rr * cols + cc] = 1;
            }
        delay[out] = (long)r;
        doppler[out] = (long)c - (long)(cols / 2);
        power[out] = v;
        ++out;
    }
    free(cells);
    free(claimed);
    return out;
}

/* periodogram.cpp:138-144 bins_to_physics (c = 3e8, waveform.hpp:14). */
void orc_bins_to_physics(long delay_bin, long doppler_bin, size_t n_prime, size_t m_prime, double df,
                         double fc, double ts, double* range_m, double* vel_mps) {
    const double c = 3.0e8;
    *range_m = c * (double)delay_bin / (2.0 * (double)n_prime * df);
    *vel_mps = c * (double)doppler_bin / (2.0 * fc * (double)m_prime * ts);
}

/* periodogram.cpp:146-152 estimate_noise_power (median / ln 2 / power factor). */
static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}
double orc_estimate_noise_power(const double* p, size_t count, double pf) {
    double* v = (double*)malloc(sizeof(double) * count);
    memcpy(v, p, sizeof(double) * count);
    qsort(v, count, sizeof(double), cmp_double);
    const double med = v[count / 2];
    free(v);
    return med / 0.6931471805599453 / pf;
}

/* ------------------------------------------------------------ pipeline -- */

typedef struct orc_rx_config {
    int32_t n, m, n_prime, m_prime;
    int32_t estimator;   /* 0 = LS (and ZCP-LS: divide by precoded x_tx), 1 = DFT-CE */
    int32_t n_cp;        /* DFT-CE truncation L (waveform.n_cp, pipeline.cpp:55) */
    int32_t window;      /* 0 rectangular, 1 Hamming */
    double pfa;
} orc_rx_config;

/* pipeline.cpp:47-58 estimate_channel + :79-92 (sigma_h^2, window, periodogram,
 * threshold, mask, extract_peaks).  y/x are the c64 frames upcast to fp64.
 * p_out (N'xM', optional) receives the map.  Returns 0, or 2 on a config error. */
int orc_receive_frame(const orc_rx_config* cfg, const float* y32, const float* x32, double sigma2,
                      int32_t max_targets, long* delay, long* doppler, double* power, long* count,
                      double* sigma2_h_out, double* eta_out, double* p_out) {
    const size_t n = (size_t)cfg->n, m = (size_t)cfg->m, np = (size_t)cfg->n_prime,
                 mp = (size_t)cfg->m_prime;
    const size_t cells = n * m;
    cd* y = (cd*)malloc(sizeof(cd) * cells);
    cd* x = (cd*)malloc(sizeof(cd) * cells);
    cd* h = (cd*)malloc(sizeof(cd) * cells);
    for (size_t i = 0; i < cells; i++) {
        y[i] = CMPLX((double)y32[2 * i], (double)y32[2 * i + 1]);
        x[i] = CMPLX((double)x32[2 * i], (double)x32[2 * i + 1]);
    }
    int rc = orc_spectral_division(y, x, h, n, m);
    if (!rc && cfg->estimator == 1) {
        cd* h2 = (cd*)malloc(sizeof(cd) * cells);
        rc = orc_dft_ce(h, h2, n, m, (size_t)cfg->n_cp);
        free(h);
        h = h2;
    }
    double* p = NULL;
    if (!rc) {
        const double s2h = orc_division_noise_power(sigma2, x, cells);
        double* wk = (double*)malloc(sizeof(double) * n);
        double* wl = (double*)malloc(sizeof(double) * m);
        orc_make_window(cfg->window, n, m, wk, wl);
        const double pf = orc_power_factor(wk, n, wl, m);
        p = p_out ? p_out : (double*)malloc(sizeof(double) * np * mp);
        rc = orc_periodogram(h, n, m, wk, wl, np, mp, p);
        double eta = 0.0;
        if (!rc) rc = orc_detection_threshold(s2h, cfg->pfa, pf, &eta);
        if (!rc) {
            uint8_t* mask = (uint8_t*)malloc(np * mp);
            for (size_t i = 0; i < np * mp; i++) mask[i] = p[i] >= eta ? 1 : 0;
            *count = orc_extract_peaks(p, np, mp, mask, (size_t)max_targets, delay, doppler, power);
            free(mask);
        }
        if (sigma2_h_out) *sigma2_h_out = s2h;
        if (eta_out) *eta_out = eta;
        free(wk);
        free(wl);
        if (!p_out) free(p);
    }
    free(y);
    free(x);
    free(h);
    return rc;
}

typedef struct {
    const orc_rx_config* cfg;
    const float *y, *x;
    const double* sigma2;
    const int32_t* k_per_frame;
    int32_t k_max;
    long *delay, *doppler;
    double* power;
    long* count;
    double *s2h, *eta;
    long next, total;
    pthread_mutex_t mtx;
    int rc;
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* j = (batch_job*)arg;
    const size_t cells = (size_t)j->cfg->n * (size_t)j->cfg->m;
    for (;;) {
        pthread_mutex_lock(&j->mtx);
        const long f = j->next++;
        pthread_mutex_unlock(&j->mtx);
        if (f >= j->total) break;
        const int32_t kf = j->k_per_frame ? j->k_per_frame[f] : j->k_max;
        const int r = orc_receive_frame(j->cfg, j->y + 2 * cells * (size_t)f, j->x + 2 * cells * (size_t)f,
                                        j->sigma2[f], kf, j->delay + (size_t)f * j->k_max,
                                        j->doppler + (size_t)f * j->k_max, j->power + (size_t)f * j->k_max,
                                        j->count + f, j->s2h ? j->s2h + f : NULL, j->eta ? j->eta + f : NULL,
                                        NULL);
        if (r) j->rc = r;
    }
    return NULL;
}

/* run_pipeline's receiver half over a batch of frames, one frame per host thread
 * (the reference is single-threaded per frame but reentrant). */
int orc_receive_batch(const orc_rx_config* cfg, const float* y, const float* x, const double* sigma2,
                      long frames, const int32_t* k_per_frame, int32_t k_max, long* delay, long* doppler,
                      double* power, long* count, double* s2h, double* eta, int nthreads) {
    batch_job j = {cfg, y, x, sigma2, k_per_frame, k_max, delay, doppler, power, count, s2h, eta, 0, frames,
                   PTHREAD_MUTEX_INITIALIZER, 0};
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, batch_worker, &j);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    return j.rc;
}

/* ---------------------------------------------------------- MT19937-64 -- */
/* std::mt19937_64 (C++ standard [rand.predef]); Rng semantics rng.hpp:20-66. */

typedef struct { uint64_t mt[312]; int mti; } orc_rng;

void orc_rng_seed(orc_rng* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; i++)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->mti = 312;
}

uint64_t orc_rng_next(orc_rng* s) {
    if (s->mti >= 312) {
        for (int i = 0; i < 312; i++) {
            const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->mti = 0;
    }
    uint64_t x = s->mt[s->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* rng.hpp:34-42 uniform_int: rejection with limit = UINT64_MAX - UINT64_MAX % n. */
uint64_t orc_rng_uniform_int(orc_rng* s, uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t v;
    do { v = orc_rng_next(s); } while (v >= limit);
    return v % n;
}

/* rng.hpp:11-16 derive_seed (SplitMix64 finaliser). */
uint64_t orc_derive_seed(uint64_t base, uint64_t stream) {
    uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void orc_rng_u64(uint64_t seed, long count, uint64_t* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (long i = 0; i < count; i++) out[i] = orc_rng_next(&r);
}

/* --------------------------------------------------------------- FPS-SFT -- */

static long gcd_l(long a, long b) {
    while (b) { long t = a % b; a = b; b = t; }
    return a < 0 ? -a : a;
}
static size_t lcm_sz(size_t a, size_t b) { return a / (size_t)gcd_l((long)a, (long)b) * b; }
static long positive_mod(long a, long m) {
    const long r = a % m;
    return r < 0 ? r + m : r;
}

/* sft.cpp:46-51 slope_admissible. */
int orc_slope_admissible(long v1, long v2, size_t n, size_t m) {
    const size_t q = lcm_sz(n, m);
    const size_t g1 = (size_t)gcd_l(positive_mod(v1, (long)n), (long)n);
    const size_t g2 = (size_t)gcd_l(positive_mod(v2, (long)m), (long)m);
    return lcm_sz(n / g1, m / g2) == q;
}

/* sft.cpp:73-83 tone_bin. */
/* pipeline.cpp:26-43 estimate_noise_from_slice (FPS-SFT estimate-noise mode): admissible
 * slope from Rng(seed) (v1 = 1 + U(N-1), v2 = 1 + U(M-1) until admissible), the slice
 * through (0, 0) of length Q = lcm(N, M), forward FFT, p = |s|^2 / Q^2, the order statistic
 * p[Q/2] (nth_element) * Q / ln 2.  Output also the slope (for the GPU path's host draws). */
static int cmp_d(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}
double orc_estimate_noise_from_slice(const cd* h, size_t n, size_t m, uint64_t seed) {
    const size_t q = lcm_sz(n, m);
    orc_rng r;
    orc_rng_seed(&r, seed);
    long v1 = 1, v2 = 1;
    do {
        v1 = (long)(1 + orc_rng_uniform_int(&r, n > 1 ? n - 1 : 1));
        v2 = (long)(1 + orc_rng_uniform_int(&r, m > 1 ? m - 1 : 1));
    } while (!orc_slope_admissible(v1, v2, n, m));
    double* s = (double*)malloc(sizeof(double) * 2 * q);
    double* p = (double*)malloc(sizeof(double) * q);
    for (size_t t = 0; t < q; t++) {
        const size_t k = (size_t)(((unsigned long long)v1 * t) % n), l = (size_t)(((unsigned long long)v2 * t) % m);
        s[2 * t] = creal(h[k * m + l]);
        s[2 * t + 1] = cimag(h[k * m + l]);
    }
    orc_fft(s, q, -1);
    for (size_t i = 0; i < q; i++) p[i] = (s[2 * i] * s[2 * i] + s[2 * i + 1] * s[2 * i + 1]) / ((double)q * (double)q);
    qsort(p, q, sizeof(double), cmp_d);
    const double out = p[q / 2] * (double)q / 0.6931471805599453;
    free(s);
    free(p);
    return out;
}

static size_t tone_bin(long k, long l, long v1, long v2, size_t n, size_t m, size_t q) {
    const unsigned long long qn = q / n, qm = q / m;
    const unsigned long long f = ((unsigned long long)v1 * (unsigned long long)k * qn +
                                  (unsigned long long)v2 * (unsigned long long)l * qm) % q;
    return (size_t)f;
}

/* sft.cpp:85-96 egcd. */
static long egcd(long a, long b, long* x, long* y) {
    if (b == 0) { *x = 1; *y = 0; return a; }
    long x1, y1;
    const long g = egcd(b, a % b, &x1, &y1);
    *x = y1;
    *y = x1 - (a / b) * y1;
    return g;
}

/* sft.cpp:98-103 wrap_dist. */
static double wrap_dist(double a, long b, size_t period) {
    double d = fmod(a - (double)b, (double)period);
    if (d > (double)period / 2) d -= (double)period;
    if (d < -(double)period / 2) d += (double)period;
    return fabs(d);
}

/* sft.cpp:105-156 lattice_decode. */
static int lattice_decode(double kap, double lam, size_t f, long v1, long v2, size_t n, size_t m, size_t q_len,
                          double tol, long* out_k, long* out_l) {
    const long q = (long)q_len;
    const long a = (long)(((unsigned long long)v2 * (q_len / m)) % q_len);
    long x, y;
    const long d = egcd(a == 0 ? q : a, q, &x, &y);
    double best = tol;
    int found = 0;
    const long k_center = llround(kap);
    for (long dk = -2; dk <= 2; ++dk) {
        const long k = positive_mod(k_center + dk, (long)n);
        const double kd = wrap_dist(kap, k, n);
        if (kd >= best) continue;
        const long fk = (long)tone_bin(k, 0, v1, v2, n, m, q_len);
        const long rhs = positive_mod((long)f - fk, q);
        if (a == 0) {
            if (rhs != 0) continue;
            const long l = positive_mod(llround(lam), (long)m);
            const double dist = hypot(kd, wrap_dist(lam, l, m));
            if (dist < best) { best = dist; *out_k = k; *out_l = l; found = 1; }
            continue;
        }
        if (rhs % d != 0) continue;
        const long qd = q / d;
        long inv, tmp;
        egcd(positive_mod(a / d, qd), qd, &inv, &tmp);
        inv = positive_mod(inv, qd);
        const long l0 = positive_mod((long)(((__int128)(rhs / d) * inv) % qd), qd);
        for (long l = l0 % (long)m; l < (long)m; l += qd) {
            if (l < 0) continue;
            if (tone_bin(k, l, v1, v2, n, m, q_len) != f) continue;
            const double dist = hypot(kd, wrap_dist(lam, l, m));
            if (dist < best) { best = dist; *out_k = k; *out_l = l; found = 1; }
        }
    }
    return found;
}

static inline cd polar1(double th) { return CMPLX(cos(th), sin(th)); }

typedef struct orc_sft_config {
    int64_t i_max;
    double detect_threshold;
    uint64_t seed;
    double sigma2;
    double pfa;
    int64_t decimation;
    double frac_tol;
    double amp_tol;
} orc_sft_config;

typedef struct orc_sft_result {
    int64_t n_entries;
    double residual_energy;
    int32_t converged;
    int64_t iterations;
    int64_t samples_used;
} orc_sft_result;

typedef struct { long k, l; cd amp; } comp_t;

/* sort candidate bins by (|spec|^2 desc, index asc) — sft.cpp:256-261 */
static void sort_bins(size_t* c, size_t count, const double* pw) {
    if (count < 2) return;
    size_t* tmp = (size_t*)malloc(sizeof(size_t) * count);
    for (size_t width = 1; width < count; width *= 2) {
        for (size_t lo = 0; lo < count; lo += 2 * width) {
            size_t mid = lo + width < count ? lo + width : count;
            size_t hi = lo + 2 * width < count ? lo + 2 * width : count;
            size_t i = lo, j = mid, o = lo;
            while (i < mid && j < hi) {
                const double a = pw[c[i]], b = pw[c[j]];
                int take_i = (a != b) ? (a > b) : (c[i] < c[j]);
                tmp[o++] = take_i ? c[i++] : c[j++];
            }
            while (i < mid) tmp[o++] = c[i++];
            while (j < hi) tmp[o++] = c[j++];
        }
        memcpy(c, tmp, sizeof(size_t) * count);
    }
    free(tmp);
}

static inline double cnorm(cd v) { return creal(v) * creal(v) + cimag(v) * cimag(v); }

/* sft.cpp:185-459 sft_iterate.  h: N x M (fp64 complex).  Entries written to
 * (ek, el, ea_re, ea_im) up to max_entries, sorted as sft.cpp:448-458. */
int orc_sft_iterate(const cd* h, size_t n, size_t m, const orc_sft_config* cfg, long max_entries, long* ek,
                    long* el, double* ea_re, double* ea_im, orc_sft_result* res) {
    if (n == 0 || m == 0) return 2;
    const size_t q_len = lcm_sz(n, m);
    /* sft.cpp:29-44 twiddle_table: rotation with an exact polar resync every 256 */
    cd* tw = (cd*)malloc(sizeof(cd) * q_len);
    {
        const cd step = polar1(-kTwoPi / (double)q_len);
        cd cur = CMPLX(1.0, 0.0);
        for (size_t j = 0; j < q_len; ++j) {
            if ((j & 255u) == 0) cur = polar1(-kTwoPi * (double)j / (double)q_len);
            tw[j] = cur;
            cur *= step;
        }
    }
    orc_rng rng;
    orc_rng_seed(&rng, orc_derive_seed(cfg->seed, 0x73667421));

    size_t ncomp = 0, capcomp = 64;
    comp_t* comps = (comp_t*)malloc(sizeof(comp_t) * capcomp);

    cd* s0 = (cd*)malloc(sizeof(cd) * q_len);
    double* spec_d = (double*)malloc(sizeof(double) * 2 * q_len);
    cd* spec = (cd*)malloc(sizeof(cd) * q_len);
    double* pw = (double*)malloc(sizeof(double) * q_len);
    size_t* cand = (size_t*)malloc(sizeof(size_t) * q_len);
    int* alias = (int*)malloc(sizeof(int) * q_len);
    cd* spec1 = (cd*)malloc(sizeof(cd) * q_len);
    cd* spec2 = (cd*)malloc(sizeof(cd) * q_len);
    cd* s1d = (cd*)malloc(sizeof(cd) * q_len);
    cd* s2d = (cd*)malloc(sizeof(cd) * q_len);
    cd* s1full = (cd*)malloc(sizeof(cd) * q_len);
    cd* s2full = (cd*)malloc(sizeof(cd) * q_len);

    memset(res, 0, sizeof(*res));
    double rel_floor = 0.0;
    double threshold = cfg->detect_threshold;
    const int threshold_fixed = cfg->detect_threshold > 0.0;
    double residual = 0.0;

    for (size_t it = 0; it < (size_t)cfg->i_max; ++it) {
        res->iterations = (int64_t)it + 1;
        long v1, v2;
        do {
            v1 = (long)(1 + orc_rng_uniform_int(&rng, n > 1 ? n - 1 : 1));
            v2 = (long)(1 + orc_rng_uniform_int(&rng, m > 1 ? m - 1 : 1));
        } while (!orc_slope_admissible(v1, v2, n, m));
        const long a1 = (long)orc_rng_uniform_int(&rng, n);
        const long a2 = (long)orc_rng_uniform_int(&rng, m);
        const size_t rs = (size_t)(v1 % (long)n), cs = (size_t)(v2 % (long)m);

        /* sft.cpp:221-229 reference slice and 1/Q-scaled spectrum */
        {
            size_t r = (size_t)a1, c = (size_t)a2;
            for (size_t q = 0; q < q_len; ++q) {
                s0[q] = h[r * m + c];
                r += rs; if (r >= n) r -= n;
                c += cs; if (c >= m) c -= m;
            }
        }
        res->samples_used += (int64_t)q_len;
        for (size_t q = 0; q < q_len; ++q) { spec_d[2 * q] = creal(s0[q]); spec_d[2 * q + 1] = cimag(s0[q]); }
        orc_fft(spec_d, q_len, -1);
        const double inv_q = 1.0 / (double)q_len;
        for (size_t q = 0; q < q_len; ++q) spec[q] = CMPLX(spec_d[2 * q], spec_d[2 * q + 1]) * inv_q;

        /* sft.cpp:232-236 subtract accepted components */
        for (size_t ci = 0; ci < ncomp; ++ci) {
            const comp_t c = comps[ci];
            const size_t f = tone_bin(c.k, c.l, v1, v2, n, m, q_len);
            spec[f] -= c.amp * polar1(kTwoPi * ((double)(a1 * c.k) / (double)n + (double)(a2 * c.l) / (double)m));
        }

        if (it == 0) {
            double peak = 0.0;
            for (size_t q = 0; q < q_len; ++q) { const double v = cnorm(spec[q]); if (v > peak) peak = v; }
            rel_floor = 1e-9 * peak;
            if (!threshold_fixed) {
                const double noise_part = cfg->sigma2 > 0.0
                    ? 4.0 * cfg->sigma2 / (double)q_len * log((double)q_len / cfg->pfa) : 0.0;
                threshold = noise_part > rel_floor ? noise_part : rel_floor;
            }
        }

        size_t ncand = 0;
        double total_power = 0.0;
        for (size_t f = 0; f < q_len; ++f) {
            const double p = cnorm(spec[f]);
            pw[f] = p;
            total_power += p;
            if (p >= threshold && p > 0.0) cand[ncand++] = f;
        }
        sort_bins(cand, ncand, pw);
        if (ncand > 256) ncand = 256;

        if (ncand == 0) {
            residual = total_power;
            res->converged = 1;
            break;
        }

        /* sft.cpp:274-289 decimation back-off */
        double weakest = pw[cand[0]];
        for (size_t i = 0; i < ncand; ++i) if (pw[cand[i]] < weakest) weakest = pw[cand[i]];
        size_t g = cfg->decimation > 1 ? (size_t)cfg->decimation : 1;
        const double dim = (double)(n > m ? n : m);
        while (g > 1) {
            const int divides = q_len % g == 0 && q_len / g >= 16;
            int quiet = 1;
            if (cfg->sigma2 > 0.0) {
                const double angle_var = cfg->sigma2 * (1.0 + (double)g) / (2.0 * (double)q_len * weakest);
                quiet = dim / kTwoPi * sqrt(angle_var) <= 0.3;
            }
            if (divides && quiet) break;
            --g;
        }
        const size_t qd = q_len / g;

        /* sft.cpp:293-295 alias counts */
        memset(alias, 0, sizeof(int) * qd);
        for (size_t i = 0; i < ncand; ++i) alias[cand[i] % qd]++;
        for (size_t ci = 0; ci < ncomp; ++ci) alias[tone_bin(comps[ci].k, comps[ci].l, v1, v2, n, m, q_len) % qd]++;

        /* sft.cpp:297-328 offset slices */
        if (g == 1) {
            size_t r = (size_t)a1, c = (size_t)a2;
            for (size_t q = 0; q < q_len; ++q) {
                const size_t r1 = r + 1 == n ? 0 : r + 1;
                const size_t c1 = c + 1 == m ? 0 : c + 1;
                spec1[q] = h[r1 * m + c];
                spec2[q] = h[r * m + c1];
                r += rs; if (r >= n) r -= n;
                c += cs; if (c >= m) c -= m;
            }
            res->samples_used += 2 * (int64_t)q_len;
            for (int which = 0; which < 2; ++which) {
                cd* sp = which ? spec2 : spec1;
                for (size_t q = 0; q < q_len; ++q) { spec_d[2 * q] = creal(sp[q]); spec_d[2 * q + 1] = cimag(sp[q]); }
                orc_fft(spec_d, q_len, -1);
                for (size_t q = 0; q < q_len; ++q) sp[q] = CMPLX(spec_d[2 * q], spec_d[2 * q + 1]) * inv_q;
            }
        } else {
            const size_t rsd = (size_t)((v1 * (long)g) % (long)n), csd = (size_t)((v2 * (long)g) % (long)m);
            size_t r = (size_t)a1, c = (size_t)a2;
            for (size_t t = 0; t < qd; ++t) {
                const size_t r1 = r + 1 == n ? 0 : r + 1;
                const size_t c1 = c + 1 == m ? 0 : c + 1;
                s1d[t] = h[r1 * m + c];
                s2d[t] = h[r * m + c1];
                r += rsd; if (r >= n) r -= n;
                c += csd; if (c >= m) c -= m;
            }
            res->samples_used += 2 * (int64_t)qd;
        }

        int have_full = 0;
        for (size_t ci2 = 0; ci2 < ncand; ++ci2) {
            const size_t f = cand[ci2];
            if (cnorm(spec[f]) < threshold) continue;
            const cd c0 = spec[f];
            if (cnorm(c0) == 0.0) continue;
            cd c1, c2;
            int full_bin = g == 1;
            if (g == 1) {
                c1 = spec1[f];
                c2 = spec2[f];
            } else {
                const cd* a_s;
                const cd* b_s;
                size_t cnt, stride;
                if (alias[f % qd] > 1) {
                    if (!have_full) {  /* sft.cpp:356-368 ensure_full */
                        size_t r = (size_t)a1, c = (size_t)a2;
                        for (size_t q = 0; q < q_len; ++q) {
                            const size_t r1 = r + 1 == n ? 0 : r + 1;
                            const size_t c1i = c + 1 == m ? 0 : c + 1;
                            s1full[q] = h[r1 * m + c];
                            s2full[q] = h[r * m + c1i];
                            r += rs; if (r >= n) r -= n;
                            c += cs; if (c >= m) c -= m;
                        }
                        res->samples_used += 2 * (int64_t)(q_len - qd);
                        have_full = 1;
                    }
                    a_s = s1full; b_s = s2full; cnt = q_len; stride = 1;
                    full_bin = 1;
                } else {
                    a_s = s1d; b_s = s2d; cnt = qd; stride = g;
                }
                /* sft.cpp:333-348 targeted DFT: incremental rotation, resync every 256 */
                for (int which = 0; which < 2; ++which) {
                    const cd* smp = which ? b_s : a_s;
                    cd acc = CMPLX(0.0, 0.0);
                    const size_t stepi = (stride * f) % q_len;
                    const cd rot = tw[stepi];
                    cd cur = CMPLX(1.0, 0.0);
                    size_t idx = 0;
                    for (size_t t = 0; t < cnt; ++t) {
                        if ((t & 255u) == 0) cur = tw[idx];
                        acc += smp[t] * cur;
                        cur *= rot;
                        idx += stepi;
                        if (idx >= q_len) idx -= q_len;
                    }
                    const cd val = acc / (double)cnt;
                    if (which) c2 = val; else c1 = val;
                }
            }
            /* sft.cpp:389-398 accepted tones still live in the raw offset slices */
            for (size_t ci = 0; ci < ncomp; ++ci) {
                const comp_t c = comps[ci];
                const size_t fc = tone_bin(c.k, c.l, v1, v2, n, m, q_len);
                if (full_bin ? (fc != f) : (fc % qd != f % qd)) continue;
                const cd psi = c.amp * polar1(kTwoPi * ((double)(a1 * c.k) / (double)n + (double)(a2 * c.l) / (double)m));
                c1 -= psi * polar1(kTwoPi * (double)c.k / (double)n);
                c2 -= psi * polar1(kTwoPi * (double)c.l / (double)m);
            }
            double kap = carg(c1 / c0) / kTwoPi * (double)n;
            if (kap < 0) kap += (double)n;
            double lam = carg(c2 / c0) / kTwoPi * (double)m;
            if (lam < 0) lam += (double)m;
            long k = 0, l = 0;
            if (!lattice_decode(kap, lam, f, v1, v2, n, m, q_len, cfg->frac_tol * 5.0, &k, &l)) continue;
            const double m0 = cabs(c0), m1 = cabs(c1), m2 = cabs(c2);
            const double mean_mag = (m0 + m1 + m2) / 3.0;
            double mx = m0, mn = m0;
            if (m1 > mx) mx = m1;
            if (m2 > mx) mx = m2;
            if (m1 < mn) mn = m1;
            if (m2 < mn) mn = m2;
            if (mx - mn > cfg->amp_tol * mean_mag) continue;

            const cd psi0 = polar1(kTwoPi * ((double)(a1 * k) / (double)n + (double)(a2 * l) / (double)m));
            const cd psi1 = psi0 * polar1(kTwoPi * (double)k / (double)n);
            const cd psi2 = psi0 * polar1(kTwoPi * (double)l / (double)m);
            const cd amp = (c0 / psi0 + c1 / psi1 + c2 / psi2) / 3.0;

            long found = -1;
            for (size_t ci = 0; ci < ncomp; ++ci)
                if (comps[ci].k == k && comps[ci].l == l) { found = (long)ci; break; }
            if (found >= 0) {
                comps[found].amp += amp;
                if (cnorm(comps[found].amp) < threshold) {
                    memmove(comps + found, comps + found + 1, sizeof(comp_t) * (ncomp - (size_t)found - 1));
                    --ncomp;
                }
            } else {
                if (ncomp == capcomp) { capcomp *= 2; comps = (comp_t*)realloc(comps, sizeof(comp_t) * capcomp); }
                comps[ncomp].k = k;
                comps[ncomp].l = l;
                comps[ncomp].amp = amp;
                ++ncomp;
            }
            total_power -= cnorm(spec[f]);
            spec[f] = CMPLX(0.0, 0.0);
        }

        residual = total_power > 0.0 ? total_power : 0.0;
        const double conv_floor = cfg->sigma2 * (1.0 + 6.0 / sqrt((double)q_len)) + rel_floor * (double)q_len;
        if (residual <= conv_floor) {
            res->converged = 1;
            break;
        }
    }

    res->residual_energy = residual;
    /* sft.cpp:448-458 sort entries by (|A|^2 desc, k asc, l asc) — insertion sort (K small) */
    for (size_t i = 1; i < ncomp; ++i) {
        comp_t key = comps[i];
        size_t j = i;
        while (j > 0) {
            const comp_t p = comps[j - 1];
            const double pa = cnorm(key.amp), pb = cnorm(p.amp);
            int before = (pa != pb) ? (pa > pb) : (key.k != p.k ? key.k < p.k : key.l < p.l);
            if (!before) break;
            comps[j] = p;
            --j;
        }
        comps[j] = key;
    }
    res->n_entries = (int64_t)ncomp;
    for (size_t i = 0; i < ncomp && (long)i < max_entries; ++i) {
        ek[i] = comps[i].k;
        el[i] = comps[i].l;
        ea_re[i] = creal(comps[i].amp);
        ea_im[i] = cimag(comps[i].amp);
    }
    free(tw); free(comps); free(s0); free(spec_d); free(spec); free(pw); free(cand); free(alias);
    free(spec1); free(spec2); free(s1d); free(s2d); free(s1full); free(s2full);
    return 0;
}

/* Convenience: FPS-SFT over a c64 frame (upcast), for batch use. */
int orc_sft_frame_c64(const float* h32, size_t n, size_t m, const orc_sft_config* cfg, long max_entries,
                      long* ek, long* el, double* ea_re, double* ea_im, orc_sft_result* res) {
    cd* h = (cd*)malloc(sizeof(cd) * n * m);
    for (size_t i = 0; i < n * m; i++) h[i] = CMPLX((double)h32[2 * i], (double)h32[2 * i + 1]);
    const int rc = orc_sft_iterate(h, n, m, cfg, max_entries, ek, el, ea_re, ea_im, res);
    free(h);
    return rc;
}

/* sft.cpp:461-490 detections_from_spectrum. Returns count (<= max_targets). */
long orc_detections_from_spectrum(const long* ek, const long* el, const double* ea_re, const double* ea_im,
                                  long n_entries, size_t n, size_t m, double sigma2, double pfa,
                                  long max_targets, long* delay, long* doppler, double* power) {
    const double nm = (double)n * (double)m;
    const double eta = -sigma2 * log(pfa) * 1.0;
    long cnt = 0;
    long* td = (long*)malloc(sizeof(long) * (size_t)(n_entries + 1));
    long* tp = (long*)malloc(sizeof(long) * (size_t)(n_entries + 1));
    double* pp = (double*)malloc(sizeof(double) * (size_t)(n_entries + 1));
    for (long i = 0; i < n_entries; i++) {
        const double pwr = (ea_re[i] * ea_re[i] + ea_im[i] * ea_im[i]) * nm;
        if (pwr < eta) continue;
        td[cnt] = ((long)n - ek[i]) % (long)n;
        const long half = (long)m / 2;
        tp[cnt] = (el[i] + half) % (long)m - half;
        pp[cnt] = pwr;
        ++cnt;
    }
    for (long i = 1; i < cnt; i++) {
        long kd = td[i], kp = tp[i];
        double kv = pp[i];
        long j = i;
        while (j > 0) {
            int before = (kv != pp[j - 1]) ? (kv > pp[j - 1])
                                           : (kd != td[j - 1] ? kd < td[j - 1] : kp < tp[j - 1]);
            if (!before) break;
            td[j] = td[j - 1]; tp[j] = tp[j - 1]; pp[j] = pp[j - 1];
            --j;
        }
        td[j] = kd; tp[j] = kp; pp[j] = kv;
    }
    if (cnt > max_targets) cnt = max_targets;
    for (long i = 0; i < cnt; i++) { delay[i] = td[i]; doppler[i] = tp[i]; power[i] = pp[i]; }
    free(td); free(tp); free(pp);
    return cnt;
}
