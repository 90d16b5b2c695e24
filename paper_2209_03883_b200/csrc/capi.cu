// C-ABI host layer (include/ofdmr_b200.h): context, argument checking with the
// reference's error semantics, chunked stream-ordered launch schedules, and the
// host-buffer (H2D/D2H inside) pipeline entry point.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ofdmr_b200.h"
#include "radar_kernels.cuh"
#include "sft_kernels.cuh"
#include "fused_args.cuh"

namespace ofdmr {
cudaError_t launch_colpass(const ColArgs& a, int n, int np, int frames, cudaStream_t st);
cudaError_t launch_rowpass(const RowArgs& a, int mp, int frames, cudaStream_t st);
cudaError_t launch_merge(const MergeArgs& a, int frames, cudaStream_t st);
int colpass_tile_cols(int np);
int rowpass_rows(int mp, int np, int m);
size_t rowpass_smem(int mp, int rows);
struct FastRowArgs {
    RowArgs r;
    const float2* tw256_t;
    int* frame_done;
    const int32_t* k_per_frame;
    int32_t* det_delay;
    int32_t* det_doppler;
    float* det_power;
    int32_t* counts;
    double* s2h_out;
};
cudaError_t launch_colpass_fast(const ColArgs& a, bool ls, bool win, const float2* tw_t, int frames, cudaStream_t st);
cudaError_t launch_rowpass_fast(const FastRowArgs& a, int frames, cudaStream_t st);
int fast_rows_per_block();
struct PersistArgs {
    ColArgs col;
    FastRowArgs row;
    const float2* tw1024_t;
    int frames, cf, ring, nchunks, nblk;
    int* ticket;
    int* done_cols;
    int* done_rows;
};
cudaError_t launch_pgram_persist(const PersistArgs& pa, bool ls, bool win, int grid, cudaStream_t st);

cudaError_t launch_fused_ce(const FusedArgs& a, bool hamming, int grid, cudaStream_t st);
size_t noise_select_scratch_bytes(int64_t frames);
cudaError_t launch_map_pgm(const float* p, int64_t count, uint8_t* out, int64_t frames, double* scratch,
                           cudaStream_t st, int64_t* launches);
cudaError_t launch_ofdm(bool inverse, const float2* in, float2* out, int n, int m, int ncp, int64_t frames,
                        const float2* tw, cudaStream_t st);
cudaError_t launch_noise_select(const float* p, int64_t count, double pf, double* sigma2_out, int64_t frames,
                                void* scratch, int sms, cudaStream_t st, int64_t* launches);
cudaError_t launch_fused_pg2(const Pg2Args& a, bool hamming, int groups, int scratch_groups, cudaStream_t st);
cudaError_t launch_fused_pg3(const Pg2Args& a, bool hamming, int groups, int scratch_groups, cudaStream_t st);
int fused_pg3_max_groups();
size_t fused_pg3_counter_ints(int groups);
size_t fused_pg3_scratch_elems(int groups);
int fused_pg2_max_groups();
bool mixed_size_supported(int len);
int mixed_col_tile(int np, int m);
cudaError_t launch_ofdm_mixed(bool inverse, const float2* in, float2* out, int n, int m, int ncp, int64_t frames,
                              const float2* tw_n, cudaStream_t st);
size_t fused_pg2_counter_ints(int groups);
size_t fused_pg2_scratch_elems(int groups);
}  // namespace ofdmr

using namespace ofdmr;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(OFDMR_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define OFDMR_CUDA(call)                                 \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

bool pow2_in(int v, int lo, int hi) { return v >= lo && v <= hi && (v & (v - 1)) == 0; }

constexpr double kTwoPi = 6.283185307179586476925286766559;

}  // namespace

struct ofdmr_context {
    ofdmr_config cfg{};
    cudaStream_t stream = nullptr;
    int device = 0;
    float2* tw = nullptr;        // 4096-entry e^{-j2pi t/4096}
    float2* zp_tw = nullptr;     // rowpass_zp twiddles (entries of tw): [4][32][16] W_2048^{j(4k1+m1)}, [128] W_128^q
    float* wk = nullptr;         // Hamming windows (fp32) or null for rectangular
    float* wk_s = nullptr;       // w_k * sqrt(1 / (N M)) for the fused kernel
    float* wl = nullptr;
    // two scheduling slots (slot 0 = the caller's stream, slot 1 = an internal stream);
    // consecutive chunks alternate so one chunk's row pass overlaps the next chunk's
    // column pass; each slot owns its L2-resident intermediate and scratch.
    struct Slot {
        cudaStream_t stream = nullptr;
        float2* gbuf = nullptr;      // k-pass intermediate for one chunk
        double* partial = nullptr;   // per (frame, tile) 1/|x|^2 partials
        unsigned long long* cand = nullptr;  // per (frame, block) top-K keys
        int* frame_done = nullptr;   // fast path: per-frame finished-block counters
        int32_t* status_scratch = nullptr;
    } slot[2];
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool fast = false;           // N = N' = 1024, M = M' = 256 specialised kernels
    bool fused = false;          // + DFT-CE with 0 < L <= 128: persistent one-frame-per-CTA kernel
    bool force_general = false;  // set by ofdmr_pipeline_general for one call
    int fused_grid = 0;
    int pg2_groups = 0;               // warp-specialised periodogram: 16-CTA frame groups
    float2* pg2_scratch = nullptr;    // per group 2 x 1024 x 256 G (L2)
    int* pg2_counters = nullptr;      // per group progress counters
    bool mixed = false;               // some size not a power of two: mixed-radix kernels (mixed_kernels.cu)
    float2* tw_n = nullptr;           // e^{-j 2 pi t / L} tables of N, N', M' (mixed path)
    float2* tw_np = nullptr;
    float2* tw_mp = nullptr;
    int pg3_groups = 0;               // split-exchange periodogram (fused_pg3.cu)
    float2* pg3_scratch = nullptr;
    int* pg3_counters = nullptr;
    void* noise_scratch = nullptr;    // estimate_noise_power radix-select histograms
    int64_t noise_cap = 0;            // frames the scratch holds
    float2* dscratch = nullptr;  // fused: per-CTA L x M compressed intermediate
    float* fedges = nullptr;               // fused: per-CTA edge columns of P (16 steps x 2)
    unsigned long long* fpend = nullptr;   // fused: per-CTA pending edge candidates
    int* fpend_loc = nullptr;
    unsigned long long* ftlist = nullptr;  // fused: per-CTA frame candidate list
    // persistent periodogram / LS pipeline (fast shapes): L2-sized ring of intermediates
    struct Persist {
        int cf = 8, ring = 4, grid = 0;
        float2* gring = nullptr;              // ring x cf x N' x M c64
        double* pring = nullptr;              // ring x cf x ntiles partials
        unsigned long long* cring = nullptr;  // ring x cf x nblk x K keys
        int* fdone = nullptr;                 // ring x cf merge counters
        int* counters = nullptr;              // ticket + done_cols[cap] + done_rows[cap]
        int64_t cap = 0;
    } ps;
    float2* tw1024_t = nullptr;  // [t1*32 + j] = W_1024^{j t1}
    float2* tw256_t = nullptr;   // [t1*16 + j] = W_256^{j t1}
    // slot-0 aliases used by the single-stream entry points
    float2* gbuf = nullptr;
    double* partial = nullptr;
    unsigned long long* cand = nullptr;
    int32_t* status_scratch = nullptr;
    int64_t chunk = 0;
    int ntiles = 0;              // M / C of the colpass
    int rows_per_block = 0;
    int nblk = 0;
    int g_rows = 0;              // rows of G (N' or L with the shortcut)
    bool shortcut = false;
    double log_pfa = 0.0, pf = 1.0, inv_count = 0.0;
    float scale = 0.f;
    int64_t launches = 0;
    // host-buffer pipeline staging (lazily allocated)
    void* dev_y[2] = {nullptr, nullptr};
    void* dev_x[2] = {nullptr, nullptr};
    double* dev_s2[2] = {nullptr, nullptr};
    int32_t* dev_k[2] = {nullptr, nullptr};
    int32_t* dev_d[2] = {nullptr, nullptr};
    int32_t* dev_dp[2] = {nullptr, nullptr};
    float* dev_pw[2] = {nullptr, nullptr};
    int32_t* dev_cnt[2] = {nullptr, nullptr};
    int32_t* dev_st[2] = {nullptr, nullptr};
    int32_t* host_st = nullptr;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr};
    cudaEvent_t ev_done[2] = {nullptr, nullptr};
    // FPS-SFT scratch
    SftScratch sft{};
    // FPS-SFT pipeline / sft_detect scratch (grown on demand): channel estimates of one chunk,
    // per-frame entries and noise powers
    struct SftPipe {
        float2* h = nullptr;
        int64_t cap_h = 0;  // frames
        int32_t* k = nullptr;
        int32_t* l = nullptr;
        double* amp = nullptr;
        int32_t* ne = nullptr;
        double* s2h = nullptr;
        double* s2u = nullptr;
        int32_t* st = nullptr;
        int64_t cap = 0;  // frames
    } sp;
    // optional per-stage event timing (bench roofline): stage 0 colpass, 1 rowpass, 2 merge
    bool profiling = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof;
    std::vector<cudaEvent_t> ev_pool;
};

namespace {

cudaEvent_t pool_event(ofdmr_context* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Brackets one kernel launch with events when profiling is on.
struct StageTimer {
    ofdmr_context* c;
    int stage;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    StageTimer(ofdmr_context* ctx, int st, cudaStream_t stream) : c(ctx), stage(st), s(stream) {
        if (c->profiling) {
            a = pool_event(c);
            cudaEventRecord(a, s);
        }
    }
    StageTimer(ofdmr_context* ctx, int st) : StageTimer(ctx, st, ctx->stream) {}
    ~StageTimer() {
        if (c->profiling) {
            cudaEvent_t b = pool_event(c);
            cudaEventRecord(b, s);
            c->prof.push_back({stage, {a, b}});
        }
    }
};

int check_cfg(const ofdmr_config* c) {
    if (!c) return fail(OFDMR_ERR_CONFIG, "ofdmr_create: null config");
    for (int v : {c->n_subcarriers, c->n_symbols, c->n_prime, c->m_prime})
        if (!mixed_size_supported(v))
            return fail(OFDMR_ERR_CONFIG,
                        "N, M, N', M' must lie in [2, 4096] and factor into 2, 3, 5, 7, 11, 13 (got " +
                            std::to_string(v) + ")");
    if (c->n_prime < c->n_subcarriers || c->m_prime < c->n_symbols)
        return fail(OFDMR_ERR_CONFIG, "periodogram: N' >= N and M' >= M required");
    if (c->window != OFDMR_WINDOW_RECT && c->window != OFDMR_WINDOW_HAMMING)
        return fail(OFDMR_ERR_CONFIG, "window must be rectangular or hamming");
    if (c->estimator != OFDMR_EST_LS && c->estimator != OFDMR_EST_DFT_CE)
        return fail(OFDMR_ERR_CONFIG, "estimator must be LS or DFT-CE");
    if (c->estimator == OFDMR_EST_DFT_CE && (c->n_cp < 0 || c->n_cp > c->n_subcarriers))
        return fail(OFDMR_ERR_CONFIG, "dft_ce: truncation length exceeds N");
    if (c->max_targets < 1 || c->max_targets > kMaxK) return fail(OFDMR_ERR_CONFIG, "max_targets must be in [1, 64]");
    if (!(c->pfa > 0.0 && c->pfa <= 1.0)) return fail(OFDMR_ERR_CONFIG, "threshold: pfa must lie in (0,1]");
    return OFDMR_OK;
}

void make_window_d(int kind, int n, int m, double* wk, double* wl) {
    for (int k = 0; k < n; ++k) wk[k] = 1.0;
    for (int l = 0; l < m; ++l) wl[l] = 1.0;
    if (kind == OFDMR_WINDOW_HAMMING) {
        for (int k = 0; k < n; ++k) wk[k] = 0.54 - 0.46 * std::cos(kTwoPi * double(k) / double(n - 1));
        for (int l = 0; l < m; ++l) wl[l] = 0.54 - 0.46 * std::cos(kTwoPi * double(l) / double(m - 1));
    }
}

double power_factor_d(int kind, int n, int m) {
    std::vector<double> wk(n), wl(m);
    make_window_d(kind, n, m, wk.data(), wl.data());
    double sk = 0.0, sl = 0.0;
    for (double v : wk) sk += v * v;
    for (double v : wl) sl += v * v;
    return sk * sl / (double(n) * double(m));
}

size_t cells(const ofdmr_context* c) { return size_t(c->cfg.n_subcarriers) * size_t(c->cfg.n_symbols); }

ColArgs base_col(ofdmr_context* c) {
    ColArgs a{};
    a.tw = c->tw;
    a.m = c->cfg.n_symbols;
    a.ntiles = c->ntiles;
    a.n = c->cfg.n_subcarriers;
    a.np = c->cfg.n_prime;
    a.tw_n = c->tw_n;    // non-null only on the mixed-radix path (launch_colpass dispatches on it)
    a.tw_np = c->tw_np;
    return a;
}

// row-pass arguments of the mixed-radix path (launch_rowpass dispatches on tw_mp)
void row_mixed(ofdmr_context* c, RowArgs& r) {
    r.mp = c->cfg.m_prime;
    r.tw_mp = c->tw_mp;
}

int launch_col(ofdmr_context* c, const ColArgs& a, int np, int64_t frames, cudaStream_t st) {
    StageTimer t(c, 0, st);
    const cudaError_t e = launch_colpass(a, c->cfg.n_subcarriers, np, int(frames), st);
    if (e != cudaSuccess) return cuda_fail(e, "colpass");
    ++c->launches;
    return OFDMR_OK;
}

int run_pipeline_chunk_fast(ofdmr_context* c, int si, const float2* y, const float2* x, const double* sigma2,
                            const int32_t* kpf, int32_t* d, int32_t* dp, float* pw, int32_t* cnt, double* s2h_out,
                            float* p_out, int32_t* status, int64_t nf) {
    const ofdmr_config& g = c->cfg;
    auto& s = c->slot[si];
    ColArgs a = base_col(c);
    a.y = y;
    a.x = x;
    a.g_out = s.gbuf;
    const bool win = g.window == OFDMR_WINDOW_HAMMING;
    if (win) {
        a.wk = c->wk;
        a.wl = c->wl;
    }
    a.inv_partial = s.partial;
    a.status = status;
    a.ce_taps = g.estimator == OFDMR_EST_DFT_CE ? g.n_cp : 0;
    a.shortcut = c->shortcut ? 1 : 0;
    a.g_rows = c->g_rows;
    cudaError_t e;
    {
        StageTimer t(c, 0, s.stream);
        e = launch_colpass_fast(a, true, win, c->tw1024_t, int(nf), s.stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "colpass_fast");
    ++c->launches;
    FastRowArgs r{};
    r.r.g = s.gbuf;
    r.r.p_out = p_out;
    r.r.inv_partial = s.partial;
    r.r.ntiles = c->ntiles;
    r.r.sigma2 = sigma2;
    r.r.log_pfa = c->log_pfa;
    r.r.power_factor = c->pf;
    r.r.inv_count = c->inv_count;
    r.r.scale = c->scale;
    r.r.n_prime = g.n_prime;
    r.r.g_rows = c->g_rows;
    r.r.m = g.n_symbols;
    r.r.kmax = g.max_targets;
    r.r.cand = s.cand;
    r.r.detect = 1;
    r.tw256_t = c->tw256_t;
    r.frame_done = s.frame_done;
    r.k_per_frame = kpf;
    r.det_delay = d;
    r.det_doppler = dp;
    r.det_power = pw;
    r.counts = cnt;
    r.s2h_out = s2h_out;
    {
        StageTimer t(c, 1, s.stream);
        e = launch_rowpass_fast(r, int(nf), s.stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "rowpass_fast");
    ++c->launches;
    return OFDMR_OK;
}

// k-pass -> row-pass (+detect) -> merge over one chunk of frames.
int run_pipeline_chunk(ofdmr_context* c, int si, const float2* y, const float2* x, const double* sigma2,
                       const int32_t* kpf, int32_t* d, int32_t* dp, float* pw, int32_t* cnt, double* s2h_out,
                       float* p_out, int32_t* status, int64_t nf) {
    if (c->fast) return run_pipeline_chunk_fast(c, si, y, x, sigma2, kpf, d, dp, pw, cnt, s2h_out, p_out, status, nf);
    const ofdmr_config& g = c->cfg;
    auto& s = c->slot[si];
    ColArgs a = base_col(c);
    a.y = y;
    a.x = x;
    a.g_out = s.gbuf;
    if (g.window == OFDMR_WINDOW_HAMMING) {
        a.wk = c->wk;
        a.wl = c->wl;
    }
    a.inv_partial = s.partial;
    a.status = status;
    a.ce_taps = g.estimator == OFDMR_EST_DFT_CE ? g.n_cp : 0;
    a.shortcut = c->shortcut ? 1 : 0;
    a.g_rows = c->g_rows;
    int rc = launch_col(c, a, g.n_prime, nf, s.stream);
    if (rc) return rc;

    RowArgs r{};
    r.g = s.gbuf;
    r.p_out = p_out;
    r.inv_partial = s.partial;
    r.ntiles = c->ntiles;
    r.sigma2 = sigma2;
    r.log_pfa = c->log_pfa;
    r.power_factor = c->pf;
    r.inv_count = c->inv_count;
    r.scale = c->scale;
    r.tw = c->tw;
    r.zp_tw = c->zp_tw;
    r.n_prime = g.n_prime;
    r.g_rows = c->g_rows;
    r.m = g.n_symbols;
    r.rows_per_block = c->rows_per_block;
    r.kmax = g.max_targets;
    r.cand = s.cand;
    r.detect = 1;
    cudaError_t e;
    {
        StageTimer t(c, 1, s.stream);
        row_mixed(c, r);
        e = launch_rowpass(r, g.m_prime, int(nf), s.stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "rowpass");
    ++c->launches;

    MergeArgs mg{};
    mg.cand = s.cand;
    mg.nblk = c->nblk;
    mg.kmax = g.max_targets;
    mg.k_per_frame = kpf;
    mg.m_prime = g.m_prime;
    mg.det_delay = d;
    mg.det_doppler = dp;
    mg.det_power = pw;
    mg.counts = cnt;
    mg.inv_partial = s.partial;
    mg.ntiles = c->ntiles;
    mg.sigma2 = sigma2;
    mg.log_pfa = c->log_pfa;
    mg.power_factor = c->pf;
    mg.inv_count = c->inv_count;
    mg.s2h_out = s2h_out;
    {
        StageTimer t(c, 2, s.stream);
        e = launch_merge(mg, int(nf), s.stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "merge");
    ++c->launches;
    return OFDMR_OK;
}

}  // namespace

namespace {

// Persistent periodogram / LS-pipeline launch over a whole batch (fast shapes).
// h != null: periodogram of H (map only).  y/x != null: LS pipeline with detection.
int run_persist(ofdmr_context* c, const float2* h, const float2* y, const float2* x, const double* sigma2,
                const int32_t* kpf, int32_t* d, int32_t* dp, float* pw, int32_t* cnt, double* s2h_out, float* p_out,
                int32_t* status, int64_t frames) {
    const ofdmr_config& g = c->cfg;
    auto& ps = c->ps;
    // frames per chunk: a batch smaller than one chunk gets a chunk of its own size (no empty
    // tickets for the CTAs to draw one by one; the ring slots are a subset of the allocated ones)
    const int cf = int(std::min<int64_t>(ps.cf, frames));
    const int nchunks = int((frames + cf - 1) / cf);
    const int64_t need = 1 + frames + nchunks;
    if (need > ps.cap) {
        cudaFree(ps.counters);
        ps.counters = nullptr;
        ps.cap = 0;
        OFDMR_CUDA(cudaMalloc(&ps.counters, sizeof(int) * size_t(need)));
        ps.cap = need;
    }
    OFDMR_CUDA(cudaMemsetAsync(ps.counters, 0, sizeof(int) * size_t(need), c->stream));
    const bool win = g.window == OFDMR_WINDOW_HAMMING;
    PersistArgs pa{};
    pa.col = base_col(c);
    pa.col.y = y;
    pa.col.x = x;
    pa.col.h = h;
    pa.col.g_out = ps.gring;
    pa.col.g_rows = g.n_prime;
    pa.col.status = status;
    pa.col.inv_partial = y ? ps.pring : nullptr;
    if (win) {
        pa.col.wk = c->wk;
        pa.col.wl = c->wl;
    }
    FastRowArgs& r = pa.row;
    r.r.g = ps.gring;
    r.r.p_out = p_out;
    r.r.inv_partial = y ? ps.pring : nullptr;
    r.r.ntiles = c->ntiles;
    r.r.sigma2 = sigma2;
    r.r.log_pfa = c->log_pfa;
    r.r.power_factor = c->pf;
    r.r.inv_count = c->inv_count;
    r.r.scale = c->scale;
    r.r.n_prime = g.n_prime;
    r.r.g_rows = g.n_prime;
    r.r.m = g.n_symbols;
    r.r.kmax = g.max_targets;
    r.r.cand = ps.cring;
    r.r.detect = y ? 1 : 0;
    r.tw256_t = c->tw256_t;
    r.frame_done = ps.fdone;
    r.k_per_frame = kpf;
    r.det_delay = d;
    r.det_doppler = dp;
    r.det_power = pw;
    r.counts = cnt;
    r.s2h_out = s2h_out;
    pa.tw1024_t = c->tw1024_t;
    pa.frames = int(frames);
    pa.cf = cf;
    pa.ring = ps.ring;
    pa.nchunks = nchunks;
    pa.nblk = c->nblk;
    pa.ticket = ps.counters;
    pa.done_cols = ps.counters + 1;
    pa.done_rows = ps.counters + 1 + frames;
    const int64_t items = int64_t(frames) * (32 + c->nblk);
    const int grid = int(std::min<int64_t>(ps.grid, items));
    cudaError_t e;
    {
        StageTimer t(c, 0, c->stream);
        e = launch_pgram_persist(pa, y != nullptr, win, grid, c->stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "pgram_persist");
    ++c->launches;
    return OFDMR_OK;
}

}  // namespace

extern "C" {

const char* ofdmr_last_error(void) { return g_last_error.c_str(); }

int ofdmr_make_window(int32_t kind, int32_t n, int32_t m, double* wk, double* wl) {
    if (n <= 0 || m <= 0) return fail(OFDMR_ERR_CONFIG, "make_window: empty");
    make_window_d(kind, n, m, wk, wl);
    return OFDMR_OK;
}

double ofdmr_window_power_factor(int32_t kind, int32_t n, int32_t m) { return power_factor_d(kind, n, m); }

int ofdmr_detection_threshold(double sigma2, double pfa, double power_factor, double* eta) {
    if (sigma2 < 0.0) return fail(OFDMR_ERR_CONFIG, "threshold: sigma2 must be >= 0");
    if (!(pfa > 0.0 && pfa <= 1.0)) return fail(OFDMR_ERR_CONFIG, "threshold: pfa must lie in (0,1]");
    *eta = -sigma2 * std::log(pfa) * power_factor;
    return OFDMR_OK;
}

void ofdmr_bins_to_physics(int64_t delay_bin, int64_t doppler_bin, int32_t n_subcarriers, int32_t n_cp,
                           int32_t n_prime, int32_t m_prime, double df_hz, double fc_hz, double* range_m,
                           double* velocity_mps) {
    const double c = 3.0e8;
    const double t_useful = 1.0 / df_hz;
    const double ts = t_useful + double(n_cp) * (t_useful / double(n_subcarriers));
    *range_m = c * double(delay_bin) / (2.0 * double(n_prime) * df_hz);
    *velocity_mps = c * double(doppler_bin) / (2.0 * fc_hz * double(m_prime) * ts);
}

int ofdmr_create(const ofdmr_config* cfg, ofdmr_context** out) {
    if (!out) return fail(OFDMR_ERR_CONFIG, "ofdmr_create: null out");
    *out = nullptr;
    int rc = check_cfg(cfg);
    if (rc) return rc;
    int ndev = 0;
    OFDMR_CUDA(cudaGetDeviceCount(&ndev));
    if (cfg->device < 0 || cfg->device >= ndev) return fail(OFDMR_ERR_CONFIG, "device ordinal out of range");
    OFDMR_CUDA(cudaSetDevice(cfg->device));
    auto* c = new ofdmr_context();
    c->cfg = *cfg;
    c->device = cfg->device;
    const int n = cfg->n_subcarriers, m = cfg->n_symbols, np = cfg->n_prime, mp = cfg->m_prime;
    // power-of-two kernels (radar_kernels.cu templates and the fused / fast specialisations) for
    // sizes in [16, 4096] with N' in {N, 2N, 4N}; every other shape runs the mixed-radix path
    c->mixed = !(pow2_in(n, 16, 4096) && pow2_in(m, 16, 4096) && pow2_in(np, 16, 4096) && pow2_in(mp, 16, 4096) &&
                 (np == n || np == 2 * n || np == 4 * n));
    c->shortcut = !c->mixed && cfg->estimator == OFDMR_EST_DFT_CE && cfg->window == OFDMR_WINDOW_RECT && np == n;
    c->g_rows = c->shortcut ? cfg->n_cp : np;
    if (c->shortcut && c->g_rows == 0) c->g_rows = 1;  // L = 0: all-zero estimate, keep one zero row
    c->ntiles = m / (c->mixed ? mixed_col_tile(np, m) : colpass_tile_cols(np));
    c->rows_per_block = c->mixed ? rowpass_rows(mp, np, 0) : rowpass_rows(mp, np, m);
    c->nblk = (np + c->rows_per_block - 1) / c->rows_per_block;
    c->log_pfa = std::log(cfg->pfa);
    c->pf = power_factor_d(cfg->window, n, m);
    c->inv_count = 1.0 / double(size_t(n) * size_t(m));
    c->scale = float(1.0 / (double(n) * double(m)));
    c->fast = !c->mixed && n == 1024 && np == 1024 && m == 256 && mp == 256;
    c->fused = c->fast && cfg->estimator == OFDMR_EST_DFT_CE && cfg->n_cp > 0 && cfg->n_cp <= 128;
    if (c->fast) {
        c->rows_per_block = fast_rows_per_block();
        c->nblk = (np + c->rows_per_block - 1) / c->rows_per_block;
    }
    const size_t gframe = size_t(c->g_rows) * size_t(m) * sizeof(float2);
    int64_t chunk = cfg->chunk_frames;
    if (chunk <= 0) {
        // two chunks in flight; keep both intermediates L2-resident (126 MB L2)
        chunk = int64_t((32ull << 20) / gframe);
        // frames whose intermediate alone is >= 8 MiB (cfg2: 16 MiB) are compute-bound, not L2-bound:
        // fill the GPU instead (8 frames per launch: whole waves, one merge launch per 8 frames)
        if (chunk < 8) chunk = 8;
        if (chunk > 256) chunk = 256;
        // the cfg2 column pass (colpass2048.cu: persistent, one CTA per SM, 8-column tiles): whole
        // rounds of items per launch -- the smallest chunk >= 8 whose tile count is a multiple of the
        // SM count (37 frames on 148 SMs; measured 30.3 k vs 28.9 k frames/s at 8)
        if (!c->mixed && n == 2048 && np == 4096 && m % 8 == 0) {
            int sms = 0;
            if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device) == cudaSuccess && sms > 0) {
                for (int64_t k = 8; k <= 64; ++k)
                    if ((k * (m / 8)) % sms == 0) {
                        chunk = k;
                        break;
                    }
            }
        }
    }
    if (c->fused && cfg->chunk_frames <= 0) chunk = 512;  // host-buffer path: fill every cluster
    c->chunk = chunk;

    std::vector<float2> tw(kTwLenHost);
    for (int t = 0; t < kTwLenHost; ++t) {
        const double a = -kTwoPi * double(t) / double(kTwLenHost);
        tw[t] = make_float2(float(std::cos(a)), float(std::sin(a)));
    }
    cudaError_t e = cudaMalloc(&c->tw, sizeof(float2) * kTwLenHost);
    if (e == cudaSuccess) e = cudaMemcpy(c->tw, tw.data(), sizeof(float2) * kTwLenHost, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        std::vector<float2> zt(4 * 512 + 128);
        for (int i = 0; i < 4 * 512; ++i) {
            const int m1 = i >> 9, k1 = (i >> 4) & 31, j = i & 15;
            zt[i] = tw[(2 * j * (4 * k1 + m1)) & (kTwLenHost - 1)];
        }
        for (int q = 0; q < 128; ++q) zt[4 * 512 + q] = tw[32 * q];
        e = cudaMalloc(&c->zp_tw, sizeof(float2) * zt.size());
        if (e == cudaSuccess) e = cudaMemcpy(c->zp_tw, zt.data(), sizeof(float2) * zt.size(), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess && c->mixed) {  // per-length twiddle tables of the mixed-radix engine
        auto table = [&](int len, float2** out) {
            std::vector<float2> t(len);
            for (int i = 0; i < len; ++i) {
                const double a = -kTwoPi * double(i) / double(len);
                t[i] = make_float2(float(std::cos(a)), float(std::sin(a)));
            }
            cudaError_t ee = cudaMalloc(out, sizeof(float2) * len);
            if (ee == cudaSuccess) ee = cudaMemcpy(*out, t.data(), sizeof(float2) * len, cudaMemcpyHostToDevice);
            return ee;
        };
        e = table(n, &c->tw_n);
        if (e == cudaSuccess) e = table(np, &c->tw_np);
        if (e == cudaSuccess) e = table(mp, &c->tw_mp);
    }
    if (e == cudaSuccess && cfg->window == OFDMR_WINDOW_HAMMING) {
        std::vector<double> wk(n), wl(m);
        make_window_d(cfg->window, n, m, wk.data(), wl.data());
        std::vector<float> fk(wk.begin(), wk.end()), fl(wl.begin(), wl.end());
        e = cudaMalloc(&c->wk, sizeof(float) * n);
        if (e == cudaSuccess) e = cudaMalloc(&c->wl, sizeof(float) * m);
        if (e == cudaSuccess) e = cudaMemcpy(c->wk, fk.data(), sizeof(float) * n, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(c->wl, fl.data(), sizeof(float) * m, cudaMemcpyHostToDevice);
        // fused kernel: w_k pre-multiplied by sqrt(1 / (N M)) (= 2^-9 at 1024 x 256, exact), so
        // |w_k X|^2 needs no separate scale
        std::vector<float> fks(n);
        const double rs = std::sqrt(1.0 / (double(n) * double(m)));
        for (int i = 0; i < n; ++i) fks[i] = float(wk[i] * rs);
        if (e == cudaSuccess) e = cudaMalloc(&c->wk_s, sizeof(float) * n);
        if (e == cudaSuccess) e = cudaMemcpy(c->wk_s, fks.data(), sizeof(float) * n, cudaMemcpyHostToDevice);
    }
    // the periodogram entry point always needs the full N' rows
    const size_t gbytes = std::max(gframe, size_t(np) * size_t(m) * sizeof(float2)) * size_t(chunk);
    for (int si = 0; si < 2 && e == cudaSuccess; ++si) {
        auto& s = c->slot[si];
        e = cudaMalloc(&s.gbuf, gbytes);
        if (e == cudaSuccess) e = cudaMalloc(&s.partial, sizeof(double) * size_t(c->ntiles) * size_t(chunk));
        if (e == cudaSuccess)
            e = cudaMalloc(&s.cand, sizeof(unsigned long long) * size_t(c->nblk) * cfg->max_targets * size_t(chunk));
        if (e == cudaSuccess) e = cudaMalloc(&s.frame_done, sizeof(int) * size_t(chunk));
        if (e == cudaSuccess) e = cudaMemset(s.frame_done, 0, sizeof(int) * size_t(chunk));
        if (e == cudaSuccess) e = cudaMalloc(&s.status_scratch, sizeof(int32_t) * size_t(chunk));
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
    if (e == cudaSuccess && c->fast) {
        std::vector<float2> t1024(1024), t256(256);
        for (int t1 = 0; t1 < 32; ++t1)
            for (int j = 0; j < 32; ++j) {
                const double a = -kTwoPi * double(t1 * j) / 1024.0;
                t1024[t1 * 32 + j] = make_float2(float(std::cos(a)), float(std::sin(a)));
            }
        for (int t1 = 0; t1 < 16; ++t1)
            for (int j = 0; j < 16; ++j) {
                const double a = -kTwoPi * double(t1 * j) / 256.0;
                t256[t1 * 16 + j] = make_float2(float(std::cos(a)), float(std::sin(a)));
            }
        e = cudaMalloc(&c->tw1024_t, sizeof(float2) * 1024);
        if (e == cudaSuccess) e = cudaMalloc(&c->tw256_t, sizeof(float2) * 256);
        if (e == cudaSuccess) e = cudaMemcpy(c->tw1024_t, t1024.data(), sizeof(float2) * 1024, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(c->tw256_t, t256.data(), sizeof(float2) * 256, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess && c->fast) {
        auto& ps = c->ps;
        int sms = 0;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device);
        ps.grid = 2 * sms;
        const size_t slots = size_t(ps.ring) * ps.cf;
        if (e == cudaSuccess) e = cudaMalloc(&ps.gring, slots * size_t(np) * size_t(m) * sizeof(float2));
        if (e == cudaSuccess) e = cudaMalloc(&ps.pring, slots * size_t(c->ntiles) * sizeof(double));
        if (e == cudaSuccess)
            e = cudaMalloc(&ps.cring, slots * size_t(c->nblk) * size_t(cfg->max_targets) * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMalloc(&ps.fdone, slots * sizeof(int));
        if (e == cudaSuccess) e = cudaMemset(ps.fdone, 0, slots * sizeof(int));
    }
    if (e == cudaSuccess && c->fused) {
        int sms = 0;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device);
        c->fused_grid = 2 * sms;  // 2 resident CTAs per SM (128 regs x 256 threads, ~102 KB smem)
        // two frames in flight per 2-CTA cluster (pass A of frame i+1 overlaps pass C of frame i)
        if (e == cudaSuccess) e = cudaMalloc(&c->dscratch, sizeof(float2) * 128 * 256 * size_t(c->fused_grid));
        if (e == cudaSuccess) e = cudaMalloc(&c->fedges, sizeof(float) * kFusedEdgeStride * size_t(c->fused_grid));
        if (e == cudaSuccess) e = cudaMalloc(&c->fpend, sizeof(unsigned long long) * kFusedPend * size_t(c->fused_grid));
        if (e == cudaSuccess) e = cudaMalloc(&c->fpend_loc, sizeof(int) * kFusedPend * size_t(c->fused_grid));
        if (e == cudaSuccess) e = cudaMalloc(&c->ftlist, sizeof(unsigned long long) * 1024 * size_t(c->fused_grid));
    }
    c->gbuf = c->slot[0].gbuf;
    c->partial = c->slot[0].partial;
    c->cand = c->slot[0].cand;
    c->status_scratch = c->slot[0].status_scratch;
    if (e != cudaSuccess) {
        ofdmr_destroy(c);
        return cuda_fail(e, "ofdmr_create: allocation");
    }
    *out = c;
    return OFDMR_OK;
}

void ofdmr_destroy(ofdmr_context* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaFree(c->tw);
    cudaFree(c->zp_tw);
    cudaFree(c->tw_n);
    cudaFree(c->tw_np);
    cudaFree(c->tw_mp);
    cudaFree(c->wk);
    cudaFree(c->wk_s);
    cudaFree(c->wl);
    for (auto& s : c->slot) {
        cudaFree(s.gbuf);
        cudaFree(s.partial);
        cudaFree(s.cand);
        cudaFree(s.frame_done);
        cudaFree(s.status_scratch);
    }
    cudaFree(c->tw1024_t);
    cudaFree(c->tw256_t);
    cudaFree(c->dscratch);
    cudaFree(c->pg2_scratch);
    cudaFree(c->pg2_counters);
    cudaFree(c->pg3_scratch);
    cudaFree(c->pg3_counters);
    cudaFree(c->noise_scratch);
    cudaFree(c->fedges);
    cudaFree(c->fpend);
    cudaFree(c->fpend_loc);
    cudaFree(c->ftlist);
    cudaFree(c->ps.gring);
    cudaFree(c->ps.pring);
    cudaFree(c->ps.cring);
    cudaFree(c->ps.fdone);
    cudaFree(c->ps.counters);
    if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    for (int i = 0; i < 2; ++i) {
        cudaFree(c->dev_y[i]);
        cudaFree(c->dev_x[i]);
        cudaFree(c->dev_s2[i]);
        cudaFree(c->dev_k[i]);
        cudaFree(c->dev_d[i]);
        cudaFree(c->dev_dp[i]);
        cudaFree(c->dev_pw[i]);
        cudaFree(c->dev_cnt[i]);
        cudaFree(c->dev_st[i]);
        if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
        if (c->ev_done[i]) cudaEventDestroy(c->ev_done[i]);
    }
    if (c->host_st) cudaFreeHost(c->host_st);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    sft_free(c->sft);
    cudaFree(c->sp.h);
    cudaFree(c->sp.k);
    cudaFree(c->sp.l);
    cudaFree(c->sp.amp);
    cudaFree(c->sp.ne);
    cudaFree(c->sp.s2h);
    cudaFree(c->sp.s2u);
    cudaFree(c->sp.st);
    for (auto& p : c->prof) {
        cudaEventDestroy(p.second.first);
        cudaEventDestroy(p.second.second);
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    delete c;
}

int ofdmr_set_stream(ofdmr_context* c, void* s) {
    if (!c) return fail(OFDMR_ERR_CONFIG, "null context");
    c->stream = static_cast<cudaStream_t>(s);
    return OFDMR_OK;
}

int64_t ofdmr_launch_count(const ofdmr_context* c) { return c ? c->launches : 0; }

int ofdmr_set_profiling(ofdmr_context* c, int32_t on) {
    if (!c) return fail(OFDMR_ERR_CONFIG, "null context");
    c->profiling = on != 0;
    return OFDMR_OK;
}

int ofdmr_get_profile(ofdmr_context* c, double* ms, int64_t* launches) {
    if (!c || !ms || !launches) return fail(OFDMR_ERR_CONFIG, "get_profile: null argument");
    for (int i = 0; i < 3; ++i) {
        ms[i] = 0.0;
        launches[i] = 0;
    }
    OFDMR_CUDA(cudaSetDevice(c->device));
    OFDMR_CUDA(cudaStreamSynchronize(c->stream));
    for (auto& p : c->prof) {
        float t = 0.f;
        OFDMR_CUDA(cudaEventElapsedTime(&t, p.second.first, p.second.second));
        ms[p.first] += t;
        launches[p.first] += 1;
        c->ev_pool.push_back(p.second.first);
        c->ev_pool.push_back(p.second.second);
    }
    c->prof.clear();
    return OFDMR_OK;
}

int ofdmr_spectral_division(ofdmr_context* c, const void* y, const void* x, void* h, int32_t* status,
                            int64_t frames) {
    if (!c || !y || !x || !h || !status) return fail(OFDMR_ERR_CONFIG, "spectral_division: null argument");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    OFDMR_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * size_t(frames), c->stream));
    const size_t fc = cells(c);
    for (int64_t f0 = 0; f0 < frames; f0 += 65535) {
        const int64_t nf = std::min<int64_t>(65535, frames - f0);
        ColArgs a = base_col(c);
        a.y = static_cast<const float2*>(y) + fc * f0;
        a.x = static_cast<const float2*>(x) + fc * f0;
        a.h_out = static_cast<float2*>(h) + fc * f0;
        a.status = status + f0;
        int rc = launch_col(c, a, c->cfg.n_subcarriers, nf, c->stream);
        if (rc) return rc;
    }
    return OFDMR_OK;
}

int ofdmr_dft_ce(ofdmr_context* c, const void* h, void* h_out, int64_t frames) {
    if (!c || !h || !h_out) return fail(OFDMR_ERR_CONFIG, "dft_ce: null argument");
    if (c->cfg.n_cp > c->cfg.n_subcarriers) return fail(OFDMR_ERR_CONFIG, "dft_ce: truncation length exceeds N");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    const size_t fc = cells(c);
    for (int64_t f0 = 0; f0 < frames; f0 += 65535) {
        const int64_t nf = std::min<int64_t>(65535, frames - f0);
        ColArgs a = base_col(c);
        a.h = static_cast<const float2*>(h) + fc * f0;
        a.h_out = static_cast<float2*>(h_out) + fc * f0;
        a.hout_after_ce = 1;
        a.ce_taps = c->cfg.n_cp;
        if (a.ce_taps == 0) {  // everything truncated: H' = 0
            OFDMR_CUDA(cudaMemsetAsync(a.h_out, 0, sizeof(float2) * fc * size_t(nf), c->stream));
            continue;
        }
        int rc = launch_col(c, a, c->cfg.n_subcarriers, nf, c->stream);
        if (rc) return rc;
    }
    return OFDMR_OK;
}

int ofdmr_estimate_channel(ofdmr_context* c, const void* y, const void* x, void* h, int32_t* status,
                           int64_t frames) {
    if (!c || !y || !x || !h || !status) return fail(OFDMR_ERR_CONFIG, "estimate_channel: null argument");
    if (frames <= 0) return OFDMR_OK;
    if (c->cfg.estimator != OFDMR_EST_DFT_CE || c->cfg.n_cp == 0) {
        int rc = ofdmr_spectral_division(c, y, x, h, status, frames);
        if (rc || c->cfg.estimator != OFDMR_EST_DFT_CE) return rc;
        return ofdmr_dft_ce(c, h, h, frames);
    }
    OFDMR_CUDA(cudaSetDevice(c->device));
    OFDMR_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * size_t(frames), c->stream));
    const size_t fc = cells(c);
    for (int64_t f0 = 0; f0 < frames; f0 += 65535) {
        const int64_t nf = std::min<int64_t>(65535, frames - f0);
        ColArgs a = base_col(c);
        a.y = static_cast<const float2*>(y) + fc * f0;
        a.x = static_cast<const float2*>(x) + fc * f0;
        a.h_out = static_cast<float2*>(h) + fc * f0;
        a.hout_after_ce = 1;
        a.ce_taps = c->cfg.n_cp;
        a.status = status + f0;
        int rc = launch_col(c, a, c->cfg.n_subcarriers, nf, c->stream);
        if (rc) return rc;
    }
    return OFDMR_OK;
}

int ofdmr_periodogram(ofdmr_context* c, const void* h, float* p, int64_t frames) {
    if (!c || !h || !p) return fail(OFDMR_ERR_CONFIG, "periodogram: null argument");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    const ofdmr_config& g = c->cfg;
    const size_t fc = cells(c);
    const size_t pframe = size_t(g.n_prime) * size_t(g.m_prime);
    // the general (non-shortcut) G layout is always N' rows; the chunk buffer holds g_rows rows
    const int64_t chunk = c->shortcut ? std::max<int64_t>(1, c->chunk * c->g_rows / g.n_prime) : c->chunk;
    (void)chunk;
    const bool pg_shape = c->fast && g.n_subcarriers == 1024 && g.n_symbols == 256 && g.n_prime == 1024 &&
                          g.m_prime == 256 && getenv("OFDMR_PG_PERSIST") == nullptr;
    if (pg_shape && getenv("OFDMR_PG2") == nullptr) {
        // split-radix exchange periodogram (fused_pg3.cu): column warps DFT_32 + twiddle, row
        // warps DFT_32 + FFT_256, 8-CTA frame groups, double-buffered G in L2
        if (!c->pg3_scratch) {
            c->pg3_groups = fused_pg3_max_groups();
            if (c->pg3_groups <= 0) return fail(OFDMR_ERR_CUDA, "fused periodogram: no co-resident frame group");
            OFDMR_CUDA(cudaMalloc(&c->pg3_scratch, sizeof(float2) * fused_pg3_scratch_elems(c->pg3_groups)));
            OFDMR_CUDA(cudaMalloc(&c->pg3_counters, sizeof(int) * fused_pg3_counter_ints(c->pg3_groups)));
        }
        const size_t cnt_bytes = sizeof(int) * fused_pg3_counter_ints(c->pg3_groups);
        Pg2Args pa{};
        const bool win = g.window == OFDMR_WINDOW_HAMMING;
        pa.wk = win ? c->wk : nullptr;
        pa.wl = win ? c->wl : nullptr;
        pa.tw1024_t = c->tw1024_t;
        pa.tw256_t = c->tw256_t;
        pa.gscratch = c->pg3_scratch;
        pa.counters = c->pg3_counters;
        pa.scale = c->scale;
        for (int64_t f0 = 0; f0 < frames; f0 += (int64_t)1 << 28) {
            const int64_t nf = std::min<int64_t>((int64_t)1 << 28, frames - f0);
            OFDMR_CUDA(cudaMemsetAsync(c->pg3_counters, 0, cnt_bytes, c->stream));
            pa.h = static_cast<const float2*>(h) + fc * f0;
            pa.p = p + pframe * f0;
            pa.frames = int(nf);
            cudaError_t e;
            {
                StageTimer t(c, 0, c->stream);
                e = launch_fused_pg3(pa, win, int(std::min<int64_t>(c->pg3_groups, nf)), c->pg3_groups, c->stream);
            }
            if (e != cudaSuccess) return cuda_fail(e, "fused_pg3");
            ++c->launches;
        }
        return OFDMR_OK;
    }
    if (pg_shape) {
        // OFDMR_PG2=1: the previous warp-specialised kernel (whole IFFT_1024 on the column warps),
        // kept as an independent cross-check of fused_pg3 (tests/test_gpu_parity.py)
        if (!c->pg2_scratch) {
            c->pg2_groups = fused_pg2_max_groups();
            if (c->pg2_groups <= 0) return fail(OFDMR_ERR_CUDA, "fused periodogram: no co-resident frame group");
            OFDMR_CUDA(cudaMalloc(&c->pg2_scratch, sizeof(float2) * fused_pg2_scratch_elems(c->pg2_groups)));
            OFDMR_CUDA(cudaMalloc(&c->pg2_counters, sizeof(int) * fused_pg2_counter_ints(c->pg2_groups)));
        }
        const size_t cnt_bytes = sizeof(int) * fused_pg2_counter_ints(c->pg2_groups);
        Pg2Args pa{};
        const bool win = g.window == OFDMR_WINDOW_HAMMING;
        pa.wk = win ? c->wk : nullptr;
        pa.wl = win ? c->wl : nullptr;
        pa.tw1024_t = c->tw1024_t;
        pa.tw256_t = c->tw256_t;
        pa.gscratch = c->pg2_scratch;
        pa.counters = c->pg2_counters;
        pa.scale = c->scale;
        for (int64_t f0 = 0; f0 < frames; f0 += (int64_t)1 << 28) {
            const int64_t nf = std::min<int64_t>((int64_t)1 << 28, frames - f0);
            OFDMR_CUDA(cudaMemsetAsync(c->pg2_counters, 0, cnt_bytes, c->stream));
            pa.h = static_cast<const float2*>(h) + fc * f0;
            pa.p = p + pframe * f0;
            pa.frames = int(nf);
            cudaError_t e;
            {
                StageTimer t(c, 0, c->stream);
                e = launch_fused_pg2(pa, win, int(std::min<int64_t>(c->pg2_groups, nf)), c->pg2_groups, c->stream);
            }
            if (e != cudaSuccess) return cuda_fail(e, "fused_pg2");
            ++c->launches;
        }
        return OFDMR_OK;
    }
    if (c->fast && getenv("OFDMR_NO_PERSIST") == nullptr)
        return run_persist(c, static_cast<const float2*>(h), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                           nullptr, nullptr, nullptr, p, nullptr, frames);
    const int64_t pchunk = c->chunk;  // slot buffers hold chunk x N' rows
    const bool two = !c->profiling;
    if (two) {
        OFDMR_CUDA(cudaEventRecord(c->ev_fork, c->stream));
        OFDMR_CUDA(cudaStreamWaitEvent(c->aux_stream, c->ev_fork, 0));
    }
    c->slot[0].stream = c->stream;
    c->slot[1].stream = c->aux_stream;
    int64_t ci = 0;
    for (int64_t f0 = 0; f0 < frames; f0 += pchunk, ++ci) {
        const int64_t nf = std::min<int64_t>(pchunk, frames - f0);
        auto& s = c->slot[two ? (ci & 1) : 0];
        ColArgs a = base_col(c);
        a.h = static_cast<const float2*>(h) + fc * f0;
        a.g_out = s.gbuf;
        a.g_rows = g.n_prime;
        const bool win = g.window == OFDMR_WINDOW_HAMMING;
        if (win) {
            a.wk = c->wk;
            a.wl = c->wl;
        }
        if (c->fast) {
            cudaError_t e;
            {
                StageTimer t(c, 0, s.stream);
                e = launch_colpass_fast(a, false, win, c->tw1024_t, int(nf), s.stream);
            }
            if (e != cudaSuccess) return cuda_fail(e, "colpass_fast");
            ++c->launches;
            FastRowArgs r{};
            r.r.g = s.gbuf;
            r.r.p_out = p + pframe * f0;
            r.r.scale = c->scale;
            r.r.n_prime = g.n_prime;
            r.r.g_rows = g.n_prime;
            r.r.m = g.n_symbols;
            r.r.kmax = g.max_targets;
            r.r.detect = 0;
            r.tw256_t = c->tw256_t;
            {
                StageTimer t(c, 1, s.stream);
                e = launch_rowpass_fast(r, int(nf), s.stream);
            }
            if (e != cudaSuccess) return cuda_fail(e, "rowpass_fast");
            ++c->launches;
            continue;
        }
        int rc = launch_col(c, a, g.n_prime, nf, s.stream);
        if (rc) return rc;
        RowArgs r{};
        r.g = s.gbuf;
        r.p_out = p + pframe * f0;
        r.scale = c->scale;
        r.tw = c->tw;
        r.zp_tw = c->zp_tw;
        r.n_prime = g.n_prime;
        r.g_rows = g.n_prime;
        r.m = g.n_symbols;
        r.rows_per_block = rowpass_rows(g.m_prime, g.n_prime, g.n_symbols);
        r.kmax = g.max_targets;
        r.detect = 0;
        cudaError_t e;
        {
            StageTimer t(c, 1, s.stream);
            row_mixed(c, r);
        e = launch_rowpass(r, g.m_prime, int(nf), s.stream);
        }
        if (e != cudaSuccess) return cuda_fail(e, "rowpass");
        ++c->launches;
    }
    if (two) {
        OFDMR_CUDA(cudaEventRecord(c->ev_join, c->aux_stream));
        OFDMR_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    }
    return OFDMR_OK;
}

static int detect_impl(ofdmr_context* c, const float* p, const double* sigma2_h, const double* eta, const int32_t* kpf,
                       int32_t* d, int32_t* dp, float* pw, int32_t* cnt, int64_t frames) {
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    const ofdmr_config& g = c->cfg;
    const size_t pframe = size_t(g.n_prime) * size_t(g.m_prime);
    const int K = g.max_targets;
    // cand buffer is sized for c->chunk frames of this context's N'
    for (int64_t f0 = 0; f0 < frames; f0 += c->chunk) {
        const int64_t nf = std::min<int64_t>(c->chunk, frames - f0);
        RowArgs r{};
        r.p_in = p + pframe * f0;
        r.sigma2 = sigma2_h ? sigma2_h + f0 : nullptr;
        r.eta_in = eta ? eta + f0 : nullptr;
        r.log_pfa = c->log_pfa;
        r.power_factor = c->pf;
        r.tw = c->tw;
        r.zp_tw = c->zp_tw;
        r.n_prime = g.n_prime;
        r.g_rows = g.n_prime;
        r.m = g.n_symbols;
        r.rows_per_block = c->rows_per_block;
        r.kmax = K;
        r.cand = c->cand;
        r.detect = 1;
        row_mixed(c, r);
        cudaError_t e = launch_rowpass(r, g.m_prime, int(nf), c->stream);
        if (e != cudaSuccess) return cuda_fail(e, "rowpass(detect)");
        ++c->launches;
        MergeArgs mg{};
        mg.cand = c->cand;
        mg.nblk = c->nblk;
        mg.kmax = K;
        mg.k_per_frame = kpf ? kpf + f0 : nullptr;
        mg.m_prime = g.m_prime;
        mg.det_delay = d + size_t(K) * f0;
        mg.det_doppler = dp + size_t(K) * f0;
        mg.det_power = pw + size_t(K) * f0;
        mg.counts = cnt + f0;
        mg.sigma2 = sigma2_h ? sigma2_h + f0 : nullptr;
        e = launch_merge(mg, int(nf), c->stream);
        if (e != cudaSuccess) return cuda_fail(e, "merge");
        ++c->launches;
    }
    return OFDMR_OK;
}

int ofdmr_map_to_pgm(ofdmr_context* c, const float* p, uint8_t* out, int64_t frames) {
    if (!c || !p || !out) return fail(OFDMR_ERR_CONFIG, "map_to_pgm: null argument");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    const int64_t count = int64_t(c->cfg.n_prime) * int64_t(c->cfg.m_prime);
    double* peak = nullptr;
    OFDMR_CUDA(cudaMallocAsync(&peak, sizeof(double) * size_t(std::min<int64_t>(frames, 65535)), c->stream));
    const cudaError_t e = ofdmr::launch_map_pgm(p, count, out, frames, peak, c->stream, &c->launches);
    cudaFreeAsync(peak, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "map_to_pgm");
    return OFDMR_OK;
}

static int ofdm_impl(ofdmr_context* c, bool inverse, const void* in, void* out, int64_t frames, const char* what) {
    if (!c || !in || !out) return fail(OFDMR_ERR_CONFIG, std::string(what) + ": null argument");
    if (frames <= 0) return OFDMR_OK;
    const ofdmr_config& g = c->cfg;
    if (g.n_cp < 0 || g.n_cp > g.n_subcarriers) return fail(OFDMR_ERR_CONFIG, "n_cp must lie in [0, N]");
    OFDMR_CUDA(cudaSetDevice(c->device));
    const cudaError_t e =
        pow2_in(g.n_subcarriers, 16, 4096)
            ? ofdmr::launch_ofdm(inverse, static_cast<const float2*>(in), static_cast<float2*>(out), g.n_subcarriers,
                                 g.n_symbols, g.n_cp, frames, c->tw, c->stream)
            : ofdmr::launch_ofdm_mixed(inverse, static_cast<const float2*>(in), static_cast<float2*>(out),
                                       g.n_subcarriers, g.n_symbols, g.n_cp, frames, c->tw_n, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, what);
    ++c->launches;
    return OFDMR_OK;
}

int ofdmr_ofdm_demodulate(ofdmr_context* c, const void* stream, void* grid, int64_t frames) {
    return ofdm_impl(c, false, stream, grid, frames, "ofdm_demodulate");
}

int ofdmr_ofdm_modulate(ofdmr_context* c, const void* grid, void* stream, int64_t frames) {
    return ofdm_impl(c, true, grid, stream, frames, "ofdm_modulate");
}

int ofdmr_estimate_noise_power(ofdmr_context* c, const float* p, double* sigma2_out, int64_t frames) {
    if (!c || !p || !sigma2_out) return fail(OFDMR_ERR_CONFIG, "estimate_noise_power: null argument");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    const int64_t count = int64_t(c->cfg.n_prime) * int64_t(c->cfg.m_prime);
    const int64_t chunk = std::min<int64_t>(frames, 4096);
    if (c->noise_cap < chunk) {
        cudaFree(c->noise_scratch);
        c->noise_scratch = nullptr;
        c->noise_cap = 0;
        OFDMR_CUDA(cudaMalloc(&c->noise_scratch, ofdmr::noise_select_scratch_bytes(chunk)));
        c->noise_cap = chunk;
    }
    int sms = 0;
    OFDMR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    for (int64_t f0 = 0; f0 < frames; f0 += chunk) {
        const int64_t nf = std::min<int64_t>(chunk, frames - f0);
        const cudaError_t e = ofdmr::launch_noise_select(p + size_t(f0) * size_t(count), count, c->pf, sigma2_out + f0,
                                                         nf, c->noise_scratch, sms, c->stream, &c->launches);
        if (e != cudaSuccess) return cuda_fail(e, "estimate_noise_power");
    }
    return OFDMR_OK;
}

int ofdmr_detect(ofdmr_context* c, const float* p, const double* sigma2_h, const int32_t* kpf, int32_t* d,
                 int32_t* dp, float* pw, int32_t* cnt, int64_t frames) {
    if (!c || !p || !sigma2_h || !d || !dp || !pw || !cnt) return fail(OFDMR_ERR_CONFIG, "detect: null argument");
    return detect_impl(c, p, sigma2_h, nullptr, kpf, d, dp, pw, cnt, frames);
}

int ofdmr_extract_peaks(ofdmr_context* c, const float* p, const double* eta, const int32_t* kpf, int32_t* d,
                        int32_t* dp, float* pw, int32_t* cnt, int64_t frames) {
    if (!c || !p || !eta || !d || !dp || !pw || !cnt) return fail(OFDMR_ERR_CONFIG, "extract_peaks: null argument");
    return detect_impl(c, p, nullptr, eta, kpf, d, dp, pw, cnt, frames);
}

int ofdmr_pipeline(ofdmr_context* c, const void* y, const void* x, const double* sigma2, const int32_t* kpf,
                   int32_t* d, int32_t* dp, float* pw, int32_t* cnt, double* s2h_out, float* p_out,
                   int32_t* status, int64_t frames) {
    if (!c || !y || !x || !sigma2 || !d || !dp || !pw || !cnt) return fail(OFDMR_ERR_CONFIG, "pipeline: null argument");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    const ofdmr_config& g = c->cfg;
    const size_t fc = cells(c);
    const size_t pframe = size_t(g.n_prime) * size_t(g.m_prime);
    const int K = g.max_targets;
    if (status) OFDMR_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * size_t(frames), c->stream));
    if (c->fused && p_out == nullptr && !c->force_general) {
        // one persistent launch over the whole batch
        FusedArgs fa{};
        fa.y = static_cast<const float2*>(y);
        fa.x = static_cast<const float2*>(x);
        fa.sigma2 = sigma2;
        fa.k_per_frame = kpf;
        fa.det_delay = d;
        fa.det_doppler = dp;
        fa.det_power = pw;
        fa.counts = cnt;
        fa.s2h_out = s2h_out;
        fa.status = status;
        const bool win = g.window == OFDMR_WINDOW_HAMMING;
        fa.wk = win ? c->wk_s : nullptr;  // sqrt-scaled copy (see ofdmr_create)
        fa.wl = win ? c->wl : nullptr;
        fa.tw1024_t = c->tw1024_t;
        fa.tw256_t = c->tw256_t;
        fa.dscratch = c->dscratch;
        fa.L = g.n_cp;
        fa.kmax = K;
        fa.log_pfa = c->log_pfa;
        fa.power_factor = c->pf;
        fa.inv_count = c->inv_count;
        fa.scale = c->scale;
        fa.edges = c->fedges;
        fa.pend = c->fpend;
        fa.pend_loc = c->fpend_loc;
        fa.tlist = c->ftlist;
        for (int64_t f0 = 0; f0 < frames; f0 += (int64_t)1 << 28) {
            const int64_t nf = std::min<int64_t>((int64_t)1 << 28, frames - f0);
            fa.frames = int(nf);
            fa.y = static_cast<const float2*>(y) + fc * f0;
            fa.x = static_cast<const float2*>(x) + fc * f0;
            fa.sigma2 = sigma2 + f0;
            fa.k_per_frame = kpf ? kpf + f0 : nullptr;
            fa.det_delay = d + f0 * K;
            fa.det_doppler = dp + f0 * K;
            fa.det_power = pw + f0 * K;
            fa.counts = cnt + f0;
            fa.s2h_out = s2h_out ? s2h_out + f0 : nullptr;
            fa.status = status ? status + f0 : nullptr;
            cudaError_t e;
            {
                StageTimer t(c, 0, c->stream);
                // two 256-thread CTAs per SM, 2-CTA cluster per frame
                e = launch_fused_ce(fa, win, int(std::min<int64_t>(c->fused_grid, 2 * nf)), c->stream);
            }
            if (e != cudaSuccess) return cuda_fail(e, "fused_ce");
            ++c->launches;
        }
        return OFDMR_OK;
    }
    if (c->fast && g.estimator == OFDMR_EST_LS && getenv("OFDMR_NO_PERSIST") == nullptr) {
        int32_t* st = status;
        if (!st) {
            // status is required by the column items; use scratch for big batches chunk-wise
            if (frames <= c->chunk) {
                OFDMR_CUDA(cudaMemsetAsync(c->status_scratch, 0, sizeof(int32_t) * size_t(frames), c->stream));
                st = c->status_scratch;
            }
        }
        if (st)
            return run_persist(c, nullptr, static_cast<const float2*>(y), static_cast<const float2*>(x), sigma2, kpf,
                               d, dp, pw, cnt, s2h_out, p_out, st, frames);
    }
    const bool two = !c->profiling && frames > c->chunk;
    if (two) {
        OFDMR_CUDA(cudaEventRecord(c->ev_fork, c->stream));
        OFDMR_CUDA(cudaStreamWaitEvent(c->aux_stream, c->ev_fork, 0));
    }
    c->slot[0].stream = c->stream;
    c->slot[1].stream = c->aux_stream;
    int64_t ci = 0;
    for (int64_t f0 = 0; f0 < frames; f0 += c->chunk, ++ci) {
        const int64_t nf = std::min<int64_t>(c->chunk, frames - f0);
        const int si = two ? int(ci & 1) : 0;
        int32_t* st = status ? status + f0 : c->slot[si].status_scratch;
        if (!status) OFDMR_CUDA(cudaMemsetAsync(st, 0, sizeof(int32_t) * size_t(nf), c->slot[si].stream));
        const int rc = run_pipeline_chunk(
            c, si, static_cast<const float2*>(y) + fc * f0, static_cast<const float2*>(x) + fc * f0, sigma2 + f0,
            kpf ? kpf + f0 : nullptr, d + size_t(K) * f0, dp + size_t(K) * f0, pw + size_t(K) * f0, cnt + f0,
            s2h_out ? s2h_out + f0 : nullptr, p_out ? p_out + pframe * f0 : nullptr, st, nf);
        if (rc) return rc;
    }
    if (two) {
        OFDMR_CUDA(cudaEventRecord(c->ev_join, c->aux_stream));
        OFDMR_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    }
    return OFDMR_OK;
}

int ofdmr_pipeline_general(ofdmr_context* c, const void* y, const void* x, const double* sigma2, const int32_t* kpf,
                           int32_t* d, int32_t* dp, float* pw, int32_t* cnt, double* s2h_out, float* p_out,
                           int32_t* status, int64_t frames) {
    if (!c) return fail(OFDMR_ERR_CONFIG, "pipeline_general: null context");
    c->force_general = true;
    const int rc = ofdmr_pipeline(c, y, x, sigma2, kpf, d, dp, pw, cnt, s2h_out, p_out, status, frames);
    c->force_general = false;
    return rc;
}

int ofdmr_pipeline_host(ofdmr_context* c, const void* y, const void* x, const double* sigma2, const int32_t* kpf,
                        int32_t* d, int32_t* dp, float* pw, int32_t* cnt, int64_t frames) {
    if (!c || !y || !x || !sigma2 || !d || !dp || !pw || !cnt)
        return fail(OFDMR_ERR_CONFIG, "pipeline_host: null argument");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    const int64_t ch = c->chunk;
    const size_t fc = cells(c);
    const size_t fbytes = fc * sizeof(float2);
    const int K = c->cfg.max_targets;
    if (!c->dev_y[0]) {
        for (int i = 0; i < 2; ++i) {
            OFDMR_CUDA(cudaMalloc(&c->dev_y[i], fbytes * size_t(ch)));
            OFDMR_CUDA(cudaMalloc(&c->dev_x[i], fbytes * size_t(ch)));
            OFDMR_CUDA(cudaMalloc(&c->dev_s2[i], sizeof(double) * size_t(ch)));
            OFDMR_CUDA(cudaMalloc(&c->dev_k[i], sizeof(int32_t) * size_t(ch)));
            OFDMR_CUDA(cudaMalloc(&c->dev_d[i], sizeof(int32_t) * size_t(ch) * K));
            OFDMR_CUDA(cudaMalloc(&c->dev_dp[i], sizeof(int32_t) * size_t(ch) * K));
            OFDMR_CUDA(cudaMalloc(&c->dev_pw[i], sizeof(float) * size_t(ch) * K));
            OFDMR_CUDA(cudaMalloc(&c->dev_cnt[i], sizeof(int32_t) * size_t(ch)));
            OFDMR_CUDA(cudaMalloc(&c->dev_st[i], sizeof(int32_t) * size_t(ch)));
            OFDMR_CUDA(cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming));
            OFDMR_CUDA(cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming));
        }
        OFDMR_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        OFDMR_CUDA(cudaMallocHost(&c->host_st, 2 * sizeof(int32_t) * size_t(ch)));
    }
    // Chunk i+1's H2D (copy stream) and compute are enqueued before chunk i's status is read back,
    // so the host check of one chunk overlaps the next chunk's transfers and kernels; a chunk
    // with status bit 1 (fused-path overflow or abnormal |x|^2) is recomputed on the exact
    // general path before its buffers are reused (chunk i+2 is enqueued only after the check).
    bool zero_cell = false;
    auto finish = [&](int64_t f0, int64_t nf, int b) -> int {
        int32_t* hs = c->host_st + size_t(b) * size_t(ch);
        OFDMR_CUDA(cudaEventSynchronize(c->ev_done[b]));
        bool redo = false;
        for (int64_t i = 0; i < nf; ++i) redo |= (hs[i] & 2) != 0;
        if (redo) {
            int rc2 = ofdmr_pipeline_general(c, c->dev_y[b], c->dev_x[b], c->dev_s2[b], kpf ? c->dev_k[b] : nullptr,
                                             c->dev_d[b], c->dev_dp[b], c->dev_pw[b], c->dev_cnt[b], nullptr, nullptr,
                                             c->dev_st[b], nf);
            if (rc2) return rc2;
            OFDMR_CUDA(cudaMemcpyAsync(d + size_t(K) * f0, c->dev_d[b], sizeof(int32_t) * K * nf,
                                       cudaMemcpyDeviceToHost, c->stream));
            OFDMR_CUDA(cudaMemcpyAsync(dp + size_t(K) * f0, c->dev_dp[b], sizeof(int32_t) * K * nf,
                                       cudaMemcpyDeviceToHost, c->stream));
            OFDMR_CUDA(cudaMemcpyAsync(pw + size_t(K) * f0, c->dev_pw[b], sizeof(float) * K * nf,
                                       cudaMemcpyDeviceToHost, c->stream));
            OFDMR_CUDA(cudaMemcpyAsync(cnt + f0, c->dev_cnt[b], sizeof(int32_t) * nf, cudaMemcpyDeviceToHost,
                                       c->stream));
            OFDMR_CUDA(cudaMemcpyAsync(hs, c->dev_st[b], sizeof(int32_t) * nf, cudaMemcpyDeviceToHost, c->stream));
            OFDMR_CUDA(cudaStreamSynchronize(c->stream));
        }
        for (int64_t i = 0; i < nf; ++i) zero_cell |= (hs[i] & 1) != 0;
        return OFDMR_OK;
    };
    int64_t idx = 0, prev_f0 = -1, prev_nf = 0;
    for (int64_t f0 = 0; f0 < frames; f0 += ch, ++idx) {
        const int b = int(idx & 1);
        const int64_t nf = std::min<int64_t>(ch, frames - f0);
        // copy stream: wait until chunk idx-2 released buffer b, then stage inputs
        OFDMR_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev_done[b], 0));
        OFDMR_CUDA(cudaMemcpyAsync(c->dev_y[b], static_cast<const char*>(y) + fbytes * f0, fbytes * nf,
                                   cudaMemcpyHostToDevice, c->copy_stream));
        OFDMR_CUDA(cudaMemcpyAsync(c->dev_x[b], static_cast<const char*>(x) + fbytes * f0, fbytes * nf,
                                   cudaMemcpyHostToDevice, c->copy_stream));
        OFDMR_CUDA(cudaMemcpyAsync(c->dev_s2[b], sigma2 + f0, sizeof(double) * nf, cudaMemcpyHostToDevice,
                                   c->copy_stream));
        if (kpf)
            OFDMR_CUDA(cudaMemcpyAsync(c->dev_k[b], kpf + f0, sizeof(int32_t) * nf, cudaMemcpyHostToDevice,
                                       c->copy_stream));
        OFDMR_CUDA(cudaEventRecord(c->ev_copied[b], c->copy_stream));
        OFDMR_CUDA(cudaStreamWaitEvent(c->stream, c->ev_copied[b], 0));
        int rc = ofdmr_pipeline(c, c->dev_y[b], c->dev_x[b], c->dev_s2[b], kpf ? c->dev_k[b] : nullptr, c->dev_d[b],
                                c->dev_dp[b], c->dev_pw[b], c->dev_cnt[b], nullptr, nullptr, c->dev_st[b], nf);
        if (rc) return rc;
        OFDMR_CUDA(cudaMemcpyAsync(d + size_t(K) * f0, c->dev_d[b], sizeof(int32_t) * K * nf, cudaMemcpyDeviceToHost,
                                   c->stream));
        OFDMR_CUDA(cudaMemcpyAsync(dp + size_t(K) * f0, c->dev_dp[b], sizeof(int32_t) * K * nf,
                                   cudaMemcpyDeviceToHost, c->stream));
        OFDMR_CUDA(cudaMemcpyAsync(pw + size_t(K) * f0, c->dev_pw[b], sizeof(float) * K * nf, cudaMemcpyDeviceToHost,
                                   c->stream));
        OFDMR_CUDA(cudaMemcpyAsync(cnt + f0, c->dev_cnt[b], sizeof(int32_t) * nf, cudaMemcpyDeviceToHost, c->stream));
        OFDMR_CUDA(cudaMemcpyAsync(c->host_st + size_t(b) * size_t(ch), c->dev_st[b], sizeof(int32_t) * nf,
                                   cudaMemcpyDeviceToHost, c->stream));
        OFDMR_CUDA(cudaEventRecord(c->ev_done[b], c->stream));
        if (prev_f0 >= 0) {
            rc = finish(prev_f0, prev_nf, b ^ 1);
            if (rc) return rc;
        }
        prev_f0 = f0;
        prev_nf = nf;
    }
    if (prev_f0 >= 0) {
        const int rc = finish(prev_f0, prev_nf, int((idx - 1) & 1));
        if (rc) return rc;
    }
    OFDMR_CUDA(cudaStreamSynchronize(c->stream));
    if (zero_cell) return fail(OFDMR_ERR_CONFIG, "spectral_division: zero cell in X");
    return OFDMR_OK;
}

int ofdmr_sft_estimate_noise(ofdmr_context* c, const void* h, int32_t n, int32_t m, const uint64_t* seeds,
                             double* sigma2_out, int64_t frames) {
    if (!c || !h || !seeds || !sigma2_out) return fail(OFDMR_ERR_CONFIG, "estimate_noise_from_slice: null argument");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    std::string err;
    const int rc = sft_slice_noise(c->sft, c->stream, static_cast<const float2*>(h), n, m, seeds, sigma2_out, frames,
                                   &c->launches, err);
    if (rc) return fail(rc, err);
    return OFDMR_OK;
}

int ofdmr_sft(ofdmr_context* c, const void* h, int32_t n, int32_t m, const ofdmr_sft_config* cfg,
              const uint64_t* seeds, const double* sigma2, int32_t* k_out, int32_t* l_out, double* amp_out,
              int32_t* n_entries, int32_t* iterations, int64_t* samples_used, int32_t* converged, double* residual,
              int32_t* status, int64_t frames) {
    if (!c || !h || !cfg || !seeds || !sigma2 || !k_out || !l_out || !amp_out || !n_entries)
        return fail(OFDMR_ERR_CONFIG, "sft: null argument");
    if (n <= 0 || m <= 0) return fail(OFDMR_ERR_CONFIG, "sft_iterate: empty grid");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    std::string err;
    if (status) OFDMR_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * size_t(frames), c->stream));
    const int rc = sft_run(c->sft, c->stream, static_cast<const float2*>(h), n, m, *cfg, seeds, sigma2, false, k_out,
                           l_out, amp_out, n_entries, iterations, samples_used, converged, residual, status, frames,
                           &c->launches, err);
    if (rc) return fail(rc, err);
    return OFDMR_OK;
}

namespace {

int sft_pipe_reserve(ofdmr_context* c, int64_t frames, int64_t h_frames, int max_entries) {
    auto& p = c->sp;
    if (h_frames > p.cap_h) {
        cudaFree(p.h);
        p.h = nullptr;
        p.cap_h = 0;
        const size_t fc = size_t(c->cfg.n_subcarriers) * size_t(c->cfg.n_symbols);
        OFDMR_CUDA(cudaMalloc(&p.h, sizeof(float2) * fc * size_t(h_frames)));
        p.cap_h = h_frames;
    }
    if (frames > p.cap) {
        cudaFree(p.k);
        cudaFree(p.l);
        cudaFree(p.amp);
        cudaFree(p.ne);
        cudaFree(p.s2h);
        cudaFree(p.s2u);
        cudaFree(p.st);
        p = ofdmr_context::SftPipe{p.h, p.cap_h};
        OFDMR_CUDA(cudaMalloc(&p.k, sizeof(int32_t) * 64 * size_t(frames)));
        OFDMR_CUDA(cudaMalloc(&p.l, sizeof(int32_t) * 64 * size_t(frames)));
        OFDMR_CUDA(cudaMalloc(&p.amp, sizeof(double) * 2 * 64 * size_t(frames)));
        OFDMR_CUDA(cudaMalloc(&p.ne, sizeof(int32_t) * size_t(frames)));
        OFDMR_CUDA(cudaMalloc(&p.s2h, sizeof(double) * size_t(frames)));
        OFDMR_CUDA(cudaMalloc(&p.s2u, sizeof(double) * size_t(frames)));
        OFDMR_CUDA(cudaMalloc(&p.st, sizeof(int32_t) * size_t(frames)));
        p.cap = frames;
    }
    (void)max_entries;
    return OFDMR_OK;
}

}  // namespace

int ofdmr_sft_detections(ofdmr_context* c, const int32_t* k, const int32_t* l, const double* amp,
                         const int32_t* n_entries, int32_t max_entries, int32_t n, int32_t m, const double* sigma2,
                         double pfa, const int32_t* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin,
                         float* peak_power, int32_t* counts, int64_t frames) {
    if (!c || !k || !l || !amp || !n_entries || !sigma2 || !delay_bin || !doppler_bin || !peak_power || !counts)
        return fail(OFDMR_ERR_CONFIG, "detections_from_spectrum: null argument");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    std::string err;
    const int rc = sft_detections(c->stream, k, l, amp, n_entries, max_entries, n, m, sigma2, pfa, k_per_frame,
                                  c->cfg.max_targets, delay_bin, doppler_bin, peak_power, counts, frames, &c->launches,
                                  err);
    return rc ? fail(rc, err) : OFDMR_OK;
}

int ofdmr_sft_detect(ofdmr_context* c, const void* h, int32_t n, int32_t m, const ofdmr_sft_config* cfg,
                     const uint64_t* seeds, const double* sigma2, const int32_t* k_per_frame, int32_t* delay_bin,
                     int32_t* doppler_bin, float* peak_power, int32_t* counts, int32_t* status, int64_t frames) {
    if (!c || !h || !cfg || !seeds || !sigma2 || !delay_bin || !doppler_bin || !peak_power || !counts || !status)
        return fail(OFDMR_ERR_CONFIG, "sft_detect: null argument");
    if (n <= 0 || m <= 0) return fail(OFDMR_ERR_CONFIG, "sft_iterate: empty grid");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    int rc = sft_pipe_reserve(c, frames, 0, cfg->max_entries);
    if (rc) return rc;
    OFDMR_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * size_t(frames), c->stream));
    ofdmr_sft_config sc = *cfg;
    sc.max_entries = 64;  // every entry reaches detections_from_spectrum (sft.cpp:467-485)
    std::string err;
    rc = sft_run(c->sft, c->stream, static_cast<const float2*>(h), n, m, sc, seeds, sigma2, true, c->sp.k, c->sp.l,
                 c->sp.amp, c->sp.ne, nullptr, nullptr, nullptr, nullptr, status, frames, &c->launches, err);
    if (rc) return fail(rc, err);
    rc = sft_detections(c->stream, c->sp.k, c->sp.l, c->sp.amp, c->sp.ne, 64, n, m, sigma2, cfg->pfa, k_per_frame,
                        c->cfg.max_targets, delay_bin, doppler_bin, peak_power, counts, frames, &c->launches, err);
    return rc ? fail(rc, err) : OFDMR_OK;
}

int ofdmr_pipeline_sft(ofdmr_context* c, const void* y, const void* x_tx, const double* sigma2,
                       const uint64_t* sft_seeds, const uint64_t* noise_seeds, const ofdmr_sft_config* cfg,
                       const int32_t* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin, float* peak_power,
                       int32_t* counts, double* sigma2_used_out, int32_t* status, int64_t frames) {
    if (!c || !y || !x_tx || !sigma2 || !sft_seeds || !cfg || !delay_bin || !doppler_bin || !peak_power || !counts ||
        !status)
        return fail(OFDMR_ERR_CONFIG, "pipeline_sft: null argument");
    if (frames <= 0) return OFDMR_OK;
    OFDMR_CUDA(cudaSetDevice(c->device));
    const int n = c->cfg.n_subcarriers, m = c->cfg.n_symbols, K = c->cfg.max_targets;
    const size_t fc = size_t(n) * size_t(m);
    // channel estimates of one chunk in scratch (<= 1 GiB)
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(frames, (int64_t(1) << 30) / int64_t(fc * 8)));
    int rc = sft_pipe_reserve(c, chunk, chunk, cfg->max_entries);
    if (rc) return rc;
    ofdmr_sft_config sc = *cfg;
    sc.max_entries = 64;
    std::string err;
    for (int64_t f0 = 0; f0 < frames; f0 += chunk) {
        const int64_t nf = std::min<int64_t>(chunk, frames - f0);
        const float2* yc = static_cast<const float2*>(y) + fc * f0;
        const float2* xc = static_cast<const float2*>(x_tx) + fc * f0;
        int32_t* stc = status + f0;
        // estimate_channel (pipeline.cpp:47-58): LS / ZCP-LS / DFT-CE per the context estimator
        rc = ofdmr_estimate_channel(c, yc, xc, c->sp.h, stc, nf);
        if (rc) return rc;
        // sigma_h^2 = division_noise_power(sigma2, x_tx) (pipeline.cpp:79)
        rc = division_noise(c->stream, xc, int64_t(fc), sigma2 + f0, c->sp.s2h, nf, &c->launches, err);
        if (rc) return fail(rc, err);
        const double* s2u = c->sp.s2h;
        if (noise_seeds) {  // estimate_noise mode: estimate_noise_from_slice (pipeline.cpp:97-98)
            rc = sft_slice_noise(c->sft, c->stream, c->sp.h, n, m, noise_seeds + f0, c->sp.s2u, nf, &c->launches, err);
            if (rc) return fail(rc, err);
            s2u = c->sp.s2u;
        }
        if (sigma2_used_out)
            OFDMR_CUDA(cudaMemcpyAsync(sigma2_used_out + f0, s2u, sizeof(double) * nf, cudaMemcpyDeviceToDevice,
                                       c->stream));
        // sft_iterate with SftConfig{i_max, seed, sigma2 = s2u, pfa} (pipeline.cpp:99-109)
        rc = sft_run(c->sft, c->stream, c->sp.h, n, m, sc, sft_seeds + f0, s2u, true, c->sp.k, c->sp.l, c->sp.amp,
                     c->sp.ne, nullptr, nullptr, nullptr, nullptr, stc, nf, &c->launches, err);
        if (rc) return fail(rc, err);
        // detections_from_spectrum(spec, N, M, w, sigma2, pfa, max_targets) (pipeline.cpp:110-111)
        rc = sft_detections(c->stream, c->sp.k, c->sp.l, c->sp.amp, c->sp.ne, 64, n, m, s2u, cfg->pfa,
                            k_per_frame ? k_per_frame + f0 : nullptr, K, delay_bin + f0 * K, doppler_bin + f0 * K,
                            peak_power + f0 * K, counts + f0, nf, &c->launches, err);
        if (rc) return fail(rc, err);
    }
    return OFDMR_OK;
}

}  // extern "C"

// Debug/introspection (tools only): integer properties of a context.
extern "C" long long ofdmr_debug_info(ofdmr_context* c, const char* key) {
    if (!c || !key) return -1;
    const std::string k(key);
    if (k == "fused_grid") return c->fused_grid;
    if (k == "pg2_max_groups") return ofdmr::fused_pg2_max_groups();
    return -1;
}
