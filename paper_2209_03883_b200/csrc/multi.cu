// Multi-device receiver: frames are independent, so a batch is split into
// contiguous shards [r F / G, (r + 1) F / G), one per device, each processed by its own context
// on its own host thread with no data-path exchange; the only exchange is the gather of the
// fixed-size detection records: to the first device with cudaMemcpyPeerAsync (NVLink /
// NVSwitch) for device-resident inputs, or straight into the caller's host arrays.  Built on the
// public single-device C-ABI (include/ofdmr_b200.h).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ofdmr_b200.h"

struct ofdmr_multi {
    ofdmr_config cfg{};
    std::vector<int32_t> devices;
    std::vector<ofdmr_context*> ctx;
    std::vector<cudaStream_t> streams;
    // per-rank record scratch for the device-resident gather (ranks > 0)
    struct Scratch {
        int32_t* d = nullptr;
        int32_t* dp = nullptr;
        float* pw = nullptr;
        int32_t* cnt = nullptr;
        int32_t* st = nullptr;
        int64_t cap = 0;
    };
    std::vector<Scratch> scratch;
};

namespace {
thread_local std::string g_multi_error;

int mfail(int code, const std::string& msg) {
    g_multi_error = msg;
    return code;
}

// fn(rank) on one host thread per device (rank 0 on the caller's thread); first error wins.
template <typename F>
int for_each_device(ofdmr_multi* m, F fn) {
    const int g = int(m->devices.size());
    std::vector<int> rc(g, OFDMR_OK);
    std::vector<std::string> err(g);
    std::vector<std::thread> th;
    for (int r = 1; r < g; ++r)
        th.emplace_back([&, r] {
            cudaSetDevice(m->devices[r]);
            rc[r] = fn(r);
            if (rc[r]) err[r] = ofdmr_last_error();
        });
    cudaSetDevice(m->devices[0]);
    rc[0] = fn(0);
    if (rc[0]) err[0] = ofdmr_last_error();
    for (auto& t : th) t.join();
    for (int r = 0; r < g; ++r)
        if (rc[r]) return mfail(rc[r], "device " + std::to_string(m->devices[r]) + ": " + err[r]);
    return OFDMR_OK;
}

int cuda_err(cudaError_t e, const char* where) {
    return e == cudaSuccess ? OFDMR_OK : mfail(OFDMR_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

void ofdmr_shard_range(int64_t frames, int32_t rank, int32_t world, int64_t* lo, int64_t* hi) {
    *lo = frames * rank / world;
    *hi = frames * (rank + 1) / world;
}

const char* ofdmr_multi_last_error(void) { return g_multi_error.c_str(); }

int ofdmr_multi_create(const ofdmr_config* cfg, const int32_t* devices, int32_t ndev, ofdmr_multi** out) {
    if (!cfg || !devices || ndev < 1 || !out) return mfail(OFDMR_ERR_CONFIG, "multi_create: bad arguments");
    auto* m = new ofdmr_multi;
    m->cfg = *cfg;
    m->devices.assign(devices, devices + ndev);
    m->scratch.resize(ndev);
    for (int r = 0; r < ndev; ++r) {
        ofdmr_config c = *cfg;
        c.device = devices[r];
        ofdmr_context* ctx = nullptr;
        const int rc = ofdmr_create(&c, &ctx);
        if (rc) {
            const std::string e = ofdmr_last_error();
            ofdmr_multi_destroy(m);
            return mfail(rc, "device " + std::to_string(devices[r]) + ": " + e);
        }
        m->ctx.push_back(ctx);
        cudaStream_t s = nullptr;
        if (cudaSetDevice(devices[r]) != cudaSuccess || cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
            ofdmr_multi_destroy(m);
            return mfail(OFDMR_ERR_CUDA, "multi_create: stream");
        }
        m->streams.push_back(s);
        ofdmr_set_stream(ctx, s);
        // direct peer writes for the gather to the first device when the link allows it
        if (r > 0 && devices[r] != devices[0]) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, devices[r], devices[0]);
            if (can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(devices[0], 0);
                if (e != cudaSuccess) cudaGetLastError();  // already enabled is fine
            }
        }
    }
    *out = m;
    return OFDMR_OK;
}

void ofdmr_multi_destroy(ofdmr_multi* m) {
    if (!m) return;
    for (std::size_t r = 0; r < m->ctx.size(); ++r) ofdmr_destroy(m->ctx[r]);
    for (std::size_t r = 0; r < m->devices.size(); ++r) {
        cudaSetDevice(m->devices[r]);
        if (r < m->streams.size()) cudaStreamDestroy(m->streams[r]);
        auto& s = m->scratch[r];
        cudaFree(s.d);
        cudaFree(s.dp);
        cudaFree(s.pw);
        cudaFree(s.cnt);
        cudaFree(s.st);
    }
    delete m;
}

int32_t ofdmr_multi_devices(const ofdmr_multi* m) { return m ? int32_t(m->devices.size()) : 0; }

ofdmr_context* ofdmr_multi_context(ofdmr_multi* m, int32_t rank) {
    return m && rank >= 0 && rank < int32_t(m->ctx.size()) ? m->ctx[rank] : nullptr;
}

int ofdmr_multi_pipeline_host(ofdmr_multi* m, const void* y, const void* x_tx, const double* sigma2,
                              const int32_t* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin, float* peak_power,
                              int32_t* counts, int64_t frames) {
    if (!m || !y || !x_tx || !sigma2 || !delay_bin || !doppler_bin || !peak_power || !counts)
        return mfail(OFDMR_ERR_CONFIG, "multi_pipeline_host: null argument");
    if (frames <= 0) return OFDMR_OK;
    const int g = int(m->devices.size());
    const size_t fb = size_t(m->cfg.n_subcarriers) * size_t(m->cfg.n_symbols) * 8;
    const int64_t K = m->cfg.max_targets;
    return for_each_device(m, [&](int r) -> int {
        int64_t lo, hi;
        ofdmr_shard_range(frames, r, g, &lo, &hi);
        if (hi <= lo) return OFDMR_OK;
        // the shard's records land directly in their slice of the caller's arrays (the gather)
        return ofdmr_pipeline_host(m->ctx[r], static_cast<const char*>(y) + fb * lo,
                                   static_cast<const char*>(x_tx) + fb * lo, sigma2 + lo,
                                   k_per_frame ? k_per_frame + lo : nullptr, delay_bin + K * lo, doppler_bin + K * lo,
                                   peak_power + K * lo, counts + lo, hi - lo);
    });
}

int ofdmr_multi_pipeline(ofdmr_multi* m, const void* const* y, const void* const* x_tx, const double* const* sigma2,
                         const int32_t* const* k_per_frame, int32_t* delay_bin, int32_t* doppler_bin,
                         float* peak_power, int32_t* counts, int32_t* status, int64_t frames) {
    if (!m || !y || !x_tx || !sigma2 || !delay_bin || !doppler_bin || !peak_power || !counts || !status)
        return mfail(OFDMR_ERR_CONFIG, "multi_pipeline: null argument");
    if (frames <= 0) return OFDMR_OK;
    const int g = int(m->devices.size());
    const int64_t K = m->cfg.max_targets;
    return for_each_device(m, [&](int r) -> int {
        int64_t lo, hi;
        ofdmr_shard_range(frames, r, g, &lo, &hi);
        const int64_t nf = hi - lo;
        if (nf <= 0) return OFDMR_OK;
        if (!y[r] || !x_tx[r] || !sigma2[r]) return mfail(OFDMR_ERR_CONFIG, "multi_pipeline: null shard input");
        const int32_t* kp = k_per_frame ? k_per_frame[r] : nullptr;
        cudaStream_t st = m->streams[r];
        if (r == 0) {  // the first device writes its shard in place
            int rc = ofdmr_pipeline(m->ctx[0], y[0], x_tx[0], sigma2[0], kp, delay_bin + K * lo, doppler_bin + K * lo,
                                    peak_power + K * lo, counts + lo, nullptr, nullptr, status + lo, nf);
            if (rc) return rc;
            return cuda_err(cudaStreamSynchronize(st), "multi_pipeline");
        }
        auto& s = m->scratch[r];
        if (s.cap < nf) {
            cudaFree(s.d);
            cudaFree(s.dp);
            cudaFree(s.pw);
            cudaFree(s.cnt);
            cudaFree(s.st);
            s = ofdmr_multi::Scratch{};
            int rc = cuda_err(cudaMalloc(&s.d, sizeof(int32_t) * K * nf), "multi_pipeline: scratch");
            if (!rc) rc = cuda_err(cudaMalloc(&s.dp, sizeof(int32_t) * K * nf), "multi_pipeline: scratch");
            if (!rc) rc = cuda_err(cudaMalloc(&s.pw, sizeof(float) * K * nf), "multi_pipeline: scratch");
            if (!rc) rc = cuda_err(cudaMalloc(&s.cnt, sizeof(int32_t) * nf), "multi_pipeline: scratch");
            if (!rc) rc = cuda_err(cudaMalloc(&s.st, sizeof(int32_t) * nf), "multi_pipeline: scratch");
            if (rc) return rc;
            s.cap = nf;
        }
        int rc = ofdmr_pipeline(m->ctx[r], y[r], x_tx[r], sigma2[r], kp, s.d, s.dp, s.pw, s.cnt, nullptr, nullptr, s.st,
                                nf);
        if (rc) return rc;
        // gather: the shard's records into their slice on the first device
        const int d0 = m->devices[0], dr = m->devices[r];
        cudaError_t e = cudaMemcpyPeerAsync(delay_bin + K * lo, d0, s.d, dr, sizeof(int32_t) * K * nf, st);
        if (e == cudaSuccess) e = cudaMemcpyPeerAsync(doppler_bin + K * lo, d0, s.dp, dr, sizeof(int32_t) * K * nf, st);
        if (e == cudaSuccess) e = cudaMemcpyPeerAsync(peak_power + K * lo, d0, s.pw, dr, sizeof(float) * K * nf, st);
        if (e == cudaSuccess) e = cudaMemcpyPeerAsync(counts + lo, d0, s.cnt, dr, sizeof(int32_t) * nf, st);
        if (e == cudaSuccess) e = cudaMemcpyPeerAsync(status + lo, d0, s.st, dr, sizeof(int32_t) * nf, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        return cuda_err(e, "multi_pipeline: gather");
    });
}

}  // extern "C"
