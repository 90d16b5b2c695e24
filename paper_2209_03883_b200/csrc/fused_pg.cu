// Persistent batched 2-D periodogram for N = N' = 1024, M = M' = 256 (H in, P out):
//   P[n][(m + M/2) mod M] = |FFT_M( IFFT_N( H .* w_k w_l ) )|^2 / (N M)
// (periodogram.cpp:39-75; the map ofdmr_periodogram returns).
//
// One group of G = 16 CTAs per frame (2 CTAs per SM, 8 warps each; a persistent grid of
// 18 groups), synchronised by a counting global-memory barrier (all CTAs are resident):
//   column pass  CTA r, step u owns symbols 8G u + 8r .. +7, so at every step the group reads
//                8G * 8 contiguous bytes of each subcarrier row of H.  H arrives through a
//                thread-private cp.async ring (4 x 8 KB); w_k w_l on the fly; each warp runs
//                one register-resident IFFT_1024; the 1024 x 8 tile of G goes to a per-group
//                2 MiB scratch as 64-B row segments.
//   group barrier (G complete)
//   row pass     CTA r owns rows 1024/G r ..: half-warp FFT_256 per row (twiddles in
//                registers), |.|^2 / (N M) with the Doppler fftshift, streamed to P; the rows
//                of the next round are loaded while the current round transforms.
//   split barrier (arrive after the last G read, wait before the first G write of the next
//                frame), so no CTA waits for its peers between frames.
// The ring keeps prefetching the next frame's H during the row pass.  Frames in flight = the
// number of groups (18), i.e. 36 MiB of G, which stays in L2: measured DRAM traffic is
// 3.7 MiB/frame against 3 MiB algorithmic (a 2-CTA hardware cluster per frame, PG_SW=0,
// PG_CLUSTER=2, runs at the same speed but spills G: 7.2 MiB/frame).
#include <cooperative_groups.h>

#include "fused_args.cuh"
#include "radar_kernels.cuh"
#include "warp_fft.cuh"

namespace cg = cooperative_groups;

namespace ofdmr {

namespace {

constexpr int kN = 1024, kM = 256;
constexpr int kVS = 1058;       // padded column stride (float2; 2 mod 8 -> conflict-free tile writes)
constexpr int kPgRing = 4;      // H staging ring depth (stages of 128 rows x 8 symbols)
#ifndef PG_CLUSTER
#define PG_CLUSTER 16
#endif
#ifndef PG_SW
#define PG_SW 1  // 1: the PG_CLUSTER CTAs of a frame are a software group (global-memory barrier)
#endif
constexpr int kPgCluster = PG_CLUSTER;  // CTAs per frame
constexpr int kPgSteps = 256 / (8 * kPgCluster);   // column tiles per CTA
constexpr int kPgRows = 1024 / kPgCluster;         // rows per CTA in the row pass

struct PgSmem {
    float2 tw[1024];
    float2 tw256[256];
    float2 cols[8 * kVS];           // column-pass tiles / row-pass half-warp scratch
    float4 stg[kPgRing][2][256];    // thread-private 16-B slots
};

__device__ __forceinline__ void pg_cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void pg_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void pg_cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
#if !PG_SW
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
#endif
#if PG_SW
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
#endif

// Frame-group barrier: a hardware cluster barrier, or (PG_SW) a monotonically counting
// global-memory barrier over the group's CTAs (all CTAs of the persistent grid are resident).
struct GroupBarrier {
    int* counter;
    int phase;
    __device__ void arrive() {
#if PG_SW
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(counter, 1);
        }
        ++phase;
#else
        cluster_arrive();
#endif
    }
    __device__ void wait() {
#if PG_SW
        if (threadIdx.x == 0) {
            const int target = kPgCluster * phase;
            while (ld_acquire(counter) < target) __nanosleep(32);
            __threadfence();
        }
        __syncthreads();
#else
        cluster_wait();
#endif
    }
};

}  // namespace

#ifdef OFDMR_PHASE_TIMING
__device__ unsigned long long g_pg_phase[8];
#define PGPH_INIT() long long _ph_t = clock64();
#define PGPH(i)                                                         \
    do {                                                                \
        if (threadIdx.x == 0) {                                         \
            const long long _n = clock64();                             \
            atomicAdd(&g_pg_phase[i], (unsigned long long)(_n - _ph_t)); \
            _ph_t = _n;                                                 \
        }                                                               \
    } while (0)
#else
#define PGPH_INIT()
#define PGPH(i)
#endif

template <bool HAMMING>
__global__ void
#if !PG_SW
__cluster_dims__(kPgCluster, 1, 1)
#endif
__launch_bounds__(256, 2) fused_pg1024_kernel(PgArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PgSmem& s = *reinterpret_cast<PgSmem*>(smem_raw);
    const int rank = (int)(blockIdx.x % kPgCluster);
    GroupBarrier bar{a.group_counters + blockIdx.x / kPgCluster, 0};
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int cid = blockIdx.x / kPgCluster, ncl = gridDim.x / kPgCluster;
    float2* g = a.gscratch + (size_t)cid * kN * kM;

    for (int i = tid; i < 1024; i += 256) s.tw[i] = a.tw1024_t[i];
    s.tw256[tid] = a.tw256_t[tid];
    __syncthreads();

    // H stream: this CTA's tiles in order (frame cid steps 0..3, frame cid + ncl steps 0..3, ..);
    // stage = 2 x 16 B per thread = rows 128 st .. 128 st + 127 of the 8-symbol tile
    int ifr = cid, iu = 0, ist = 0, islot = 0, cslot = 0;
    const size_t lane_off = (size_t)(tid >> 2) * kM + 8 * rank + (tid & 3) * 2;
    auto issue = [&]() {
        if (ifr < a.frames) {
            const float2* src = a.h + (size_t)ifr * kN * kM + (size_t)ist * 128 * kM + 8 * kPgCluster * iu + lane_off;
            pg_cp_async16(&s.stg[islot][0][tid], src);
            pg_cp_async16(&s.stg[islot][1][tid], src + (size_t)64 * kM);
        }
        pg_cp_commit();
        islot = islot + 1 == kPgRing ? 0 : islot + 1;
        if (++ist == 8) {
            ist = 0;
            if (++iu == kPgSteps) {
                iu = 0;
                ifr += ncl;
            }
        }
    };
    for (int i = 0; i < kPgRing; ++i) issue();
    PGPH_INIT();

    bool first = true;
    for (int f = cid; f < a.frames; f += ncl) {
        // ------------------------------------------------------------ column pass
        for (int u = 0; u < kPgSteps; ++u) {
            const int c0 = 8 * kPgCluster * u + 8 * rank;
            float wl0 = 1.f, wl1 = 1.f;
            if (HAMMING) {
                wl0 = __ldg(a.wl + c0 + (tid & 3) * 2);
                wl1 = __ldg(a.wl + c0 + (tid & 3) * 2 + 1);
            }
#pragma unroll 2
            for (int st = 0; st < 8; ++st) {
                pg_cp_wait<kPgRing - 1>();
                const float4 h0 = s.stg[cslot][0][tid];
                const float4 h1 = s.stg[cslot][1][tid];
                cslot = cslot + 1 == kPgRing ? 0 : cslot + 1;
                const int k0 = (tid >> 2) + 128 * st, k1 = k0 + 64;
                const int c = (tid & 3) * 2;
                float a0 = 1.f, b0 = 1.f, a1 = 1.f, b1 = 1.f;
                if (HAMMING) {
                    const float wk0 = __ldg(a.wk + k0), wk1 = __ldg(a.wk + k1);
                    a0 = wk0 * wl0;
                    b0 = wk0 * wl1;
                    a1 = wk1 * wl0;
                    b1 = wk1 * wl1;
                }
                const int p0 = k0 + (k0 >> 5), p1 = k1 + (k1 >> 5);
                s.cols[c * kVS + p0] = make_float2(h0.x * a0, h0.y * a0);
                s.cols[(c + 1) * kVS + p0] = make_float2(h0.z * b0, h0.w * b0);
                s.cols[c * kVS + p1] = make_float2(h1.x * a1, h1.y * a1);
                s.cols[(c + 1) * kVS + p1] = make_float2(h1.z * b1, h1.w * b1);
                issue();
            }
            __syncthreads();
            PGPH(0);
            {
                float2* col = s.cols + w * kVS;
                float2 v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = col[lane + 33 * i];
                warp_fft1024<true, 32>(v, col, s.tw);  // lane t1: G[t1 + 32 t2]
                __syncwarp();
#pragma unroll
                for (int t2 = 0; t2 < 32; ++t2) col[lane + 33 * t2] = v[t2];
            }
            __syncthreads();
            PGPH(1);
            if (u == 0 && !first) bar.wait();  // peers finished reading the previous frame's G
            first = false;
            PGPH(2);
#pragma unroll 4
            for (int q = 0; q < 16; ++q) {
                const int idx = tid + q * 256;
                const int k = idx >> 2, c = (idx & 3) * 2;
                const int pk = k + (k >> 5);
                const float2 v0 = s.cols[c * kVS + pk];
                const float2 v1 = s.cols[(c + 1) * kVS + pk];
                __stcg(reinterpret_cast<float4*>(g + (size_t)k * kM + c0 + c), make_float4(v0.x, v0.y, v1.x, v1.y));
            }
            __syncthreads();
            PGPH(3);
        }
        __threadfence();
        bar.arrive();  // G of frame f complete
        bar.wait();
        PGPH(4);

        // ------------------------------------------------------------ row pass
        {
            const int hw = tid >> 4, j = tid & 15;
            float2* tb = s.cols + hw * (16 * 17);
            float* pf = a.p + (size_t)f * kN * kM;
            float2 v[16], vn[16], twr[16];
#pragma unroll
            for (int t1 = 0; t1 < 16; ++t1) twr[t1] = s.tw256[t1 * 16 + j];
            const int rbase = kPgRows * rank + hw;
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = __ldcg(g + (size_t)rbase * kM + j + 16 * i);
            for (int q = 0; q < kPgRows / 16; ++q) {
                const int n = rbase + 16 * q;
                if (q < kPgRows / 16 - 1) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) vn[i] = __ldcg(g + (size_t)(n + 16) * kM + j + 16 * i);
                }
                halfwarp_fft256_rt<false>(v, tb, twr);
                float* prow = pf + (size_t)n * kM;
#pragma unroll
                for (int t2 = 0; t2 < 16; ++t2) __stcs(prow + ((j + 16 * t2 + 128) & 255), cnorm(v[t2]) * a.scale);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = vn[i];
            }
        }
        __syncthreads();   // row-pass scratch (cols) free before the next frame's tiles land in it
        PGPH(5);
        bar.arrive();  // our G reads are done (matched by the wait before the next G write)
    }
    if (!first) bar.wait();  // balance the last arrive before exit
}

}  // namespace ofdmr

extern "C" int ofdmr_debug_pg_phase_cycles(unsigned long long* out, int reset) {
#ifdef OFDMR_PHASE_TIMING
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, ofdmr::g_pg_phase, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(ofdmr::g_pg_phase, z, sizeof(z));
    }
    return 8;
#else
    (void)out;
    (void)reset;
    return 0;
#endif
}

namespace ofdmr {

size_t fused_pg_smem() { return sizeof(PgSmem); }
int fused_pg_cluster() { return kPgCluster; }

cudaError_t launch_fused_pg(const PgArgs& a, bool hamming, int grid, cudaStream_t st) {
    const size_t smem = sizeof(PgSmem);
    grid -= grid % kPgCluster;
    if (grid < kPgCluster) grid = kPgCluster;
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
#if PG_SW
        // software frame-group barriers: every CTA must be co-resident (cooperative launch)
        PgArgs aa = a;
        void* args[] = {&aa};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(256), args, smem, st);
#else
        kern<<<grid, 256, smem, st>>>(a);
        return cudaGetLastError();
#endif
    };
    return hamming ? go(fused_pg1024_kernel<true>) : go(fused_pg1024_kernel<false>);
}

// Co-resident 8-CTA clusters of the kernel (the persistent grid is this many clusters).
int fused_pg_max_clusters() {
    const size_t smem = sizeof(PgSmem);
#if PG_SW
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaFuncSetAttribute(fused_pg1024_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_pg1024_kernel<false>, 256, smem) != cudaSuccess)
        return 0;
    return per_sm * sms / kPgCluster;
#endif
    if (cudaFuncSetAttribute(fused_pg1024_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kPgCluster * 64, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = kPgCluster;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fused_pg1024_kernel<false>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // namespace ofdmr
