// Probe: how many thread-block clusters of size C (one CTA per SM, ~216 KB shared memory)
// can be co-resident on this GPU (cudaOccupancyMaxActiveClusters), and the DSMEM remote-store
// bandwidth of a 16-CTA cluster (each CTA writes 128 KiB into the other CTAs' shared memory).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void dummy(int* out) {
    extern __shared__ int s[];
    s[threadIdx.x] = threadIdx.x;
    if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

__global__ void __cluster_dims__(16, 1, 1) dsmem_bw(float4* out, int reps) {
    extern __shared__ float4 sm[];  // 128 KiB slice
    cg::cluster_group cl = cg::this_cluster();
    const unsigned r = cl.block_rank();
    float4 v = make_float4(r, threadIdx.x, 0, 0);
    for (int it = 0; it < reps; ++it) {
        cl.sync();
        // each CTA writes 8 KiB into each of the 16 slices (incl. its own) = 128 KiB out
        for (int q = 0; q < 16; ++q) {
            float4* dst = cl.map_shared_rank(sm, (r + q) & 15);
            for (int i = threadIdx.x; i < 512; i += blockDim.x) dst[r * 512 + i] = v;
        }
    }
    cl.sync();
    if (threadIdx.x == 0) out[blockIdx.x] = sm[threadIdx.x];
}

int main() {
    int dev = 0, sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = 216 * 1024;
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {1, 2, 4, 8, 12, 16}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(c * 16);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d SMs (%s)\n", c, n, n * c, cudaGetErrorString(e));
    }
    // DSMEM bandwidth
    cudaFuncSetAttribute(dsmem_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    cudaFuncSetAttribute(dsmem_bw, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    float4* out;
    cudaMalloc(&out, 1 << 20);
    for (int nc : {1, 8}) {
        const int reps = 2000;
        dsmem_bw<<<16 * nc, 512, 128 * 1024>>>(out, 10);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        dsmem_bw<<<16 * nc, 512, 128 * 1024>>>(out, reps);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = 16.0 * nc * reps * 128 * 1024;
        printf("dsmem %d clusters: %.3f ms, %.1f GB/s total, %.1f GB/s per SM out, %.2f us per 128 KiB round (%s)\n", nc, ms,
               bytes / ms / 1e6, bytes / ms / 1e6 / (16 * nc), ms * 1e3 / reps, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
