// probes.cu -- micro-benchmarks that decide the fused-kernel design
// (round-2 planning): DSMEM (distributed shared memory) bandwidth inside a
// thread-block cluster, and whether an intermediate written by one kernel is
// re-read from L2 by the next.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 scripts/probes.cu -o build/probes
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                               \
        }                                                                           \
    } while (0)

constexpr int kSmemFloats = 64 * 1024 / 4;  // 64 KB per CTA

// Each CTA reads `iters` x 64 KB of another CTA's shared memory (rank + dist).
__global__ void dsmem_read(float* out, int iters, int dist) {
    extern __shared__ float4 sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int n4 = kSmemFloats / 4;
    for (int i = threadIdx.x; i < n4; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
    cl.sync();
    const unsigned peer = (cl.block_rank() + dist) % cl.num_blocks();
    const float4* remote = cl.map_shared_rank(sm, peer);
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int i = threadIdx.x; i < n4; i += blockDim.x) {
            const float4 v = remote[(i + it * 64) & (n4 - 1)];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
    }
    cl.sync();
    if (acc.x == -1.f) out[0] = acc.y + acc.z + acc.w;
}

__global__ void stream_write(float4* dst, const float4* src, size_t n4, int read_src) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) {
        float4 v = read_src ? __ldcs(src + i) : make_float4(i, 0, 0, 0);
        dst[i] = v;
    }
}

__global__ void stream_read(const float4* src, size_t n4, float* out) {
    float s = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x)
        s += __ldcs(src + i).x;
    if (s == -1.f) out[0] = s;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float* out;
    CK(cudaMalloc(&out, 4));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaFuncSetAttribute(dsmem_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    CK(cudaFuncSetAttribute(dsmem_read, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int cs : {2, 4, 8}) {
        for (int dist : {0, 1}) {
            cudaLaunchConfig_t cfg{};
            const int clusters = sms / cs;
            cfg.gridDim = dim3(clusters * cs);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = 64 * 1024;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            const int iters = 200;
            CK(cudaLaunchKernelEx(&cfg, dsmem_read, out, 10, dist));
            CK(cudaEventRecord(a));
            CK(cudaLaunchKernelEx(&cfg, dsmem_read, out, iters, dist));
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            const double bytes = double(clusters * cs) * iters * 64.0 * 1024;
            std::printf("dsmem cluster=%d dist=%d (%s): %.1f GB/s aggregate over %d CTAs = %.1f GB/s per SM "
                        "(%.1f B/clk at 1.965 GHz)\n",
                        cs, dist, dist ? "remote" : "local", bytes / ms / 1e6, clusters * cs,
                        bytes / ms / 1e6 / (clusters * cs), bytes / ms / 1e6 / (clusters * cs) / 1.965);
        }
    }
    // L2 round trip: kernel A writes an intermediate (optionally while
    // streaming a same-size input), kernel B reads it back.
    for (size_t mb : {16, 32, 48, 64, 96, 256}) {
        const size_t bytes = mb << 20, n4 = bytes / 16;
        float4 *x, *y;
        CK(cudaMalloc(&x, bytes));
        CK(cudaMalloc(&y, bytes));
        CK(cudaMemset(y, 0, bytes));
        for (int with_input : {0, 1}) {
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                stream_write<<<sms * 4, 512>>>(x, y, n4, with_input);
                CK(cudaEventRecord(a));
                stream_read<<<sms * 4, 512>>>(x, n4, out);
                CK(cudaEventRecord(b));
                CK(cudaEventSynchronize(b));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, a, b));
                best = ms < best ? ms : best;
            }
            std::printf("L2 round trip %4zu MB (writer %s): re-read at %.0f GB/s\n", mb,
                        with_input ? "also streams an input" : "write only", bytes / best / 1e6);
        }
        cudaFree(x);
        cudaFree(y);
    }
    int persist = 0;
    cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, 0);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    std::printf("L2 size %d MB, max persisting %d MB\n", l2 >> 20, persist >> 20);
    return 0;
}
