// Launch cost of thread-block clusters on B200: an (almost) empty kernel with
// the cluster kernel's launch shape, timed over back-to-back launches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_launch cluster_launch.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_empty(int* out, int sync_cluster) {
    if (sync_cluster) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0 && out) out[blockIdx.x] = blockIdx.x;
}

static float run(int cl, int ctas, int smem, int threads, int sync, int reps, bool graph) {
    cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_empty, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int* out;
    cudaMalloc(&out, ctas * 4);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = cl > 1 ? 1 : 0;
    cudaGraphExec_t ge = nullptr;
    if (graph) {
        cudaGraph_t g;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        cudaLaunchKernelEx(&cfg, k_empty, out, sync);
        cudaError_t e1 = cudaStreamEndCapture(s, &g);
        cudaError_t e2 = e1 == cudaSuccess ? cudaGraphInstantiate(&ge, g, 0) : e1;
        if (e2 != cudaSuccess || !ge) {
            printf("graph capture failed: %s\n", cudaGetErrorString(e2));
            cudaGetLastError();
            return -1.f;
        }
    }
    auto once = [&] {
        if (graph) cudaGraphLaunch(ge, s);
        else cudaLaunchKernelEx(&cfg, k_empty, out, sync);
    };
    for (int i = 0; i < 20; ++i) once();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int i = 0; i < reps; ++i) once();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        exit(1);
    }
    cudaFree(out);
    cudaStreamDestroy(s);
    return ms * 1000.f / reps;
}

int main() {
    struct C { int cl, ctas, smem, threads, sync; const char* name; } cs[] = {
        {1, 128, 0, 256, 0, "no cluster, 128 CTAs, 0 smem"},
        {1, 128, 110 * 1024, 256, 0, "no cluster, 128 CTAs, 110KB smem"},
        {8, 128, 110 * 1024, 256, 1, "cluster 8, 128 CTAs, 110KB, cluster barrier"},
        {16, 128, 110 * 1024, 256, 1, "cluster 16, 128 CTAs, 110KB, cluster barrier"},
        {16, 128, 110 * 1024, 256, 0, "cluster 16, 128 CTAs, 110KB, no barrier"},
        {16, 16, 110 * 1024, 256, 1, "cluster 16, 16 CTAs, 110KB, cluster barrier"},
        {8, 128, 200 * 1024, 512, 1, "cluster 8, 128 CTAs, 200KB, 512 thr"},
    };
    setvbuf(stdout, nullptr, _IONBF, 0);
    for (auto& c : cs) {
        const float a = run(c.cl, c.ctas, c.smem, c.threads, c.sync, 500, false);
        printf("%-50s stream %.2f us", c.name, a);
        const float b = run(c.cl, c.ctas, c.smem, c.threads, c.sync, 500, true);
        printf("   graph %.2f us\n", b);
    }
}
