// Pinned H2D bandwidth with 1..4 concurrent streams (copy engines), and H2D
// concurrent with D2H.  nvcc -O2 -o h2d_engines h2d_engines.cu
#include <cstdio>
#include <cuda_runtime.h>

int main() {
    const size_t N = size_t(512) << 20;
    char *h, *h2, *d, *d2;
    cudaHostAlloc(&h, N, cudaHostAllocDefault);
    cudaHostAlloc(&h2, N / 32, cudaHostAllocDefault);
    cudaMalloc(&d, N);
    cudaMalloc(&d2, N / 32);
    cudaStream_t s[4];
    for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int k : {1, 2, 4}) {
        for (int chunk_mb : {16, 64}) {
            const size_t chunk = size_t(chunk_mb) << 20;
            float best = 1e9f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaDeviceSynchronize();
                cudaEventRecord(a, s[0]);
                for (int i = 1; i < k; ++i) cudaStreamWaitEvent(s[i], a, 0);
                size_t off = 0;
                for (int c = 0; off < N; ++c, off += chunk)
                    cudaMemcpyAsync(d + off, h + off, chunk, cudaMemcpyHostToDevice, s[c % k]);
                for (int i = 1; i < k; ++i) {
                    cudaEvent_t e;
                    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
                    cudaEventRecord(e, s[i]);
                    cudaStreamWaitEvent(s[0], e, 0);
                    cudaEventDestroy(e);
                }
                cudaEventRecord(b, s[0]);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("H2D %d stream(s), %3d MB chunks: %.1f GB/s\n", k, chunk_mb, N / best / 1e6);
        }
    }
    // H2D with a concurrent small D2H stream (as in the recon pipeline)
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaDeviceSynchronize();
        cudaEventRecord(a, s[0]);
        cudaStreamWaitEvent(s[1], a, 0);
        cudaMemcpyAsync(d, h, N, cudaMemcpyHostToDevice, s[0]);
        cudaMemcpyAsync(h2, d2, N / 32, cudaMemcpyDeviceToHost, s[1]);
        cudaEvent_t e;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        cudaEventRecord(e, s[1]);
        cudaStreamWaitEvent(s[0], e, 0);
        cudaEventRecord(b, s[0]);
        cudaEventSynchronize(b);
        cudaEventDestroy(e);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    printf("H2D 512 MB + D2H 16 MB concurrently: %.1f GB/s H2D\n", N / best / 1e6);
    int ce = 0;
    cudaDeviceGetAttribute(&ce, cudaDevAttrAsyncEngineCount, 0);
    printf("async engines: %d\n", ce);
    return 0;
}
