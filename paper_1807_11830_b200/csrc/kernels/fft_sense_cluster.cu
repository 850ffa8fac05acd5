// fft_sense_cluster.cu -- the front half of the SENSE normal operator E^H E
// at 256 x 256 as ONE thread-block-cluster kernel:
//
//   z[:, :, c, f] = F_y^-1 P F_y F_x ( S[:, :, c] . M[:, :, f] )
//
// which the default graph runs as two kernels with a global round trip in
// between (fft_sense_model.cu: k_fft_expand, then k_fft_strided_masked in
// roundtrip mode).  Here a 16-CTA cluster owns one coil image (512 KB, spread
// over its 16 SMs):
//
//   phase 1 : CTA r expands and x-transforms rows 16r .. 16r+15 (16 threads
//             per row, the expand kernel's arithmetic and rounding);
//   transpose: every thread st.async's its 16 results straight into the
//             shared memory of the CTA that owns their columns (x' / 16),
//             completing on that CTA's mbarrier -- the DSMEM all-to-all
//             replaces the HBM/L2 round trip of the intermediate;
//   phase 2 : CTA q y-transforms columns 16q .. 16q+15, applies the sampling
//             mask, inverse-transforms in registers (the roundtrip kernel's
//             arithmetic) and stores z.
//
// The coil-parallel x-IFFT + conj(S) combine (fft_combine_cp.cu) then runs
// as before, so E^H E keeps its coil-ordered deterministic sum.  Per-line
// arithmetic (LineFFT plan, twiddles, slot order, cmul rounding) is exactly
// that of the two kernels it replaces: z, and the final image, are
// bit-identical.  Clusters loop over coil images w = k, k + K, ... (K
// resident clusters); a cluster barrier per image keeps the receive buffer
// single.
//
// Reference semantics: complex_element_prod.cl.src:9-19 (S . m, kernel_abi.h
// :123-125 rounding) and fft_radix2_pass.cl.src:22-69 (the transforms).
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "cluster.cuh"
#include "fft_kernels.cuh"

namespace hetreco::dev {

namespace {

using namespace cl;

constexpr int kN = 256;
constexpr int kCL = 16;            // CTAs per cluster (non-portable size)
constexpr int kRows = kN / kCL;    // rows (phase 1) / columns (phase 2) per CTA
using LS = LineFFT<kN>;            // R = 16 samples per thread, T = 16 threads per line
constexpr int kThreads = kRows * LS::T;
constexpr int kBuf = kN * kRows;   // phase-2 tile [256 rows][16 columns] (float2)
constexpr int kLS = line_stride<kN>();
constexpr int kLinesLen = kRows * (kLS > row_stride<kN>() ? kLS : row_stride<kN>());
constexpr int kSmem = (kBuf + kLinesLen) * 8 + 16;
constexpr std::uint32_t kRecvBytes = std::uint32_t(kBuf) * 8;
static_assert(kThreads == 256 && LS::R == 16 && LS::T == 16, "plan of the 256-point lines");

__device__ __forceinline__ float2 cmul_ref(float2 a, float2 b) {
    return make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                       __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
}

__global__ void __launch_bounds__(kThreads, 1) k_sense_normal_front(SenseFrontArgs a) {
    pdl_launch_dependents();
    constexpr int R = LS::R, T = LS::T;
    extern __shared__ __align__(16) float2 sm[];
    float2* buf = sm;          // [256 rows][16 columns]: this CTA's columns, all rows
    float2* lines = sm + kBuf;  // exchange lines of both phases
    const std::uint32_t rbar = smem_u32(lines + kLinesLen);
    const int tid = threadIdx.x;
    const std::uint32_t r = cluster_rank();
    const std::uint32_t k = blockIdx.x / kCL, K = gridDim.x / kCL;
    const std::uint32_t C = a.coils, W = a.coils * a.frames;
    const bool sh = a.shift;

    // phase 1: lines-major (row l1 of the CTA's 16, thread j1 of 16)
    const int l1 = tid / T, j1 = tid % T;
    float2* line1 = lines + l1 * row_stride<kN>();
    // phase 2: column tile (column l2 of 16, thread j2 of 16), as k_fft_strided_masked
    const int l2 = tid % kRows, j2 = tid / kRows;
    float2* line2 = lines + l2 * kLS;
    typename LS::Twiddles tw1, tw2;  // forward W_256^t, scale 1
    LS::load_twiddles(tw1, a.tw, j1, 1.0f);
    LS::load_twiddles(tw2, a.tw, j2, 1.0f);
    const std::uint32_t col = r * kRows + std::uint32_t(l2);
    if (tid == 0) mbar_init(rbar, 1);
    __syncthreads();  // the initialised barrier is visible to every thread before first use
    if (tid == 0) mbar_expect_tx(rbar, kRecvBytes);
    cluster_arrive();  // every CTA's barrier is armed before any DSMEM store
    cluster_wait();
    pdl_wait();  // inputs may come from the previous kernel
    float mk[R];  // mask of this thread's column samples (displayed k-space positions)
    sfor<R>([&](auto m) { mk[m.value] = 1.0f; });
    if (a.mask) slots<R>(sh, [&](auto m, auto ms) { mk[m.value] = __ldg(a.mask + col + (j2 + T * ms.value) * kN); });

    const std::uint32_t buf_u32 = smem_u32(buf);
    std::uint32_t parity = 0;
    for (std::uint32_t w = k; w < W; w += K) {
        if (w != k) cluster_wait();  // every CTA has read the previous image out of its tile
        const std::uint32_t c = w % C, f = w / C;
        // ---- phase 1: expand + x-FFT of row y, then scatter by column block ----
        {
            const std::uint32_t y = r * kRows + std::uint32_t(l1);
            const float2* mrow = a.m + (std::uint64_t(f) * kN + y) * kN + j1;
            const float2* srow = a.smap + (std::uint64_t(c) * kN + y) * kN + j1;
            float2 v[R];
            slots_ld<R>(sh, (long long)(R / 2) * T, [&](auto m, long long d) {
                v[m.value] = cmul_ref(__ldg(srow + T * m.value + d), __ldg(mrow + T * m.value + d));
            });
            LS::template run<-1>(v, tw1, line1, j1, [] { line_sync<T>(); }, 1.0f);
            // x' = j1 + 16 ms -> CTA ms, tile column j1, row y
            const std::uint32_t off = (y * kRows + std::uint32_t(j1)) * 8u;
            slots<R>(sh, [&](auto m, auto ms) {
                st_async(mapa(buf_u32 + off, std::uint32_t(ms.value)), v[m.value], mapa(rbar, std::uint32_t(ms.value)));
            });
        }
        mbar_wait(rbar, parity);
        parity ^= 1u;
        // ---- phase 2: y-FFT, mask, y-IFFT of this CTA's 16 columns ----
        float2 v[R];
        slots_ld<R>(sh, (long long)(R / 2) * T * kRows,
                    [&](auto m, long long d) { v[m.value] = buf[(j2 + T * m.value) * kRows + l2 + d]; });
        __syncthreads();  // tile reads done (the exchanges below reuse `lines`, not `buf`)
        if (tid == 0 && w + K < W) mbar_expect_tx(rbar, kRecvBytes);  // arm for the next image
        cluster_arrive_relaxed();  // this CTA's tile may be refilled
        LS::template run<-1>(v, tw2, line2, j2, [] { __syncthreads(); });
        slots<R>(sh, [&](auto m, auto ms) { v[m.value] = make_float2(v[m.value].x * mk[m.value], -v[m.value].y * mk[m.value]); });
        LS::template run<-1>(v, tw2, line2, j2, [] { __syncthreads(); });
        float2* dst = a.out + std::uint64_t(c + C * f) * kN * kN + col + std::uint32_t(j2) * kN;
        slots<R>(sh, [&](auto m, auto ms) {
            dst[ms.value * T * kN] = make_float2(v[m.value].x * a.scale, -v[m.value].y * a.scale);
        });
        __syncthreads();  // phase-2 exchanges done before the next image's phase 1 reuses `lines`
    }
    if (k < W) cluster_wait();  // pairs the last arrive
}

cudaLaunchConfig_t front_config(int clusters, cudaLaunchAttribute* at) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(kCL * clusters));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
}

int front_capacity() {
    static int cap = -1;
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (cap >= 0) return cap;
    cudaFuncSetAttribute(k_sense_normal_front, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(k_sense_normal_front, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = front_config(16, at);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_sense_normal_front, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cap = n;
    return cap;
}

}  // namespace

int plan_sense_front(std::uint64_t nx, std::uint64_t ny, std::uint64_t coil_images) {
    if (nx != std::uint64_t(kN) || ny != std::uint64_t(kN) || coil_images == 0) return 0;
    // opt-in: measured slower than the two-kernel front on B200 (16.6 vs 12.7 us
    // per C4 launch: only 7 16-CTA clusters fit, so 8 coil images take two
    // rounds, and one image is ~5 us of dependent latency per cluster;
    // profiles/round2_c4.md)
    const char* e = std::getenv("HETRECO_NORMAL_CLUSTER");
    if (!(e && *e == '1')) return 0;
    const int cap = front_capacity();
    if (std::getenv("HETRECO_DEBUG"))
        std::fprintf(stderr, "plan_sense_front: capacity %d clusters of %d\n", cap, kCL);
    return int(std::min<std::uint64_t>(std::uint64_t(cap), coil_images));
}

cudaError_t launch_sense_front(const SenseFrontArgs& a, int clusters, cudaStream_t st) {
    if (clusters <= 0) return cudaErrorInvalidConfiguration;
    front_capacity();  // kernel attributes
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = front_config(clusters, at);
    cfg.stream = st;
    return cudaLaunchKernelEx(&cfg, k_sense_normal_front, a);
}

}  // namespace hetreco::dev
