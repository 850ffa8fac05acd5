// fft_cluster.cu -- single-pass fused reconstruction (IFFT2 + coil combine)
// for square 256x256 images on one 8-CTA thread-block cluster per coil image.
//
// The two-pass chain (fft_kernels.cuh: axis-1 pass to an HBM intermediate,
// then axis-0 pass + combine) moves every coil image through HBM three
// times.  Here a cluster keeps the whole 512 KB coil image on chip, spread
// over its 8 SMs:
//
//   TMA      : CTA r pulls its 32-column tile of Y_c (256 rows x 256 B, one
//              cp.async.bulk.tensor per coil) into shared memory; the next
//              coil's tile is in flight while this one is transformed.
//   phase A  : axis-1 (y) IFFT of the 32 columns (16 threads per column,
//              radix-16 x 16 Stockham, one shared-memory exchange).
//   transpose: every thread stores its 16 results straight into the shared
//              memory of the CTA that owns their rows (st.shared::cluster,
//              256 B per warp store) -- the DSMEM all-to-all replaces the
//              intermediate's HBM round trip; one cluster barrier per coil,
//              receive buffers double-buffered so it is the only one.
//   phase B  : axis-0 (x) IFFT of the CTA's 32 rows (16 threads per row,
//              warp-synchronous), scale 1/(nx*ny) folded into the last-pass
//              twiddles, then conj(S_c) . X_c (or |X_c|^2) accumulated in
//              registers across the coils.
//
// Work split: the W = frames*coils coil images are cut into K contiguous
// ranges, one per resident cluster (persistent grid), so every SM does the
// same amount of work whatever F and C are.  A frame whose coils straddle two
// ranges is finished by whichever piece arrives last (per-CTA arrival
// counter, no spinning): it adds the pieces' partial sums in range order, so
// the result is deterministic for a given K.
//
// Arithmetic per coil image is exactly the two-pass kernels' (same LineFFT
// plan and twiddles, same fused fp32 coil-ordered accumulation),
// so outputs are bit-identical to them except where a frame is split.
// Reference semantics: complex_element_prod.cl.src:9-19 (conj product),
// ximage_sum.cl.src:6-23 (coil sum), rss_combine.cl.src:5-20 (RSS),
// fft_radix2_pass.cl.src:22-69 (the transform it replaces).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "cluster.cuh"
#include "fft_kernels.cuh"

namespace hetreco::dev {

namespace {

using namespace cl;

constexpr int kCN = 256;     // image side
using CL256 = LineFFT<kCN>;  // R = 16 points/thread, T = 16 threads/line

// Geometry for a cluster of CL CTAs (8 = portable, 16 = non-portable; at 16
// a CTA needs half the shared memory, so two clusters' CTAs share an SM and
// one's DSMEM exchange overlaps the other's arithmetic).
template <int CL>
struct Geo {
    static constexpr int TX = kCN / CL;             // phase A: columns per CTA
    static constexpr int RY = kCN / CL;             // phase B: rows per CTA
    static constexpr int threads = TX * CL256::T;   // 512 at CL=8, 256 at CL=16
    static constexpr int LS = line_stride<kCN>();   // padded line stride (float2)
    static constexpr int buf = TX * LS;             // one buffer (float2), >= staging tile
    static constexpr int smem = (3 * buf + 2 * kCN) * 8 + 32;  // tile, 2 receive buffers, tables, barriers
    static constexpr int min_blocks = CL >= 16 ? 2 : 1;
    static_assert(RY * CL256::T == threads, "phase B mapping");
    static_assert(buf >= kCN * TX, "staging tile must fit in a buffer");
    static_assert(RY % CL256::T == 0 || CL256::T % RY == 0, "row blocks");
};

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_load_2d(std::uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            std::uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

struct ClusterArgs {
    const float2* smap;  // S [N, N, C] (Sense)
    void* out;           // M [N, N, F] complex64 (Sense) / float32 (Rss)
    float2* ws;          // split-frame partials [K][2][N*N]
    unsigned* cnt;       // split-frame arrival counters [F][kCL], zero between launches
    const float2* tw;    // W_N^t, t < N, inverse direction
    std::uint32_t coils, frames;
    int shift;
    float scale;
};

template <int MODE, int kCL>
__global__ void __launch_bounds__(Geo<kCL>::threads, Geo<kCL>::min_blocks)
    k_recon_cluster(const __grid_constant__ CUtensorMap ymap, ClusterArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    using L = CL256;
    using G = Geo<kCL>;
    constexpr int kTX = G::TX, kRY = G::RY, kThreads = G::threads, kLS = G::LS, kBuf = G::buf;
    constexpr int N = kCN, R = L::R, T = L::T;
    constexpr bool SENSE = MODE == int(Combine::Sense);
    constexpr std::uint32_t kRecvBytes = std::uint32_t(kRY) * N * 8;
    extern __shared__ __align__(1024) float2 sm[];
    float2* stg = sm;              // TMA tile [N rows][kTX], then the phase-A exchange lines
    float2* recv = sm + kBuf;      // 2 x [kRY lines][kLS]: phase-B input (st.async from all CTAs),
                                   // then the phase-B exchange lines in place
    float2* twA = sm + 3 * kBuf;   // W_N^t
    float2* twB = twA + N;         // scale * W_N^t (last pass of phase B)
    const std::uint32_t bar = smem_u32(twB + N);  // TMA tile landed
    const std::uint32_t rbar0 = bar + 8;          // rbar0 + 8*b: receive buffer b complete
    int* s_flag = reinterpret_cast<int*>(twB + N) + 6;

    const int tid = threadIdx.x;
    const std::uint32_t r = cluster_rank();
    const std::uint64_t k = blockIdx.x / kCL, K = gridDim.x / kCL;
    const std::uint32_t C = a.coils;
    const std::uint64_t W = std::uint64_t(C) * a.frames;
    const std::uint64_t w0 = k * W / K, w1 = (k + 1) * W / K;
    auto cluster_of = [&](std::uint64_t w) { return ((w + 1) * K - 1) / W; };
    auto first_frame = [&](std::uint64_t kk) { return (kk * W / K) / C; };

    for (int t = tid; t < N; t += kThreads) {
        const float2 w = a.tw[t];
        twA[t] = w;
        twB[t] = make_float2(w.x * a.scale, w.y * a.scale);
    }
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(rbar0, 1);
        mbar_init(rbar0 + 8, 1);
    }
    __syncthreads();
    cluster_arrive();  // every CTA of the cluster is running before any DSMEM store
    cluster_wait();

    const bool sh = a.shift;
    // ifftshift along x = load the tile half an image away
    const int xtile = sh ? int((r + kCL / 2) % kCL) : int(r);
    auto issue = [&](std::uint64_t w) {
        mbar_expect_tx(bar, std::uint32_t(kTX * N * 8));
        tma_load_2d(smem_u32(stg), &ymap, xtile * kTX * 2, int(w * N), bar);
    };
    if (tid == 0 && w0 < w1) {
        issue(w0);
        mbar_expect_tx(rbar0, kRecvBytes);
        if (w0 + 1 < w1) mbar_expect_tx(rbar0 + 8, kRecvBytes);
    }

    const int l = tid % kTX, jA = tid / kTX;  // phase A: column l, thread jA of 16
    const int yl = tid / T, jB = tid % T;     // phase B: row yl, thread jB of 16
    float2* lineA = stg + l * kLS;
    const std::uint32_t recv_u32 = smem_u32(recv) + std::uint32_t(L::pad(kTX * int(r) + l)) * 8;
    const std::uint32_t row = kRY * r + yl;  // output row of this thread in phase B
    const std::uint64_t pix = std::uint64_t(row) * N + jB;

    float acc_re[R], acc_im[R];
    sfor<R>([&](auto m) {
        acc_re[m.value] = 0.f;
        acc_im[m.value] = 0.f;
    });

    auto store_final = [&](std::uint32_t f, const float (&re)[R], const float (&im)[R]) {
        if constexpr (SENSE) {
            float2* dst = static_cast<float2*>(a.out) + std::uint64_t(f) * N * N + pix;
            slots<R>(sh, [&](auto m, auto ms) { dst[T * ms.value] = make_float2(re[m.value], im[m.value]); });
        } else {
            float* dst = static_cast<float*>(a.out) + std::uint64_t(f) * N * N + pix;
            slots<R>(sh, [&](auto m, auto ms) { dst[T * ms.value] = float(sqrt(double(re[m.value]))); });
        }
    };

    // frame f's coils end at this thread's current position: write M, or
    // hand in a partial sum if the frame is shared with other clusters
    auto finish_frame = [&](std::uint32_t f) {
        const std::uint64_t fc0 = std::uint64_t(f) * C;
        const std::uint64_t kf = cluster_of(fc0), kl = cluster_of(fc0 + C - 1);
        if (kf == kl) {
            store_final(f, acc_re, acc_im);
            return;
        }
        const std::uint64_t slot = f == first_frame(k) ? 0 : 1;
        float2* mine = a.ws + (k * 2 + slot) * N * N + pix;
        slots<R>(sh, [&](auto m, auto ms) { __stcg(mine + T * ms.value, make_float2(acc_re[m.value], acc_im[m.value])); });
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            unsigned* c = a.cnt + std::uint64_t(f) * kCL + r;
            const unsigned old = atomicAdd(c, 1u);
            const bool last = old == unsigned(kl - kf);
            if (last) *c = 0u;  // ready for the next launch
            *s_flag = last;
        }
        __syncthreads();
        if (*s_flag) {
            __threadfence();
            float re[R], im[R];
            sfor<R>([&](auto m) {
                re[m.value] = 0.f;
                im[m.value] = 0.f;
            });
            for (std::uint64_t kk = kf; kk <= kl; ++kk) {
                const std::uint64_t sl = f == first_frame(kk) ? 0 : 1;
                const float2* p = a.ws + (kk * 2 + sl) * N * N + pix;
                slots<R>(sh, [&](auto m, auto ms) {
                    const float2 v = __ldcg(p + T * ms.value);
                    re[m.value] = __fadd_rn(re[m.value], v.x);
                    im[m.value] = __fadd_rn(im[m.value], v.y);
                });
            }
            store_final(f, re, im);
        }
    };

    // ---- phase A of coil w: axis-1 IFFT of this CTA's columns, then the
    // DSMEM transpose into receive buffer b (row y' -> CTA y'/kRY, line
    // y' mod kRY), counted on that CTA's receive barrier b ----
    std::uint32_t parity = 0;
    auto phase_a = [&](std::uint64_t w, int b) {
        mbar_wait(bar, parity);
        parity ^= 1;
        float2 v[R];
        slots_ld<R>(sh, (long long)(R / 2) * T * kTX,
                    [&](auto m, long long d) { v[m.value] = stg[(jA + T * m.value) * kTX + l + d]; });
        // the first exchange barrier inside run_f also retires every read of the tile
        L::template run_f<+1>(
            v, [&](auto pc, auto sc, auto qc) { return twA[L::template tw_index<pc.value, sc.value, qc.value>(jA)]; },
            lineA, jA, [] { __syncthreads(); }, 1.0f);
        __syncthreads();  // exchange reads done: the tile buffer is free
        if (tid == 0 && w + 1 < w1) {
            fence_proxy_async();
            issue(w + 1);
        }
        const std::uint32_t dst = recv_u32 + std::uint32_t(b * kBuf) * 8;
        const std::uint32_t rb = rbar0 + 8 * b;
        slots<R>(sh, [&](auto m, auto ms) {
            constexpr int y0 = T * ms.value;  // y' = jA + y0, jA < T <= kRY
            constexpr int q = y0 / kRY;       // destination CTA (compile time)
            const int y = jA + y0;
            st_async(mapa(dst + std::uint32_t((y % kRY) * kLS) * 8, q), v[m.value], mapa(rb, q));
        });
    };

    // ---- phase B of coil w: axis-0 IFFT of this CTA's rows + combine ----
    std::uint32_t rpar = 0;  // bit b: phase parity of receive barrier b
    auto phase_b = [&](std::uint64_t w, int b) {
        const std::uint32_t f = std::uint32_t(w / C), c = std::uint32_t(w % C);
        float2 sv[SENSE ? R : 1];
        if constexpr (SENSE) {
            const float2* sp = a.smap + std::uint64_t(c) * N * N + pix;
            slots_ld<R>(sh, (long long)(R / 2) * T, [&](auto m, long long d) { sv[m.value] = __ldg(sp + T * m.value + d); });
        }
        mbar_wait(rbar0 + 8 * b, (rpar >> b) & 1u);
        rpar ^= 1u << b;
        if (tid == 0 && w + 2 < w1) mbar_expect_tx(rbar0 + 8 * b, kRecvBytes);  // coil w+2's phase
        float2* lineB = recv + b * kBuf + yl * kLS;
        float2 v[R];
        sfor<R>([&](auto m) { v[m.value] = lineB[L::pad(jB + T * m.value)]; });
        L::template run_f<+1>(
            v, [&](auto pc, auto sc, auto qc) { return twB[L::template tw_index<pc.value, sc.value, qc.value>(jB)]; },
            lineB, jB, [] { __syncwarp(); }, a.scale);
        // bar.sync performs every access of the CTA to buffer b before the
        // (relaxed) cluster arrive that lets coil w+2's stores into it
        __syncthreads();
        cluster_arrive_relaxed();
        if constexpr (SENSE) {
            sfor<R>([&](auto m) { mac_conj(acc_re[m.value], acc_im[m.value], v[m.value], sv[m.value]); });
        } else {
            sfor<R>([&](auto m) { mac_abs2(acc_re[m.value], v[m.value]); });
        }
        if (c + 1 == C || w + 1 == w1) {
            finish_frame(f);
            sfor<R>([&](auto m) {
                acc_re[m.value] = 0.f;
                acc_im[m.value] = 0.f;
            });
        }
    };

    // Two-stage software pipeline: iteration i transposes coil i into buffer
    // i%2 and finishes coil i-1 from the other buffer, so a CTA only waits
    // for data its peers sent one iteration earlier.  Cluster barrier: arrive
    // after each phase B, wait before each reuse of a buffer (i >= 2) --
    // strictly alternating per thread.
    const std::uint64_t n = w1 - w0;
    for (std::uint64_t i = 0; i <= n; ++i) {
        if (i >= 2) cluster_wait();  // coil i-2's buffer has been consumed by every CTA
        if (i < n) phase_a(w0 + i, int(i & 1));
        if (i >= 1) phase_b(w0 + i - 1, int((i - 1) & 1));
    }
    if (n >= 1) cluster_wait();  // pairs the last arrive
}

template <int MODE, int CL>
cudaLaunchConfig_t cluster_config(int clusters, cudaLaunchAttribute* at) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CL * clusters);
    cfg.blockDim = dim3(Geo<CL>::threads);
    cfg.dynamicSmemBytes = Geo<CL>::smem;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    at[1].val.clusterSchedulingPolicyPreference =
        std::getenv("HETRECO_CLUSTER_SPREAD") ? cudaClusterSchedulingPolicySpread
                                              : cudaClusterSchedulingPolicyLoadBalancing;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cfg;
}

// Resident clusters of size CL (0 when the configuration cannot launch).
// Also sets the kernel's shared-memory / cluster-size attributes.
template <int MODE, int CL>
int cluster_capacity() {
    static int cap = -1;
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (cap >= 0) return cap;
    auto kern = k_recon_cluster<MODE, CL>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<CL>::smem);
    if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchAttribute at[2];
    cudaLaunchConfig_t cfg = cluster_config<MODE, CL>(32, at);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cap = n;
    return cap;
}

template <int MODE>
int capacity_of(int cl) {
    return cl == 16 ? cluster_capacity<MODE, 16>() : cluster_capacity<MODE, 8>();
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q{};
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    });
    return fn;
}

}  // namespace

bool cluster_supported(std::uint64_t nx, std::uint64_t ny, Combine mode) {
    return nx == kCN && ny == kCN && (mode == Combine::Sense || mode == Combine::Rss);
}

int cluster_smem_bytes(int cl) { return cl == 16 ? Geo<16>::smem : Geo<8>::smem; }

ClusterPlan plan_cluster(Combine mode, std::uint64_t coils, std::uint64_t frames, int max_clusters, int cluster_size) {
    ClusterPlan p;
    if (cluster_size == 0) {
        if (const char* v = std::getenv("HETRECO_CLUSTER_SIZE")) cluster_size = std::atoi(v);
    }
    auto cap_of = [&](int cl) {
        return mode == Combine::Sense ? capacity_of<int(Combine::Sense)>(cl) : capacity_of<int(Combine::Rss)>(cl);
    };
    int cl = cluster_size;
    if (cl == 0) cl = cap_of(16) > 0 ? 16 : 8;  // default: two CTAs per SM
    if (cl != 8 && cl != 16) return p;
    const int cap = cap_of(cl);
    const std::uint64_t W = coils * frames;
    std::uint64_t k = cap;
    if (max_clusters > 0) k = std::min<std::uint64_t>(k, std::uint64_t(max_clusters));
    k = std::min<std::uint64_t>(k, W);
    p.cl = cl;
    p.clusters = int(k);
    p.ws_bytes = std::uint64_t(k) * 2 * kCN * kCN * 8;
    p.cnt_bytes = frames * cl * 4;
    if (std::getenv("HETRECO_DEBUG"))
        std::fprintf(stderr, "plan_cluster: %d-CTA clusters, capacity %d, launching %d for %llu coil images\n", cl, cap,
                     p.clusters, static_cast<unsigned long long>(W));
    return p;
}

cudaError_t make_cluster_map(ClusterMap& m, const float2* y, std::uint64_t rows, int cl) {
    auto enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    if (cl != 8 && cl != 16) return cudaErrorInvalidValue;
    static_assert(sizeof(CUtensorMap) == sizeof(m.bytes), "tensor map size");
    cuuint64_t dims[2] = {cuuint64_t(2 * kCN), cuuint64_t(rows)};  // float32 elements
    cuuint64_t strides[1] = {cuuint64_t(kCN) * 8};
    cuuint32_t box[2] = {cuuint32_t(2 * (kCN / cl)), cuuint32_t(kCN)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap*>(m.bytes), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                     const_cast<float2*>(y), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

namespace {
template <int MODE, int CL>
cudaError_t launch_as(const CUtensorMap& map, const ClusterArgs& ka, int clusters, cudaStream_t st) {
    cluster_capacity<MODE, CL>();  // sets the kernel attributes once
    cudaLaunchAttribute at[2];
    cudaLaunchConfig_t cfg = cluster_config<MODE, CL>(clusters, at);
    cfg.stream = st;
    return cudaLaunchKernelEx(&cfg, k_recon_cluster<MODE, CL>, map, ka);
}
}  // namespace

cudaError_t launch_cluster(Combine mode, const ClusterMap& m, const ClusterLaunch& a, const ClusterPlan& p,
                           cudaStream_t st) {
    if (p.clusters <= 0) return cudaErrorInvalidConfiguration;
    ClusterArgs ka{a.smap, a.out, a.ws, a.cnt, a.tw, std::uint32_t(a.coils), std::uint32_t(a.frames), a.shift,
                   a.scale};
    const CUtensorMap& map = *reinterpret_cast<const CUtensorMap*>(m.bytes);
    const bool sense = mode == Combine::Sense;
    if (p.cl == 16)
        return sense ? launch_as<int(Combine::Sense), 16>(map, ka, p.clusters, st)
                     : launch_as<int(Combine::Rss), 16>(map, ka, p.clusters, st);
    return sense ? launch_as<int(Combine::Sense), 8>(map, ka, p.clusters, st)
                 : launch_as<int(Combine::Rss), 8>(map, ka, p.clusters, st);
}

}  // namespace hetreco::dev
