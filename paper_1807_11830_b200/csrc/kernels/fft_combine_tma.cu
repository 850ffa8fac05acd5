// fft_combine_tma.cu -- axis-0 IFFT + coil combine fed by a TMA bulk-copy ring
// (opt-in: HETRECO_COMBINE_TMA=1).
//
// Hypothesis tested: the register-prefetch combine (fft_kernels.cuh
// k_fft_combine) keeps one coil ahead in registers, ~16 KB in flight per SM,
// and might be short of memory parallelism.  Result (profiles/round1_combine.md):
// it is not -- that kernel is issue-bound (62 % issue-active, 'selected' the
// top stall, 37.5 warp instructions per sample), and this ring version is
// slower (165 vs 130 us at C3, K=2; more stages cost CTAs per SM and get
// slower still) because the coil's map row is no longer a coil ahead and the
// per-coil CTA barrier adds stalls.  Kept, tested, as the measured
// alternative.
//
// Here a CTA owns LPB consecutive rows (y0..y0+LPB-1) of one frame, and the
// rows of one coil are one contiguous LPB*N*8-byte tile of X.  Thread 0 keeps
// K tiles in flight with cp.async.bulk (global -> shared, mbarrier
// complete_tx), so bytes in flight scale with shared memory instead of
// registers; the CTA walks (row group, coil) pairs as one stream, so the ring
// stays full across row groups.  Per coil: wait the tile, copy it to
// registers, release the slot (one bar.sync, then the refill is issued), load
// the coil's map row (L2), transform, accumulate in fp32 (fused products).
//
// Same semantics as k_fft_combine (complex_element_prod.cl.src:9-19,
// ximage_sum.cl.src:6-23, rss_combine.cl.src:5-20); fp32 accumulation only.
#include "fft_kernels.cuh"

namespace hetreco::dev {

namespace {

__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(std::uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_expect(std::uint32_t bar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(std::uint32_t bar, std::uint32_t parity) {
    std::uint32_t ok;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(std::uint32_t dst, const void* src, std::uint32_t bytes, std::uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

template <int N>
constexpr int tma_rows() {  // rows per CTA: a ~16 KB tile
    return (16384 / (N * 8)) >= 1 ? ((16384 / (N * 8)) > 32 ? 32 : 16384 / (N * 8)) : 1;
}

template <int N, int MODE, int LPB, int K>
__global__ void __launch_bounds__(LPB * LineFFT<N>::T)
    k_fft_combine_tma(ContigArgs a, std::uint32_t groups_per_frame, std::uint32_t groups) {
    pdl_launch_dependents();
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T;
    constexpr bool SENSE = MODE == int(Combine::Sense);
    constexpr int TILE = LPB * N;  // float2 per ring slot
    extern __shared__ __align__(128) float2 sm[];
    float2* ring = sm;                              // K x [LPB rows][N]
    float2* xch = sm + K * TILE;                    // LPB exchange lines
    const std::uint32_t bars = smem_addr(xch + LPB * row_stride<N>());
    const int tid = threadIdx.x;
    const int j = tid % T, l = tid / T;
    float2* line = xch + l * row_stride<N>();
    typename L::Twiddles tw;
    L::load_twiddles(tw, a.tw, j, a.scale);
    pdl_wait();  // twiddle tables are init-time constants
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    const std::uint32_t C = std::uint32_t(a.coils), ny = std::uint32_t(a.ny);
    const std::uint64_t coil_elems = std::uint64_t(ny) * N;

    // stream element t -> (row group, coil); false past the CTA's last group
    auto locate = [&](std::uint32_t t, std::uint32_t& g, std::uint32_t& c) {
        g = blockIdx.x + (t / C) * gridDim.x;
        c = t % C;
        return g < groups;
    };
    auto rows_of = [&](std::uint32_t g, std::uint32_t& f, std::uint32_t& y0) {
        f = g / groups_per_frame;
        y0 = (g - f * groups_per_frame) * LPB;
        return std::min<std::uint32_t>(LPB, ny - y0);
    };
    auto issue = [&](std::uint32_t t) {
        std::uint32_t g, c, f, y0;
        if (!locate(t, g, c)) return;
        const std::uint32_t rows = rows_of(g, f, y0);
        const std::uint32_t bytes = rows * N * 8;
        const std::uint32_t bar = bars + 8 * (t % K);
        bar_expect(bar, bytes);
        bulk_g2s(smem_addr(ring + (t % K) * TILE), a.in + (std::uint64_t(f) * C + c) * coil_elems + std::uint64_t(y0) * N,
                 bytes, bar);
    };
    if (tid == 0) {
        for (int k = 0; k < K; ++k) bar_init(bars + 8 * k);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int k = 0; k < K; ++k) issue(std::uint32_t(k));

    float acc_re[R], acc_im[R];
    std::uint32_t f = 0, y0 = 0, rows = 0;
    for (std::uint32_t t = 0;; ++t) {
        std::uint32_t g, c;
        if (!locate(t, g, c)) break;
        if (c == 0) {
            rows = rows_of(g, f, y0);
            sfor<R>([&](auto m) {
                acc_re[m.value] = 0.f;
                acc_im[m.value] = 0.f;
            });
        }
        const bool active = std::uint32_t(l) < rows;
        const std::uint32_t y = active ? y0 + l : y0;
        // the map row of this coil (L2-resident across frames), in flight during the wait + FFT
        float2 sv[SENSE ? R : 1];
        if constexpr (SENSE) {
            const float2* sp = a.smap + (std::uint64_t(c) * ny + y) * N + j;
            slots_ld<R>(sh_out, (long long)(R / 2) * T, [&](auto m, long long d) { sv[m.value] = __ldg(sp + T * m.value + d); });
        }
        const int slot = int(t % K);
        bar_wait(bars + 8 * slot, (t / K) & 1u);
        float2 v[R];
        const float2* src = ring + slot * TILE + (active ? l : 0) * N + j;
        slots_ld<R>(sh_in, (long long)(R / 2) * T, [&](auto m, long long d) { v[m.value] = src[T * m.value + d]; });
        __syncthreads();  // every thread holds its row: the slot can be refilled
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(t + K);
        }
        L::template run<+1>(v, tw, line, j, [] { line_sync<T>(); }, a.scale);
        if constexpr (SENSE) {
            sfor<R>([&](auto m) { mac_conj(acc_re[m.value], acc_im[m.value], v[m.value], sv[m.value]); });
        } else {
            sfor<R>([&](auto m) { mac_abs2(acc_re[m.value], v[m.value]); });
        }
        if (c + 1 == C && active) {
            if constexpr (SENSE) {
                float2* dst = static_cast<float2*>(a.out) + (std::uint64_t(f) * ny + y) * N + j;
                slots<R>(sh_out, [&](auto m, auto ms) { dst[T * ms.value] = make_float2(acc_re[m.value], acc_im[m.value]); });
            } else {
                float* dst = static_cast<float*>(a.out) + (std::uint64_t(f) * ny + y) * N + j;
                slots<R>(sh_out, [&](auto m, auto ms) { dst[T * ms.value] = float(sqrt(double(acc_re[m.value]))); });
            }
        }
    }
}

template <int N, int MODE, int LPB, int K>
constexpr int tma_smem() {
    return (K * LPB * N + LPB * row_stride<N>()) * 8 + K * 8;
}

template <int N, int MODE, int K>
int tma_occupancy(int sms_unused) {
    constexpr int LPB = tma_rows<N>();
    auto kern = k_fft_combine_tma<N, MODE, LPB, K>;
    (void)sms_unused;
    return blocks_per_sm(kern, LPB * LineFFT<N>::T, tma_smem<N, MODE, LPB, K>());
}

template <int N, int MODE>
cudaError_t tma_go(int stages, const ContigArgs& a, const LaunchShape& s, std::uint32_t gpf, std::uint32_t groups,
                   cudaStream_t st) {
    constexpr int LPB = tma_rows<N>();
    switch (stages) {
#define S(k)                                                                                            \
    case k:                                                                                             \
        tma_occupancy<N, MODE, k>(0);                                                                   \
        k_fft_combine_tma<N, MODE, LPB, k><<<s.grid, s.block, s.smem, st>>>(a, gpf, groups);             \
        break;
        S(2) S(3) S(4) S(6)
#undef S
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

int tma_stages() {
    const int k = env_int("HETRECO_TMA_STAGES", 4);
    return (k == 2 || k == 3 || k == 4 || k == 6) ? k : 4;
}

}  // namespace

bool combine_tma_supported(std::uint64_t N) {
    switch (N) {
#define X(n) \
    case n: return n >= 16;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return false;
}

LaunchShape plan_combine_tma(std::uint64_t N, Combine mode, std::uint64_t ny, std::uint64_t frames, int sms) {
    LaunchShape s;
    if (!combine_tma_supported(N) || mode == Combine::None) return s;
    const int K = tma_stages();
    int occ = 1;
    switch (N) {
#define X(n)                                                                                                    \
    case n:                                                                                                     \
        if constexpr (n >= 16) {                                                                                \
            constexpr int LPB = tma_rows<n>();                                                                  \
            s.rq = LineFFT<n>::R;                                                                               \
            s.block = LPB * LineFFT<n>::T;                                                                      \
            switch (K) {                                                                                        \
                case 2: s.smem = tma_smem<n, 1, LPB, 2>(); break;                                               \
                case 3: s.smem = tma_smem<n, 1, LPB, 3>(); break;                                               \
                case 6: s.smem = tma_smem<n, 1, LPB, 6>(); break;                                               \
                default: s.smem = tma_smem<n, 1, LPB, 4>(); break;                                              \
            }                                                                                                   \
            const std::uint64_t gpf = (ny + LPB - 1) / LPB;                                                     \
            const std::uint64_t groups = gpf * frames;                                                          \
            if (mode == Combine::Sense)                                                                         \
                occ = K == 2 ? tma_occupancy<n, 1, 2>(0) : K == 3 ? tma_occupancy<n, 1, 3>(0)                   \
                    : K == 6 ? tma_occupancy<n, 1, 6>(0) : tma_occupancy<n, 1, 4>(0);                           \
            else                                                                                                \
                occ = K == 2 ? tma_occupancy<n, 2, 2>(0) : K == 3 ? tma_occupancy<n, 2, 3>(0)                   \
                    : K == 6 ? tma_occupancy<n, 2, 6>(0) : tma_occupancy<n, 2, 4>(0);                           \
            s.grid = int(std::min<std::uint64_t>(groups, std::uint64_t(sms) * occ));                            \
            s.variant = 64 | K;                                                                                 \
        }                                                                                                       \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    if (s.grid < 1) s.grid = 1;
    return s;
}

cudaError_t launch_combine_tma(std::uint64_t N, Combine mode, const ContigArgs& a, const LaunchShape& s,
                               cudaStream_t st) {
    if (s.block == 0 || !(s.variant & 64)) return cudaErrorInvalidValue;
    const int K = s.variant & 63;
    switch (N) {
#define X(n)                                                                                     \
    case n:                                                                                      \
        if constexpr (n >= 16) {                                                                 \
            constexpr int LPB = tma_rows<n>();                                                   \
            const std::uint64_t gpf = (a.ny + LPB - 1) / LPB;                                    \
            const std::uint64_t groups = gpf * a.frames;                                         \
            if (groups >= (std::uint64_t(1) << 32)) return cudaErrorInvalidValue;                \
            return mode == Combine::Sense                                                        \
                       ? tma_go<n, 1>(K, a, s, std::uint32_t(gpf), std::uint32_t(groups), st)    \
                       : tma_go<n, 2>(K, a, s, std::uint32_t(gpf), std::uint32_t(groups), st);   \
        }                                                                                        \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

}  // namespace hetreco::dev
