// fft_combine_cp.cu -- coil-parallel axis-0 IFFT + combine for small problems.
//
// The coil-serial combine (k_fft_combine) gives each output line (y, f) to T
// threads that walk all C coils in turn: at one or a few frames (the paper's
// single-frame 8-coil case C2, the iterative normal operator C4) that is only
// ny*F*T threads -- 4096 at 256^2 x 1 frame, a fraction of one wave -- and the
// C coil transforms run back to back on each of them.  Here a CTA owns one
// output line and G coil groups of T threads; group g transforms coils g,
// g+G, ... in parallel, keeps fp32 partial sums in registers, and the CTA adds
// the G partials in group order through shared memory (deterministic).  Same
// semantics as k_fft_combine's fp32 variant (complex_element_prod.cl.src:9-19,
// ximage_sum.cl.src:6-23, rss_combine.cl.src:5-20), different fp32 summation
// order (within the 1e-5 tolerance).
#include <cstdlib>

#include "fft_kernels.cuh"

namespace hetreco::dev {

namespace {

template <int T>
__device__ __forceinline__ unsigned group_mask(int tid) {
    if constexpr (T >= 32) {
        return 0xffffffffu;
    } else {
        const int lane = tid & 31;
        return ((1u << T) - 1u) << (lane / T * T);
    }
}

// Synchronises the T threads of coil group g.  Groups of <= 32 threads sit in
// one warp (__syncwarp with the group's lane mask); wider groups (T = 64/128/256
// at N = 1024/2048/4096) span several warps, so they use named barrier 1 + g
// with a T-thread count (barrier 0 is __syncthreads), or the CTA barrier when
// the CTA is a single group.
template <int T, int G>
__device__ __forceinline__ void group_sync(unsigned mask, int g) {
    if constexpr (T <= 32) {
        __syncwarp(mask);
    } else if constexpr (G == 1) {
        __syncthreads();
    } else {
        static_assert(T % 32 == 0 && G < 16, "named barriers need whole warps and ids < 16");
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(T) : "memory");
    }
}

template <int N>
constexpr int cp_groups() {  // coil groups per CTA: ~128 threads
    constexpr int T = LineFFT<N>::T;
    return T >= 128 ? 1 : 128 / T;
}

// No resident-CTA floor: a 128-register cap (4 CTAs/SM) once made the 20-point
// 5*2^k SENSE lines faster (160^2: 160 -> 150 us, profiles/round1_combine.md)
// while their exchanges ran 3.4x over the ideal shared-memory wavefronts; with
// the conflict-free mixed-radix layout (fft_core.cuh pad, row_stride) the
// uncapped kernel is the faster one (150 -> 106 us,
// profiles/round2_mixed_radix.md).
template <int N, int MODE, int G>
__global__ void __launch_bounds__(G * LineFFT<N>::T) k_fft_combine_cp(ContigArgs a, std::uint32_t items) {
    pdl_launch_dependents();
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T;
    constexpr bool SENSE = MODE == int(Combine::Sense);
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int j = tid % T, g = tid / T;
    float2* line = smem + g * row_stride<N>();
    const unsigned mask = group_mask<T>(tid);
    typename L::Twiddles tw;
    L::load_twiddles(tw, a.tw, j, a.scale);
    pdl_wait();  // twiddle tables are init-time constants
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    const std::uint32_t C = std::uint32_t(a.coils), ny = std::uint32_t(a.ny);
    const IndexSplit ysplit(ny);
    const std::uint64_t coil_stride = std::uint64_t(ny) * N;
    for (std::uint32_t item = blockIdx.x; item < items; item += gridDim.x) {
        std::uint32_t f, y;
        ysplit.split(item, f, y);
        const float2* xbase = a.in + (std::uint64_t(f) * C * ny + y) * N + j;
        const float2* sbase = a.smap + std::uint64_t(y) * N + j;
        float acc_re[R], acc_im[R];
        sfor<R>([&](auto m) {
            acc_re[m.value] = 0.f;
            acc_im[m.value] = 0.f;
        });
        for (std::uint32_t c = g; c < C; c += G) {
            float2 v[R];
            const float2* src = xbase + c * coil_stride;
            slots_ld<R>(sh_in, (long long)(R / 2) * T, [&](auto m, long long d) { v[m.value] = __ldcs(src + T * m.value + d); });
            // map row: issued before the transform (in flight during it) for
            // powers of two; at the point of use for mixed radix, whose 20-point
            // threads cannot hold another R registers across the transform
            constexpr bool kEarlyMap = !is_mixed_size(N);
            float2 sv[SENSE ? R : 1];
            const float2* sp = sbase + c * coil_stride;
            auto load_map = [&] {
                slots_ld<R>(sh_out, (long long)(R / 2) * T, [&](auto m, long long d) { sv[m.value] = __ldg(sp + T * m.value + d); });
            };
            if constexpr (SENSE && kEarlyMap) load_map();
            L::template run<+1>(v, tw, line, j, [mask, g] { group_sync<T, G>(mask, g); }, a.scale);
            if constexpr (SENSE && !kEarlyMap) load_map();
            if constexpr (SENSE) {
                sfor<R>([&](auto m) { mac_conj(acc_re[m.value], acc_im[m.value], v[m.value], sv[m.value]); });
            } else {
                sfor<R>([&](auto m) { mac_abs2(acc_re[m.value], v[m.value]); });
            }
        }
        // partials -> shared memory at their output positions, then the CTA
        // sums the G groups in order
        __syncthreads();  // every group is done with its exchange line
        slots<R>(sh_out, [&](auto m, auto ms) {
            line[L::pad(j + T * ms.value)] = make_float2(acc_re[m.value], acc_im[m.value]);
        });
        __syncthreads();
        for (int p = tid; p < N; p += G * T) {
            float re = 0.f, im = 0.f;
            for (int q = 0; q < G; ++q) {
                const float2 w = smem[q * row_stride<N>() + L::pad(p)];
                re += w.x;
                im += w.y;
            }
            if constexpr (SENSE)
                static_cast<float2*>(a.out)[(std::uint64_t(f) * ny + y) * N + p] = make_float2(re, im);
            else
                static_cast<float*>(a.out)[(std::uint64_t(f) * ny + y) * N + p] = float(sqrt(double(re)));
        }
        __syncthreads();  // the partial buffers are reused by the next line
    }
}

template <int N, int MODE>
int cp_occ(int smem) {
    constexpr int G = cp_groups<N>();
    return blocks_per_sm(k_fft_combine_cp<N, MODE, G>, G * LineFFT<N>::T, smem);
}

template <int n>
LaunchShape plan_cp_n(Combine mode, std::uint64_t items, int sms) {
    LaunchShape s;
    if constexpr (n >= 16) {
        constexpr int G = cp_groups<n>();
        s.rq = LineFFT<n>::R;
        s.block = G * LineFFT<n>::T;
        s.smem = G * row_stride<n>() * 8;
        const int occ = mode == Combine::Sense ? cp_occ<n, 1>(s.smem) : cp_occ<n, 2>(s.smem);
        s.grid = int(std::min<std::uint64_t>(items, std::uint64_t(sms) * occ));
        s.variant = 128;
    }
    return s;
}

template <int n>
cudaError_t launch_cp_n(Combine mode, const ContigArgs& a, const LaunchShape& s, std::uint32_t items, cudaStream_t st) {
    if constexpr (n >= 16) {
        constexpr int G = cp_groups<n>();
        if (mode == Combine::Sense)
            k_fft_combine_cp<n, 1, G><<<s.grid, s.block, s.smem, st>>>(a, items);
        else
            k_fft_combine_cp<n, 2, G><<<s.grid, s.block, s.smem, st>>>(a, items);
        return cudaGetLastError();
    } else {
        return cudaErrorInvalidValue;
    }
}

}  // namespace

bool combine_cp_preferred(std::uint64_t N, std::uint64_t items, std::uint64_t coils, int sms) {
    if (!fft_size_supported(N) || N < 16 || coils < 2) return false;
    if (const char* e = std::getenv("HETRECO_COMBINE_CP"); e && *e) return *e == '1';  // force on / off
    const int R = points_for(N, 0);
    const std::uint64_t T = N / std::uint64_t(R);
    // warps of lines per SM the coil-serial kernel would have.  Measured:
    // C2/C4 (0.9 warps/SM) coil-parallel 22 % faster; 512^2 x 2-frame chunk
    // (7 warps/SM, T = 32) coil-serial 18 % faster; 256^2 C3 (26 warps/SM)
    // coil-serial 5 % faster; 160^2 C3 (8 warps/SM, T = 8 threads per line)
    // coil-parallel 12 % faster (SENSE), 19 % (RSS).
    const std::uint64_t warps = items * T / 32 / std::uint64_t(sms);
    return warps < 2 || (T < 16 && warps < 16);
}

LaunchShape plan_combine_cp(std::uint64_t N, Combine mode, std::uint64_t items, int sms) {
    LaunchShape s;
    if (!fft_size_supported(N) || N < 16 || mode == Combine::None) return s;
    switch (N) {
#define X(n) \
    case n: s = plan_cp_n<n>(mode, items, sms); break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    if (s.grid < 1) s.grid = 1;
    return s;
}

cudaError_t launch_combine_cp(std::uint64_t N, Combine mode, const ContigArgs& a, const LaunchShape& s,
                              cudaStream_t st) {
    if (s.block == 0 || !(s.variant & 128)) return cudaErrorInvalidValue;
    const std::uint64_t items64 = a.ny * a.frames;
    if (items64 >= (std::uint64_t(1) << 32)) return cudaErrorInvalidValue;
    const std::uint32_t items = std::uint32_t(items64);
    switch (N) {
#define X(n) \
    case n: return launch_cp_n<n>(mode, a, s, items, st);
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

}  // namespace hetreco::dev
