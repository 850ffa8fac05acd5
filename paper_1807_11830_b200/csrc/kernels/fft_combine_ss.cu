// fft_combine_ss.cu -- SENSE axis-0 IFFT + combine with the map row staged in
// shared memory (the default SENSE fp32 combine).
//
// In k_fft_combine every thread prefetches the next coil's map row S[:, y, c]
// into 32 registers (and holds the current one in another 32): 216 registers,
// 8 warps per SM, and the SENSE pass runs 30 % slower than the RSS pass that
// reads no maps (profiles/round1_combine.md).  Here the LPB lines of a CTA are
// one row y of LPB consecutive frames, so they share S[:, y, c]: the CTA
// stages that row into shared memory one coil ahead, every line reads it at the point of use, and the register budget
// drops to the transform + X prefetch + accumulators.  One bar.sync per coil.
//
// Same semantics as k_fft_combine's fp32 SENSE variant (complex_element_prod
// .cl.src:9-19, ximage_sum.cl.src:6-23): out[x,y,f] = sum_c conj(S) X,
// coil-ordered fp32 accumulation with fused products -- bit-identical to it.
#include "fft_kernels.cuh"

namespace hetreco::dev {

namespace {

// Frames per CTA.  Measured at C3 shapes (profiles/round1_combine.md):
// 256^2 -> 16: 168 us, 8: 121, 4: 114, 2: 113; 512^2 x 8 -> 8: 203, 4: 172,
// 2: 159 (register-prefetch kernel 162).  HETRECO_SS_LINES = 2|4|8|16 overrides.
constexpr int kSsLines = 8;

int ss_lines(std::uint64_t N) {
    const int v = env_int("HETRECO_SS_LINES", N >= 512 ? 2 : 4);
    return (v == 2 || v == 4 || v == 6 || v == 8 || v == 16) ? v : kSsLines;
}

template <int N, int LPB>
__global__ void __launch_bounds__(LPB * LineFFT<N>::T) k_fft_combine_ss(ContigArgs a, std::uint32_t gpy,
                                                                        std::uint32_t groups) {
    pdl_launch_dependents();
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T, NT = LPB * T;
    constexpr int NS = (N + NT - 1) / NT;  // map elements staged per thread
    extern __shared__ float2 smem[];
    float2* sbuf = smem + LPB * line_stride<N>();  // 2 x [N]
    const int tid = threadIdx.x;
    const int j = tid % T, l = tid / T;
    float2* line = smem + l * line_stride<N>();
    typename L::Twiddles tw;
    L::load_twiddles(tw, a.tw, j, a.scale);
    pdl_wait();  // twiddle tables are init-time constants
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    const std::uint32_t C = std::uint32_t(a.coils), ny = std::uint32_t(a.ny), F = std::uint32_t(a.frames);
    const std::uint64_t coil_stride = std::uint64_t(ny) * N;
    for (std::uint32_t grp = blockIdx.x; grp < groups; grp += gridDim.x) {
        const std::uint32_t y = grp / gpy;
        const std::uint32_t f0 = (grp - y * gpy) * LPB;
        const std::uint32_t f = f0 + l;
        const bool active = f < F;
        // inactive lines re-read frame f0 (valid memory) and skip the store
        const float2* xbase = a.in + (std::uint64_t(active ? f : f0) * C * ny + y) * N + j;
        const float2* srow = a.smap + std::uint64_t(y) * N;
        auto load_x = [&](std::uint32_t c, float2(&d)[R]) {
            const float2* src = xbase + c * coil_stride;
            slots_ld<R>(sh_in, (long long)(R / 2) * T, [&](auto m, long long o) { d[m.value] = __ldcs(src + T * m.value + o); });
        };
        float2 sn[NS];
        auto load_s = [&](std::uint32_t c) {
            sfor<NS>([&](auto k) {
                const int i = tid + k.value * NT;
                if (NS * NT == N || i < N) sn[k.value] = __ldg(srow + c * coil_stride + i);
            });
        };
        auto put_s = [&](int b) {
            sfor<NS>([&](auto k) {
                const int i = tid + k.value * NT;
                if (NS * NT == N || i < N) sbuf[b * N + i] = sn[k.value];
            });
        };
        float acc_re[R], acc_im[R];
        sfor<R>([&](auto m) {
            acc_re[m.value] = 0.f;
            acc_im[m.value] = 0.f;
        });
        float2 xn[R];
        load_s(0);
        load_x(0, xn);
        put_s(0);
        __syncthreads();
        for (std::uint32_t c = 0; c < C; ++c) {
            float2 v[R];
            sfor<R>([&](auto m) { v[m.value] = xn[m.value]; });
            const bool more = c + 1 < C;
            if (more) {
                load_x(c + 1, xn);
                load_s(c + 1);
            }
            L::template run<+1>(v, tw, line, j, [] { line_sync<T>(); }, a.scale);
            const float2* sb = sbuf + (c & 1) * N + j;
            slots_ld<R>(sh_out, (long long)(R / 2) * T, [&](auto m, long long o) {
                mac_conj(acc_re[m.value], acc_im[m.value], v[m.value], sb[T * m.value + o]);
            });
            if (more) put_s(int((c + 1) & 1));
            __syncthreads();  // next row staged; this row's readers done
        }
        if (active) {
            float2* dst = static_cast<float2*>(a.out) + (std::uint64_t(f) * ny + y) * N + j;
            slots<R>(sh_out, [&](auto m, auto ms) { dst[T * ms.value] = make_float2(acc_re[m.value], acc_im[m.value]); });
        }
    }
}

template <int N, int LPB>
constexpr int ss_smem() {
    return (LPB * line_stride<N>() + 2 * N) * 8;
}

template <int n, int LPB>
LaunchShape plan_ss_nl(std::uint64_t ny, std::uint64_t frames, int sms) {
    LaunchShape s;
    if constexpr (n >= 64 && LPB * LineFFT<n>::T <= 1024) {
        s.rq = LineFFT<n>::R;
        s.block = LPB * LineFFT<n>::T;
        s.smem = ss_smem<n, LPB>();
        const std::uint64_t groups = ny * ((frames + LPB - 1) / LPB);
        const int occ = blocks_per_sm(k_fft_combine_ss<n, LPB>, s.block, s.smem);
        const int per_sm = env_int("HETRECO_SS_CTAS_PER_SM", occ);  // experiments (profiles/round1_combine.md)
        s.grid = int(std::min<std::uint64_t>(groups, std::uint64_t(sms) * std::uint64_t(per_sm > 0 ? per_sm : occ)));
        s.variant = 256 | (LPB << 10);
    }
    return s;
}

template <int n>
LaunchShape plan_ss_n(std::uint64_t ny, std::uint64_t frames, int sms) {
    switch (ss_lines(std::uint64_t(n))) {
        case 2: return plan_ss_nl<n, 2>(ny, frames, sms);
        case 4: return plan_ss_nl<n, 4>(ny, frames, sms);
        case 6: return plan_ss_nl<n, 6>(ny, frames, sms);
        case 16: return plan_ss_nl<n, 16>(ny, frames, sms);
        default: return plan_ss_nl<n, 8>(ny, frames, sms);
    }
}

template <int n, int LPB>
cudaError_t launch_ss_nl(const ContigArgs& a, const LaunchShape& s, cudaStream_t st) {
    if constexpr (n >= 64 && LPB * LineFFT<n>::T <= 1024) {
        const std::uint64_t gpy = (a.frames + LPB - 1) / LPB;
        const std::uint64_t groups = a.ny * gpy;
        if (groups >= (std::uint64_t(1) << 32)) return cudaErrorInvalidValue;
        k_fft_combine_ss<n, LPB><<<s.grid, s.block, s.smem, st>>>(a, std::uint32_t(gpy), std::uint32_t(groups));
        return cudaGetLastError();
    } else {
        return cudaErrorInvalidValue;
    }
}

template <int n>
cudaError_t launch_ss_n(const ContigArgs& a, const LaunchShape& s, cudaStream_t st) {
    switch (s.variant >> 10) {
        case 2: return launch_ss_nl<n, 2>(a, s, st);
        case 4: return launch_ss_nl<n, 4>(a, s, st);
        case 6: return launch_ss_nl<n, 6>(a, s, st);
        case 16: return launch_ss_nl<n, 16>(a, s, st);
        default: return launch_ss_nl<n, 8>(a, s, st);
    }
}

}  // namespace

bool combine_ss_supported(std::uint64_t N) {
    switch (N) {
#define X(n) \
    case n: return n >= 64;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return false;
}

LaunchShape plan_combine_ss(std::uint64_t N, std::uint64_t ny, std::uint64_t frames, int sms) {
    LaunchShape s;
    if (combine_tc_enabled(N)) return plan_combine_tc(N, ny, frames, sms);  // experiment (profiles/round2_dft_gemm.md)
    switch (N) {
#define X(n) \
    case n: s = plan_ss_n<n>(ny, frames, sms); break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    if (s.grid < 1) s.grid = 1;
    return s;
}

cudaError_t launch_combine_ss(std::uint64_t N, const ContigArgs& a, const LaunchShape& s, cudaStream_t st) {
    if (s.block == 0 || !(s.variant & 256)) return cudaErrorInvalidValue;
    switch (N) {
#define X(n) \
    case n: return launch_ss_n<n>(a, s, st);
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

}  // namespace hetreco::dev
