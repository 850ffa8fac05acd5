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

__device__ __forceinline__ std::uint32_t smem_u32addr(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float2 lds_f2(std::uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

// Pass twiddles from shared memory (TWS) at 256 points: A/B switch
// HETRECO_SS_TWSMEM=0|1 (profiles/round2_summary.md).
bool ss_tws(std::uint64_t N) { return N == 256 && env_int("HETRECO_SS_TWSMEM", 0) == 1; }

// Line exchange by warp shuffles instead of shared memory at 256 points
// (north_star's "warp-shuffle butterflies"): A/B switch HETRECO_SS_SHFL=1.
bool ss_shfl(std::uint64_t N) { return N == 256 && env_int("HETRECO_SS_SHFL", 0) == 1; }

// run_f of the 2-pass 256-point plan (16 x 16) with the pass-0 -> pass-1
// exchange done in registers: the exchange is the 16 x 16 transpose
// v'[m] (lane j) = v[j] (lane m) among the line's 16 lanes, as four butterfly
// stages (lane ^ 1, 2, 4, 8), each swapping 8 value pairs; which value of a
// pair a lane sends depends on its lane bit, hence the selects.
template <int DIR, class Twiddles>
__device__ __forceinline__ void run_shfl(float2 (&v)[16], const Twiddles& twd, int j, float scale) {
    using L = LineFFT<256>;
    static_assert(L::P == 2 && L::R == 16 && L::T == 16, "256 = 16 x 16");
    dft_regs<16, DIR, 1, 0>(v);  // pass 0
    sfor<4>([&](auto sc) {
        constexpr int d = 1 << sc.value;
        const bool hi = (j >> sc.value) & 1;
        sfor<16>([&](auto qc) {
            constexpr int q = qc.value;
            if constexpr ((q & d) == 0) {
                const float2 snd = hi ? v[q] : v[q | d];
                const float2 rcv = make_float2(__shfl_xor_sync(0xffffffffu, snd.x, d), __shfl_xor_sync(0xffffffffu, snd.y, d));
                if (hi)
                    v[q] = rcv;
                else
                    v[q | d] = rcv;
            }
        });
    });
    // pass 1: twiddles (the last pass: pre-scaled), the q = 0 slot scaled, DFT
    sfor<15>([&](auto qc) { v[qc.value + 1] = cmul(v[qc.value + 1], twd.w[L::tw_offset(1) + qc.value]); });
    if (scale != 1.0f) v[0] = cscale(v[0], scale);
    dft_regs<16, DIR, 1, 0>(v);
}

int ss_lines(std::uint64_t N) {
    const int v = env_int("HETRECO_SS_LINES", N >= 512 ? 2 : 4);
    return (v == 2 || v == 4 || v == 6 || v == 8 || v == 16) ? v : kSsLines;
}

// TWS (two-pass lengths, 256 = 16 x 16): the pass-1 twiddles W^{j q} (x
// scale, q = 1..15) come from a per-CTA shared table laid out [j][q - 1] --
// row stride 15 float2, so the 16 threads of a line hit 16 distinct bank
// pairs -- read at the point of use, instead of 30 registers per thread.
template <int N>
constexpr bool tws_ok() {
    using L = LineFFT<N>;
    return L::P == 2 && !L::kTableTw && L::R == L::radix(1) && L::R == L::T;
}
template <int N>
constexpr int tws_len() {
    return tws_ok<N>() ? LineFFT<N>::T * (LineFFT<N>::R - 1) : 0;
}

template <int N, int LPB, int XV>
__global__ void __launch_bounds__(LPB * LineFFT<N>::T) k_fft_combine_ss(ContigArgs a, std::uint32_t gpy,
                                                                        std::uint32_t groups) {
    pdl_launch_dependents();
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T, NT = LPB * T;
    constexpr int NS = (N + NT - 1) / NT;  // map elements staged per thread
    extern __shared__ float2 smem[];
    float2* sbuf = smem + LPB * row_stride<N>();  // 2 x [N]
    constexpr bool TWS = XV == 1, SHF = XV == 2;
    float2* twt = sbuf + 2 * N;                    // TWS: [T][R - 1]
    const int tid = threadIdx.x;
    const int j = tid % T, l = tid / T;
    float2* line = smem + l * row_stride<N>();
    typename L::Twiddles tw;
    if constexpr (TWS) {
        static_assert(tws_ok<N>(), "shared pass twiddles need a 2-pass plan with R = T");
        for (int i = tid; i < tws_len<N>(); i += NT) {
            const int jj = i / (R - 1), q = i % (R - 1) + 1;
            const float2 w = __ldg(a.tw + L::template tw_index<1, 0, 0>(jj) * q);
            twt[i] = make_float2(w.x * a.scale, w.y * a.scale);
        }
    } else {
        L::load_twiddles(tw, a.tw, j, a.scale);
    }
    const std::uint32_t tws_row = smem_u32addr(twt + j * (R - 1));
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
            if constexpr (SHF) {
                run_shfl<+1>(v, tw, j, a.scale);
            } else if constexpr (TWS) {
                // volatile shared loads: re-read per coil, never hoisted into registers
                L::template run_f<+1>(
                    v, [&](auto, auto, auto qc) { return lds_f2(tws_row + 8u * qc.value); }, line, j,
                    [] { line_sync<T>(); }, a.scale);
            } else {
                L::template run<+1>(v, tw, line, j, [] { line_sync<T>(); }, a.scale);
            }
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

template <int N, int LPB, int XV>
constexpr int ss_smem() {
    return (LPB * row_stride<N>() + 2 * N + (XV == 1 ? tws_len<N>() : 0)) * 8;
}

template <int n, int LPB, int XV>
LaunchShape plan_ss_nlt(std::uint64_t ny, std::uint64_t frames, int sms) {
    LaunchShape s;
    if constexpr (n >= 64 && LPB * LineFFT<n>::T <= 1024 && (XV == 0 || (XV == 1 && tws_ok<n>()) || (XV == 2 && n == 256))) {
        s.rq = LineFFT<n>::R;
        s.block = LPB * LineFFT<n>::T;
        s.smem = ss_smem<n, LPB, XV>();
        const std::uint64_t groups = ny * ((frames + LPB - 1) / LPB);
        const int occ = blocks_per_sm(k_fft_combine_ss<n, LPB, XV>, s.block, s.smem);
        const int per_sm = env_int("HETRECO_SS_CTAS_PER_SM", occ);  // experiments (profiles/round1_combine.md)
        s.grid = int(std::min<std::uint64_t>(groups, std::uint64_t(sms) * std::uint64_t(per_sm > 0 ? per_sm : occ)));
        s.variant = 256 | (LPB << 10) | (XV == 1 ? (1 << 15) : 0) | (XV == 2 ? (1 << 16) : 0);
    }
    return s;
}

template <int n, int LPB>
LaunchShape plan_ss_nl(std::uint64_t ny, std::uint64_t frames, int sms) {
    if (ss_tws(n)) return plan_ss_nlt<n, LPB, 1>(ny, frames, sms);
    if (ss_shfl(n)) return plan_ss_nlt<n, LPB, 2>(ny, frames, sms);
    return plan_ss_nlt<n, LPB, 0>(ny, frames, sms);
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

template <int n, int LPB, int XV>
cudaError_t launch_ss_nlt(const ContigArgs& a, const LaunchShape& s, cudaStream_t st) {
    if constexpr (n >= 64 && LPB * LineFFT<n>::T <= 1024 && (XV == 0 || (XV == 1 && tws_ok<n>()) || (XV == 2 && n == 256))) {
        const std::uint64_t gpy = (a.frames + LPB - 1) / LPB;
        const std::uint64_t groups = a.ny * gpy;
        if (groups >= (std::uint64_t(1) << 32)) return cudaErrorInvalidValue;
        k_fft_combine_ss<n, LPB, XV><<<s.grid, s.block, s.smem, st>>>(a, std::uint32_t(gpy), std::uint32_t(groups));
        return cudaGetLastError();
    } else {
        return cudaErrorInvalidValue;
    }
}

template <int n, int LPB>
cudaError_t launch_ss_nl(const ContigArgs& a, const LaunchShape& s, cudaStream_t st) {
    if (s.variant & (1 << 15)) return launch_ss_nlt<n, LPB, 1>(a, s, st);
    if (s.variant & (1 << 16)) return launch_ss_nlt<n, LPB, 2>(a, s, st);
    return launch_ss_nlt<n, LPB, 0>(a, s, st);
}

template <int n>
cudaError_t launch_ss_n(const ContigArgs& a, const LaunchShape& s, cudaStream_t st) {
    switch ((s.variant >> 10) & 31) {
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
