// fft_kernels.cu -- batched 2-D FFT as two HBM passes, with the coil combine
// fused into the second.
//
//   k_fft_strided : axis 1 (stride nx).  A CTA owns a tile of tx adjacent
//                   columns of one plane (tx*8 B contiguous per row, so every
//                   warp load is a run of full 32-B sectors), transforms all of
//                   them along y with the LineFFT passes (block barriers between
//                   exchanges since a column's threads span warps).
//   k_fft_contig  : axis 0 (contiguous lines).  T <= 32 threads own a line, so
//                   exchanges need only __syncwarp.  Optional epilogues:
//                   SENSE  M = sum_c conj(S_c) . X_c   and   RSS  sqrt(sum |X_c|^2)
//                   accumulated in registers across the coil loop, written once.
//
// fftshift/ifftshift are index permutations applied on store/load along each
// kernel's own axis (exact).  The inverse scale 1/(nx*ny) is applied once, in
// the second pass.  Twiddles W_N^t are a per-direction device table baked at
// init (double -> float, as the reference bakes its pass payloads,
// fft_radix2_pass.cl.src:15-16) and held in registers for the CTA's lifetime.
#include <cstdlib>

#include "fft_core.cuh"
#include "launch.hpp"

namespace hetreco::dev {

namespace {

template <int N>
constexpr int line_stride() {
    return (LineFFT<N>::padded_len) | 1;  // odd: spreads lines over banks
}

// ---- axis 1 ------------------------------------------------------------------------------

template <int N, int DIR>
__global__ void __launch_bounds__(512) k_fft_strided(StridedArgs a, int tx, std::uint64_t ntiles) {
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T;
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int l = tid % tx, j = tid / tx;
    float2* line = smem + l * line_stride<N>();
    float2 tw[L::NTW];
    L::load_twiddles(tw, a.tw, j);
    const std::uint64_t xtiles = a.nx / std::uint64_t(tx);
    const std::uint64_t plane_elems = a.nx * std::uint64_t(N);
    const int sh_in = a.shift_in ? N / 2 : 0;
    const int sh_out = a.shift_out ? N / 2 : 0;
    for (std::uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const std::uint64_t plane = tile / xtiles;
        const std::uint64_t x = (tile % xtiles) * tx + l;
        const float2* src = a.in + plane * plane_elems + x;
        float2 v[R];
        sfor<R>([&](auto m) {
            const int p = (j + T * m.value + sh_in) & (N - 1);
            v[m.value] = src[std::uint64_t(p) * a.nx];
        });
        L::template run<DIR>(v, tw, line, j, [] { __syncthreads(); });
        float2* dst = a.out + plane * plane_elems + x;
        const float s = a.scale;
        sfor<R>([&](auto m) {
            const int p = (j + T * m.value + sh_out) & (N - 1);
            dst[std::uint64_t(p) * a.nx] = cscale(v[m.value], s);
        });
    }
}

// ---- axis 0 -------------------------------------------------------------------------------

template <int N, int DIR>
__global__ void __launch_bounds__(256) k_fft_contig(ContigArgs a, int lpb, std::uint64_t items) {
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T;
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int j = tid % T, l = tid / T;
    float2* line = smem + l * line_stride<N>();
    float2 tw[L::NTW];
    L::load_twiddles(tw, a.tw, j);
    auto sync = [] {
        if constexpr (T <= 32)
            __syncwarp();
        else
            __syncthreads();
    };
    const int sh_in = a.shift_in ? N / 2 : 0;
    const int sh_out = a.shift_out ? N / 2 : 0;
    const float scale = a.scale;
    for (std::uint64_t grp = blockIdx.x; grp * lpb < items; grp += gridDim.x) {
        const std::uint64_t item = grp * lpb + l;
        const bool active = item < items;
        float2 v[R];
        const float2* src = a.in + item * N;
        sfor<R>([&](auto m) {
            const int p = (j + T * m.value + sh_in) & (N - 1);
            v[m.value] = active ? src[p] : make_float2(0.f, 0.f);
        });
        L::template run<DIR>(v, tw, line, j, sync);
        float2* dst = static_cast<float2*>(a.out) + item * N;
        if (active)
            sfor<R>([&](auto m) {
                const int p = (j + T * m.value + sh_out) & (N - 1);
                dst[p] = cscale(v[m.value], scale);
            });
    }
}

// ---- axis 0 + coil combine -------------------------------------------------------------------
//
// Output line (y, f) is owned by T threads; they loop over the coils, each
// iteration = load the coil's line of X (axis-1 transformed k-space) and the
// matching line of S, inverse-transform X along x, multiply by conj(S) (or
// take |X|^2) and accumulate.  ACCF selects fp32 instead of fp64
// accumulators; PF double-buffers the next coil's X and S in registers so
// their HBM/L2 latency overlaps the current coil's FFT.

template <int N, int MODE, bool ACCF, bool PF>
__global__ void __launch_bounds__(256) k_fft_combine(ContigArgs a, int lpb, std::uint64_t items) {
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T;
    constexpr bool SENSE = MODE == int(Combine::Sense);
    using Acc = std::conditional_t<ACCF, float, double>;
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int j = tid % T, l = tid / T;
    float2* line = smem + l * line_stride<N>();
    float2 tw[L::NTW];
    L::load_twiddles(tw, a.tw, j);
    auto sync = [] {
        if constexpr (T <= 32)
            __syncwarp();
        else
            __syncthreads();
    };
    const int sh_in = a.shift_in ? N / 2 : 0;
    const int sh_out = a.shift_out ? N / 2 : 0;
    const float scale = a.scale;
    const std::uint64_t C = a.coils;
    for (std::uint64_t grp = blockIdx.x; grp * lpb < items; grp += gridDim.x) {
        const std::uint64_t item = grp * lpb + l;
        const bool active = item < items;
        const std::uint64_t y = active ? item % a.ny : 0;
        const std::uint64_t f = active ? item / a.ny : 0;
        auto load_x = [&](std::uint64_t c, float2(&d)[R]) {
            const float2* src = a.in + ((f * C + c) * a.ny + y) * N;
            sfor<R>([&](auto m) {
                const int p = (j + T * m.value + sh_in) & (N - 1);
                d[m.value] = active ? __ldcs(src + p) : make_float2(0.f, 0.f);
            });
        };
        auto load_s = [&](std::uint64_t c, float2(&d)[R]) {
            if constexpr (SENSE) {
                const float2* srow = a.smap + (c * a.ny + y) * N;
                sfor<R>([&](auto m) {
                    const int p = (j + T * m.value + sh_out) & (N - 1);
                    d[m.value] = active ? __ldg(srow + p) : make_float2(0.f, 0.f);
                });
            }
        };
        Acc acc_re[R], acc_im[R];
        sfor<R>([&](auto m) {
            acc_re[m.value] = Acc(0);
            acc_im[m.value] = Acc(0);
        });
        float2 xn[PF ? R : 1], sn[(PF && SENSE) ? R : 1];
        if constexpr (PF) {
            load_x(0, xn);
            if constexpr (SENSE) load_s(0, sn);
        }
        for (std::uint64_t c = 0; c < C; ++c) {
            float2 v[R], sv[(PF && SENSE) ? R : 1];
            if constexpr (PF) {
                sfor<R>([&](auto m) { v[m.value] = xn[m.value]; });
                if constexpr (SENSE) sfor<R>([&](auto m) { sv[m.value] = sn[m.value]; });
                if (c + 1 < C) {
                    load_x(c + 1, xn);
                    if constexpr (SENSE) load_s(c + 1, sn);
                }
            } else {
                load_x(c, v);
            }
            L::template run<+1>(v, tw, line, j, sync);
            if constexpr (SENSE) {
                const float2* srow = a.smap + (c * a.ny + y) * N;
                sfor<R>([&](auto m) {
                    const float2 x = cscale(v[m.value], scale);
                    float2 s;
                    if constexpr (PF) {
                        s = sv[m.value];
                    } else {
                        const int p = (j + T * m.value + sh_out) & (N - 1);
                        s = active ? __ldg(srow + p) : make_float2(0.f, 0.f);
                    }
                    // x * conj(s) with the reference's rounding (kernel_abi.h:123-125)
                    const float nsi = -s.y;
                    const float re = __fsub_rn(__fmul_rn(x.x, s.x), __fmul_rn(x.y, nsi));
                    const float im = __fadd_rn(__fmul_rn(x.x, nsi), __fmul_rn(x.y, s.x));
                    if constexpr (ACCF) {
                        acc_re[m.value] = __fadd_rn(acc_re[m.value], re);
                        acc_im[m.value] = __fadd_rn(acc_im[m.value], im);
                    } else {
                        acc_re[m.value] = __dadd_rn(acc_re[m.value], double(re));
                        acc_im[m.value] = __dadd_rn(acc_im[m.value], double(im));
                    }
                });
            } else {
                sfor<R>([&](auto m) {
                    const float2 x = cscale(v[m.value], scale);
                    if constexpr (ACCF) {
                        acc_re[m.value] = __fadd_rn(acc_re[m.value], __fadd_rn(__fmul_rn(x.x, x.x), __fmul_rn(x.y, x.y)));
                    } else {
                        const double re = x.x, im = x.y;
                        acc_re[m.value] =
                            __dadd_rn(acc_re[m.value], __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
                    }
                });
            }
        }
        if (active) {
            if constexpr (SENSE) {
                float2* dst = static_cast<float2*>(a.out) + (f * a.ny + y) * N;
                sfor<R>([&](auto m) {
                    const int p = (j + T * m.value + sh_out) & (N - 1);
                    dst[p] = make_float2(float(acc_re[m.value]), float(acc_im[m.value]));
                });
            } else {
                float* dst = static_cast<float*>(a.out) + (f * a.ny + y) * N;
                sfor<R>([&](auto m) {
                    const int p = (j + T * m.value + sh_out) & (N - 1);
                    dst[p] = float(sqrt(double(acc_re[m.value])));
                });
            }
        }
    }
}

// ---- dispatch -----------------------------------------------------------------------------

#define HETRECO_FFT_SIZES(X) \
    X(1) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)

template <int N>
constexpr int threads_per_line() {
    return LineFFT<N>::T;
}

int tpl_of(std::uint64_t N) {
    switch (N) {
#define X(n) \
    case n: return threads_per_line<n>();
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return 0;
}

int stride_of(std::uint64_t N) {
    switch (N) {
#define X(n) \
    case n: return line_stride<n>();
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return 0;
}

template <class K>
int blocks_per_sm(K kernel, int block, int smem) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, smem) != cudaSuccess) {
        cudaGetLastError();
        n = 1;
    }
    return n > 0 ? n : 1;
}

template <int N, int DIR>
int strided_occ(int block, int smem) {
    return blocks_per_sm(k_fft_strided<N, DIR>, block, smem);
}

template <int N, int DIR>
int contig_occ(int block, int smem) {
    return blocks_per_sm(k_fft_contig<N, DIR>, block, smem);
}

// Combine-kernel variants: bit 0 = fp32 accumulators, bit 1 = register
// prefetch of the next coil.  All four are built for the benchmark sizes
// (256, 512); other sizes use variant 0.
template <int N>
constexpr bool has_variants() {
    return N == 256 || N == 512;
}

template <int N, int MODE>
int combine_occ(int variant, int block, int smem) {
    if constexpr (has_variants<N>()) {
        switch (variant) {
            case 1: return blocks_per_sm(k_fft_combine<N, MODE, true, false>, block, smem);
            case 2: return blocks_per_sm(k_fft_combine<N, MODE, false, true>, block, smem);
            case 3: return blocks_per_sm(k_fft_combine<N, MODE, true, true>, block, smem);
            default: break;
        }
    }
    return blocks_per_sm(k_fft_combine<N, MODE, false, false>, block, smem);
}

template <int N, int MODE>
void combine_launch(int variant, const ContigArgs& a, const LaunchShape& s, int lpb, std::uint64_t items,
                    cudaStream_t st) {
    if constexpr (has_variants<N>()) {
        switch (variant) {
            case 1: k_fft_combine<N, MODE, true, false><<<s.grid, s.block, s.smem, st>>>(a, lpb, items); return;
            case 2: k_fft_combine<N, MODE, false, true><<<s.grid, s.block, s.smem, st>>>(a, lpb, items); return;
            case 3: k_fft_combine<N, MODE, true, true><<<s.grid, s.block, s.smem, st>>>(a, lpb, items); return;
            default: break;
        }
    }
    k_fft_combine<N, MODE, false, false><<<s.grid, s.block, s.smem, st>>>(a, lpb, items);
}

int env_int(const char* name, int fallback) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : fallback;
}

}  // namespace

bool fft_size_supported(std::uint64_t n) { return tpl_of(n) != 0; }

LaunchShape plan_strided(std::uint64_t N, std::uint64_t nx, std::uint64_t planes, int sms) {
    LaunchShape s;
    const int T = tpl_of(N);
    if (T == 0) return s;
    const int ls_bytes = stride_of(N) * 8;
    // columns per tile: >= 16 (128-B rows) when possible, bounded by 1024
    // threads and ~100 KB of shared memory.
    std::uint64_t tx = std::max(16, 256 / T);
    tx = std::min<std::uint64_t>(tx, std::uint64_t(std::max(1, 512 / T)));
    tx = std::min<std::uint64_t>(tx, std::uint64_t(std::max(1, (100 * 1024) / ls_bytes)));
    tx = std::min<std::uint64_t>(tx, nx);
    while (tx > 1 && nx % tx) tx >>= 1;  // both powers of two in practice
    s.block = int(tx) * T;
    s.smem = int(tx) * ls_bytes;
    const std::uint64_t tiles = (nx / tx) * planes;
    int occ = 1;
    switch (N) {
#define X(n) \
    case n: occ = strided_occ<n, 1>(s.block, s.smem); strided_occ<n, -1>(s.block, s.smem); break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    s.grid = int(std::min<std::uint64_t>(tiles, std::uint64_t(sms) * occ));
    if (s.grid < 1) s.grid = 1;
    return s;
}

LaunchShape plan_contig(std::uint64_t N, Combine mode, std::uint64_t items, int sms) {
    LaunchShape s;
    const int T = tpl_of(N);
    if (T == 0) return s;
    int lpb = std::max(1, env_int("HETRECO_LINES_PER_BLOCK", 128) / T);  // lines per block
    // small problems: fewer lines per block so every SM gets work
    while (lpb > 1 && (items + lpb - 1) / lpb < std::uint64_t(2 * sms)) lpb >>= 1;
    s.block = lpb * T;
    s.smem = lpb * stride_of(N) * 8;
    s.variant = mode == Combine::None ? 0 : env_int("HETRECO_COMBINE_VARIANT", 0);
    int occ = 1;
    switch (N) {
#define X(n)                                                                            \
    case n:                                                                             \
        if (mode == Combine::None) {                                                    \
            occ = contig_occ<n, 1>(s.block, s.smem);                                    \
            contig_occ<n, -1>(s.block, s.smem);                                         \
        } else if (mode == Combine::Sense) {                                            \
            occ = combine_occ<n, 1>(s.variant, s.block, s.smem);                        \
        } else {                                                                        \
            occ = combine_occ<n, 2>(s.variant, s.block, s.smem);                        \
        }                                                                               \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    const std::uint64_t groups = (items + lpb - 1) / lpb;
    s.grid = int(std::min<std::uint64_t>(groups, std::uint64_t(sms) * occ));
    if (s.grid < 1) s.grid = 1;
    return s;
}

cudaError_t launch_strided(std::uint64_t N, int dir, const StridedArgs& a, const LaunchShape& s,
                           cudaStream_t st) {
    const int T = tpl_of(N);
    if (T == 0 || s.block == 0) return cudaErrorInvalidValue;
    const int tx = s.block / T;
    const std::uint64_t tiles = (a.nx / tx) * a.planes;
    switch (N) {
#define X(n)                                                                                 \
    case n:                                                                                  \
        if (dir > 0)                                                                         \
            k_fft_strided<n, 1><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);              \
        else                                                                                 \
            k_fft_strided<n, -1><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);             \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return cudaGetLastError();
}

cudaError_t launch_contig(std::uint64_t N, int dir, Combine mode, const ContigArgs& a,
                          const LaunchShape& s, cudaStream_t st) {
    const int T = tpl_of(N);
    if (T == 0 || s.block == 0) return cudaErrorInvalidValue;
    const int lpb = s.block / T;
    const std::uint64_t items = mode == Combine::None ? a.ny * a.frames : a.ny * a.frames;
    if (mode != Combine::None && dir < 0) return cudaErrorInvalidValue;
    switch (N) {
#define X(n)                                                                                   \
    case n:                                                                                    \
        if (mode == Combine::None) {                                                           \
            if (dir > 0)                                                                       \
                k_fft_contig<n, 1><<<s.grid, s.block, s.smem, st>>>(a, lpb, items);            \
            else                                                                               \
                k_fft_contig<n, -1><<<s.grid, s.block, s.smem, st>>>(a, lpb, items);           \
        } else if (mode == Combine::Sense) {                                                   \
            combine_launch<n, 1>(s.variant, a, s, lpb, items, st);                             \
        } else {                                                                               \
            combine_launch<n, 2>(s.variant, a, s, lpb, items, st);                             \
        }                                                                                      \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return cudaGetLastError();
}

}  // namespace hetreco::dev
