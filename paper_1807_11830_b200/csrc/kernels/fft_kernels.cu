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

// ---- axis 0 (+ combine) ---------------------------------------------------------------------

template <int N, int DIR, int MODE>
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
        if constexpr (MODE == int(Combine::None)) {
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
        } else {
            const std::uint64_t y = active ? item % a.ny : 0;
            const std::uint64_t f = active ? item / a.ny : 0;
            double acc_re[R], acc_im[R];
            sfor<R>([&](auto m) {
                acc_re[m.value] = 0.0;
                acc_im[m.value] = 0.0;
            });
            for (std::uint64_t c = 0; c < a.coils; ++c) {
                const float2* src = a.in + ((f * a.coils + c) * a.ny + y) * N;
                float2 v[R];
                sfor<R>([&](auto m) {
                    const int p = (j + T * m.value + sh_in) & (N - 1);
                    v[m.value] = active ? __ldcs(src + p) : make_float2(0.f, 0.f);
                });
                L::template run<DIR>(v, tw, line, j, sync);
                if constexpr (MODE == int(Combine::Sense)) {
                    const float2* srow = a.smap + (c * a.ny + y) * N;
                    sfor<R>([&](auto m) {
                        const int p = (j + T * m.value + sh_out) & (N - 1);
                        const float2 x = cscale(v[m.value], scale);
                        const float2 s = active ? __ldg(srow + p) : make_float2(0.f, 0.f);
                        // x * conj(s) with the reference's rounding (kernel_abi.h:123-125)
                        const float nsi = -s.y;
                        const float re = __fsub_rn(__fmul_rn(x.x, s.x), __fmul_rn(x.y, nsi));
                        const float im = __fadd_rn(__fmul_rn(x.x, nsi), __fmul_rn(x.y, s.x));
                        acc_re[m.value] = __dadd_rn(acc_re[m.value], double(re));
                        acc_im[m.value] = __dadd_rn(acc_im[m.value], double(im));
                    });
                } else {
                    sfor<R>([&](auto m) {
                        const float2 x = cscale(v[m.value], scale);
                        const double re = x.x, im = x.y;
                        acc_re[m.value] =
                            __dadd_rn(acc_re[m.value], __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
                    });
                }
            }
            if (active) {
                if constexpr (MODE == int(Combine::Sense)) {
                    float2* dst = static_cast<float2*>(a.out) + (f * a.ny + y) * N;
                    sfor<R>([&](auto m) {
                        const int p = (j + T * m.value + sh_out) & (N - 1);
                        dst[p] = make_float2(float(acc_re[m.value]), float(acc_im[m.value]));
                    });
                } else {
                    float* dst = static_cast<float*>(a.out) + (f * a.ny + y) * N;
                    sfor<R>([&](auto m) {
                        const int p = (j + T * m.value + sh_out) & (N - 1);
                        dst[p] = float(sqrt(acc_re[m.value]));
                    });
                }
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

template <int N, int DIR, int MODE>
int contig_occ(int block, int smem) {
    return blocks_per_sm(k_fft_contig<N, DIR, MODE>, block, smem);
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
    int lpb = std::max(1, 128 / T);  // lines per block
    // small problems: fewer lines per block so every SM gets work
    while (lpb > 1 && (items + lpb - 1) / lpb < std::uint64_t(2 * sms)) lpb >>= 1;
    s.block = lpb * T;
    s.smem = lpb * stride_of(N) * 8;
    int occ = 1;
    switch (N) {
#define X(n)                                                                            \
    case n:                                                                             \
        if (mode == Combine::None) {                                                    \
            occ = contig_occ<n, 1, 0>(s.block, s.smem);                                 \
            contig_occ<n, -1, 0>(s.block, s.smem);                                      \
        } else if (mode == Combine::Sense) {                                            \
            occ = contig_occ<n, 1, 1>(s.block, s.smem);                                 \
        } else {                                                                        \
            occ = contig_occ<n, 1, 2>(s.block, s.smem);                                 \
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
                k_fft_contig<n, 1, 0><<<s.grid, s.block, s.smem, st>>>(a, lpb, items);         \
            else                                                                               \
                k_fft_contig<n, -1, 0><<<s.grid, s.block, s.smem, st>>>(a, lpb, items);        \
        } else if (mode == Combine::Sense) {                                                   \
            k_fft_contig<n, 1, 1><<<s.grid, s.block, s.smem, st>>>(a, lpb, items);             \
        } else {                                                                               \
            k_fft_contig<n, 1, 2><<<s.grid, s.block, s.smem, st>>>(a, lpb, items);             \
        }                                                                                      \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return cudaGetLastError();
}

}  // namespace hetreco::dev
