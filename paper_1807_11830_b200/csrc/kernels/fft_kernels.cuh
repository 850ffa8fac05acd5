// fft_kernels.cuh -- batched 2-D FFT as two HBM passes, with the coil combine
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
#pragma once

#include <cstdlib>

#include "fft_core.cuh"
#include "launch.hpp"

namespace hetreco::dev {

// item -> (item / d, item % d): shift/mask when d is a power of two (the
// common case), a 32-bit division otherwise (mixed-radix image sides).
struct IndexSplit {
    std::uint32_t d;
    int shift;  // -1: not a power of two
    __host__ __device__ __forceinline__ explicit IndexSplit(std::uint32_t d_) : d(d_), shift(-1) {
        if (d_ && !(d_ & (d_ - 1))) {
            shift = 0;
            while ((1u << shift) < d_) ++shift;
        }
    }
    __device__ __forceinline__ void split(std::uint32_t item, std::uint32_t& q, std::uint32_t& r) const {
        if (shift >= 0) {
            q = item >> shift;
            r = item & (d - 1);
        } else {
            q = item / d;
            r = item - q * d;
        }
    }
};

// Line stride (float2) when a warp's lanes run across lines (column tiles of
// the axis-1 kernels: lane = line + TX * thread): odd, so consecutive lines
// start on different banks.
template <int N>
constexpr int line_stride() {
    return (LineFFT<N>::padded_len) | 1;  // odd: spreads lines over banks
}

// Line stride when a warp holds 32/T whole lines (lines-major: lane = line * T
// + thread; the axis-0, combine and expand kernels).  Powers of two: as
// line_stride.  Mixed radix with T <= 8 threads per line (96, 160): the first
// stride >= N that is 8 mod 16, which puts the 4 lines of a warp on
// complementary bank halves; with an odd stride the lines collide
// (scripts/tools/bank_sim.py at 160: 624 -> 288 wavefronts per exchange round,
// ideal 240).
template <int N>
constexpr int row_stride() {
    if constexpr (!is_mixed_size(N) || LineFFT<N>::T > 8)
        return line_stride<N>();
    else
        return N + (24 - N % 16) % 16;
}

// ---- axis 1 ------------------------------------------------------------------------------
//
// NXC = compile-time row length (square images) so every slot address is a
// base register + immediate offset; NXC = 0 is the generic runtime-stride
// variant.  Indices are 32-bit and power-of-two divisions are shifts (a
// 64-bit division is an emulated call on the GPU).

// MINB > 1 asks ptxas for MINB resident 256-thread CTAs per SM (register cap).
// TWR: pass twiddles in registers also for mixed radix (default: table).
template <int N, int DIR, int NXC, int RQ = default_points(N), bool PFS = false, int MINB = 1, bool TWR = false>
__global__ void __launch_bounds__((MINB > 1 || TWR) ? 256 : 512, MINB > 1 ? MINB : 0) k_fft_strided(StridedArgs a, int tx, std::uint32_t ntiles) {
    pdl_launch_dependents();
    using L = LineFFT<N, RQ, !is_mixed_size(N) || TWR>;
    constexpr int R = L::R, T = L::T;
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int l = tid % tx, j = tid / tx;
    float2* line = smem + l * line_stride<N>();
    typename L::Twiddles tw;
    L::load_twiddles(tw, a.tw, j, a.scale);
    pdl_wait();  // twiddle tables are init-time constants
    const std::uint32_t nx = NXC ? std::uint32_t(NXC) : std::uint32_t(a.nx);
    const std::uint32_t xtiles = nx / std::uint32_t(tx);
    const IndexSplit xsplit(xtiles);
    const std::uint64_t plane_elems = std::uint64_t(nx) * N;
    const std::uint32_t step = std::uint32_t(T) * nx;  // slot-to-slot distance (runtime variant)
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    auto tile_off = [&](std::uint32_t tile) {
        std::uint32_t plane, xt;
        xsplit.split(tile, plane, xt);
        const std::uint32_t col = xt * std::uint32_t(tx) + std::uint32_t(l);
        return std::uint64_t(plane) * plane_elems + col + std::uint32_t(j) * nx;
    };
    auto load = [&](std::uint64_t off, float2(&v)[R]) {
        const float2* src = a.in + off;
        if constexpr (NXC > 0 && !PFS) {
            // consumed at once: duplicated code paths with immediate offsets
            // beat a moving base under the MINB register cap (measured)
            slots<R>(sh_in, [&](auto m, auto ms) { v[m.value] = __ldcs(src + ms.value * T * NXC); });
        } else if constexpr (NXC > 0) {
            slots_ld<R>(sh_in, (long long)(R / 2) * T * NXC,
                        [&](auto m, long long d) { v[m.value] = __ldcs(src + m.value * T * NXC + d); });
        } else {
            slots_ld<R>(sh_in, (long long)(R / 2) * step,
                        [&](auto m, long long d) { v[m.value] = __ldcs(src + std::uint64_t(m.value) * step + d); });
        }
    };
    auto store = [&](std::uint64_t off, float2(&v)[R]) {
        float2* dst = a.out + off;
        if constexpr (NXC > 0) {
            slots<R>(sh_out, [&](auto m, auto ms) { dst[ms.value * T * NXC] = v[m.value]; });
        } else {
            slots<R>(sh_out, [&](auto m, auto ms) { dst[ms.value * step] = v[m.value]; });
        }
    };
    if constexpr (PFS) {
        // the next tile's column samples are in flight while this tile is
        // transformed (tiles are disjoint, so in-place use stays safe)
        float2 nxt[R];
        std::uint32_t tile = blockIdx.x;
        if (tile < ntiles) load(tile_off(tile), nxt);
        for (; tile < ntiles; tile += gridDim.x) {
            float2 v[R];
            sfor<R>([&](auto m) { v[m.value] = nxt[m.value]; });
            const std::uint64_t off = tile_off(tile);
            if (tile + gridDim.x < ntiles) load(tile_off(tile + gridDim.x), nxt);
            L::template run<DIR>(v, tw, line, j, [] { __syncthreads(); }, a.scale);
            store(off, v);
        }
    } else {
        for (std::uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            float2 v[R];
            const std::uint64_t off = tile_off(tile);
            load(off, v);
            L::template run<DIR>(v, tw, line, j, [] { __syncthreads(); }, a.scale);
            store(off, v);
        }
    }
}

// ---- axis 0 -------------------------------------------------------------------------------

template <int T>
__device__ __forceinline__ void line_sync() {
    if constexpr (T <= 32)
        __syncwarp();
    else
        __syncthreads();
}

template <int N, int DIR>
__global__ void __launch_bounds__(256) k_fft_contig(ContigArgs a, int lpb, std::uint32_t items) {
    pdl_launch_dependents();
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T;
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int j = tid % T, l = tid / T;
    float2* line = smem + l * row_stride<N>();
    typename L::Twiddles tw;
    L::load_twiddles(tw, a.tw, j, a.scale);
    pdl_wait();  // twiddle tables are init-time constants
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    for (std::uint32_t grp = blockIdx.x; grp * lpb < items; grp += gridDim.x) {
        const std::uint32_t item = grp * lpb + l;
        const bool active = item < items;
        float2 v[R];
        const float2* src = a.in + std::uint64_t(item) * N + j;
        slots_ld<R>(sh_in, (long long)(R / 2) * T,
                    [&](auto m, long long d) { v[m.value] = active ? src[T * m.value + d] : make_float2(0.f, 0.f); });
        L::template run<DIR>(v, tw, line, j, [] { line_sync<T>(); }, a.scale);
        float2* dst = static_cast<float2*>(a.out) + std::uint64_t(item) * N + j;
        if (active) slots<R>(sh_out, [&](auto m, auto ms) { dst[T * ms.value] = v[m.value]; });
    }
}

// ---- axis 0 + coil combine -------------------------------------------------------------------
//
// Output line (y, f) is owned by T threads; they loop over the coils, each
// iteration = load the coil's line of X (axis-1 transformed k-space) and the
// matching line of S, inverse-transform X along x (scale folded into the last
// pass), multiply by conj(S) (or take |X|^2) and accumulate.  ACCF selects
// fp32 instead of fp64 accumulators; PF double-buffers the next coil's X and
// S in registers so their HBM/L2 latency overlaps the current coil's FFT.

// PF: 0 = no prefetch, 1 = next coil copied into registers at the top of each
// iteration, 2 = ping-pong register buffers (loop unrolled by two).
template <int N, int MODE, bool ACCF, int PF, int RQ = default_points(N), int MINB = 1>
__global__ void __launch_bounds__(MINB > 1 ? 128 : 256, MINB > 1 ? MINB : 0) k_fft_combine(ContigArgs a, int lpb, std::uint32_t items) {
    pdl_launch_dependents();
    using L = LineFFT<N, RQ>;
    constexpr int R = L::R, T = L::T;
    constexpr bool SENSE = MODE == int(Combine::Sense);
    using Acc = std::conditional_t<ACCF, float, double>;
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int j = tid % T, l = tid / T;
    float2* line = smem + l * row_stride<N>();
    typename L::Twiddles tw;
    L::load_twiddles(tw, a.tw, j, a.scale);
    pdl_wait();  // twiddle tables are init-time constants
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    const std::uint32_t C = std::uint32_t(a.coils);
    const std::uint32_t ny = std::uint32_t(a.ny);
    const IndexSplit ysplit(ny);
    const std::uint64_t coil_stride = std::uint64_t(ny) * N;  // elements between coils (X and S)
    for (std::uint32_t grp = blockIdx.x; grp * lpb < items; grp += gridDim.x) {
        const std::uint32_t item = grp * lpb + l;
        const bool active = item < items;
        // inactive lines re-read line 0 (valid memory) and skip the store
        std::uint32_t f, y;
        ysplit.split(active ? item : 0u, f, y);
        const float2* xbase = a.in + (std::uint64_t(f) * C * ny + y) * N + j;
        const float2* sbase = a.smap + std::uint64_t(y) * N + j;
        auto load_x = [&](std::uint32_t c, float2(&d)[R]) {
            const float2* src = xbase + c * coil_stride;
            slots_ld<R>(sh_in, (long long)(R / 2) * T, [&](auto m, long long o) { d[m.value] = __ldcs(src + T * m.value + o); });
        };
        auto load_s = [&](std::uint32_t c, float2(&d)[R]) {
            const float2* src = sbase + c * coil_stride;
            slots_ld<R>(sh_out, (long long)(R / 2) * T, [&](auto m, long long o) { d[m.value] = __ldg(src + T * m.value + o); });
        };
        Acc acc_re[R], acc_im[R];
        sfor<R>([&](auto m) {
            acc_re[m.value] = Acc(0);
            acc_im[m.value] = Acc(0);
        });
        // one coil: inverse FFT of x (in place) and accumulate against s
        using SBuf = float2[SENSE ? R : 1];
        auto process = [&](float2(&x)[R], SBuf& sv, std::uint32_t c) {
            L::template run<+1>(x, tw, line, j, [] { line_sync<T>(); }, a.scale);
            if constexpr (SENSE) {
                if constexpr (!PF) {
                    asm volatile("" ::: "memory");  // keep S loads after the FFT (register pressure)
                    load_s(c, sv);
                }
                sfor<R>([&](auto m) {
                    const float2 xv = x[m.value];
                    const float2 s = sv[m.value];
                    if constexpr (ACCF) {
                        mac_conj(acc_re[m.value], acc_im[m.value], xv, s);
                    } else {
                        // x * conj(s) with the reference's rounding (kernel_abi.h:123-125)
                        const float nsi = -s.y;
                        const float re = __fsub_rn(__fmul_rn(xv.x, s.x), __fmul_rn(xv.y, nsi));
                        const float im = __fadd_rn(__fmul_rn(xv.x, nsi), __fmul_rn(xv.y, s.x));
                        acc_re[m.value] = __dadd_rn(acc_re[m.value], double(re));
                        acc_im[m.value] = __dadd_rn(acc_im[m.value], double(im));
                    }
                });
            } else {
                sfor<R>([&](auto m) {
                    const float2 xv = x[m.value];
                    if constexpr (ACCF) {
                        mac_abs2(acc_re[m.value], xv);
                    } else {
                        const double re = xv.x, im = xv.y;
                        acc_re[m.value] =
                            __dadd_rn(acc_re[m.value], __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
                    }
                });
            }
        };
        if constexpr (PF == 1) {
            float2 xn[R];
            SBuf sn;
            load_x(0, xn);
            if constexpr (SENSE) load_s(0, sn);
            for (std::uint32_t c = 0; c < C; ++c) {
                float2 v[R];
                SBuf sv;
                sfor<R>([&](auto m) { v[m.value] = xn[m.value]; });
                if constexpr (SENSE) sfor<R>([&](auto m) { sv[m.value] = sn[m.value]; });
                if (c + 1 < C) {
                    load_x(c + 1, xn);
                    if constexpr (SENSE) load_s(c + 1, sn);
                }
                process(v, sv, c);
            }
        } else if constexpr (PF == 2) {
            // ping-pong register buffers: coil c+1 is in flight while c is transformed
            float2 xa[R], xb[R];
            SBuf sa, sb;
            load_x(0, xa);
            if constexpr (SENSE) load_s(0, sa);
            for (std::uint32_t c = 0; c < C; c += 2) {
                const bool has_b = c + 1 < C;
                if (has_b) {
                    load_x(c + 1, xb);
                    if constexpr (SENSE) load_s(c + 1, sb);
                }
                process(xa, sa, c);
                if (has_b) {
                    if (c + 2 < C) {
                        load_x(c + 2, xa);
                        if constexpr (SENSE) load_s(c + 2, sa);
                    }
                    process(xb, sb, c + 1);
                }
            }
        } else {
            for (std::uint32_t c = 0; c < C; ++c) {
                float2 v[R];
                SBuf sv;
                load_x(c, v);
                process(v, sv, c);
            }
        }
        if (active) {
            if constexpr (SENSE) {
                float2* dst = static_cast<float2*>(a.out) + (std::uint64_t(f) * ny + y) * N + j;
                slots<R>(sh_out, [&](auto m, auto ms) {
                    dst[T * ms.value] = make_float2(float(acc_re[m.value]), float(acc_im[m.value]));
                });
            } else {
                float* dst = static_cast<float*>(a.out) + (std::uint64_t(f) * ny + y) * N + j;
                slots<R>(sh_out, [&](auto m, auto ms) { dst[T * ms.value] = float(sqrt(double(acc_re[m.value]))); });
            }
        }
    }
}

// ---- shared dispatch helpers ----------------------------------------------------------------

// Powers of two, plus the mixed-radix sides 3*2^k / 5*2^k of common MR
// matrices (96, 160 -- the paper's cine --, 192, 320, 384).
#define HETRECO_FFT_SIZES(X) \
    X(1) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) \
    X(96) X(160) X(192) X(320) X(384)

// Sizes that also get the tuning variants (R = 8 plans, register prefetch).
template <int N>
constexpr bool has_variants() {
    return N == 256 || N == 512;
}

template <class K>
inline int blocks_per_sm(K kernel, int block, int smem) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, smem) != cudaSuccess) {
        cudaGetLastError();
        n = 1;
    }
    return n > 0 ? n : 1;
}

inline int env_int(const char* name, int fallback) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : fallback;
}

// points per thread actually used for size N when `rq` is requested
inline int points_for(std::uint64_t N, int rq) {
    switch (N) {
#define X(n) \
    case n: return (rq == 8 && has_variants<n>()) ? 8 : LineFFT<n>::R;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return 0;
}

inline int stride_of(std::uint64_t N) {
    switch (N) {
#define X(n) \
    case n: return line_stride<n>();
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return 0;
}

inline int row_stride_of(std::uint64_t N) {
    switch (N) {
#define X(n) \
    case n: return row_stride<n>();
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return 0;
}

// Combine kernels (fft_combine_*.cu).  variant bit 0 = fp32 accumulators,
// bit 1 = register prefetch, bit 2 = 8 points per thread.
int combine_occupancy(Combine mode, std::uint64_t N, int variant, int block, int smem);
cudaError_t combine_launch(Combine mode, std::uint64_t N, int variant, const ContigArgs& a, const LaunchShape& s,
                           int lpb, std::uint32_t items, cudaStream_t st);

}  // namespace hetreco::dev
