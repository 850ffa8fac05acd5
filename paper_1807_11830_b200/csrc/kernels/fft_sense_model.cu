// fft_sense_model.cu -- the SENSE forward model E = P F S and the pieces of
// the normal operator E^H E used by iterative reconstruction (SURVEY.md
// §8 f.1; the reference has no such process -- its building blocks are
// complex_element_prod.cl.src (S . m) and fft_radix2_pass.cl.src (F)).
//
//   k_fft_expand          : line (y, c, f) = F_x( S[:, y, c] * M[:, y, f] ), the
//                           coil expansion fused into the axis-0 forward pass
//                           (the product uses the reference rounding,
//                           kernel_abi.h:123-125).
//   k_fft_strided_masked  : axis-1 forward FFT with the k-space sampling mask
//                           applied at the store; or (roundtrip) forward FFT,
//                           mask, inverse FFT in registers -- F_y^-1 P F_y with
//                           no k-space round trip through HBM.  The inverse uses
//                           the forward twiddles via F^-1(z) = conj(F(conj z)).
#include "fft_kernels.cuh"

namespace hetreco::dev {

namespace {

__device__ __forceinline__ float2 cmul_ref(float2 a, float2 b) {
    return make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                       __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
}

template <int N>
__global__ void __launch_bounds__(256) k_fft_expand(ContigArgs a, int lpb, std::uint32_t items) {
    pdl_launch_dependents();
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T;
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int j = tid % T, l = tid / T;
    float2* line = smem + l * row_stride<N>();
    typename L::Twiddles tw;
    L::load_twiddles(tw, a.tw, j, 1.0f);
    pdl_wait();  // twiddle tables are init-time constants
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    const std::uint32_t ny = std::uint32_t(a.ny), C = std::uint32_t(a.coils);
    const IndexSplit ysplit(ny);
    for (std::uint32_t grp = blockIdx.x; grp * lpb < items; grp += gridDim.x) {
        const std::uint32_t item = grp * lpb + l;  // = y + ny * (c + C * f)
        const bool active = item < items;
        const std::uint32_t it = active ? item : 0;
        std::uint32_t y, rest;
        ysplit.split(it, rest, y);
        const std::uint32_t c = rest % C, f = rest / C;
        const float2* mrow = a.in + (std::uint64_t(f) * ny + y) * N + j;
        const float2* srow = a.smap + (std::uint64_t(c) * ny + y) * N + j;
        float2 v[R];
        slots_ld<R>(sh_in, (long long)(R / 2) * T, [&](auto m, long long d) {
            v[m.value] = cmul_ref(__ldg(srow + T * m.value + d), mrow[T * m.value + d]);
        });
        L::template run<-1>(v, tw, line, j, [] { line_sync<T>(); }, 1.0f);
        float2* dst = static_cast<float2*>(a.out) + std::uint64_t(it) * N + j;
        if (active) slots<R>(sh_out, [&](auto m, auto ms) { dst[T * ms.value] = v[m.value]; });
    }
}

template <int N, bool RT>
__global__ void __launch_bounds__(256) k_fft_strided_masked(StridedArgs a, int tx, std::uint32_t ntiles) {
    pdl_launch_dependents();
    using L = LineFFT<N>;
    constexpr int R = L::R, T = L::T;
    constexpr std::uint32_t NX = N;  // square images
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int l = tid % tx, j = tid / tx;
    float2* line = smem + l * line_stride<N>();
    typename L::Twiddles tw;  // forward twiddles, scale 1
    L::load_twiddles(tw, a.tw, j, 1.0f);
    pdl_wait();  // twiddle tables are init-time constants
    const std::uint32_t xtiles = NX / std::uint32_t(tx);
    const IndexSplit xsplit(xtiles);
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    const float scale = a.scale;
    for (std::uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        std::uint32_t plane, xt;
        xsplit.split(tile, plane, xt);
        const std::uint32_t col = xt * std::uint32_t(tx) + std::uint32_t(l);
        const std::uint64_t off = std::uint64_t(plane) * NX * N + col + std::uint32_t(j) * NX;
        const float2* src = a.in + off;
        float2 v[R];
        slots_ld<R>(sh_in, (long long)(R / 2) * T * NX,
                    [&](auto m, long long d) { v[m.value] = __ldcs(src + m.value * T * NX + d); });
        L::template run<-1>(v, tw, line, j, [] { __syncthreads(); });
        // mask at the displayed k-space position (fftshift'ed when shifting)
        const float* mrow = a.mask ? a.mask + col + std::uint32_t(j) * NX : nullptr;
        if constexpr (RT) {
            // conj(mask . X): the forward FFT of it, conjugated, is the inverse
            slots<R>(sh_out, [&](auto m, auto ms) {
                const float mk = mrow ? __ldg(mrow + ms.value * T * NX) : 1.0f;
                v[m.value] = make_float2(v[m.value].x * mk, -v[m.value].y * mk);
            });
            L::template run<-1>(v, tw, line, j, [] { __syncthreads(); });
            float2* dst = a.out + off;
            slots<R>(sh_out, [&](auto m, auto ms) {
                dst[ms.value * T * NX] = make_float2(v[m.value].x * scale, -v[m.value].y * scale);
            });
        } else {
            float2* dst = a.out + off;
            slots<R>(sh_out, [&](auto m, auto ms) {
                const float mk = mrow ? __ldg(mrow + ms.value * T * NX) : 1.0f;
                dst[ms.value * T * NX] = make_float2(v[m.value].x * mk * scale, v[m.value].y * mk * scale);
            });
        }
    }
}

}  // namespace

LaunchShape plan_strided_masked(std::uint64_t N, bool rt, std::uint64_t planes, int sms) {
    LaunchShape s;
    const int R = points_for(N, 0);
    if (R == 0) return s;
    s.rq = R;
    const int T = int(N) / R;
    const int ls_bytes = stride_of(N) * 8;
    std::uint64_t tx = std::max(16, 256 / T);
    tx = std::min<std::uint64_t>(tx, std::uint64_t(std::max(1, 256 / T)));
    tx = std::min<std::uint64_t>(tx, std::uint64_t(std::max(1, (100 * 1024) / ls_bytes)));
    tx = std::max<std::uint64_t>(1, std::min<std::uint64_t>(tx, N));
    s.block = int(tx) * T;
    s.smem = int(tx) * ls_bytes;
    int occ = 1;
    switch (N) {
#define X(n)                                                                                        \
    case n:                                                                                         \
        occ = rt ? blocks_per_sm(k_fft_strided_masked<n, true>, s.block, s.smem)                    \
                 : blocks_per_sm(k_fft_strided_masked<n, false>, s.block, s.smem);                  \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    const std::uint64_t tiles = (N / tx) * planes;
    s.grid = int(std::max<std::uint64_t>(1, std::min<std::uint64_t>(tiles, std::uint64_t(sms) * occ)));
    return s;
}

LaunchShape plan_expand(std::uint64_t N, std::uint64_t items, int sms) {
    LaunchShape s;
    const int R = points_for(N, 0);
    if (R == 0) return s;
    s.rq = R;
    const int T = int(N) / R;
    int lpb = std::max(1, 128 / T);
    const int min_lpb = std::max(1, 32 / T);
    while (lpb > min_lpb && (items + lpb - 1) / lpb < std::uint64_t(2 * sms)) lpb >>= 1;
    s.block = lpb * T;
    s.smem = lpb * row_stride_of(N) * 8;
    int occ = 1;
    switch (N) {
#define X(n) \
    case n: occ = blocks_per_sm(k_fft_expand<n>, s.block, s.smem); break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    const std::uint64_t groups = (items + lpb - 1) / lpb;
    s.grid = int(std::max<std::uint64_t>(1, std::min<std::uint64_t>(groups, std::uint64_t(sms) * occ)));
    return s;
}

cudaError_t launch_expand(std::uint64_t N, const ContigArgs& a, const LaunchShape& s, cudaStream_t st) {
    if (s.block == 0 || s.rq == 0) return cudaErrorInvalidValue;
    const int T = int(N) / s.rq;
    const int lpb = s.block / T;
    const std::uint64_t items64 = a.ny * a.coils * a.frames;
    if (items64 >= (std::uint64_t(1) << 32)) return cudaErrorInvalidValue;
    const std::uint32_t items = std::uint32_t(items64);
    switch (N) {
#define X(n) \
    case n: k_fft_expand<n><<<s.grid, s.block, s.smem, st>>>(a, lpb, items); break;
        HETRECO_FFT_SIZES(X)
#undef X
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_strided_masked(std::uint64_t N, bool rt, const StridedArgs& a, const LaunchShape& s,
                                  cudaStream_t st) {
    if (s.block == 0 || s.rq == 0 || a.nx != N) return cudaErrorInvalidValue;
    const int T = int(N) / s.rq;
    const int tx = s.block / T;
    const std::uint64_t tiles64 = (a.nx / tx) * a.planes;
    if (tiles64 >= (std::uint64_t(1) << 32)) return cudaErrorInvalidValue;
    const std::uint32_t tiles = std::uint32_t(tiles64);
    switch (N) {
#define X(n)                                                                              \
    case n:                                                                               \
        if (rt)                                                                           \
            k_fft_strided_masked<n, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);  \
        else                                                                              \
            k_fft_strided_masked<n, false><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles); \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace hetreco::dev
