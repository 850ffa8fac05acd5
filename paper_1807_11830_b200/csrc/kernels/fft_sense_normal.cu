// fft_sense_normal.cu -- the SENSE normal operator E^H E m in ONE persistent
// cooperative kernel (C4, the iterative loop: VERDICT r1 next #5).
//
// The three-kernel form (fft_sense_model.cu: expand + x-FFT, y-FFT . mask .
// y-IFFT, x-IFFT + conj(S) combine) moves 3 x 4 MiB at 256^2 x 8 coils and
// is latency-bound: each pass is a fraction of a wave and every kernel
// boundary drains the GPU.  MEASURED SLOWER (profiles/round2_c4.md): the
// cooperative launch + two grid barriers alone cost 4.6 us, so this path is
// opt-in (HETRECO_NORMAL_FUSED=1) and the PDL-linked three-kernel graph stays
// the default (12.8 us per launch).  Here one grid of resident CTAs runs the three
// phases back to back, separated by grid-wide barriers; the 4 MiB coil-image
// scratch stays in L2 between phases (reads after a barrier bypass L1 with
// ld.global.cg, since other SMs wrote the lines).
//
//   phase A  z[:, y, c, f] = F_x( S[:, y, c] . m[:, y, f] )      (lines of x)
//   phase B  z[x, :, c, f] = F_y^-1 P F_y z[x, :, c, f]           (tiles of columns)
//   phase C  out[:, y, f]  = 1/(nx ny) sum_c conj(S_c) F_x^-1 z   (coil groups in parallel,
//                                                                   partials summed in group order)
// Same arithmetic as the three kernels (the S . m product with the reference
// rounding, complex_element_prod.cl.src:9-19; the FFT butterflies of
// fft_radix2_pass.cl.src:29-49 as radix-16 Stockham passes).
#include <cooperative_groups.h>

#include "fft_kernels.cuh"

namespace hetreco::dev {

namespace {

namespace cg = cooperative_groups;

constexpr int kNormThreads = 256;

__device__ __forceinline__ float2 cmul_rn(float2 a, float2 b) {
    return make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                       __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
}

template <int N, int RQ>
__global__ void __launch_bounds__(kNormThreads, N <= 256 ? 2 : 1) k_sense_normal_fused(SenseNormalArgs a) {
    using L = LineFFT<N, RQ>;
    constexpr int R = L::R, T = L::T;
    constexpr int LPB = kNormThreads / T;  // lines (phases A, C: coil groups; B: columns) per CTA
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const bool sh = a.shift;
    const std::uint32_t C = a.coils, F = a.frames;
    constexpr std::uint32_t NY = N;
    const std::uint32_t planes = C * F;
    float2* z = a.z;
    typename L::Twiddles tw;
    cg::grid_group grid = cg::this_grid();

    // ---- phase A: coil expansion + forward x-FFT, one line per T threads ----
    if (a.phases & 1) {
        const int j = tid % T, l = tid / T;
        float2* line = smem + l * (L::padded_len | 1);
        L::load_twiddles(tw, a.tw_fwd, j, 1.0f);
        const std::uint32_t items = NY * planes;  // item = y + NY * (c + C * f)
        for (std::uint32_t base = blockIdx.x * LPB; base < items; base += gridDim.x * LPB) {
            const std::uint32_t item = base + std::uint32_t(l);
            const bool active = item < items;
            const std::uint32_t it = active ? item : 0;
            const std::uint32_t y = it % NY, rest = it / NY;
            const std::uint32_t c = rest % C, f = rest / C;
            const float2* mrow = a.m + (std::uint64_t(f) * NY + y) * N + j;
            const float2* srow = a.s + (std::uint64_t(c) * NY + y) * N + j;
            float2 v[R];
            slots_ld<R>(sh, (long long)(R / 2) * T, [&](auto m, long long d) {
                v[m.value] = cmul_rn(__ldg(srow + T * m.value + d), __ldg(mrow + T * m.value + d));
            });
            L::template run<-1>(v, tw, line, j, [] { line_sync<T>(); }, 1.0f);
            float2* dst = z + std::uint64_t(it) * N + j;
            if (active) slots<R>(sh, [&](auto m, auto ms) { dst[T * ms.value] = v[m.value]; });
        }
    }
    grid.sync();

    // ---- phase B: y-FFT, k-space mask, y-IFFT of LPB-column tiles (in place) ----
    if (a.phases & 2) {
        constexpr int TX = LPB;
        const int l = tid % TX, j = tid / TX;
        float2* line = smem + l * (L::padded_len | 1);
        L::load_twiddles(tw, a.tw_fwd, j, 1.0f);
        const std::uint32_t xtiles = N / TX;
        const std::uint32_t tiles = xtiles * planes;
        for (std::uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const std::uint32_t plane = tile / xtiles, xt = tile % xtiles;
            const std::uint32_t col = xt * TX + std::uint32_t(l);
            float2* col0 = z + std::uint64_t(plane) * N * NY + col + std::uint32_t(j) * N;
            float2 v[R];
            slots_ld<R>(sh, (long long)(R / 2) * T * N,
                        [&](auto m, long long d) { v[m.value] = __ldcg(col0 + m.value * T * N + d); });
            L::template run<-1>(v, tw, line, j, [] { __syncthreads(); });
            const float* mrow = a.mask ? a.mask + col + std::uint32_t(j) * N : nullptr;
            // conj(mask . X): its forward FFT, conjugated, is the inverse
            slots<R>(sh, [&](auto m, auto ms) {
                const float mk = mrow ? __ldg(mrow + ms.value * T * N) : 1.0f;
                v[m.value] = make_float2(v[m.value].x * mk, -v[m.value].y * mk);
            });
            L::template run<-1>(v, tw, line, j, [] { __syncthreads(); });
            slots<R>(sh, [&](auto m, auto ms) { col0[ms.value * T * N] = make_float2(v[m.value].x, -v[m.value].y); });
        }
    }
    grid.sync();

    // ---- phase C: inverse x-FFT + conj(S) combine, LPB coil groups per line ----
    if (a.phases & 4) {
        constexpr int G = LPB;
        const int j = tid % T, g = tid / T;
        float2* line = smem + g * (L::padded_len | 1);
        L::load_twiddles(tw, a.tw_inv, j, a.scale);
        const std::uint32_t items = NY * F;
        for (std::uint32_t item = blockIdx.x; item < items; item += gridDim.x) {
            const std::uint32_t y = item % NY, f = item / NY;
            float acc_re[R], acc_im[R];
            sfor<R>([&](auto m) {
                acc_re[m.value] = 0.f;
                acc_im[m.value] = 0.f;
            });
            // coil groups of T <= 32 threads share warps with idle groups when
            // C % G != 0: exchange syncs use the group's own lane mask
            const unsigned gmask = T >= 32 ? 0xffffffffu : (((1u << (T & 31)) - 1u) << ((tid & 31) / T * T));
            for (std::uint32_t c = std::uint32_t(g); c < C; c += G) {
                const float2* src = z + (std::uint64_t(f * C + c) * NY + y) * N + j;
                const float2* sp = a.s + (std::uint64_t(c) * NY + y) * N + j;
                float2 v[R], sv[R];
                slots_ld<R>(sh, (long long)(R / 2) * T, [&](auto m, long long d) { v[m.value] = __ldcg(src + T * m.value + d); });
                slots_ld<R>(sh, (long long)(R / 2) * T, [&](auto m, long long d) { sv[m.value] = __ldg(sp + T * m.value + d); });
                L::template run<+1>(v, tw, line, j, [gmask] { __syncwarp(gmask); }, a.scale);
                sfor<R>([&](auto m) { mac_conj(acc_re[m.value], acc_im[m.value], v[m.value], sv[m.value]); });
            }
            __syncthreads();  // every group is done with its exchange line
            slots<R>(sh, [&](auto m, auto ms) { line[L::pad(j + T * ms.value)] = make_float2(acc_re[m.value], acc_im[m.value]); });
            __syncthreads();
            for (int p = tid; p < N; p += kNormThreads) {
                float re = 0.f, im = 0.f;
                for (int q = 0; q < G; ++q) {
                    const float2 w = smem[q * (L::padded_len | 1) + L::pad(p)];
                    re += w.x;
                    im += w.y;
                }
                a.out[(std::uint64_t(f) * NY + y) * N + p] = make_float2(re, im);
            }
            __syncthreads();  // partial buffers are reused by the next line
        }
    }
}

template <int N>
constexpr bool normal_fused_size() {
    return N >= 64 && N <= 256 && (N & (N - 1)) == 0;  // coil groups within one warp (T <= 32)
}

}  // namespace

// Points per thread: 8 by default (one warp per 256-point line, half the
// serial work of the 16-point threads the streaming kernels use -- these
// phases are latency-bound); HETRECO_NORMAL_POINTS=16 for the A/B.
int normal_points() { return env_int("HETRECO_NORMAL_POINTS", 8) == 16 ? 16 : 8; }

template <int n, int RQ>
void plan_normal_nr(LaunchShape& s, int sms) {
    using L = LineFFT<n, RQ>;
    s.rq = L::R;
    s.block = kNormThreads;
    s.smem = (kNormThreads / L::T) * (L::padded_len | 1) * 8;
    int occ = 0;
    if (s.smem > 48 * 1024)
        cudaFuncSetAttribute(k_sense_normal_fused<n, RQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, s.smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sense_normal_fused<n, RQ>, s.block, s.smem);
    s.grid = sms * occ;
    if (occ < 1) s.block = 0;
}

template <int n>
void plan_normal_n(LaunchShape& s, int sms) {
    if constexpr (normal_fused_size<n>()) {
        if (normal_points() == 16)
            plan_normal_nr<n, 16>(s, sms);
        else
            plan_normal_nr<n, 8>(s, sms);
    }
}

template <int n>
void* normal_kernel(int rq) {
    if constexpr (normal_fused_size<n>()) {
        return rq == LineFFT<n, 16>::R ? (void*)&k_sense_normal_fused<n, 16> : (void*)&k_sense_normal_fused<n, 8>;
    } else {
        return nullptr;
    }
}

LaunchShape plan_sense_normal_fused(std::uint64_t N, std::uint64_t planes, int sms) {
    LaunchShape s;
    (void)planes;
    if (const char* e = std::getenv("HETRECO_NORMAL_FUSED"); !(e && *e == '1')) return s;
    switch (N) {
#define X(n) \
    case n: plan_normal_n<n>(s, sms); break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return s;
}

cudaError_t launch_sense_normal_fused(std::uint64_t N, const SenseNormalArgs& a, const LaunchShape& s,
                                      cudaStream_t st) {
    if (s.block == 0) return cudaErrorInvalidValue;
    void* kern = nullptr;
    switch (N) {
#define X(n) \
    case n: kern = normal_kernel<n>(s.rq); break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    if (!kern) return cudaErrorInvalidValue;
    // cooperative launch: the runtime guarantees every CTA is resident (the
    // grid barriers cannot deadlock) or fails the launch
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(s.grid));
    cfg.blockDim = dim3(unsigned(s.block));
    cfg.dynamicSmemBytes = std::size_t(s.smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SenseNormalArgs args = a;
    void* params[] = {&args};
    return cudaLaunchKernelExC(&cfg, kern, params);
}

}  // namespace hetreco::dev
