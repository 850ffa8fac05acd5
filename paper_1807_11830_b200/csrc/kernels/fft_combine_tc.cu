// fft_combine_tc.cu -- SENSE axis-0 IFFT + combine with the DFTs on the
// tcgen05 tensor cores (the "DFT-as-GEMM" variant north_star asks to be
// measured against the radix path; HETRECO_COMBINE_TC=1, 256-point lines).
//
// 256 = 16 x 16 Cooley-Tukey with n = 16a + b, k = p + 16q:
//   stage 1  Y[c,b,p] = sum_a x_c[16a+b] W16^{ap}        (GEMM, K = a)
//   twiddle  Y'       = Y . W256^{bp}                    (CUDA cores)
//   stage 2  Z[c,p,q] = sum_b Y'[c,b,p] W16^{bq}         (GEMM, K = b)
//   combine  M[p+16q] = scale . sum_c conj(S_c[p+16q]) Z[c,p,q]
// Each stage is a real GEMM D[128 x 32] = A[128 x 32] . B[32 x 32]: rows =
// 8 coils x 16 (b or p), K = 16 complex inputs as (re, im), N = 16 complex
// outputs as (re, im), B = the real form of the 16-point DFT matrix
// [[cos, sin], [-sin, cos]].  fp32 accuracy from tf32 operands by the
// 3-term split (x = hi + lo, hi tf32-exact): A.B ~ Ahi.Bhi + Ahi.Blo + Alo.Bhi,
// per-product error ~2^-21 (the dropped Alo.Blo term and lo's own rounding).
//
// CTA = 128 threads = the 128 TMEM lanes; unit = one output line (y, f),
// coils in groups of 8:
//   - thread (c, b) loads x_c[16a+b] (a = 0..15), splits, tcgen05.st's hi/lo
//     into TMEM columns [0,32) / [32,64) -> stage-1 A;
//   - one thread issues 12 tcgen05.mma (4 K-steps x 3 split terms) into D1,
//     commit -> mbarrier;
//   - thread (c, b) tcgen05.ld's its D1 row, twiddles, splits and stores
//     the transposed rows (c, p) into the stage-2 A tile in shared memory
//     (K-chunk stride padded by 16 B so the 16 b-threads hit 16 banks);
//   - 12 more MMAs into D2; thread (c, p) tcgen05.ld's its row and
//     accumulates conj(S) Z over its coils; the 32 coil partials are summed
//     through shuffles and shared memory at the end of the line.
// Reference arithmetic being matched: kernels/fft_radix2_pass.cl.src:29-49
// (the butterflies), complex_element_prod.cl.src:9-19 + ximage_sum.cl.src:
// 6-23 (the combine); tolerance max|d|/max|ref| <= 1e-5 (north_star).
#include "fft_kernels.cuh"
#include "tcgen05.cuh"

namespace hetreco::dev {

namespace {

constexpr int kTcThreads = 128;
constexpr std::uint32_t kA2Lbo = 128 * 16 + 16;  // stage-2 A: K-chunk stride (128 rows x 16 B + pad)
constexpr std::uint32_t kOffBhi = 0, kOffBlo = 4096, kOffA2hi = 8192;
constexpr std::uint32_t kOffA2lo = kOffA2hi + 8 * kA2Lbo;
constexpr std::uint32_t kOffTw = kOffA2lo + 8 * kA2Lbo;
constexpr std::uint32_t kOffBar = kOffTw + 16 * 17 * 8;  // W256 table, rows padded to 17 (bank spread)
constexpr std::uint32_t kOffSlot = kOffBar + 8;
constexpr std::uint32_t kSmemUsed = kOffSlot + 8;
// 56 KiB per CTA: at most 4 CTAs per SM, so 4 x 128 TMEM columns never oversubscribe
constexpr int kTcSmem = 56 * 1024;
static_assert(kSmemUsed <= std::uint32_t(kTcSmem), "smem layout");
constexpr std::uint32_t kTmemCols = 128;  // A1 hi | A1 lo | D1 | D2, 32 columns each

template <bool SHIN, bool SHOUT>
__global__ void __launch_bounds__(kTcThreads, 3) k_fft_combine_tc(ContigArgs a, std::uint32_t units) {
    pdl_launch_dependents();
    extern __shared__ __align__(1024) unsigned char sm[];
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    float* bhi = reinterpret_cast<float*>(sm + kOffBhi);
    float* blo = reinterpret_cast<float*>(sm + kOffBlo);
    unsigned char* a2hi = sm + kOffA2hi;
    unsigned char* a2lo = sm + kOffA2lo;
    float2* tw = reinterpret_cast<float2*>(sm + kOffTw);
    std::uint32_t* slot = reinterpret_cast<std::uint32_t*>(sm + kOffSlot);
    const std::uint32_t bar = tc::smem_u32(sm + kOffBar);

    // B = real form of the 16-point inverse DFT, K-major core matrices:
    // element (n, k) at float offset (k/4)*128 + n*4 + k%4  (LBO 512 B, SBO 128 B)
    for (int e = tid; e < 1024; e += kTcThreads) {
        const int n = e >> 5, k = e & 31;
        const int p = n >> 1, ro = n & 1, ai = k >> 1, ri = k & 1;
        double s, c;
        sincospi(double((ai * p) & 15) / 8.0, &s, &c);
        const float v = float(ro == 0 ? (ri == 0 ? c : -s) : (ri == 0 ? s : c));
        std::uint32_t h, lo;
        tc::split_tf32(v, h, lo);
        const int off = (k >> 2) * 128 + n * 4 + (k & 3);
        bhi[off] = __uint_as_float(h);
        blo[off] = __uint_as_float(lo);
    }
    for (int e = tid; e < 256; e += kTcThreads) {  // W256^{b p} at tw[17 b + p]
        double s, c;
        sincospi(double((e >> 4) * (e & 15)) / 128.0, &s, &c);
        tw[17 * (e >> 4) + (e & 15)] = make_float2(float(c), float(s));
    }
    if (w == 0) tc::tmem_alloc(slot, kTmemCols);
    if (tid == 0) tc::mbar_init(bar, 1);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    pdl_wait();

    const std::uint32_t tbase = *slot;
    const std::uint32_t lane = std::uint32_t(w * 32) << 16;
    const std::uint32_t tA1 = tbase, tD1 = tbase + 64, tD2 = tbase + 96;
    constexpr std::uint32_t idesc = tc::idesc_tf32(128, 32);
    const std::uint32_t sb_hi = tc::smem_u32(bhi), sb_lo = tc::smem_u32(blo);
    const std::uint32_t sa_hi = tc::smem_u32(a2hi), sa_lo = tc::smem_u32(a2lo);
    const std::uint32_t C = std::uint32_t(a.coils), ny = std::uint32_t(a.ny), F = std::uint32_t(a.frames);
    const std::uint32_t groups = (C + 7) / 8;
    const int b = l & 15;       // stage 1: this thread's row is (coil 2w + l/16 of the group, b)
    const int p = l & 15;       // stage 2: (coil 2w + l/16, p)
    const int cl = 2 * w + (l >> 4);
    std::uint32_t phase = 0;

    for (std::uint32_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
        // concurrently resident CTAs share y (so S rows are L2 hits)
        const std::uint32_t y = unit / F, f = unit - (unit / F) * F;
        float acr[16], aci[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) acr[q] = aci[q] = 0.f;

        float xv[32];
        auto load_x = [&](std::uint32_t gg) {
            const std::uint32_t cc = 8 * gg + std::uint32_t(cl);
            if (gg < groups && cc < C) {
                const float2* src = a.in + (std::uint64_t(f * C + cc) * ny + y) * 256 + b;
#pragma unroll
                for (int ai = 0; ai < 16; ++ai) {
                    const float2 v = __ldcs(src + 16 * (SHIN ? ((ai + 8) & 15) : ai));
                    xv[2 * ai] = v.x;
                    xv[2 * ai + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k) xv[k] = 0.f;
            }
        };
        load_x(0);
        for (std::uint32_t g = 0; g < groups; ++g) {
            const std::uint32_t c = 8 * g + std::uint32_t(cl);
            // ---- stage 1: A1 rows (c, b), K = (a, re/im), into TMEM ----
            {
                std::uint32_t hi[32], lo[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) tc::split_tf32(xv[k], hi[k], lo[k]);
                tc::st32(tA1 + lane, hi);
                tc::st32(tA1 + 32 + lane, lo);
            }
            load_x(g + 1);  // next group's samples in flight during this group's MMAs
            tc::wait_st();
            tc::fence_before();
            __syncthreads();
            if (tid == 0) {
                tc::fence_after();
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const std::uint64_t bh = tc::sdesc(sb_hi + kk * 1024, 512, 128);
                    const std::uint64_t bl = tc::sdesc(sb_lo + kk * 1024, 512, 128);
                    tc::mma_ts(tD1, tA1 + 8 * kk, bh, idesc, kk > 0);
                    tc::mma_ts(tD1, tA1 + 8 * kk, bl, idesc, 1);
                    tc::mma_ts(tD1, tA1 + 32 + 8 * kk, bh, idesc, 1);
                }
                tc::commit(bar);
            }
            tc::mbar_wait(bar, phase);
            phase ^= 1;
            tc::fence_after();
            // ---- twiddle, split, transpose into the stage-2 A tile (smem) ----
            {
                std::uint32_t d[32];
                tc::ld32(tD1 + lane, d);
                tc::wait_ld();
                const float2* twb = tw + 17 * b;
                const std::uint32_t rowbase = std::uint32_t(cl) * 16;
                const std::uint32_t kofs = std::uint32_t(b >> 1) * kA2Lbo + std::uint32_t(b & 1) * 8;
#pragma unroll
                for (int pp = 0; pp < 16; ++pp) {
                    const float2 t = twb[pp];
                    const float yr = __uint_as_float(d[2 * pp]), yi = __uint_as_float(d[2 * pp + 1]);
                    const float zr = fmaf(yr, t.x, -yi * t.y), zi = fmaf(yr, t.y, yi * t.x);
                    std::uint32_t hr, lr, hi_, li;
                    tc::split_tf32(zr, hr, lr);
                    tc::split_tf32(zi, hi_, li);
                    const std::uint32_t m2 = rowbase + std::uint32_t(pp);
                    const std::uint32_t off = kofs + (m2 >> 3) * 128 + (m2 & 7) * 16;
                    *reinterpret_cast<uint2*>(a2hi + off) = make_uint2(hr, hi_);
                    *reinterpret_cast<uint2*>(a2lo + off) = make_uint2(lr, li);
                }
            }
            tc::fence_proxy_async();
            tc::fence_before();
            __syncthreads();
            // this group's map samples S_c[p + 16q] in flight during the stage-2 MMAs
            float2 sv[16];
            if (c < C) {
                const float2* srow = a.smap + (std::uint64_t(c) * ny + y) * 256 + p;
#pragma unroll
                for (int q = 0; q < 16; ++q) sv[q] = __ldg(srow + 16 * (SHOUT ? ((q + 8) & 15) : q));
            }
            if (tid == 0) {
                tc::fence_after();
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const std::uint64_t ah = tc::sdesc(sa_hi + kk * 2 * kA2Lbo, kA2Lbo, 128);
                    const std::uint64_t al = tc::sdesc(sa_lo + kk * 2 * kA2Lbo, kA2Lbo, 128);
                    const std::uint64_t bh = tc::sdesc(sb_hi + kk * 1024, 512, 128);
                    const std::uint64_t bl = tc::sdesc(sb_lo + kk * 1024, 512, 128);
                    tc::mma_ss(tD2, ah, bh, idesc, kk > 0);
                    tc::mma_ss(tD2, ah, bl, idesc, 1);
                    tc::mma_ss(tD2, al, bh, idesc, 1);
                }
                tc::commit(bar);
            }
            tc::mbar_wait(bar, phase);
            phase ^= 1;
            tc::fence_after();
            // ---- combine: row (c, p) holds Z[c, p, q], q = 0..15 ----
            {
                std::uint32_t d[32];
                tc::ld32(tD2 + lane, d);
                tc::wait_ld();
                if (c < C) {
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        mac_conj(acr[q], aci[q], make_float2(__uint_as_float(d[2 * q]), __uint_as_float(d[2 * q + 1])), sv[q]);
                }
            }
            tc::fence_before();  // this group's TMEM reads precede the next group's MMAs
        }
        // ---- sum the 32 coil partials of each output sample ----
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            acr[q] += __shfl_xor_sync(0xffffffffu, acr[q], 16);
            aci[q] += __shfl_xor_sync(0xffffffffu, aci[q], 16);
        }
        float2* red = reinterpret_cast<float2*>(a2hi);  // free: the last stage-2 MMA has completed
        if (l < 16) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
                red[w * 256 + p + 16 * (SHOUT ? ((q + 8) & 15) : q)] = make_float2(acr[q], aci[q]);
        }
        __syncthreads();
        float2* dst = static_cast<float2*>(a.out) + (std::uint64_t(f) * ny + y) * 256;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = tid + h * kTcThreads;
            float2 s = red[e];
#pragma unroll
            for (int ww = 1; ww < 4; ++ww) s = cadd(s, red[ww * 256 + e]);
            dst[e] = cscale(s, a.scale);
        }
        __syncthreads();  // red (the stage-2 A tile) is rewritten by the next line
    }
    tc::fence_before();
    __syncthreads();
    if (w == 0) {
        tc::fence_after();
        tc::tmem_free(tbase, kTmemCols);
    }
}

}  // namespace

bool combine_tc_enabled(std::uint64_t N) {
    if (N != 256) return false;
    const char* e = std::getenv("HETRECO_COMBINE_TC");
    return e && *e == '1';
}

LaunchShape plan_combine_tc(std::uint64_t N, std::uint64_t ny, std::uint64_t frames, int sms) {
    LaunchShape s;
    if (N != 256) return s;
    s.block = kTcThreads;
    s.smem = kTcSmem;
    s.rq = 16;
    const std::uint64_t units = ny * frames;
    s.grid = int(std::max<std::uint64_t>(1, std::min<std::uint64_t>(units, std::uint64_t(sms) * 3)));
    s.variant = 512;
    // per device: plans are made at init() on the process' GPU
    for (auto k : {k_fft_combine_tc<false, false>, k_fft_combine_tc<false, true>, k_fft_combine_tc<true, false>,
                   k_fft_combine_tc<true, true>})
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem) != cudaSuccess) s.block = 0;
    return s;
}

cudaError_t launch_combine_tc(std::uint64_t N, const ContigArgs& a, const LaunchShape& s, cudaStream_t st) {
    if (N != 256 || s.block != kTcThreads || !(s.variant & 512)) return cudaErrorInvalidValue;
    const std::uint64_t units = a.ny * a.frames;
    if (units >= (std::uint64_t(1) << 32)) return cudaErrorInvalidValue;
    const std::uint32_t u = std::uint32_t(units);
    if (a.shift_in)
        a.shift_out ? k_fft_combine_tc<true, true><<<s.grid, s.block, s.smem, st>>>(a, u)
                    : k_fft_combine_tc<true, false><<<s.grid, s.block, s.smem, st>>>(a, u);
    else
        a.shift_out ? k_fft_combine_tc<false, true><<<s.grid, s.block, s.smem, st>>>(a, u)
                    : k_fft_combine_tc<false, false><<<s.grid, s.block, s.smem, st>>>(a, u);
    return cudaGetLastError();
}

}  // namespace hetreco::dev
