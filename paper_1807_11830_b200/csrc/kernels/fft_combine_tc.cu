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
// CTA = 128 threads = the 128 TMEM lanes.  A "step" is one group of 8 coils
// of one output line (y, f); a CTA walks its lines' steps as a 3-deep
// software pipeline, one block barrier per step:
//   P1(k)   thread (c, b) splits x_c[16a+b] (prefetched a step earlier) and
//           tcgen05.st's hi/lo into TMEM A1[k%2];
//   P2(k-1) waits MMA1(k-1), tcgen05.ld's D1, twiddles, splits and stores the
//           transposed rows (c, p) into the shared-memory A2[(k-1)%2] (K-chunk
//           stride padded by 16 B: the 16 b-threads hit 16 banks);
//   P3(k-2) waits MMA2(k-2), tcgen05.ld's D2 row (c, p) and accumulates
//           conj(S) Z (S prefetched by P2 a step earlier; P3 runs before P2);
//   barrier; one thread issues MMA1(k) (12 tcgen05.mma: 4 K-steps x 3 split
//   terms, A from TMEM) and MMA2(k-1) (A from shared memory), each committed
//   to its buffer's mbarrier.  Nobody waits for an MMA issued in the same
//   step.  At the end of a line the 32 coil partials are summed through
//   shuffles and a (line-parity double-buffered) shared tile, finalised one
//   step later.
// Reference arithmetic being matched: kernels/fft_radix2_pass.cl.src:29-49
// (the butterflies), complex_element_prod.cl.src:9-19 + ximage_sum.cl.src:
// 6-23 (the combine); tolerance max|d|/max|ref| <= 1e-5 (north_star).
#include "fft_kernels.cuh"
#include "tcgen05.cuh"

namespace hetreco::dev {

namespace {

constexpr int kTcThreads = 128;
constexpr std::uint32_t kA2Lbo = 128 * 16 + 16;  // stage-2 A: K-chunk stride (128 rows x 16 B + pad)
constexpr std::uint32_t kA2Bytes = 8 * kA2Lbo;    // one A2 tile (hi or lo)
constexpr std::uint32_t kOffBhi = 0, kOffBlo = 4096;
constexpr std::uint32_t kOffA2 = 8192;                        // [2 buffers][hi, lo]
constexpr std::uint32_t kOffTw = kOffA2 + 4 * kA2Bytes;       // W256 table, rows padded to 17
constexpr std::uint32_t kOffRed = kOffTw + 16 * 17 * 8;       // [2][4 warps][256] float2
constexpr std::uint32_t kOffBar = kOffRed + 2 * 4 * 256 * 8;  // bar1[2], bar2[2]
constexpr std::uint32_t kOffSlot = kOffBar + 4 * 8;
constexpr std::uint32_t kSmemUsed = kOffSlot + 8;
// > 228 KB / 3: at most 2 CTAs per SM, so 2 x 256 TMEM columns never oversubscribe
constexpr int kTcSmem = 96 * 1024;
static_assert(kSmemUsed <= std::uint32_t(kTcSmem), "smem layout");
constexpr std::uint32_t kTmemCols = 256;  // A1 (hi|lo) x2 @0,64 | D1 x2 @128,160 | D2 x2 @192,224

template <bool SHIN, bool SHOUT>
__global__ void __launch_bounds__(kTcThreads, 2) k_fft_combine_tc(ContigArgs a, std::uint32_t units) {
    pdl_launch_dependents();
    extern __shared__ __align__(1024) unsigned char sm[];
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    float* bhi = reinterpret_cast<float*>(sm + kOffBhi);
    float* blo = reinterpret_cast<float*>(sm + kOffBlo);
    float2* tw = reinterpret_cast<float2*>(sm + kOffTw);
    float2* red = reinterpret_cast<float2*>(sm + kOffRed);
    std::uint32_t* slot = reinterpret_cast<std::uint32_t*>(sm + kOffSlot);
    const std::uint32_t bar1 = tc::smem_u32(sm + kOffBar), bar2 = bar1 + 16;  // [2] each, 8 B apart

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
    if (tid == 0)
        for (int i = 0; i < 4; ++i) tc::mbar_init(bar1 + 8 * i, 1);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    pdl_wait();

    const std::uint32_t tbase = *slot;
    const std::uint32_t lane = std::uint32_t(w * 32) << 16;
    constexpr std::uint32_t idesc = tc::idesc_tf32(128, 32);
    const std::uint32_t sb_hi = tc::smem_u32(bhi), sb_lo = tc::smem_u32(blo);
    const std::uint32_t sa = tc::smem_u32(sm + kOffA2);
    const std::uint32_t C = std::uint32_t(a.coils), ny = std::uint32_t(a.ny), F = std::uint32_t(a.frames);
    const std::uint32_t G = (C + 7) / 8;  // coil groups (steps) per line
    const int b = l & 15;                 // P1/P2 row (coil cl of the group, b); P3 row (cl, p = b)
    const int cl = 2 * w + (l >> 4);
    const float2* twb = tw + 17 * b;
    const std::uint32_t my_units = blockIdx.x < units ? (units - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const std::uint32_t steps = my_units * G;

    // step -> (line y, f; coil group g)
    auto line_of = [&](std::uint32_t s, std::uint32_t& y, std::uint32_t& f, std::uint32_t& g) {
        const std::uint32_t i = s / G;
        g = s - i * G;
        const std::uint32_t unit = blockIdx.x + i * gridDim.x;
        y = unit / F;  // concurrently resident CTAs share y (S rows are L2 hits)
        f = unit - y * F;
    };
    float xv[32];
    auto load_x = [&](std::uint32_t s) {
        std::uint32_t y, f, g;
        line_of(s, y, f, g);
        const std::uint32_t c = 8 * g + std::uint32_t(cl);
        if (s < steps && c < C) {
            const float2* src = a.in + (std::uint64_t(f * C + c) * ny + y) * 256 + b;
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
    float2 sv[16];
    auto load_s = [&](std::uint32_t s) {
        std::uint32_t y, f, g;
        line_of(s, y, f, g);
        const std::uint32_t c = 8 * g + std::uint32_t(cl);
        if (s < steps && c < C) {
            const float2* srow = a.smap + (std::uint64_t(c) * ny + y) * 256 + b;
#pragma unroll
            for (int q = 0; q < 16; ++q) sv[q] = __ldg(srow + 16 * (SHOUT ? ((q + 8) & 15) : q));
        } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) sv[q] = make_float2(0.f, 0.f);
        }
    };
    auto finalise = [&](int i) {  // sum line i's 4 warp partials -> out
        const std::uint32_t unit = blockIdx.x + std::uint32_t(i) * gridDim.x;
        const std::uint32_t y = unit / F, f = unit - y * F;
        const float2* rb = red + (i & 1) * 1024;
        float2* dst = static_cast<float2*>(a.out) + (std::uint64_t(f) * ny + y) * 256;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = tid + h * kTcThreads;
            float2 s = rb[e];
#pragma unroll
            for (int ww = 1; ww < 4; ++ww) s = cadd(s, rb[ww * 256 + e]);
            dst[e] = cscale(s, a.scale);
        }
    };
    float acr[16], aci[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acr[q] = aci[q] = 0.f;
    int pending_line = -1;  // line whose partials sit in red[line & 1], finalised after the next barrier

    load_x(0);
    for (std::uint32_t k = 0; k < steps + 2; ++k) {
        if (pending_line >= 0) {
            finalise(pending_line);
            pending_line = -1;
        }
        // ---- P1(k): split + tcgen05.st into A1[k % 2] ----
        if (k < steps) {
            std::uint32_t hi[32], lo[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) tc::split_tf32(xv[q], hi[q], lo[q]);
            const std::uint32_t tA1 = tbase + (k & 1) * 64;
            tc::st32(tA1 + lane, hi);
            tc::st32(tA1 + 32 + lane, lo);
            load_x(k + 1);  // next step's samples in flight
        }
        // ---- P3(k-2): D2 row (c, p) -> conj(S) Z accumulation (before P2 reloads sv) ----
        if (k >= 2) {
            const std::uint32_t s = k - 2, buf = s & 1;
            tc::mbar_wait(bar2 + 8 * buf, (s >> 1) & 1);
            tc::fence_after();
            std::uint32_t d[32];
            tc::ld32(tbase + 192 + buf * 32 + lane, d);
            tc::wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q)
                mac_conj(acr[q], aci[q], make_float2(__uint_as_float(d[2 * q]), __uint_as_float(d[2 * q + 1])), sv[q]);
            const std::uint32_t i = s / G;
            if (s - i * G == G - 1) {  // last coil group of line i: warp partials -> red[i & 1]
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    acr[q] += __shfl_xor_sync(0xffffffffu, acr[q], 16);
                    aci[q] += __shfl_xor_sync(0xffffffffu, aci[q], 16);
                }
                float2* rb = red + (i & 1) * 1024 + w * 256 + b;
                if (l < 16) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) rb[16 * (SHOUT ? ((q + 8) & 15) : q)] = make_float2(acr[q], aci[q]);
                }
#pragma unroll
                for (int q = 0; q < 16; ++q) acr[q] = aci[q] = 0.f;
                pending_line = int(i);
            }
        }
        // ---- P2(k-1): D1 -> twiddle -> split -> A2[(k-1) % 2] ----
        if (k >= 1 && k - 1 < steps) {
            const std::uint32_t s = k - 1, buf = s & 1;
            tc::mbar_wait(bar1 + 8 * buf, (s >> 1) & 1);
            tc::fence_after();
            std::uint32_t d[32];
            tc::ld32(tbase + 128 + buf * 32 + lane, d);
            load_s(s);  // this step's maps, consumed in P3 next iteration
            tc::wait_ld();
            unsigned char* a2hi = sm + kOffA2 + buf * 2 * kA2Bytes;
            unsigned char* a2lo = a2hi + kA2Bytes;
            const std::uint32_t kofs = std::uint32_t(b >> 1) * kA2Lbo + std::uint32_t(b & 1) * 8;
            const std::uint32_t rowbase = std::uint32_t(cl) * 16;
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
        // ---- barrier, then one thread issues MMA1(k) and MMA2(k-1) ----
        tc::wait_st();
        tc::fence_proxy_async();
        tc::fence_before();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            if (k < steps) {
                const std::uint32_t buf = k & 1, tA1 = tbase + buf * 64, tD1 = tbase + 128 + buf * 32;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const std::uint64_t bh = tc::sdesc(sb_hi + kk * 1024, 512, 128);
                    const std::uint64_t bl = tc::sdesc(sb_lo + kk * 1024, 512, 128);
                    tc::mma_ts(tD1, tA1 + 8 * kk, bh, idesc, kk > 0);
                    tc::mma_ts(tD1, tA1 + 8 * kk, bl, idesc, 1);
                    tc::mma_ts(tD1, tA1 + 32 + 8 * kk, bh, idesc, 1);
                }
                tc::commit(bar1 + 8 * buf);
            }
            if (k >= 1 && k - 1 < steps) {
                const std::uint32_t buf = (k - 1) & 1, tD2 = tbase + 192 + buf * 32;
                const std::uint32_t ahi = sa + buf * 2 * kA2Bytes, alo = ahi + kA2Bytes;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const std::uint64_t ah = tc::sdesc(ahi + kk * 2 * kA2Lbo, kA2Lbo, 128);
                    const std::uint64_t al = tc::sdesc(alo + kk * 2 * kA2Lbo, kA2Lbo, 128);
                    const std::uint64_t bh = tc::sdesc(sb_hi + kk * 1024, 512, 128);
                    const std::uint64_t bl = tc::sdesc(sb_lo + kk * 1024, 512, 128);
                    tc::mma_ss(tD2, ah, bh, idesc, kk > 0);
                    tc::mma_ss(tD2, ah, bl, idesc, 1);
                    tc::mma_ss(tD2, al, bh, idesc, 1);
                }
                tc::commit(bar2 + 8 * buf);
            }
        }
        __syncwarp();
    }
    if (pending_line >= 0) finalise(pending_line);  // written in the final step, before its barrier
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
    s.grid = int(std::max<std::uint64_t>(1, std::min<std::uint64_t>(units, std::uint64_t(sms) * 2)));
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
