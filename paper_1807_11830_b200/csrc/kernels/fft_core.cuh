// fft_core.cuh -- register/shared-memory building blocks of the batched FFT.
//
// A line of N = 2^n complex samples is owned by T = N/R threads; thread j
// keeps R samples in registers, slot m <-> position j + T*m.  The transform
// is a Stockham autosort sequence of radix passes (radix list per N below):
// in a pass of radix Rp after `Ns` points have been combined, thread j runs
// R/Rp in-register DFT_Rp's (groups g = j + s*T), each on slots
// m = s + q*(R/Rp), after multiplying by W_{Ns*Rp}^{(g mod Ns) q}; results go
// to shared position (g/Ns)*Ns*Rp + g%Ns + q*Ns.  Every pass reads slot m from
// position j + T*m, so only passes 2.. touch shared memory, and the last
// pass leaves the output in natural order in the same slots -- first-pass
// loads and last-pass stores are the coalesced pattern j + T*m.
//
// The in-register DFTs are radix-2 DIT with compile-time twiddles; trivial
// twiddles (1, -1, +-i) cost nothing and the (1 +- i)/sqrt2 ones cost 2 FMUL.
//
// This replaces the reference's per-pass, one-butterfly-per-work-item
// formulation (kernels/fft_radix2_pass.cl.src:22-69), which sweeps the whole
// array log2(N)+1 times per axis, with one HBM read and one HBM write per axis.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>
#include <utility>

#include "pdl.cuh"

namespace hetreco::dev {

// ---- compile-time helpers ---------------------------------------------------------

template <class F, int... Is>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
// Calls f(std::integral_constant<int, i>) for i = 0..N-1 (fully unrolled).
template <int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
    sfor_impl(f, std::make_integer_sequence<int, N>{});
}

constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }

constexpr int bitrev_c(int v, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b)
        if (v & (1 << b)) r |= 1 << (bits - 1 - b);
    return r;
}

// cos(2 pi k / 64): first quadrant literal values (17 significant digits),
// the rest by symmetry.
constexpr double kQuarterCos[17] = {
    1.0, 0.9951847266721969, 0.9807852804032304, 0.9569403357322088, 0.9238795325112867,
    0.881921264348355, 0.8314696123025452, 0.773010453362737, 0.7071067811865476,
    0.6343932841636455, 0.5555702330196023, 0.4713967368259978, 0.38268343236508984,
    0.29028467725446233, 0.19509032201612833, 0.09801714032956077, 0.0};

constexpr double cos64(int k) {
    k = ((k % 64) + 64) % 64;
    return k <= 16 ? kQuarterCos[k]
         : k <= 32 ? -kQuarterCos[32 - k]
         : k <= 48 ? -kQuarterCos[k - 32]
                   : kQuarterCos[64 - k];
}
constexpr double sin64(int k) { return cos64(k - 16); }

// ---- complex arithmetic ---------------------------------------------------------------

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

// fp32 coil-combine accumulation, products fused into the sums (4 FFMA per
// sample instead of 4 FMUL + 4 FADD).  acc += x * conj(s)  /  acc += |x|^2.
// The fp64 combine variants keep the reference's separately rounded products
// (complex_element_prod.cl.src + ximage_sum.cl.src) instead.
__device__ __forceinline__ void mac_conj(float& re, float& im, float2 x, float2 s) {
    re = fmaf(x.x, s.x, fmaf(x.y, s.y, re));
    im = fmaf(x.y, s.x, fmaf(-x.x, s.y, im));
}
__device__ __forceinline__ void mac_abs2(float& acc, float2 x) { acc = fmaf(x.x, x.x, fmaf(x.y, x.y, acc)); }

// v * W_N^K with W_N = exp(DIR * 2 pi i / N), N | 64, all at compile time.
template <int N, int K, int DIR>
__device__ __forceinline__ float2 wmul(float2 v) {
    constexpr int k = ((K % N) + N) % N;
    if constexpr (k == 0) {
        return v;
    } else if constexpr (2 * k == N) {
        return make_float2(-v.x, -v.y);
    } else if constexpr (4 * k == N) {  // angle DIR*pi/2
        return DIR > 0 ? make_float2(-v.y, v.x) : make_float2(v.y, -v.x);
    } else if constexpr (4 * k == 3 * N) {  // angle DIR*3pi/2
        return DIR > 0 ? make_float2(v.y, -v.x) : make_float2(-v.y, v.x);
    } else {
        constexpr int idx = k * (64 / N);
        constexpr float c = float(cos64(idx));
        constexpr float s = float(DIR * sin64(idx));
        if constexpr ((8 * k) % N == 0) {
            // odd multiple of pi/4: |c| == |s| == sqrt(2)/2
            constexpr float h = c;  // c = +-h
            constexpr float r = s / c;  // +-1
            return make_float2(h * (v.x - r * v.y), h * (v.y + r * v.x));
        } else {
            return make_float2(fmaf(c, v.x, -s * v.y), fmaf(c, v.y, s * v.x));
        }
    }
}

// Radix-2 butterfly with a compile-time twiddle: (u, b) <- (u + W b, u - W b),
// W = W_N^K (N | 64).  Trivial twiddles (+-1, +-i) cost 4 FADD.  Others use
// the factored form W b = c (b.x - t b.y, b.y + t b.x) with |t| <= 1 (t = s/c,
// or the roles of c and s swapped when |s| > |c|): 2 FFMA for the bracket and
// 4 FFMA for u +- c (.), i.e. 6 FP32 instructions instead of 4 (W b) + 4 (u +- .).
template <int N, int K, int DIR>
__device__ __forceinline__ void bfly_tw(float2& u, float2& b) {
    constexpr int k = ((K % N) + N) % N;
    if constexpr (k == 0 || 2 * k == N || 4 * k == N || 4 * k == 3 * N) {
        const float2 t = wmul<N, K, DIR>(b);
        const float2 x = u;
        u = cadd(x, t);
        b = csub(x, t);
    } else {
        constexpr int idx = k * (64 / N);
        constexpr double c = cos64(idx), s = DIR * sin64(idx);
        constexpr bool cos_major = (c < 0 ? -c : c) >= (s < 0 ? -s : s);
        constexpr float f = float(cos_major ? c : s);        // common factor
        constexpr float t = float(cos_major ? s / c : c / s);  // |t| <= 1
        float2 r;
        if constexpr (cos_major)  // W b = c (b.x - t b.y, b.y + t b.x)
            r = make_float2(fmaf(-t, b.y, b.x), fmaf(t, b.x, b.y));
        else                      // W b = s (t b.x - b.y, t b.y + b.x)
            r = make_float2(fmaf(t, b.x, -b.y), fmaf(t, b.y, b.x));
        const float2 x = u;
        u = make_float2(fmaf(f, r.x, x.x), fmaf(f, r.y, x.y));
        b = make_float2(fmaf(-f, r.x, x.x), fmaf(-f, r.y, x.y));
    }
}

// i * DIR * v  (multiplication by +-i)
template <int DIR>
__device__ __forceinline__ float2 mul_i(float2 v) {
    return DIR > 0 ? make_float2(-v.y, v.x) : make_float2(v.y, -v.x);
}

// In-register DFT of Rp points stored at v[OFF + q*STR], q = 0..Rp-1, natural
// order in and out.  Radix-2 decimation in time for powers of two; direct
// symmetric butterflies for 3 and 5 (W = e^{DIR 2 pi i / Rp}).
template <int Rp, int DIR, int STR, int OFF, int R>
__device__ __forceinline__ void dft_regs(float2 (&v)[R]) {
    if constexpr (Rp == 1) {
        return;
    } else if constexpr (Rp == 3) {
        constexpr float c = -0.5f, sn = 0.86602540378443864676f;  // cos, sin(2 pi / 3)
        const float2 a0 = v[OFF], a1 = v[OFF + STR], a2 = v[OFF + 2 * STR];
        const float2 t1 = cadd(a1, a2), t2 = csub(a1, a2);
        const float2 m = make_float2(fmaf(c, t1.x, a0.x), fmaf(c, t1.y, a0.y));
        const float2 r = mul_i<DIR>(cscale(t2, sn));
        v[OFF] = cadd(a0, t1);
        v[OFF + STR] = cadd(m, r);
        v[OFF + 2 * STR] = csub(m, r);
    } else if constexpr (Rp == 5) {
        constexpr float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;  // cos(2pi/5), cos(4pi/5)
        constexpr float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;   // sin(2pi/5), sin(4pi/5)
        const float2 a0 = v[OFF], a1 = v[OFF + STR], a2 = v[OFF + 2 * STR], a3 = v[OFF + 3 * STR],
                     a4 = v[OFF + 4 * STR];
        const float2 t1 = cadd(a1, a4), t2 = cadd(a2, a3), t3 = csub(a1, a4), t4 = csub(a2, a3);
        const float2 m1 = make_float2(fmaf(c1, t1.x, fmaf(c2, t2.x, a0.x)), fmaf(c1, t1.y, fmaf(c2, t2.y, a0.y)));
        const float2 m2 = make_float2(fmaf(c2, t1.x, fmaf(c1, t2.x, a0.x)), fmaf(c2, t1.y, fmaf(c1, t2.y, a0.y)));
        const float2 r1 = mul_i<DIR>(make_float2(fmaf(s1, t3.x, s2 * t4.x), fmaf(s1, t3.y, s2 * t4.y)));
        const float2 r2 = mul_i<DIR>(make_float2(fmaf(s2, t3.x, -s1 * t4.x), fmaf(s2, t3.y, -s1 * t4.y)));
        v[OFF] = cadd(a0, cadd(t1, t2));
        v[OFF + STR] = cadd(m1, r1);
        v[OFF + 4 * STR] = csub(m1, r1);
        v[OFF + 2 * STR] = cadd(m2, r2);
        v[OFF + 3 * STR] = csub(m2, r2);
    } else {
        constexpr int bits = ilog2c(Rp);
        float2 a[Rp];
        sfor<Rp>([&](auto i) { a[i.value] = v[OFF + bitrev_c(i.value, bits) * STR]; });
        sfor<bits>([&](auto st) {
            constexpr int m = 2 << st.value;  // span of this stage
            constexpr int h = m / 2;
            sfor<Rp / m>([&](auto b) {
                sfor<h>([&](auto kk) {
                    constexpr int i0 = b.value * m + kk.value;
                    bfly_tw<m, kk.value, DIR>(a[i0], a[i0 + h]);
                });
            });
        });
        sfor<Rp>([&](auto i) { v[OFF + i.value * STR] = a[i.value]; });
    }
}

// Visits the line positions j + T*ms in increasing ms with the register
// slot m that pairs with it: m = ms, or m = (ms + R/2) mod R when `rot` (a
// cyclic shift by N/2 along the line, i.e. fftshift/ifftshift for even N;
// the rotation is an involution so the pairing is symmetric).  Both branches
// keep compile-time slot offsets, so addresses stay affine.
template <int R, class F>
__device__ __forceinline__ void slots(bool rot, F&& fn) {
    if (rot)
        sfor<R>([&](auto ms) { fn(std::integral_constant<int, (ms.value + R / 2) % R>{}, ms); });
    else
        sfor<R>([&](auto ms) { fn(ms, ms); });
}

// Loads for the same rotation as slots(), written as addresses: slot m reads
// position m + R/2 (m < R/2) or m - R/2 (m >= R/2) when `rot`.  fn(m, d)
// receives d = +-half (the element offset of half a line, or 0): the
// destination register stays compile-time, only the address moves, so a
// prefetching load never needs a data-dependent register permutation (which
// would make the consumer wait for the load right where it is issued).
template <int R, class F>
__device__ __forceinline__ void slots_ld(bool rot, long long half, F&& fn) {
    const long long d = rot ? half : 0;
    sfor<R>([&](auto m) { fn(m, m.value < R / 2 ? d : -d); });
}

// ---- per-size plan ------------------------------------------------------------------------

// Radix lists are derived from (N, R): R points per thread, passes of radix R
// while they divide the remaining length, then one remainder pass.  The
// default R is 16 for N >= 128 (two passes at 256, one shared-memory
// exchange) and 8 below; kernels may ask for R = 8 at N >= 128 (more passes,
// fewer registers per thread).
//
// Mixed radix (N = 3 * 2^k or 5 * 2^k, e.g. the paper's 160 x 160 cine; the
// reference is radix-2 only): one radix-3/5 pass, then
// radix-4 passes and a remainder, with R = 3*4 or 5*4 points per thread so
// every pass radix divides R.  The pass twiddles of these sizes are read from
// the (L1-resident) W_N^t table at the point of use instead of being held in
// registers.
constexpr int default_points(int N) { return N <= 16 ? N : (N <= 64 ? 8 : 16); }

constexpr int odd_part(int N) { return (N > 0 && N % 2 == 0) ? odd_part(N / 2) : N; }
constexpr bool is_mixed_size(int N) { return odd_part(N) != 1; }

template <int N, int RQ>
struct Plan {
    static constexpr int M = odd_part(N);  // 1 (power of two), 3 or 5
    static_assert(M == 1 || M == 3 || M == 5, "FFT sizes are 2^k, 3*2^k or 5*2^k");
    static constexpr int Q = M == 1 ? 0 : (N / M >= 4 ? 4 : N / M);
    static constexpr int R = M == 1 ? (RQ < N ? RQ : N) : M * Q;
    static constexpr int first = M == 1 ? R : M;  // radix of pass 0
    static constexpr int step = M == 1 ? R : Q;   // radix of the passes after it
    static constexpr int radix(int p) {
        int n = N;
        for (int i = 0; i <= p; ++i) {
            const int r = i == 0 ? (first < n ? first : n) : (n >= step ? step : n);
            if (i == p) return r;
            n /= r;
        }
        return 1;
    }
    static constexpr int count_passes() {
        int n = N, p = 0;
        while (n > 1) {
            n /= radix(p);
            ++p;
        }
        return p;
    }
    static constexpr int P = count_passes();
};

// TWREG: pass twiddles held in registers (default for powers of two) or read
// from the W_N^t table at the point of use (default for mixed radix, whose
// plans need up to 40 twiddles per thread).
template <int N, int RQ = default_points(N), bool TWREG = !is_mixed_size(N)>
struct LineFFT {
    using PL = Plan<N, RQ>;
    static constexpr int R = PL::R;
    static constexpr int T = N / R;
    static constexpr int P = PL::P;

    static constexpr int radix(int p) { return PL::radix(p); }
    static constexpr int ns(int p) { return p == 0 ? 1 : ns(p - 1) * radix(p - 1); }
    // twiddle registers needed by pass p (p >= 1) and their offset
    static constexpr int tw_count(int p) { return p == 0 ? 0 : (R / radix(p)) * (radix(p) - 1); }
    static constexpr int tw_offset(int p) { return p <= 1 ? 0 : tw_offset(p - 1) + tw_count(p - 1); }
    static constexpr int NTW = P == 0 ? 1 : tw_offset(P - 1) + tw_count(P - 1) + 1;
    static constexpr bool kTableTw = !TWREG;  // table twiddles

    // Pass twiddles of a thread: registers (powers of two) or a reference to
    // the W_N^t table (mixed radix).
    struct RegTwiddles {
        float2 w[NTW];
    };
    struct TableTwiddles {
        const float2* __restrict__ table;
        float scale;
    };
    using Twiddles = std::conditional_t<kTableTw, TableTwiddles, RegTwiddles>;

    // Shared-memory index of line position p.  Powers of two: one 8-byte pad
    // per 16 samples (their exchange strides are powers of two).  Mixed radix
    // 96 / 160 / 320: no pad -- their strides (5, 20, 80 ... at 160) already
    // spread over the banks, and the inter-line offset is chosen by the line
    // stride instead (row_stride<N>(), fft_kernels.cuh; the model is
    // scripts/tools/bank_sim.py).  192 and 384 keep the pad: unpadded they
    // have fewer bank conflicts too, but ptxas then schedules their combine
    // with ~60 fewer registers and fewer loads in flight, and it runs slower
    // (profiles/round2_mixed_radix.md).
    static constexpr bool kPadded = !is_mixed_size(N) || N == 192 || N == 384;
    __device__ __forceinline__ static int pad(int p) {
        if constexpr (kPadded)
            return p + (p >> 4);
        else
            return p;
    }
    static constexpr int padded_len = kPadded ? N + (N >> 4) : N;

    // Loads this thread's pass twiddles from the W_N^t table (DIR applied).
    // The last pass' twiddles are pre-multiplied by `scale` so run() applies
    // the normalisation for free (only the q = 0 slots need an explicit FMUL).
    __device__ __forceinline__ static void load_twiddles(Twiddles& twd, const float2* __restrict__ table, int j,
                                                         float scale = 1.0f) {
        if constexpr (kTableTw) {
            twd.table = table;
            twd.scale = scale;
            return;
        } else {
            load_twiddles_regs(twd.w, table, j, scale);
        }
    }
    __device__ __forceinline__ static void load_twiddles_regs(float2 (&tw)[NTW], const float2* __restrict__ table,
                                                              int j, float scale) {
        sfor<P>([&](auto pc) {
            constexpr int p = pc.value;
            if constexpr (p >= 1) {
                constexpr int Rp = radix(p), Ns = ns(p), S = R / Rp;
                constexpr int stride = N / (Ns * Rp);
                sfor<S>([&](auto sc) {
                    const int g = j + sc.value * T;
                    const int gm = g % Ns;
                    sfor<Rp - 1>([&](auto qc) {
                        constexpr int q = qc.value + 1;
                        float2 w = __ldg(&table[gm * q * stride]);
                        if constexpr (p == P - 1) w = make_float2(w.x * scale, w.y * scale);
                        tw[tw_offset(p) + sc.value * (Rp - 1) + qc.value] = w;
                    });
                });
            }
        });
    }

    // Runs all passes.  `line` is this line's shared buffer (padded_len
    // float2), `sync` a callable that synchronises the threads of the line.
    // The output is multiplied by `scale`, which must be the value the
    // twiddles were loaded with.
    template <int DIR, class Sync>
    __device__ __forceinline__ static void run(float2 (&v)[R], const Twiddles& twd, float2* line, int j,
                                               Sync&& sync, float scale = 1.0f) {
        if constexpr (kTableTw) {
            run_f<DIR>(
                v,
                [&](auto pc, auto sc, auto qc) {
                    float2 w = __ldg(twd.table + tw_index<pc.value, sc.value, qc.value>(j));
                    if constexpr (pc.value == P - 1) w = make_float2(w.x * twd.scale, w.y * twd.scale);
                    return w;
                },
                line, j, sync, scale);
        } else {
            run_f<DIR>(
                v,
                [&](auto pc, auto sc, auto qc) {
                    return twd.w[tw_offset(pc.value) + sc.value * (radix(pc.value) - 1) + qc.value];
                },
                line, j, sync, scale);
        }
    }

    // Twiddle for pass p (>= 1), sub-group s, q = qc + 1 of thread j from a
    // W_N^t table (shared or global): table[(g mod Ns) * q * N/(Ns*Rp)].
    template <int p, int s, int qc>
    __device__ __forceinline__ static int tw_index(int j) {
        constexpr int Rp = radix(p), Ns = ns(p), stride = N / (Ns * Rp);
        return ((j + s * T) % Ns) * (qc + 1) * stride;
    }

    // As run(), with the pass twiddles supplied by `twf(pass, s, qc)` (all
    // three std::integral_constant) -- e.g. read from a shared-memory table
    // at the point of use instead of held in registers.
    template <int DIR, class TwF, class Sync>
    __device__ __forceinline__ static void run_f(float2 (&v)[R], TwF&& twf, float2* line, int j, Sync&& sync,
                                                 float scale = 1.0f) {
        sfor<P>([&](auto pc) {
            constexpr int p = pc.value;
            constexpr int Rp = radix(p), Ns = ns(p), S = R / Rp;
            if constexpr (p >= 1) {
                // exchange: write previous pass' outputs, read this pass' inputs
                constexpr int Rq = radix(p - 1), Nq = ns(p - 1), Sq = R / Rq;
                sync();
                sfor<Sq>([&](auto sc) {
                    const int g = j + sc.value * T;
                    const int base = (g / Nq) * Nq * Rq + (g % Nq);
                    sfor<Rq>([&](auto qc) { line[pad(base + qc.value * Nq)] = v[sc.value + qc.value * Sq]; });
                });
                sync();
                sfor<R>([&](auto m) { v[m.value] = line[pad(j + T * m.value)]; });
                // twiddles
                sfor<S>([&](auto sc) {
                    sfor<Rp - 1>([&](auto qc) {
                        constexpr int m = sc.value + (qc.value + 1) * S;
                        v[m] = cmul(v[m], twf(pc, sc, qc));
                    });
                });
            }
            if constexpr (p == P - 1) {
                if (scale != 1.0f) {
                    if constexpr (p == 0)
                        sfor<R>([&](auto m) { v[m.value] = cscale(v[m.value], scale); });
                    else  // q = 0 slots; the others went through scaled twiddles
                        sfor<S>([&](auto sc) { v[sc.value] = cscale(v[sc.value], scale); });
                }
            }
            sfor<S>([&](auto sc) { dft_regs<Rp, DIR, S, sc.value>(v); });
            (void)Ns;
        });
        if constexpr (P == 0)
            if (scale != 1.0f) v[0] = cscale(v[0], scale);
    }
};

}  // namespace hetreco::dev
