/*
 * hetreco_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see hetreco_oracle.h).  Compiled with
 * -O2 -ffp-contract=off so that every float expression rounds exactly where
 * the reference kernels round (the reference is built as ISO C++20, which
 * also implies -ffp-contract=off under g++).
 *
 * Each loop body restates the per-work-item function of one reference kernel;
 * the loop over `gid` replaces WorkerPool::run (src/backend.cpp:95-127),
 * whose contiguous chunking never changes results because every work item
 * writes only its own outputs (src/backend_internal.hpp:29-31).
 */
#include "hetreco_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    float re, im;
} cf32; /* kernel_abi.h:106-109 (hetreco_cfloat) */

/* kernel_abi.h:123-125: (a.re*b.re - a.im*b.im, a.re*b.im + a.im*b.re) */
static inline cf32 cf_mul(cf32 a, cf32 b) {
    cf32 r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}

/* ---- negate: kernels/negate.cl.src:6-22 ------------------------------------ */

void oracle_negate_u8(const uint8_t* in, uint8_t* out, uint64_t n, double max_value) {
    for (uint64_t g = 0; g < n; ++g) {
        double v = max_value - (double)in[g]; /* :13 */
        v = v < 0.0 ? 0.0 : v;                /* :14 */
        v = v > 255.0 ? 255.0 : v;            /* :15 */
        out[g] = (uint8_t)(v + 0.5);          /* :16 */
    }
}

void oracle_negate_f32(const float* in, float* out, uint64_t n, double max_value) {
    const float mv = (float)max_value; /* :20 casts before subtracting */
    for (uint64_t g = 0; g < n; ++g) out[g] = mv - in[g];
}

/* ---- fft_radix2_pass: kernels/fft_radix2_pass.cl.src:22-69 ------------------ */

void oracle_fft_radix2_pass(const float* data_in, float* data_out, uint64_t n, uint32_t mode,
                            uint64_t L, uint64_t S, uint64_t m, float scale,
                            const void* payload) {
    cf32* out = (cf32*)data_out;
    if (mode == 2) {
        /* butterflies: gsize = n/2, one per work item (:29-49) */
        const float* tw = (const float*)payload;
        const uint64_t half = L / 2;
        const uint64_t tstep = L / (2 * m);
        for (uint64_t g = 0; g < n / 2; ++g) {
            const uint64_t line = g / half, j = g % half;
            const uint64_t grp = j / m, k = j % m;
            const uint64_t base = (line % S) + (line / S) * (S * L);
            const uint64_t i0 = base + (grp * 2 * m + k) * S;
            const uint64_t i1 = i0 + m * S;
            const uint64_t t = k * tstep;
            cf32 w = {tw[2 * t], tw[2 * t + 1]};
            cf32 a = out[i0];
            cf32 b = cf_mul(out[i1], w);
            cf32 lo = {a.re + b.re, a.im + b.im};
            cf32 hi = {a.re - b.re, a.im - b.im};
            out[i0].re = lo.re * scale;
            out[i0].im = lo.im * scale;
            out[i1].re = hi.re * scale;
            out[i1].im = hi.im * scale;
        }
        return;
    }
    const uint32_t* rev = (const uint32_t*)payload;
    const cf32* in = (const cf32*)data_in;
    for (uint64_t g = 0; g < n; ++g) {
        const uint64_t k = g % L, line = g / L;
        const uint64_t base = (line % S) + (line / S) * (S * L);
        if (mode == 0) { /* gather (:56-58) */
            out[base + k * S] = in[base + (uint64_t)rev[k] * S];
        } else { /* in-place swap, k < rev[k] only (:59-67) */
            const uint64_t r = rev[k];
            if (k < r) {
                cf32 tmp = out[base + k * S];
                out[base + k * S] = out[base + r * S];
                out[base + r * S] = tmp;
            }
        }
    }
}

/* ---- restated FFT plan --------------------------------- */

static int is_pow2(uint64_t v) { return v != 0 && (v & (v - 1)) == 0; }

static unsigned log2u(uint64_t v) {
    unsigned b = 0;
    while ((UINT64_C(1) << b) < v) ++b;
    return b;
}

static void make_bitrev(uint32_t* rev, uint64_t L) {
    const unsigned bits = log2u(L);
    for (uint64_t k = 0; k < L; ++k) {
        uint32_t r = 0;
        for (unsigned b = 0; b < bits; ++b)
            if (k & (UINT64_C(1) << b)) r |= 1u << (bits - 1 - b);
        rev[k] = r;
    }
}

/* W_L^t for t < L/2, theta = -/+ 2 pi t / L in double, rounded to float
 * (payload convention of fft_radix2_pass.cl.src:15-16). */
static void make_twiddles(float* tw, uint64_t L, int inverse) {
    const double sign = inverse ? 1.0 : -1.0;
    for (uint64_t t = 0; t < L / 2; ++t) {
        const double th = sign * 2.0 * M_PI * (double)t / (double)L;
        tw[2 * t] = (float)cos(th);
        tw[2 * t + 1] = (float)sin(th);
    }
}

int oracle_fft2d(const float* in, float* out, uint64_t nx, uint64_t ny, uint64_t batch,
                 int inverse) {
    if (!is_pow2(nx) || !is_pow2(ny) || batch == 0) return -1;
    const uint64_t n = nx * ny * batch;
    const uint64_t lmax = nx > ny ? nx : ny;
    uint32_t* rev = (uint32_t*)malloc(sizeof(uint32_t) * lmax);
    float* tw = (float*)malloc(sizeof(float) * (lmax > 1 ? lmax : 2));
    const unsigned bx = log2u(nx), by = log2u(ny);
    const float final_scale = inverse ? (float)(1.0 / ((double)nx * (double)ny)) : 1.0f;

    /* axis 0: L = nx, S = 1 -- gather then butterflies */
    make_bitrev(rev, nx);
    oracle_fft_radix2_pass(in, out, n, 0, nx, 1, 0, 1.0f, rev);
    make_twiddles(tw, nx, inverse);
    for (unsigned p = 0; p < bx; ++p) {
        const int last = (by == 0) && (p + 1 == bx);
        oracle_fft_radix2_pass(NULL, out, n, 2, nx, 1, UINT64_C(1) << p,
                               last ? final_scale : 1.0f, tw);
    }
    /* axis 1: L = ny, S = nx -- in-place swap then butterflies */
    make_bitrev(rev, ny);
    oracle_fft_radix2_pass(NULL, out, n, 1, ny, nx, 0, 1.0f, rev);
    make_twiddles(tw, ny, inverse);
    for (unsigned p = 0; p < by; ++p) {
        const int last = (p + 1 == by);
        oracle_fft_radix2_pass(NULL, out, n, 2, ny, nx, UINT64_C(1) << p,
                               last ? final_scale : 1.0f, tw);
    }
    free(rev);
    free(tw);
    return 0;
}

/* ---- combine kernels ------------------------------------------------------------ */

void oracle_complex_element_prod(const float* x, uint64_t nx_elems, const float* s,
                                 uint64_t ns_elems, float* out, int conjugate) {
    const cf32* xv = (const cf32*)x;
    const cf32* sv = (const cf32*)s;
    cf32* ov = (cf32*)out;
    for (uint64_t g = 0; g < nx_elems; ++g) {
        cf32 b = sv[g % ns_elems]; /* cyclic broadcast (:16) */
        if (conjugate) b.im = -b.im;
        ov[g] = cf_mul(xv[g], b);
    }
}

void oracle_ximage_sum(const float* in, float* out, uint64_t plane, uint64_t ncoils,
                       uint64_t nframes) {
    const cf32* iv = (const cf32*)in;
    cf32* ov = (cf32*)out;
    for (uint64_t g = 0; g < plane * nframes; ++g) {
        const uint64_t f = g / plane, p = g % plane;
        double re = 0.0, im = 0.0; /* double accumulation in coil order (:17-21) */
        for (uint64_t c = 0; c < ncoils; ++c) {
            const cf32 v = iv[p + plane * (c + ncoils * f)];
            re += v.re;
            im += v.im;
        }
        ov[g].re = (float)re;
        ov[g].im = (float)im;
    }
}

void oracle_rss_combine(const float* in, float* out, uint64_t plane, uint64_t ncoils,
                        uint64_t nframes) {
    const cf32* iv = (const cf32*)in;
    for (uint64_t g = 0; g < plane * nframes; ++g) {
        const uint64_t f = g / plane, p = g % plane;
        double acc = 0.0;
        for (uint64_t c = 0; c < ncoils; ++c) {
            const cf32 v = iv[p + plane * (c + ncoils * f)];
            acc += (double)v.re * v.re + (double)v.im * v.im; /* :16 */
        }
        out[g] = (float)sqrt(acc);
    }
}

void oracle_matrix_add_f32(const float* a, const float* b, float* out, uint64_t n) {
    for (uint64_t g = 0; g < n; ++g) out[g] = a[g] + b[g];
}

/* ---- compositions -------------------------------------------- */

int oracle_sens_recon(const float* Y, const float* S, float* M, uint64_t nx, uint64_t ny,
                      uint64_t C, uint64_t F, float* scratch) {
    const uint64_t n = nx * ny * C * F;
    float* X = scratch;
    float* P = scratch + 2 * n;
    if (oracle_fft2d(Y, X, nx, ny, C * F, 1) != 0) return -1;
    oracle_complex_element_prod(X, n, S, nx * ny * C, P, 1);
    oracle_ximage_sum(P, M, nx * ny, C, F);
    return 0;
}

int oracle_sense_forward(const float* M, const float* S, const float* mask, float* Y, uint64_t nx,
                         uint64_t ny, uint64_t C, uint64_t F, float* scratch) {
    const uint64_t plane = nx * ny;
    for (uint64_t f = 0; f < F; ++f) {
        for (uint64_t c = 0; c < C; ++c) {
            /* S_c . M_f (complex_element_prod, conjugate = 0) */
            oracle_complex_element_prod(M + 2 * plane * f, plane, S + 2 * plane * c, plane, scratch, 0);
            float* y = Y + 2 * plane * (c + C * f);
            if (oracle_fft2d(scratch, y, nx, ny, 1, 0) != 0) return -1;
            if (mask)
                for (uint64_t p = 0; p < plane; ++p) {
                    y[2 * p] *= mask[p];
                    y[2 * p + 1] *= mask[p];
                }
        }
    }
    return 0;
}

int oracle_rss_recon(const float* Y, float* R, uint64_t nx, uint64_t ny, uint64_t C,
                     uint64_t F, float* scratch) {
    if (oracle_fft2d(Y, scratch, nx, ny, C * F, 1) != 0) return -1;
    oracle_rss_combine(scratch, R, nx * ny, C, F);
    return 0;
}
