/*
 * hetreco_oracle.h -- CPU restatement of the reference's hot-path arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1807_11830_b200/,
 * include/) links, loads or calls this code.  It is imported only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg, always as the
 * checker, never as the thing measured or shipped.
 *
 * Every function restates one reference routine, cited by file:line relative
 * to /root/reference/proj/core.  Arithmetic is written in the same operation
 * order as the reference kernels and this file is compiled with
 * -ffp-contract=off, so the results are bit-identical to the reference CPU
 * backend (pinned against oracle/_ref in tests/test_oracle.py and against the
 * committed fixtures in tests/golden/).
 *
 * Layout convention (include/hetreco/ndarray.hpp:61-67 of the reference):
 * column-major, dims fastest first; COMPLEX64 is interleaved (re, im) float.
 */
#ifndef HETRECO_ORACLE_H
#define HETRECO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* kernels/negate.cl.src:6-22 */
void oracle_negate_u8(const uint8_t* in, uint8_t* out, uint64_t n, double max_value);
void oracle_negate_f32(const float* in, float* out, uint64_t n, double max_value);

/* kernels/fft_radix2_pass.cl.src:22-69, one pass over the whole array.
 * `data_in` is only read in mode 0; modes 1/2 work in place on `data_out`.
 * `n` is the element count of the array (gsize = n for modes 0/1, n/2 for 2).
 * `payload` points at the pass payload (u32 rev[L] or f32 (re,im)[L/2]). */
void oracle_fft_radix2_pass(const float* data_in, float* data_out, uint64_t n, uint32_t mode,
                            uint64_t L, uint64_t S, uint64_t m, float scale,
                            const void* payload);

/* Restated FFT plan:
 * bit-reversal gather + log2(nx) butterfly passes on axis 0, bit-reversal
 * swap + log2(ny) butterfly passes on axis 1, twiddles W_L^t computed in
 * double and rounded to float, inverse scaled by 1/(nx*ny) in the last
 * butterfly pass.  in/out are COMPLEX64 [nx, ny, batch]; they may not alias.
 * Returns 0, or -1 when nx or ny is not a power of two (ShapeMismatch). */
int oracle_fft2d(const float* in, float* out, uint64_t nx, uint64_t ny, uint64_t batch,
                 int inverse);

/* kernels/complex_element_prod.cl.src:9-19 */
void oracle_complex_element_prod(const float* x, uint64_t nx_elems, const float* s,
                                 uint64_t ns_elems, float* out, int conjugate);

/* kernels/ximage_sum.cl.src:6-23; in [plane, coils, frames] -> out [plane, frames] */
void oracle_ximage_sum(const float* in, float* out, uint64_t plane, uint64_t ncoils,
                       uint64_t nframes);

/* kernels/rss_combine.cl.src:5-20; in COMPLEX64 [plane, coils, frames] -> FLOAT32 */
void oracle_rss_combine(const float* in, float* out, uint64_t plane, uint64_t ncoils,
                        uint64_t nframes);

/* kernels/matrix_add.cl.src:5-24 (f32 path) */
void oracle_matrix_add_f32(const float* a, const float* b, float* out, uint64_t n);

/* sens_recon = chain(fft2d INVERSE, complex_element_prod
 * conj=1, ximage_sum).  Y [nx,ny,C,F], S [nx,ny,C] -> M [nx,ny,F] (COMPLEX64).
 * `scratch` must hold 2*nx*ny*C*F complex values. */
int oracle_sens_recon(const float* Y, const float* S, float* M, uint64_t nx, uint64_t ny,
                      uint64_t C, uint64_t F, float* scratch);

/* rss_recon = fft2d INVERSE + rss_combine.  Y -> R [nx,ny,F]
 * FLOAT32.  `scratch` must hold nx*ny*C*F complex values. */
int oracle_rss_recon(const float* Y, float* R, uint64_t nx, uint64_t ny, uint64_t C,
                     uint64_t F, float* scratch);

/* SENSE forward model (no reference kernel exists; composed from the
 * reference's own operations): Y[:,:,c,f] = mask . fft2d_FORWARD(S_c . M_f),
 * S_c . M_f as complex_element_prod (conj = 0, complex_element_prod.cl.src:9-19),
 * mask FLOAT32 [nx,ny] or NULL.  M [nx,ny,F], S [nx,ny,C], Y [nx,ny,C,F].
 * `scratch` holds nx*ny complex values. */
int oracle_sense_forward(const float* M, const float* S, const float* mask, float* Y, uint64_t nx,
                         uint64_t ny, uint64_t C, uint64_t F, float* scratch);

#ifdef __cplusplus
}
#endif

#endif
