/*
 * device_abi.h -- the kernel argument record and layout-header decoders,
 * shared by host C++ and sm_100a device code.
 *
 * Replaces include/hetreco/kernel_abi.h:23-103 of the reference: the same
 * five-field argument convention (input, input header, output, output
 * header, parameter block) and the same header wire format (u64 words:
 * [A, {offset, type, rank, d0..d7} x A]).  Differences that follow from the
 * device model: every pointer is a device pointer, and the parameter block is
 * a device copy staged by the backend (the reference borrows the host span
 * for the duration of a synchronous call, backend.hpp:31).
 */
#ifndef HETRECO_B200_DEVICE_ABI_H
#define HETRECO_B200_DEVICE_ABI_H

#include <stdint.h>

#if defined(__CUDACC__)
#define HETRECO_HD __host__ __device__ __forceinline__
#else
#define HETRECO_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* kernel_abi.h:23-30 */
typedef struct hetreco_kernel_args {
    const void* in;
    const uint64_t* in_layout;
    void* out;
    const uint64_t* out_layout;
    const void* params;
    uint64_t params_size;
} hetreco_kernel_args;

/* kernel_abi.h:32-33: host-side entry point type.  In this build the
 * registry's `fn` is a host stub that reports the kernel as device-only
 * (see src/registry.cpp); execution always goes through the CUDA backend. */
typedef void (*hetreco_kernel_fn)(const hetreco_kernel_args* args, uint64_t gid, uint64_t gsize);

/* kernel_abi.h:36-41 -- wire-format element type codes */
#define HETRECO_UINT8 1
#define HETRECO_INT32 2
#define HETRECO_FLOAT32 3
#define HETRECO_COMPLEX64 4
#define HETRECO_FLOAT64 5
#define HETRECO_COMPLEX128 6

#define HETRECO_HEADER_WORDS_PER_ARRAY 11

HETRECO_HD uint64_t hetreco_type_size(uint64_t code) {
    return code == HETRECO_UINT8 ? 1
         : (code == HETRECO_INT32 || code == HETRECO_FLOAT32) ? 4
         : (code == HETRECO_COMPLEX64 || code == HETRECO_FLOAT64) ? 8
         : code == HETRECO_COMPLEX128 ? 16 : 0;
}

/* kernel_abi.h:57-81: header record accessors */
HETRECO_HD uint64_t hetreco_hdr_word(const uint64_t* h, uint64_t arr, uint64_t field) {
    return h[1 + HETRECO_HEADER_WORDS_PER_ARRAY * arr + field];
}
HETRECO_HD uint64_t hetreco_hdr_offset(const uint64_t* h, uint64_t arr) { return hetreco_hdr_word(h, arr, 0); }
HETRECO_HD uint64_t hetreco_hdr_type(const uint64_t* h, uint64_t arr) { return hetreco_hdr_word(h, arr, 1); }
HETRECO_HD uint64_t hetreco_hdr_dim(const uint64_t* h, uint64_t arr, uint64_t d) {
    return hetreco_hdr_word(h, arr, 3 + d);
}
HETRECO_HD uint64_t hetreco_hdr_elements(const uint64_t* h, uint64_t arr) {
    uint64_t n = 1;
    for (uint64_t d = 0; d < 8; ++d) n *= hetreco_hdr_dim(h, arr, d);
    return n;
}

#ifdef __cplusplus
}
#endif

#endif
