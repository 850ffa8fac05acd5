// tcgen05.cuh -- the few sm_100a tensor-core primitives the DFT-as-GEMM
// combine uses (fft_combine_tc.cu): TMEM allocation, tcgen05.ld/st of 32
// columns per thread, single-thread tcgen05.mma (kind::tf32, A from TMEM or
// shared memory, B from shared memory), commit to an mbarrier, and the
// shared-memory matrix descriptor (no swizzle, K-major core matrices of
// 8 rows x 16 B).
#pragma once

#include <cstdint>

namespace hetreco::dev::tc {

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return std::uint32_t(__cvta_generic_to_shared(p));
}

// One full warp.  Writes the TMEM base address to *slot (shared memory).
__device__ __forceinline__ void tmem_alloc(std::uint32_t* slot, std::uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(std::uint32_t taddr, std::uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Thread i of warp w reads TMEM lane 32*(w%4)+i, columns [col, col+32).
__device__ __forceinline__ void ld32(std::uint32_t taddr, std::uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
}
__device__ __forceinline__ void st32(std::uint32_t taddr, const std::uint32_t (&r)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
                 : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]   (kind::tf32, fp32 accumulate)
__device__ __forceinline__ void mma_ts(std::uint32_t d, std::uint32_t a, std::uint64_t bdesc, std::uint32_t idesc,
                                       std::uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]
__device__ __forceinline__ void mma_ss(std::uint32_t d, std::uint64_t adesc, std::uint64_t bdesc, std::uint32_t idesc,
                                       std::uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive (once) on the mbarrier when every previously issued MMA of this thread completes.
__device__ __forceinline__ void commit(std::uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_init(std::uint32_t bar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint32_t bar, std::uint32_t parity) {
    std::uint32_t done = 0;
    while (!done)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_NONE, K-major: core matrix =
// 8 rows x 16 B stored contiguously (128 B); `lbo` = byte distance between
// core matrices adjacent in K, `sbo` = between core matrices adjacent in M/N.
__device__ __forceinline__ std::uint64_t sdesc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
    return std::uint64_t((saddr >> 4) & 0x3FFFu) | (std::uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
           (std::uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (std::uint64_t(1) << 46);  // version 1 (sm_100)
}

// Instruction descriptor: tf32 x tf32 -> f32, both operands K-major, M x N.
__host__ __device__ constexpr std::uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)                          // D format f32
           | (2u << 7) | (2u << 10)           // A, B format tf32
           | (std::uint32_t(N >> 3) << 17)    // N / 8
           | (std::uint32_t(M >> 4) << 24);   // M / 16
}

// x = hi + lo with hi exactly representable in tf32 (low 13 mantissa bits clear).
__device__ __forceinline__ void split_tf32(float x, std::uint32_t& hi, std::uint32_t& lo) {
    hi = __float_as_uint(x) & 0xFFFFE000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

}  // namespace hetreco::dev::tc
