// fft_strided.cu -- host plan/launch for the axis-1 (strided) pass.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "fft_kernels.cuh"

namespace hetreco::dev {

bool fft_size_supported(std::uint64_t n) { return points_for(n, 0) != 0; }

namespace {

// ---- column tiles through a shared-memory ring (256/512-point columns, default) ----
//
// At 512^2 the register-prefetch kernel holds one 512-thread CTA per SM
// (8 columns x 64 threads, 96 registers): ~32 KB per SM in flight in 64-byte
// row segments, 0.63 of the HBM peak (profiles/round1_summary.md).  Here the
// CTA keeps K-1 column tiles in flight with cp.async (16-byte chunks,
// row-major [N rows][TX columns] per stage), then each thread reads its
// column samples from the landed stage and runs the same transform and
// stores as k_fft_strided -- bit-identical output.  Square images only.
// Default: 16 columns (128-byte row segments), 2 stages, 1024 threads at
// 512^2; 32 columns, 2 stages, 512 threads at 256^2.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<std::uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(PENDING) : "memory");
}

template <int N, int DIR, int RQ, int K, int TX>
__global__ void __launch_bounds__(TX * (N / RQ)) k_fft_strided_ring(StridedArgs a, std::uint32_t ntiles) {
    pdl_launch_dependents();
    using L = LineFFT<N, RQ>;
    constexpr int R = L::R, T = L::T, NT = TX * T;
    constexpr int TILE = N * TX;        // float2 per stage
    constexpr int CPR = TX / 2;         // 16-byte chunks per tile row
    extern __shared__ __align__(16) float2 smem[];
    const int tid = threadIdx.x;
    const int l = tid % TX, j = tid / TX;
    float2* ring = smem;
    float2* line = smem + K * TILE + l * line_stride<N>();
    typename L::Twiddles tw;
    L::load_twiddles(tw, a.tw, j, a.scale);
    pdl_wait();  // twiddle tables are init-time constants
    constexpr std::uint32_t nx = N, xtiles = N / TX;
    constexpr std::uint64_t plane_elems = std::uint64_t(N) * N;
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    auto tile_base = [&](std::uint32_t tile) {
        const std::uint32_t plane = tile / xtiles, xt = tile % xtiles;
        return std::uint64_t(plane) * plane_elems + xt * std::uint32_t(TX);
    };
    auto issue = [&](std::uint32_t tile, int stage) {
        if (tile < ntiles) {
            const float2* src = a.in + tile_base(tile);
            float2* dst = ring + stage * TILE;
            sfor<N * CPR / NT>([&](auto k) {
                const int q = tid + k.value * NT;
                const int row = q / CPR, cc = q % CPR;
                cp_async16(dst + row * TX + 2 * cc, src + std::uint64_t(row) * nx + 2 * cc);
            });
        }
        cp_async_commit();
    };
    std::uint32_t tile = blockIdx.x;
    sfor<K - 1>([&](auto k) { issue(tile + std::uint32_t(k.value) * gridDim.x, k.value); });
    for (int i = 0; tile < ntiles; ++i, tile += gridDim.x) {
        const int stage = i % K;
        cp_async_wait<K - 2>();
        __syncthreads();  // stage landed for every thread; stage i-1 free
        issue(tile + std::uint32_t(K - 1) * gridDim.x, (i + K - 1) % K);
        const float2* t = ring + stage * TILE + l;
        float2 v[R];
        slots_ld<R>(sh_in, (long long)(R / 2) * T,
                    [&](auto m, long long d) { v[m.value] = t[(j + T * m.value + int(d)) * TX]; });
        L::template run<DIR>(v, tw, line, j, [] { __syncthreads(); }, a.scale);
        float2* dst = a.out + tile_base(tile) + l + std::uint32_t(j) * nx;
        slots<R>(sh_out, [&](auto m, auto ms) { dst[ms.value * T * N] = v[m.value]; });
    }
    cp_async_wait<0>();
}

// ---- the same column-tile ring fed by TMA (cp.async.bulk.tensor.2d) ------------------
//
// one elected thread issues the tile as 2-D tensor-map boxes
// ([TX columns x <=256 rows] of the [planes*N rows, N] view; two boxes at
// 512 rows) completing on the stage's mbarrier, instead of 1024 threads
// issuing 16-byte cp.async chunks.  Shared-memory layout, consumer reads,
// transform and stores are those of k_fft_strided_ring (bit-identical).
// The stage a TMA refills was last read before the previous iteration's
// transform, whose block barriers every thread has passed -- no extra barrier.
__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

template <int N, int DIR, int RQ, int K, int TX>
__global__ void __launch_bounds__(TX * (N / RQ)) k_fft_strided_tma(const __grid_constant__ CUtensorMap map,
                                                                   StridedArgs a, std::uint32_t ntiles) {
    pdl_launch_dependents();
    using L = LineFFT<N, RQ>;
    constexpr int R = L::R, T = L::T;
    constexpr int TILE = N * TX;  // float2 per stage
    constexpr int BOX_ROWS = N < 256 ? N : 256;
    constexpr std::uint32_t STAGE_BYTES = std::uint32_t(TILE) * 8;
    extern __shared__ __align__(128) float2 smem[];
    const int tid = threadIdx.x;
    const int l = tid % TX, j = tid / TX;
    float2* ring = smem;
    float2* line = smem + K * TILE + l * line_stride<N>();
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + K * TILE + TX * line_stride<N>());
    typename L::Twiddles tw;
    L::load_twiddles(tw, a.tw, j, a.scale);
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&map)) : "memory");
        for (int k = 0; k < K; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(full + k)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();  // the input is the previous kernel's output
    constexpr std::uint32_t xtiles = N / TX;
    const bool sh_in = a.shift_in, sh_out = a.shift_out;
    auto issue = [&](std::uint32_t tile, int stage) {  // thread 0 only
        if (tile >= ntiles) return;
        const std::uint32_t plane = tile / xtiles, xt = tile % xtiles;
        const std::uint32_t bar = smem_addr(full + stage);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(STAGE_BYTES) : "memory");
        for (int b = 0; b < N / BOX_ROWS; ++b) {
            const std::uint32_t dst = smem_addr(ring + stage * TILE + b * BOX_ROWS * TX);
            const int c0 = int(xt) * 2 * TX, c1 = int(plane) * N + b * BOX_ROWS;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(dst),
                "l"(reinterpret_cast<std::uint64_t>(&map)), "r"(c0), "r"(c1), "r"(bar)
                : "memory");
        }
    };
    std::uint32_t tile = blockIdx.x;
    if (tid == 0)
        for (int k = 0; k < K - 1; ++k) issue(tile + std::uint32_t(k) * gridDim.x, k);
    for (int i = 0; tile < ntiles; ++i, tile += gridDim.x) {
        const int stage = i % K;
        const std::uint32_t parity = std::uint32_t(i / K) & 1u;
        std::uint32_t ok = 0;
        do {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                : "=r"(ok)
                : "r"(smem_addr(full + stage)), "r"(parity)
                : "memory");
        } while (!ok);
        if (tid == 0) issue(tile + std::uint32_t(K - 1) * gridDim.x, (i + K - 1) % K);
        const float2* t = ring + stage * TILE + l;
        float2 v[R];
        slots_ld<R>(sh_in, (long long)(R / 2) * T,
                    [&](auto m, long long d) { v[m.value] = t[(j + T * m.value + int(d)) * TX]; });
        L::template run<DIR>(v, tw, line, j, [] { __syncthreads(); }, a.scale);
        float2* dst = a.out + std::uint64_t(tile / xtiles) * N * N + (tile % xtiles) * TX + l + std::uint32_t(j) * N;
        slots<R>(sh_out, [&](auto m, auto ms) { dst[ms.value * T * N] = v[m.value]; });
    }
}

PFN_cuTensorMapEncodeTiled_v12000 strided_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q{};
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    });
    return fn;
}

template <int N, int RQ, int K, int TX>
cudaError_t tma_ring_launch(int dir, const StridedArgs& a, const LaunchShape& s, std::uint32_t tiles, cudaStream_t st) {
    auto enc = strided_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap map;
    cuuint64_t dims[2] = {cuuint64_t(2 * N), cuuint64_t(a.planes) * N};  // float32 elements, rows
    cuuint64_t strides[1] = {cuuint64_t(N) * 8};
    cuuint32_t box[2] = {cuuint32_t(2 * TX), cuuint32_t(N < 256 ? N : 256)};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float2*>(a.in), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    if (dir > 0)
        k_fft_strided_tma<N, 1, RQ, K, TX><<<s.grid, s.block, s.smem, st>>>(map, a, tiles);
    else
        k_fft_strided_tma<N, -1, RQ, K, TX><<<s.grid, s.block, s.smem, st>>>(map, a, tiles);
    return cudaGetLastError();
}

template <int N, int RQ, int K, int TX>
int tma_ring_smem() {
    return (K * N * TX + TX * line_stride<N>()) * 8 + K * 8;
}

template <int N, int RQ, int K, int TX>
int tma_ring_occ(int block, int smem) {
    return std::max(blocks_per_sm(k_fft_strided_tma<N, 1, RQ, K, TX>, block, smem),
                    blocks_per_sm(k_fft_strided_tma<N, -1, RQ, K, TX>, block, smem));
}

// TMA boxes instead of cp.async chunks (profiles/round2_tma_axis1.md): the
// default at 512^2 (axis-1 184 -> 170 us at 512^2 x 32 coils x 8 frames, ncu
// 185 -> 166 us, same DRAM bytes); at 256^2 the cp.async ring stays (162 vs
// 165 us).  HETRECO_STRIDED_TMA=0|1 forces it off / on at both sizes.
bool tma_ring_enabled(std::uint64_t N) { return env_int("HETRECO_STRIDED_TMA", N == 512 ? 1 : 0) == 1; }

// Stages K and columns per tile.  Measured (profiles/round1_summary.md),
// axis-1 us at 512^2 x 32 coils x 8 frames: register prefetch 260; 8 columns
// with K = 3/4/5 stages 252/240/240; 16 columns (128-byte row segments,
// 1024 threads, 64 registers) with K = 2: 187 -- the default.  At 256^2 C3:
// register prefetch 173, 32 columns x 2 stages (512 threads) 160-163 -- the
// default.  HETRECO_STRIDED_RING = 0 selects the register-prefetch kernel.
int ring_tx(int K) {
    const int tx = env_int("HETRECO_RING_TX", 16);
    if (tx == 16) return K == 2 ? 16 : 0;
    return (K >= 3 && K <= 5) ? 8 : 0;
}

int ring_smem_bytes(int K, int tx) { return (K * 512 * tx + tx * line_stride<512>()) * 8; }

int ring_stages() { return env_int("HETRECO_STRIDED_RING", 2); }

template <int N, int RQ, int K, int TX>
int ring_occ_k(int block, int smem) {
    return std::max(blocks_per_sm(k_fft_strided_ring<N, 1, RQ, K, TX>, block, smem),
                    blocks_per_sm(k_fft_strided_ring<N, -1, RQ, K, TX>, block, smem));
}

template <int N, int RQ>
int ring_occ(int K, int tx, int block, int smem) {
    if (tx == 16) return ring_occ_k<N, RQ, 2, 16>(block, smem);
    switch (K) {
        case 3: return ring_occ_k<N, RQ, 3, 8>(block, smem);
        case 4: return ring_occ_k<N, RQ, 4, 8>(block, smem);
        default: return ring_occ_k<N, RQ, 5, 8>(block, smem);
    }
}

template <int N, int RQ, int K, int TX>
void ring_launch(int dir, const StridedArgs& a, const LaunchShape& s, std::uint32_t tiles, cudaStream_t st) {
    if (dir > 0)
        k_fft_strided_ring<N, 1, RQ, K, TX><<<s.grid, s.block, s.smem, st>>>(a, tiles);
    else
        k_fft_strided_ring<N, -1, RQ, K, TX><<<s.grid, s.block, s.smem, st>>>(a, tiles);
}

template <int N, int RQ>
void ring_go(int dir, int K, int tx, const StridedArgs& a, const LaunchShape& s, std::uint32_t tiles, cudaStream_t st) {
    if (tx == 16) return ring_launch<N, RQ, 2, 16>(dir, a, s, tiles, st);
    switch (K) {
        case 3: return ring_launch<N, RQ, 3, 8>(dir, a, s, tiles, st);
        case 4: return ring_launch<N, RQ, 4, 8>(dir, a, s, tiles, st);
        default: return ring_launch<N, RQ, 5, 8>(dir, a, s, tiles, st);
    }
}

template <int N, int RQ>
int strided_occ(int block, int smem, int variant) {
    // the generic (non-square) instantiations run whatever the variant: give
    // them the shared-memory attribute too
    blocks_per_sm(k_fft_strided<N, -1, 0, RQ>, block, smem);
    blocks_per_sm(k_fft_strided<N, 1, 0, RQ>, block, smem);
    if constexpr (is_mixed_size(N)) {
        // both directions: blocks_per_sm also sets the shared-memory attribute
        if (variant & 256) {
            if (variant & 1) {
                blocks_per_sm(k_fft_strided<N, -1, N, RQ, true, 1, true>, block, smem);
                return blocks_per_sm(k_fft_strided<N, 1, N, RQ, true, 1, true>, block, smem);
            }
            blocks_per_sm(k_fft_strided<N, -1, N, RQ, false, 1, true>, block, smem);
            return blocks_per_sm(k_fft_strided<N, 1, N, RQ, false, 1, true>, block, smem);
        }
        if (variant & 1) {
            blocks_per_sm(k_fft_strided<N, -1, N, RQ, true>, block, smem);
            return blocks_per_sm(k_fft_strided<N, 1, N, RQ, true>, block, smem);
        }
    }
    if constexpr (has_variants<N>()) {
        if ((variant & 2) && !(variant & 1)) {
            blocks_per_sm(k_fft_strided<N, -1, N, RQ, false, 3>, block, smem);
            return blocks_per_sm(k_fft_strided<N, 1, N, RQ, false, 3>, block, smem);
        }
        if (variant & 1) {
            blocks_per_sm(k_fft_strided<N, -1, N, RQ, true>, block, smem);
            return blocks_per_sm(k_fft_strided<N, 1, N, RQ, true>, block, smem);
        }
    }
    blocks_per_sm(k_fft_strided<N, -1, N, RQ>, block, smem);
    blocks_per_sm(k_fft_strided<N, -1, 0, RQ>, block, smem);
    blocks_per_sm(k_fft_strided<N, 1, N, RQ>, block, smem);
    return blocks_per_sm(k_fft_strided<N, 1, 0, RQ>, block, smem);
}

template <int N, int RQ>
cudaError_t strided_go(int dir, bool sq, const StridedArgs& a, const LaunchShape& s, int tx, std::uint32_t tiles,
                cudaStream_t st) {
    if constexpr (N == 512 && RQ == 8) {
        if (sq && (s.variant & 64)) {
            return tma_ring_launch<512, 8, 2, 16>(dir, a, s, tiles, st);
        }
    }
    if constexpr (N == 256 && RQ == 16) {
        if (sq && (s.variant & 64)) {
            switch ((s.variant >> 3) & 7) {  // stages; columns per tile from the block size
                case 3: return tma_ring_launch<256, 16, 3, 16>(dir, a, s, tiles, st);
                case 4: return tma_ring_launch<256, 16, 4, 16>(dir, a, s, tiles, st);
                default:
                    return s.block == 16 * 16 ? tma_ring_launch<256, 16, 2, 16>(dir, a, s, tiles, st)
                                              : tma_ring_launch<256, 16, 2, 32>(dir, a, s, tiles, st);
            }
        }
    }
    if constexpr (is_mixed_size(N)) {
        // mixed-radix experiment bits (HETRECO_STRIDED_MIXED): 1 = next-tile
        // prefetch, 256 = pass twiddles in registers
        if (sq && (s.variant & 256)) {
            if (s.variant & 1) {
                if (dir > 0) k_fft_strided<N, 1, N, RQ, true, 1, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
                else k_fft_strided<N, -1, N, RQ, true, 1, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            } else {
                if (dir > 0) k_fft_strided<N, 1, N, RQ, false, 1, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
                else k_fft_strided<N, -1, N, RQ, false, 1, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            }
            return cudaSuccess;
        }
        if (sq && (s.variant & 1)) {
            if (dir > 0) k_fft_strided<N, 1, N, RQ, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            else k_fft_strided<N, -1, N, RQ, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            return cudaSuccess;
        }
    }
    if constexpr (N == 512 && RQ == 8) {
        if (sq && (s.variant & 4)) {
            ring_go<N, RQ>(dir, (s.variant >> 3) & 7, tx, a, s, tiles, st);
            return cudaSuccess;
        }
    }
    if constexpr (N == 256 && RQ == 16) {
        if (sq && (s.variant & 4)) {
            ring_launch<N, RQ, 2, 32>(dir, a, s, tiles, st);
            return cudaSuccess;
        }
    }
    if constexpr (has_variants<N>()) {
        if (sq && (s.variant & 2) && !(s.variant & 1)) {  // 3 CTAs/SM register cap
            if (dir > 0)
                k_fft_strided<N, 1, N, RQ, false, 3><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            else
                k_fft_strided<N, -1, N, RQ, false, 3><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            return cudaSuccess;
        }
        if (sq && (s.variant & 1)) {  // register prefetch of the next tile (square fast path)
            if (dir > 0)
                k_fft_strided<N, 1, N, RQ, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            else
                k_fft_strided<N, -1, N, RQ, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            return cudaSuccess;
        }
    }
    if (dir > 0) {
        if (sq)
            k_fft_strided<N, 1, N, RQ><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
        else
            k_fft_strided<N, 1, 0, RQ><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
    } else {
        if (sq)
            k_fft_strided<N, -1, N, RQ><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
        else
            k_fft_strided<N, -1, 0, RQ><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
    }
    return cudaSuccess;
}

}  // namespace

LaunchShape plan_strided(std::uint64_t N, std::uint64_t nx, std::uint64_t planes, int sms) {
    LaunchShape s;
    // measured defaults (profiles/round1_summary.md): 512-point columns run
    // best with 8 points/thread, 8-column tiles and next-tile prefetch.
    const int rq = env_int("HETRECO_STRIDED_POINTS", N == 512 ? 8 : 0);
    const int R = points_for(N, rq);
    if (R == 0) return s;
    s.rq = R;
    // bit 0 next-tile prefetch, bit 1 three CTAs per SM register cap.
    // Measured on B200 (profiles/round1_summary.md): 256 -> 32-column tiles
    // with next-tile prefetch (170 us vs 181 us for 16 columns under the
    // 3-CTA register cap at C3); 512 -> 8-column tiles with prefetch.
    s.variant = env_int("HETRECO_STRIDED_PF", (N == 512 || N == 256) ? 1 : 0);
    const int T = int(N) / R;
    const int ls_bytes = stride_of(N) * 8;
    // columns per tile: >= 16 (128-B rows) when possible, bounded by 512
    // threads and ~100 KB of shared memory.
    std::uint64_t tx = std::max(16, 256 / T);
    tx = std::min<std::uint64_t>(tx, std::uint64_t(std::max(1, 512 / T)));
    tx = std::min<std::uint64_t>(tx, std::uint64_t(std::max(1, (100 * 1024) / ls_bytes)));
    // mixed-radix columns (8 threads each): 16-column tiles (160^2 C3: 91 vs 97 us at 32)
    const bool mixed = (N & (N - 1)) != 0;
    // Few planes (C2: 256^2 x 8 coils x 1 frame = 64 wide tiles for 148 SMs):
    // narrower tiles without prefetch or ring fill more SMs (C2 axis-1 kernel
    // 11.1 -> 9.9 us with 16 columns).
    const int ring_cols = N == 256 ? 32 : (N == 512 ? 16 : 0);
    const bool few_tiles = ring_cols && nx == N && (nx / std::uint64_t(ring_cols)) * planes < std::uint64_t(sms);
    int tx_default = N == 512 ? 8 : (N == 256 ? 32 : (mixed ? 16 : 0));
    if (few_tiles) {
        tx_default = 16;
        while (tx_default > 8 && (nx / std::uint64_t(tx_default)) * planes < std::uint64_t(sms)) tx_default >>= 1;
        s.variant = env_int("HETRECO_STRIDED_PF", 0);
    }
    // mixed radix, square: next-tile prefetch + pass twiddles in registers
    // (bits 1 | 256; measured 3-21 % faster at 96..320, profiles/round2_mixed_radix.md)
    if (mixed && nx == N) s.variant = env_int("HETRECO_STRIDED_MIXED", 257);
    if (const int e = env_int("HETRECO_STRIDED_TX", tx_default)) tx = std::uint64_t(e);
    tx = std::min<std::uint64_t>(tx, nx);
    tx = std::min<std::uint64_t>(tx, std::uint64_t(std::max(1, 512 / T)));  // the kernels' 512-thread bound
    while (tx > 1 && nx % tx) tx >>= 1;  // both powers of two in practice
    s.block = int(tx) * T;
    s.smem = int(tx) * ls_bytes;
    if ((s.variant & 256) && (!mixed || s.block > 256)) s.variant &= ~256;  // register twiddles: <= 256 threads
    const std::uint64_t tiles = (nx / tx) * planes;
    int occ = 1;
    if (N == 256 && R == 16 && nx == 256 && ring_stages() && !few_tiles && tma_ring_enabled(256)) {
        // stages x columns: 2 x 32 (default), or 16-column tiles with 2-4
        // stages (HETRECO_TMA_STAGES256 = 2|3|4 with HETRECO_TMA_TX256 = 16)
        const int k = env_int("HETRECO_TMA_STAGES256", 2), ttx = env_int("HETRECO_TMA_TX256", 32);
        const int K = (ttx == 16 && k >= 2 && k <= 4) ? k : 2, TXc = (ttx == 16) ? 16 : 32;
        s.variant = 64 | (K << 3);
        s.block = TXc * T;
        if (TXc == 32) {
            s.smem = tma_ring_smem<256, 16, 2, 32>();
            occ = tma_ring_occ<256, 16, 2, 32>(s.block, s.smem);
        } else if (K == 2) {
            s.smem = tma_ring_smem<256, 16, 2, 16>();
            occ = tma_ring_occ<256, 16, 2, 16>(s.block, s.smem);
        } else if (K == 3) {
            s.smem = tma_ring_smem<256, 16, 3, 16>();
            occ = tma_ring_occ<256, 16, 3, 16>(s.block, s.smem);
        } else {
            s.smem = tma_ring_smem<256, 16, 4, 16>();
            occ = tma_ring_occ<256, 16, 4, 16>(s.block, s.smem);
        }
        s.grid = int(std::min<std::uint64_t>((nx / std::uint64_t(TXc)) * planes, std::uint64_t(sms) * occ));
        return s;
    }
    if (N == 512 && R == 8 && nx == 512 && ring_stages() && !few_tiles && tma_ring_enabled(512)) {
        s.variant = 64 | (2 << 3);
        s.block = 16 * T;
        s.smem = tma_ring_smem<512, 8, 2, 16>();
        occ = tma_ring_occ<512, 8, 2, 16>(s.block, s.smem);
        s.grid = int(std::min<std::uint64_t>((nx / 16) * planes, std::uint64_t(sms) * occ));
        return s;
    }
    if (N == 256 && R == 16 && nx == 256 && ring_stages() && !few_tiles) {  // 32 columns (256-B rows), 2 stages
        s.variant = 4 | (2 << 3);
        s.block = 32 * T;
        s.smem = (2 * 256 * 32 + 32 * line_stride<256>()) * 8;
        occ = ring_occ_k<256, 16, 2, 32>(s.block, s.smem);
        s.grid = int(std::min<std::uint64_t>((nx / 32) * planes, std::uint64_t(sms) * occ));
        return s;
    }
    if (const int K = ring_stages(); K && N == 512 && R == 8 && nx == 512 && !few_tiles) {
        const int rtx = ring_tx(K);
        if (rtx) {
            s.variant = 4 | (K << 3);
            s.block = rtx * T;
            s.smem = ring_smem_bytes(K, rtx);
            occ = ring_occ<512, 8>(K, rtx, s.block, s.smem);
            s.grid = int(std::min<std::uint64_t>((nx / std::uint64_t(rtx)) * planes, std::uint64_t(sms) * occ));
            return s;
        }
    }
    switch (N) {
#define X(n)                                                              \
    case n:                                                               \
        if constexpr (has_variants<n>())                                  \
            if (R == 8 && LineFFT<n>::R != 8) {                           \
                occ = strided_occ<n, 8>(s.block, s.smem, s.variant);                 \
                break;                                                    \
            }                                                             \
        occ = strided_occ<n, default_points(n)>(s.block, s.smem, s.variant);         \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
    }
    s.grid = int(std::min<std::uint64_t>(tiles, std::uint64_t(sms) * occ));
    if (s.grid < 1) s.grid = 1;
    return s;
}

cudaError_t launch_strided(std::uint64_t N, int dir, const StridedArgs& a, const LaunchShape& s, cudaStream_t st) {
    if (s.block == 0 || s.rq == 0) return cudaErrorInvalidValue;
    const int T = int(N) / s.rq;
    const int tx = s.block / T;
    const std::uint64_t tiles64 = (a.nx / tx) * a.planes;
    if (tiles64 >= (std::uint64_t(1) << 32)) return cudaErrorInvalidValue;
    const std::uint32_t tiles = std::uint32_t(tiles64);
    const bool sq = a.nx == N;  // square image: compile-time row stride
    switch (N) {
#define X(n)                                                              \
    case n:                                                               \
        if constexpr (has_variants<n>())                                  \
            if (s.rq == 8 && LineFFT<n>::R != 8) {                        \
                if (auto e = strided_go<n, 8>(dir, sq, a, s, tx, tiles, st)) return e; \
                break;                                                    \
            }                                                             \
        if (auto e = strided_go<n, default_points(n)>(dir, sq, a, s, tx, tiles, st)) return e; \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace hetreco::dev
