// fft_strided.cu -- host plan/launch for the axis-1 (strided) pass.
#include "fft_kernels.cuh"

namespace hetreco::dev {

bool fft_size_supported(std::uint64_t n) { return points_for(n, 0) != 0; }

namespace {

template <int N, int RQ>
int strided_occ(int block, int smem, int variant) {
    // the generic (non-square) instantiations run whatever the variant: give
    // them the shared-memory attribute too
    blocks_per_sm(k_fft_strided<N, -1, 0, RQ>, block, smem);
    blocks_per_sm(k_fft_strided<N, 1, 0, RQ>, block, smem);
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
void strided_go(int dir, bool sq, const StridedArgs& a, const LaunchShape& s, int tx, std::uint32_t tiles,
                cudaStream_t st) {
    if constexpr (has_variants<N>()) {
        if (sq && (s.variant & 2) && !(s.variant & 1)) {  // 3 CTAs/SM register cap
            if (dir > 0)
                k_fft_strided<N, 1, N, RQ, false, 3><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            else
                k_fft_strided<N, -1, N, RQ, false, 3><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            return;
        }
        if (sq && (s.variant & 1)) {  // register prefetch of the next tile (square fast path)
            if (dir > 0)
                k_fft_strided<N, 1, N, RQ, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            else
                k_fft_strided<N, -1, N, RQ, true><<<s.grid, s.block, s.smem, st>>>(a, tx, tiles);
            return;
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
    if (const int e = env_int("HETRECO_STRIDED_TX", N == 512 ? 8 : (N == 256 ? 32 : (mixed ? 16 : 0))))
        tx = std::uint64_t(e);
    tx = std::min<std::uint64_t>(tx, nx);
    while (tx > 1 && nx % tx) tx >>= 1;  // both powers of two in practice
    s.block = int(tx) * T;
    s.smem = int(tx) * ls_bytes;
    const std::uint64_t tiles = (nx / tx) * planes;
    int occ = 1;
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
                strided_go<n, 8>(dir, sq, a, s, tx, tiles, st);           \
                break;                                                    \
            }                                                             \
        strided_go<n, default_points(n)>(dir, sq, a, s, tx, tiles, st);   \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace hetreco::dev
