// fft_contig.cu -- host plan/launch for the axis-0 (contiguous) pass; the
// coil-combine epilogues are dispatched to fft_combine_*.cu.
#include "fft_kernels.cuh"

namespace hetreco::dev {

int combine_occupancy_sense(std::uint64_t N, int variant, int block, int smem);
int combine_occupancy_rss(std::uint64_t N, int variant, int block, int smem);
cudaError_t combine_launch_sense(std::uint64_t N, int variant, const ContigArgs& a, const LaunchShape& s, int lpb,
                                 std::uint32_t items, cudaStream_t st);
cudaError_t combine_launch_rss(std::uint64_t N, int variant, const ContigArgs& a, const LaunchShape& s, int lpb,
                               std::uint32_t items, cudaStream_t st);

int combine_occupancy(Combine mode, std::uint64_t N, int variant, int block, int smem) {
    return mode == Combine::Sense ? combine_occupancy_sense(N, variant, block, smem)
                                  : combine_occupancy_rss(N, variant, block, smem);
}

cudaError_t combine_launch(Combine mode, std::uint64_t N, int variant, const ContigArgs& a, const LaunchShape& s,
                           int lpb, std::uint32_t items, cudaStream_t st) {
    return mode == Combine::Sense ? combine_launch_sense(N, variant, a, s, lpb, items, st)
                                  : combine_launch_rss(N, variant, a, s, lpb, items, st);
}

namespace {

template <int N>
int contig_occ(int block, int smem) {
    blocks_per_sm(k_fft_contig<N, -1>, block, smem);
    return blocks_per_sm(k_fft_contig<N, 1>, block, smem);
}

}  // namespace

LaunchShape plan_contig(std::uint64_t N, Combine mode, std::uint64_t items, int sms, int variant) {
    LaunchShape s;
    if (points_for(N, 0) == 0) return s;
    s.variant = mode == Combine::None ? 0 : (variant >= 0 ? variant : env_int("HETRECO_COMBINE_VARIANT", N == 512 ? 3 : 11));
    const int R = points_for(N, (s.variant & 4) ? 8 : 0);
    s.rq = R;
    const int T = int(N) / R;
    int lpb = std::max(1, env_int("HETRECO_LINES_PER_BLOCK", 128) / T);  // lines per block
    // small problems: fewer lines per block so every SM gets work
    // (never below one full warp per block)
    const int min_lpb = std::max(1, 32 / T);
    while (lpb > min_lpb && (items + lpb - 1) / lpb < std::uint64_t(2 * sms)) lpb >>= 1;
    s.block = lpb * T;
    s.smem = lpb * row_stride_of(N) * 8;
    int occ = 1;
    if (mode == Combine::None) {
        switch (N) {
#define X(n) \
    case n: occ = contig_occ<n>(s.block, s.smem); break;
            HETRECO_FFT_SIZES(X)
#undef X
        }
    } else {
        occ = combine_occupancy(mode, N, s.variant, s.block, s.smem);
    }
    const std::uint64_t groups = (items + lpb - 1) / lpb;
    s.grid = int(std::min<std::uint64_t>(groups, std::uint64_t(sms) * occ));
    if (s.grid < 1) s.grid = 1;
    return s;
}

cudaError_t launch_contig(std::uint64_t N, int dir, Combine mode, const ContigArgs& a, const LaunchShape& s,
                          cudaStream_t st) {
    if (s.block == 0 || s.rq == 0) return cudaErrorInvalidValue;
    const int T = int(N) / s.rq;
    const int lpb = s.block / T;
    const std::uint64_t items64 = a.ny * a.frames;
    if (items64 >= (std::uint64_t(1) << 32)) return cudaErrorInvalidValue;
    const std::uint32_t items = std::uint32_t(items64);
    if (mode != Combine::None) {
        if (dir < 0) return cudaErrorInvalidValue;
        if (s.variant & 128) return launch_combine_cp(N, mode, a, s, st);
        if (s.variant & 512) return mode == Combine::Sense ? launch_combine_tc(N, a, s, st) : cudaErrorInvalidValue;
        if (s.variant & 256) return mode == Combine::Sense ? launch_combine_ss(N, a, s, st) : cudaErrorInvalidValue;
        return combine_launch(mode, N, s.variant, a, s, lpb, items, st);
    }
    switch (N) {
#define X(n)                                                                  \
    case n:                                                                   \
        if (dir > 0)                                                          \
            k_fft_contig<n, 1><<<s.grid, s.block, s.smem, st>>>(a, lpb, items);  \
        else                                                                  \
            k_fft_contig<n, -1><<<s.grid, s.block, s.smem, st>>>(a, lpb, items); \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace hetreco::dev
