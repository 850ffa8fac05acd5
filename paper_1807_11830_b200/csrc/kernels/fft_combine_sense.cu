// fft_combine_sense.cu -- Sense coil-combine kernels (all sizes and
// the tuning variants), split from the other translation units for build
// parallelism.
#include "fft_kernels.cuh"

namespace hetreco::dev {

namespace {

constexpr int M = 1;

template <int N, int V>
struct CombineK {
    static constexpr bool R8 = has_variants<N>() && (V & 4) && LineFFT<N>::R != 8;
    // bit 1: prefetch; bit 3 selects the copy form over the ping-pong form
    static constexpr int PF = (has_variants<N>() && (V & 2)) ? ((V & 8) ? 1 : 2) : 0;
    static constexpr auto kernel() {
        return &k_fft_combine<N, M, (V & 1) != 0, PF, R8 ? 8 : default_points(N), (V & 16) ? 3 : 1>;
    }
};

template <int N, int V = 0>
auto pick(int v) {
    if constexpr (V == 0)
        if (has_variants<N>() && (v & 31) == 27) return CombineK<N, 27>::kernel();  // copy-PF fp32, 3 CTAs/SM
    if constexpr (V == 15) {
        return CombineK<N, 15>::kernel();
    } else {
        if ((v & 15) == V) return CombineK<N, V>::kernel();
        return pick<N, V + 1>(v);
    }
}

}  // namespace

int combine_occupancy_sense(std::uint64_t N, int variant, int block, int smem) {
    switch (N) {
#define X(n) \
    case n: return blocks_per_sm(pick<n>(variant), block, smem);
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return 1;
}

cudaError_t combine_launch_sense(std::uint64_t N, int variant, const ContigArgs& a, const LaunchShape& s,
                                 int lpb, std::uint32_t items, cudaStream_t st) {
    switch (N) {
#define X(n)                                                            \
    case n:                                                             \
        pick<n>(variant)<<<s.grid, s.block, s.smem, st>>>(a, lpb, items); \
        break;
        HETRECO_FFT_SIZES(X)
#undef X
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace hetreco::dev
