// fft_combine_rss.cu -- Rss coil-combine kernels (all sizes and
// the tuning variants), split from the other translation units for build
// parallelism.
#include "fft_kernels.cuh"

namespace hetreco::dev {

namespace {

constexpr int M = 2;

template <int N, int V>
struct CombineK {
    static constexpr bool R8 = has_variants<N>() && (V & 4) && LineFFT<N>::R != 8;
    static constexpr bool PF = has_variants<N>() && (V & 2);
    static constexpr auto kernel() {
        return &k_fft_combine<N, M, (V & 1) != 0, PF, R8 ? 8 : default_points(N)>;
    }
};

template <int N>
auto pick(int v) {
    switch (v & 7) {
        case 1: return CombineK<N, 1>::kernel();
        case 2: return CombineK<N, 2>::kernel();
        case 3: return CombineK<N, 3>::kernel();
        case 4: return CombineK<N, 4>::kernel();
        case 5: return CombineK<N, 5>::kernel();
        case 6: return CombineK<N, 6>::kernel();
        case 7: return CombineK<N, 7>::kernel();
        default: return CombineK<N, 0>::kernel();
    }
}

}  // namespace

int combine_occupancy_rss(std::uint64_t N, int variant, int block, int smem) {
    switch (N) {
#define X(n) \
    case n: return blocks_per_sm(pick<n>(variant), block, smem);
        HETRECO_FFT_SIZES(X)
#undef X
    }
    return 1;
}

cudaError_t combine_launch_rss(std::uint64_t N, int variant, const ContigArgs& a, const LaunchShape& s,
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
