// fused_recon.hpp -- the fused reconstruction chains as layer-1 kernels.
//
// The reference session reaches device code only through
// Backend::intrinsic_kernels()/execute() (include/hetreco/backend.hpp:64-75,
// src/session.cpp:139-169), whose builtin bundle is the six per-element
// kernels: a reference user driving the B200 through that interface runs the
// 18-launch radix-2 chain.  CudaBackend therefore also registers two fused
// kernels under the reference ABI:
//
//   "sens_recon"  in = Data [Y [nx,ny,C(,F)] c64, S [nx,ny,C] c64]  out = [M [nx,ny,F] c64]
//   "rss_recon"   in = Data [Y]                                     out = [R [nx,ny,F] f32]
//
// params: empty, or one u32 flag word (bit 0: ifftshift in / fftshift out);
// global size: nx*ny*F (one work item per output pixel, like ximage_sum /
// rss_combine).  Each launch is the axis-1 IFFT pass into a cached scratch
// buffer and the fused axis-0 IFFT + coil combine (fp32 accumulation, within
// the north_star 1e-5 of the reference chain), with plans and twiddle tables
// cached per shape -- the layer-2 sens_recon / rss_recon processes' kernels.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <span>
#include <string>
#include <string_view>

#include "hetreco_b200/data.hpp"

typedef struct CUstream_st* cudaStream_t;

namespace hetreco::detail {

class FusedReconKernels {
public:
    static constexpr const char* kSense = "sens_recon";
    static constexpr const char* kRss = "rss_recon";
    static bool is_fused(std::string_view name);

    explicit FusedReconKernels(int ordinal);
    ~FusedReconKernels();
    FusedReconKernels(const FusedReconKernels&) = delete;
    FusedReconKernels& operator=(const FusedReconKernels&) = delete;

    // Validates the layouts (ShapeMismatch / UnsupportedElementType /
    // InvalidArgument) and enqueues the two kernels on `stream`.
    void launch(std::string_view name, const LayoutDescriptor& in, const LayoutDescriptor& out, const void* in_base,
                void* out_base, std::span<const std::byte> params, std::uint64_t gsize, cudaStream_t stream);

private:
    struct Plan;
    int ordinal_;
    std::map<std::string, std::unique_ptr<Plan>> plans_;
    void* scratch_ = nullptr;
    std::uint64_t scratch_bytes_ = 0;
};

}  // namespace hetreco::detail
