// phantom.cu -- synthetic cine phantom + coil sensitivities on the device
// (gen_phantom).  One thread per pixel
// writes M_true for every frame and S for every coil (x-fastest, coalesced).
// Double-precision arithmetic, rounded once to complex64, so the CPU port
// (oracle/oracle.py gen_phantom_port) agrees to ~1 ulp.
#include <cuda_runtime.h>

#include "launch.hpp"
#include "pdl.cuh"

namespace hetreco::dev {

namespace {

__global__ void k_phantom(PhantomArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    const std::uint64_t npix = std::uint64_t(a.nx) * a.ny;
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    for (std::uint64_t p = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; p < npix;
         p += std::uint64_t(gridDim.x) * blockDim.x) {
        const double u = double(p % a.nx) - 0.5 * a.nx;
        const double v = double(p / a.nx) - 0.5 * a.ny;
        // M_true: three Gaussian blobs rotated by 2 pi f / F about the centre
        for (std::uint32_t f = 0; f < a.frames; ++f) {
            const double th = kTwoPi * double(f) / double(a.frames);
            double m = 0.0;
            for (int b = 0; b < 3; ++b) {
                const double cu = a.blob[b].radius * cos(a.blob[b].angle + th);
                const double cv = a.blob[b].radius * sin(a.blob[b].angle + th);
                const double du = u - cu, dv = v - cv, s = a.blob[b].sigma;
                m += a.blob[b].amp * exp(-(du * du + dv * dv) / (2.0 * s * s));
            }
            a.truth[std::uint64_t(f) * npix + p] = make_float2(float(m), 0.0f);
        }
        // coil maps: Gaussian centred at angle 2 pi i / C on the boundary
        // circle, constant phase e^{i 2 pi i / C}, normalised so sum |S|^2 = 1
        double norm = 0.0;
        for (std::uint32_t c = 0; c < a.coils; ++c) {
            const double be = kTwoPi * double(c) / double(a.coils);
            const double du = u - a.coil_radius * cos(be), dv = v - a.coil_radius * sin(be);
            const double g = exp(-(du * du + dv * dv) / (2.0 * a.coil_width * a.coil_width));
            norm += g * g;
        }
        const double inv = 1.0 / sqrt(norm);
        for (std::uint32_t c = 0; c < a.coils; ++c) {
            const double be = kTwoPi * double(c) / double(a.coils);
            const double du = u - a.coil_radius * cos(be), dv = v - a.coil_radius * sin(be);
            const double g = exp(-(du * du + dv * dv) / (2.0 * a.coil_width * a.coil_width)) * inv;
            a.smaps[std::uint64_t(c) * npix + p] = make_float2(float(g * cos(be)), float(g * sin(be)));
        }
    }
}

}  // namespace

cudaError_t launch_phantom(const PhantomArgs& a, int device_sms, cudaStream_t st) {
    const std::uint64_t npix = std::uint64_t(a.nx) * a.ny;
    const int block = 256;
    const std::uint64_t want = (npix + block - 1) / block;
    const int grid = int(std::min<std::uint64_t>(want, std::uint64_t(device_sms) * 8));
    k_phantom<<<grid > 0 ? grid : 1, block, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace hetreco::dev
