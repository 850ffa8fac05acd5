// phantom.cpp -- gen_phantom on the device (include/hetreco_b200/phantom.hpp).
#include "hetreco_b200/phantom.hpp"

#include <cuda_runtime.h>

#include <random>
#include <string>

#include "../kernels/launch.hpp"
#include "hetreco_b200/processes.hpp"

namespace hetreco {

namespace {
bool pow2(std::uint64_t v) { return v >= 2 && v <= 4096 && (v & (v - 1)) == 0; }
}  // namespace

std::array<std::array<double, 4>, 3> phantom_blobs(const PhantomSpec& spec) {
    std::mt19937_64 g(spec.seed);
    auto uni = [&] { return double(g() >> 11) * (1.0 / 9007199254740992.0); };  // [0, 1), 53 bits
    const double L = double(std::min(spec.nx, spec.ny));
    std::array<std::array<double, 4>, 3> b{};
    for (auto& blob : b) {
        blob[0] = 0.5 + 0.5 * uni();              // amplitude
        blob[1] = 0.25 * L * uni();               // distance of the centre from the image centre
        blob[2] = 6.283185307179586 * uni();      // angle of the centre at frame 0
        blob[3] = L * (0.04 + 0.08 * uni());      // Gaussian width
    }
    return b;
}

Phantom gen_phantom(ComputeSession& s, const PhantomSpec& spec, HostMemory memory) {
    if (!pow2(spec.nx) || !pow2(spec.ny))
        throw InvalidParams("gen_phantom: nx and ny must be powers of two in [2, 4096], got " +
                            std::to_string(spec.nx) + "x" + std::to_string(spec.ny));
    if (spec.frames < 1 || spec.coils < 1 || spec.frames > (1u << 20) || spec.coils > 4096)
        throw InvalidParams("gen_phantom: frames and coils must be >= 1");
    const auto blobs = phantom_blobs(spec);
    CudaBackend& cb = s.cuda();
    cb.make_current();
    const ArrayShape model_shapes[2] = {{ElementType::Complex64, {spec.nx, spec.ny, spec.frames}},
                                        {ElementType::Complex64, {spec.nx, spec.ny, spec.coils}}};
    const DataHandle model = s.allocate_data(model_shapes, DataKind::XData);
    const ArrayShape k_shape[1] = {{ElementType::Complex64, {spec.nx, spec.ny, spec.coils, spec.frames}}};
    const DataHandle kd = s.allocate_data(k_shape, DataKind::KData);
    try {
        dev::PhantomArgs a{};
        a.truth = static_cast<float2*>(s.device_array(model, 0));
        a.smaps = static_cast<float2*>(s.device_array(model, 1));
        a.nx = std::uint32_t(spec.nx);
        a.ny = std::uint32_t(spec.ny);
        a.frames = std::uint32_t(spec.frames);
        a.coils = std::uint32_t(spec.coils);
        for (int i = 0; i < 3; ++i) a.blob[i] = {blobs[i][0], blobs[i][1], blobs[i][2], blobs[i][3]};
        const double L = double(std::min(spec.nx, spec.ny));
        a.coil_radius = 0.5 * L;
        a.coil_width = 0.4 * L;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cb.ordinal());
        cb.note_work();
        const cudaError_t e = dev::launch_phantom(a, sms, cb.compute_stream());
        if (e != cudaSuccess) throw DeviceError("gen_phantom", cudaGetErrorString(e));
        // Y_i = F(S_i . M_true): the forward model process, unmasked
        auto fwd = make_process(s, "sense_forward", "gen_phantom/forward");
        fwd->set_input(model);
        fwd->set_output(kd);
        fwd->init();
        fwd->launch();
        Phantom out;
        Data m = s.fetch_data(model, memory);
        out.truth.kind = DataKind::XData;
        out.truth.arrays.push_back(std::move(m.arrays[0]));
        out.smaps.arrays.push_back(std::move(m.arrays[1]));
        out.kdata = s.fetch_data(kd, memory);
        s.release_data(model);
        s.release_data(kd);
        return out;
    } catch (...) {
        s.release_data(model);
        s.release_data(kd);
        throw;
    }
}

}  // namespace hetreco
