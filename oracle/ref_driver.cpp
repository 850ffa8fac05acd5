// ref_driver.cpp -- drives the UNMODIFIED reference library (built from
// /root/reference/proj/core by oracle/build_ref.sh into oracle/_ref/) through
// its own public API: ComputeSession::register_data / launch_kernel /
// fetch_data on the `reference` CPU backend (src/session.cpp:60-169,
// src/backend.cpp:223-249).
//
// TEST INFRASTRUCTURE ONLY: used to pin the C oracle and to generate the
// golden fixtures (tests/golden/make_golden.py), and as bench.py's
// `--impl reference` / cpu_baseline arm.  Never linked into the product.
//
// The reference ships no FFT host plan (process.hpp declares Process but no
// process.cpp exists), so the plan is the restatement of SURVEY.md Appendix B,
// expressed purely as launches of the reference's own `fft_radix2_pass` kernel.
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "hetreco/backend.hpp"
#include "hetreco/session.hpp"

// Built twice by build_ref.sh: as libhetreco_refdrv.so on the reference CPU
// backend (entry points refdrv_*), and with -DHETRECO_REF_ON_B200 as
// libhetreco_ref_on_b200.so, where the SAME reference session code runs on the
// B200 through integration/reference_cuda_backend.cpp (entry points refcuda_*).
#ifdef HETRECO_REF_ON_B200
#define REFDRV(name) refcuda_##name
namespace hetreco_b200_integration {
std::unique_ptr<hetreco::Backend> make_cuda_backend(int ordinal, std::uint64_t capacity, bool source_kernels);
}
#else
#define REFDRV(name) refdrv_##name
#endif

using namespace hetreco;

namespace {

using cf = std::complex<float>;

thread_local std::string g_err;

// Process-lifetime backend, deliberately leaked (no static destructor runs
// after the CUDA runtime has torn itself down at exit).
int g_source_mode = 0;  // B200 adapter: 1 = builtins compiled from the reference's sources by NVRTC

std::unique_ptr<Backend>& backend() {
#ifdef HETRECO_REF_ON_B200
    static auto* pre = new std::unique_ptr<Backend>(hetreco_b200_integration::make_cuda_backend(0, 0, false));
    if (g_source_mode) {
        static auto* src = new std::unique_ptr<Backend>(hetreco_b200_integration::make_cuda_backend(0, 0, true));
        return *src;
    }
    return *pre;
#else
    static auto* b = new std::unique_ptr<Backend>(make_reference_backend());
    return *b;
#endif
}

std::vector<std::byte> fft_params(uint32_t mode, uint64_t L, uint64_t S, uint64_t m, float scale,
                                  const void* payload, size_t payload_bytes) {
    std::vector<std::byte> p(40 + payload_bytes);
    std::memcpy(p.data() + 0, &mode, 4);
    std::memcpy(p.data() + 8, &L, 8);
    std::memcpy(p.data() + 16, &S, 8);
    std::memcpy(p.data() + 24, &m, 8);
    std::memcpy(p.data() + 32, &scale, 4);
    if (payload_bytes) std::memcpy(p.data() + 40, payload, payload_bytes);
    return p;
}

unsigned ilog2(uint64_t v) {
    unsigned b = 0;
    while ((uint64_t{1} << b) < v) ++b;
    return b;
}

// One baked FFT plan = list of (params, is_gather) launches (Appendix B).
struct Launch {
    std::vector<std::byte> params;
    uint64_t gsize;
    bool gather;  // mode 0 reads input, writes output; others in place on output
};

std::vector<Launch> bake_fft_plan(uint64_t nx, uint64_t ny, uint64_t batch, bool inverse) {
    const uint64_t n = nx * ny * batch;
    std::vector<Launch> plan;
    const float fs = inverse ? float(1.0 / (double(nx) * double(ny))) : 1.0f;
    const unsigned bx = ilog2(nx), by = ilog2(ny);
    for (int axis = 0; axis < 2; ++axis) {
        const uint64_t L = axis == 0 ? nx : ny;
        const uint64_t S = axis == 0 ? 1 : nx;
        const unsigned bits = ilog2(L);
        std::vector<uint32_t> rev(L);
        for (uint64_t k = 0; k < L; ++k) {
            uint32_t r = 0;
            for (unsigned b = 0; b < bits; ++b)
                if (k & (uint64_t{1} << b)) r |= 1u << (bits - 1 - b);
            rev[k] = r;
        }
        plan.push_back({fft_params(axis == 0 ? 0u : 1u, L, S, 0, 1.0f, rev.data(), 4 * L), n,
                        axis == 0});
        std::vector<float> tw(std::max<uint64_t>(L, 2));
        const double sg = inverse ? 1.0 : -1.0;
        for (uint64_t t = 0; t < L / 2; ++t) {
            const double th = sg * 2.0 * M_PI * double(t) / double(L);
            tw[2 * t] = float(std::cos(th));
            tw[2 * t + 1] = float(std::sin(th));
        }
        for (unsigned p = 0; p < bits; ++p) {
            const bool last = axis == 0 ? (by == 0 && p + 1 == bx) : (p + 1 == by);
            plan.push_back({fft_params(2u, L, S, uint64_t{1} << p, last ? fs : 1.0f, tw.data(),
                                       4 * L),
                            n / 2, false});
        }
    }
    return plan;
}

NDArray c64(std::vector<uint64_t> dims, const float* src) {
    NDArray a(ElementType::Complex64, std::move(dims));
    if (src) std::memcpy(a.bytes().data(), src, a.byte_size());
    return a;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // namespace

extern "C" {

const char* REFDRV(last_error)() { return g_err.c_str(); }

// WorkerPool size used by the reference backend (src/backend.cpp:73-79).
int REFDRV(pool_threads)() {
    unsigned hw = std::thread::hardware_concurrency();
    if (hw == 0) hw = 1;
    return int(hw > 16 ? 16 : hw);
}

// Runs any builtin kernel once: in/out are single-array Data of the given
// type/dims; `extra_in` (optional) is appended as array 1 of the input
// (complex_element_prod's s).  Output array is overwritten with the result.
int REFDRV(run_kernel)(const char* name, int in_type, int in_rank, const uint64_t* in_dims,
                      const void* in_data, int extra_type, int extra_rank,
                      const uint64_t* extra_dims, const void* extra_data, int out_type,
                      int out_rank, const uint64_t* out_dims, void* out_data, int in_place,
                      const void* params, uint64_t params_size, uint64_t gsize) {
    return guarded([&] {
        ComputeSession s(*backend());
        s.load_builtin_kernels();
        auto mk = [](int t, int r, const uint64_t* d, const void* src) {
            NDArray a(ElementType(t), std::vector<uint64_t>(d, d + r));
            if (src) std::memcpy(a.bytes().data(), src, a.byte_size());
            return a;
        };
        std::vector<NDArray> ins;
        ins.push_back(mk(in_type, in_rank, in_dims, in_data));
        if (extra_data) ins.push_back(mk(extra_type, extra_rank, extra_dims, extra_data));
        DataHandle hin = s.register_data(Data(std::move(ins)));
        DataHandle hout = hin;
        if (!in_place) {
            std::vector<NDArray> outs;
            outs.push_back(mk(out_type, out_rank, out_dims, nullptr));
            hout = s.register_data(Data(std::move(outs)));
        }
        s.launch_kernel(name, hin, hout,
                        std::span<const std::byte>((const std::byte*)params, params_size), gsize);
        Data res = s.fetch_data(hout);
        std::memcpy(out_data, res.arrays[0].bytes().data(), res.arrays[0].byte_size());
    });
}

// 2-D FFT of COMPLEX64 [nx, ny, batch] with the restated plan.
int REFDRV(fft2d)(const float* in, float* out, uint64_t nx, uint64_t ny, uint64_t batch,
                 int inverse) {
    return guarded([&] {
        ComputeSession s(*backend());
        s.load_builtin_kernels();
        std::vector<NDArray> a1;
        a1.push_back(c64({nx, ny, batch}, in));
        DataHandle hk = s.register_data(Data(std::move(a1), DataKind::KData));
        std::vector<NDArray> a2;
        a2.push_back(c64({nx, ny, batch}, nullptr));
        DataHandle hx = s.register_data(Data(std::move(a2), DataKind::XData));
        for (const Launch& l : bake_fft_plan(nx, ny, batch, inverse != 0))
            s.launch_kernel("fft_radix2_pass", l.gather ? hk : hx, hx, l.params, l.gsize);
        Data res = s.fetch_data(hx);
        std::memcpy(out, res.arrays[0].bytes().data(), res.arrays[0].byte_size());
    });
}

// SENSE (method 0: ifft -> complex_element_prod(conj) -> ximage_sum)
// or RSS (method 1: ifft -> rss_combine) over Y [nx,ny,C,F].
// Runs `reps` launches of the baked chain after one init; writes the last
// result to `out` and the mean seconds per launch (each launch followed by
// synchronize(), init excluded) to *mean_s, init seconds to *init_s.
int REFDRV(recon)(int method, const float* Y, const float* S, void* out, uint64_t nx,
                 uint64_t ny, uint64_t C, uint64_t F, int reps, double* mean_s,
                 double* init_s) {
    return guarded([&] {
        const double t0 = now_s();
        ComputeSession s(*backend());
        s.load_builtin_kernels();
        std::vector<NDArray> ak;
        ak.push_back(c64({nx, ny, C, F}, Y));
        DataHandle hk = s.register_data(Data(std::move(ak), DataKind::KData));
        // FFT output: XData [X, S] so complex_element_prod reads arrays 0 and 1
        // (complex_element_prod.cl.src:12-13).
        std::vector<NDArray> ax;
        ax.push_back(c64({nx, ny, C, F}, nullptr));
        if (method == 0) ax.push_back(c64({nx, ny, C}, S));
        DataHandle hx = s.register_data(Data(std::move(ax), DataKind::XData));
        DataHandle hp{}, hm{};
        if (method == 0) {
            std::vector<NDArray> ap;
            ap.push_back(c64({nx, ny, C, F}, nullptr));
            hp = s.register_data(Data(std::move(ap), DataKind::XData));
            std::vector<NDArray> am;
            am.push_back(c64({nx, ny, F}, nullptr));
            hm = s.register_data(Data(std::move(am), DataKind::XData));
        } else {
            std::vector<NDArray> am;
            am.push_back(NDArray(ElementType::Float32, {nx, ny, F}));
            hm = s.register_data(Data(std::move(am), DataKind::XData));
        }
        const std::vector<Launch> plan = bake_fft_plan(nx, ny, C * F, true);
        const uint32_t conj = 1;
        std::vector<std::byte> cep_params(4);
        std::memcpy(cep_params.data(), &conj, 4);
        const uint64_t n = nx * ny * C * F;
        *init_s = now_s() - t0;
        double total = 0;
        for (int r = 0; r < reps; ++r) {
            const double a = now_s();
            for (const Launch& l : plan)
                s.launch_kernel("fft_radix2_pass", l.gather ? hk : hx, hx, l.params, l.gsize);
            if (method == 0) {
                s.launch_kernel("complex_element_prod", hx, hp, cep_params, n);
                s.launch_kernel("ximage_sum", hp, hm, {}, nx * ny * F);
            } else {
                s.launch_kernel("rss_combine", hx, hm, {}, nx * ny * F);
            }
            s.synchronize();
            total += now_s() - a;
        }
        *mean_s = reps > 0 ? total / reps : 0.0;
        Data res = s.fetch_data(hm);
        std::memcpy(out, res.arrays[0].bytes().data(), res.arrays[0].byte_size());
    });
}

// End-to-end per step through the reference API, the CPU analogue of the
// B200 e2e measurement: S and the plan are set up once (excluded, like the
// B200 arm's init), then every step registers the k-space (the reference's
// "send the data to the computing device", session.cpp:60-83), runs the
// chain, fetches the images (session.cpp:85-98) and releases the k-space.
// Writes the last result to `out`, mean seconds per step to *mean_s.
int REFDRV(recon_e2e)(int method, const float* Y, const float* S, void* out, uint64_t nx, uint64_t ny,
                     uint64_t C, uint64_t F, int reps, double* mean_s) {
    return guarded([&] {
        ComputeSession s(*backend());
        s.load_builtin_kernels();
        std::vector<NDArray> ax;
        ax.push_back(c64({nx, ny, C, F}, nullptr));
        if (method == 0) ax.push_back(c64({nx, ny, C}, S));
        DataHandle hx = s.register_data(Data(std::move(ax), DataKind::XData));
        DataHandle hp{}, hm{};
        if (method == 0) {
            std::vector<NDArray> ap;
            ap.push_back(c64({nx, ny, C, F}, nullptr));
            hp = s.register_data(Data(std::move(ap), DataKind::XData));
            std::vector<NDArray> am;
            am.push_back(c64({nx, ny, F}, nullptr));
            hm = s.register_data(Data(std::move(am), DataKind::XData));
        } else {
            std::vector<NDArray> am;
            am.push_back(NDArray(ElementType::Float32, {nx, ny, F}));
            hm = s.register_data(Data(std::move(am), DataKind::XData));
        }
        const std::vector<Launch> plan = bake_fft_plan(nx, ny, C * F, true);
        const uint32_t conj = 1;
        std::vector<std::byte> cep_params(4);
        std::memcpy(cep_params.data(), &conj, 4);
        const uint64_t n = nx * ny * C * F;
        double total = 0;
        for (int r = 0; r < reps; ++r) {
            const double a = now_s();
            std::vector<NDArray> ak;
            ak.push_back(c64({nx, ny, C, F}, Y));
            DataHandle hk = s.register_data(Data(std::move(ak), DataKind::KData));
            for (const Launch& l : plan)
                s.launch_kernel("fft_radix2_pass", l.gather ? hk : hx, hx, l.params, l.gsize);
            if (method == 0) {
                s.launch_kernel("complex_element_prod", hx, hp, cep_params, n);
                s.launch_kernel("ximage_sum", hp, hm, {}, nx * ny * F);
            } else {
                s.launch_kernel("rss_combine", hx, hm, {}, nx * ny * F);
            }
            Data res = s.fetch_data(hm);
            std::memcpy(out, res.arrays[0].bytes().data(), res.arrays[0].byte_size());
            s.release_data(hk);
            total += now_s() - a;
        }
        *mean_s = reps > 0 ? total / reps : 0.0;
    });
}

// Layout header bytes exactly as the reference serializes them
// (src/layout.cpp:89-102) for a Data of `count` arrays.
int REFDRV(layout_header)(int count, const int* types, const int* ranks, const uint64_t* dims8,
                         uint64_t alignment, uint64_t* out_words, uint64_t* total_bytes) {
    return guarded([&] {
        std::vector<NDArray> arrs;
        for (int i = 0; i < count; ++i)
            arrs.push_back(NDArray(ElementType(types[i]),
                                   std::vector<uint64_t>(dims8 + 8 * i, dims8 + 8 * i + ranks[i])));
        LayoutDescriptor l = pack(Data(std::move(arrs)), alignment);
        std::vector<std::byte> h = serialize_layout_header(l);
        std::memcpy(out_words, h.data(), h.size());
        *total_bytes = l.total_bytes;
    });
}

// The reference's embedded builtin kernel sources (kernels.hpp:52-57,
// builtin_kernel_sources()) -- fed to the B200 NVRTC path by the tests to
// pin source-kernel equivalence with the precompiled builtins.
int REFDRV(builtin_source_count)() { return int(builtin_kernel_sources().size()); }
const char* REFDRV(builtin_source_name)(int i) { return builtin_kernel_sources()[std::size_t(i)].unit_name.c_str(); }
const char* REFDRV(builtin_source_text)(int i) { return builtin_kernel_sources()[std::size_t(i)].source_text.c_str(); }

// Selects the adapter flavour used by the following calls (B200 build only):
// 0 = precompiled sm_100a builtins, 1 = the reference's embedded sources
// compiled by NVRTC through Backend::compile.  Returns the backend's
// supports_source_kernels().
int REFDRV(set_source_mode)(int mode) {
#ifdef HETRECO_REF_ON_B200
    g_source_mode = mode;
#else
    (void)mode;
#endif
    return backend()->supports_source_kernels() ? 1 : 0;
}

}  // extern "C"
