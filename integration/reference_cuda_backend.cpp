// reference_cuda_backend.cpp -- the binding a maintainer adds to the
// REFERENCE code base to run it on a B200: a hetreco::Backend (the reference's
// own interface, include/hetreco/backend.hpp:44-79) implemented over the
// C-ABI of libhetreco_b200.so (include/hetreco_b200.h, layer 1).
//
// It is compiled against the unmodified reference headers and linked with
// the unmodified reference library by oracle/build_ref.sh (output in
// oracle/_ref/, never committed).  tests/test_gpu_integration.py then drives
// the reference's own ComputeSession (src/session.cpp) on it through
// ComputeSession(Backend&) (session.hpp:59-61) and checks the results against
// the reference CPU backend bit for bit.  To make it the default device a
// maintainer appends `make_cuda_backends()` to owned_backends()
// (src/backend.cpp:294-302); device ranking (GPU > CPU, device.cpp:48-55)
// then selects it with an empty DeviceFilter.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hetreco/backend.hpp"
#include "hetreco/errors.hpp"
#include "hetreco/kernels.hpp"
#include "hetreco_b200.h"

namespace hetreco_b200_integration {

using namespace hetreco;

// ErrorCode values of the C-ABI (include/hetreco_b200/error_types.hpp).
enum : int { kAllocationFailure = 8, kUnknownHandle = 9, kInvalidArgument = 4, kUnsupportedSource = 13 };

[[noreturn]] void rethrow(int rc, const std::string& kernel = {}) {
    const std::string msg = hetreco_last_error();
    switch (rc) {
        case kAllocationFailure: throw AllocationFailure(msg);
        case kUnknownHandle: throw UnknownHandle(msg);
        case kInvalidArgument: throw InvalidArgument(msg);
        case kUnsupportedSource: throw UnsupportedSource(msg);
        default: throw DeviceError(kernel.empty() ? "<cuda>" : kernel, msg);
    }
}

inline void ck(int rc, const std::string& kernel = {}) {
    if (rc != HETRECO_OK) rethrow(rc, kernel);
}

// The registry requires a non-null host entry point (src/kernels.cpp:13);
// these kernels only exist on the GPU, so a host call fails loudly.
void device_only(const hetreco_kernel_args*, std::uint64_t, std::uint64_t) {
    throw DeviceError("<sm_100a>", "device kernel invoked on the host");
}

class CudaBackend final : public Backend {
public:
    // source_kernels: report supports_source_kernels() when NVRTC is present,
    // so the reference session's load_builtin_kernels compiles its embedded
    // sources for sm_100a (session.cpp:139-148); false = precompiled builtins.
    explicit CudaBackend(int ordinal, std::uint64_t capacity = 0, bool source_kernels = true) {
        ck(hetreco_cuda_backend_create(ordinal, capacity, &h_));
        hetreco_device_desc d{};
        ck(hetreco_cuda_backend_device(h_, &d));
        id_ = d.backend_id;
        desc_.backend_id = id_;
        desc_.device_index = 0;
        desc_.device_type = DeviceType::Gpu;
        desc_.vendor = d.vendor;
        desc_.name = d.name;
        desc_.api_version = d.api_version;
        desc_.global_memory_bytes = d.global_memory_bytes;
        desc_.base_alignment_bytes = d.base_alignment_bytes;
        int src = 0;
        ck(hetreco_cuda_supports_source(h_, &src));
        desc_.supports_source_kernels = source_kernels && src != 0;
    }
    ~CudaBackend() override { hetreco_cuda_backend_destroy(h_); }

    std::string_view id() const override { return id_; }
    std::vector<DeviceDescriptor> devices() const override { return {desc_}; }
    TransferPath transfer_path() const override { return TransferPath::Staged; }
    bool supports_source_kernels() const override { return desc_.supports_source_kernels; }

    BufferId allocate(std::uint64_t bytes) override {
        std::uint64_t id = 0;
        ck(hetreco_cuda_allocate(h_, bytes, &id));
        return id;
    }
    void release(BufferId b) override { ck(hetreco_cuda_release(h_, b)); }
    void upload(BufferId b, std::uint64_t off, std::span<const std::byte> bytes) override {
        ck(hetreco_cuda_upload(h_, b, off, bytes.data(), bytes.size()));
    }
    void download(BufferId b, std::uint64_t off, std::span<std::byte> into) const override {
        ck(hetreco_cuda_download(h_, b, off, into.data(), into.size()));
    }
    void copy(BufferId s, std::uint64_t so, BufferId d, std::uint64_t doff, std::uint64_t n) override {
        ck(hetreco_cuda_copy(h_, s, so, d, doff, n));
    }
    std::vector<CompiledKernel> intrinsic_kernels() override {
        int n = 0;
        ck(hetreco_cuda_kernel_count(&n));
        std::vector<CompiledKernel> ks;
        for (int i = 0; i < n; ++i) {
            const std::string name = hetreco_cuda_kernel_name(i);
            ks.push_back({name, "sm_100a:" + name, &device_only});
        }
        return ks;
    }
    // Source units are compiled by NVRTC for sm_100a inside the B200 library
    // (the role cpujit_backend.cpp:121-177 plays on the CPU); one call per
    // unit so a failure reports that unit's own log.
    std::vector<CompiledKernel> compile(std::span<const ProgramSource> units) override {
        if (!desc_.supports_source_kernels)
            throw UnsupportedSource("backend '" + id_ + "': NVRTC is not available");
        std::vector<CompiledKernel> out;
        std::vector<BuildDiagnostic> failures;
        for (const ProgramSource& u : units) {
            const char* name = u.unit_name.c_str();
            const char* text = u.source_text.c_str();
            std::string listing(1 << 16, '\0');
            const int rc = hetreco_cuda_compile(h_, 1, &name, &text, listing.data(), listing.size());
            if (rc != HETRECO_OK) {
                // keep the unit's own compiler log (drop the library's header line)
                std::string log = hetreco_last_error();
                const std::string head = "--- unit '" + u.unit_name + "' ---\n";
                if (const std::size_t at = log.find(head); at != std::string::npos) log = log.substr(at + head.size());
                failures.push_back({u.unit_name, log});
                continue;
            }
            listing.resize(std::strlen(listing.c_str()));
            std::size_t at = 0;
            while (at < listing.size()) {
                const std::size_t tab = listing.find('\t', at), nl = listing.find('\n', at);
                out.push_back({listing.substr(tab + 1, nl - tab - 1), listing.substr(at, tab - at), &device_only});
                at = nl + 1;
            }
        }
        if (!failures.empty()) throw CompileError(std::move(failures));
        // The reference's builtin bundle (kernels.hpp:52-57) compiled from
        // source: append the precompiled fused chains (sens_recon, rss_recon;
        // csrc/host/fused_recon.hpp), which have no kernel-source form, so
        // load_builtin_kernels (session.cpp:139-148) registers them in both modes.
        if (is_builtin_bundle(units)) {
            int n = 0;
            ck(hetreco_cuda_kernel_count(&n));
            for (int i = 0; i < n; ++i) {
                const std::string name = hetreco_cuda_kernel_name(i);
                bool have = false;
                for (const CompiledKernel& k : out) have = have || k.name == name;
                if (!have) out.push_back({name, "sm_100a:" + name, &device_only});
            }
        }
        return out;
    }
    static bool is_builtin_bundle(std::span<const ProgramSource> units) {
        const auto builtins = builtin_kernel_sources();
        if (units.size() != builtins.size()) return false;
        for (std::size_t i = 0; i < units.size(); ++i)
            if (units[i].unit_name != builtins[i].unit_name) return false;
        return true;
    }
    void execute(const CompiledKernel& k, const KernelBinding& b, std::uint64_t gsize) override {
        if (k.unit_name.rfind("nvrtc#", 0) == 0) {
            ck(hetreco_cuda_execute_unit(h_, k.unit_name.c_str(), k.name.c_str(), b.input, b.input_header, b.output,
                                         b.output_header, b.params.data(), b.params.size(), gsize),
               k.name);
            return;
        }
        ck(hetreco_cuda_execute(h_, k.name.c_str(), b.input, b.input_header, b.output, b.output_header,
                                b.params.data(), b.params.size(), gsize),
           k.name);
    }
    void synchronize() override { ck(hetreco_cuda_synchronize(h_)); }

private:
    hetreco_cuda_backend h_ = nullptr;
    std::string id_;
    DeviceDescriptor desc_;
};

// One backend per visible GPU, for owned_backends() (src/backend.cpp:294-302).
std::vector<std::unique_ptr<Backend>> make_cuda_backends() {
    std::vector<std::unique_ptr<Backend>> v;
    int n = 0;
    if (hetreco_cuda_device_count(&n) != HETRECO_OK) return v;
    for (int i = 0; i < n; ++i) v.push_back(std::make_unique<CudaBackend>(i));
    return v;
}

std::unique_ptr<Backend> make_cuda_backend(int ordinal, std::uint64_t capacity, bool source_kernels) {
    return std::make_unique<CudaBackend>(ordinal, capacity, source_kernels);
}

}  // namespace hetreco_b200_integration
