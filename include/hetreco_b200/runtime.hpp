// runtime.hpp -- devices, the backend contract, the CUDA backend and the
// kernel registry.
//
// API-compatible with the reference's include/hetreco/device.hpp:15-114,
// include/hetreco/backend.hpp:16-102 and include/hetreco/kernels.hpp:15-54.
// The backend list of this build holds one CudaBackend per visible GPU
// (ids "cuda0".."cudaN-1", device type Gpu, vendor "NVIDIA", api_version =
// compute capability).  The reference's CPU backends are deliberately not
// part of the product: the CPU implementation is the test oracle (oracle/),
// and a host without GPUs therefore enumerates no devices and select_device
// throws NoMatchingDevice.
#pragma once

#include <atomic>
#include <compare>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "hetreco_b200/data.hpp"
#include "hetreco_b200/device_abi.h"

typedef struct CUstream_st* cudaStream_t;
typedef struct CUevent_st* cudaEvent_t;
typedef struct CUkern_st* cudaKernel_t;
typedef struct CUlib_st* cudaLibrary_t;

namespace hetreco {

namespace detail {
class HostStager;         // pinned-ring staging of pageable transfers (csrc/host/host_stager.hpp)
class FusedReconKernels;  // sens_recon / rss_recon as layer-1 kernels (csrc/host/fused_recon.hpp)
}

// ---- devices (device.hpp:15-114) ---------------------------------------------------

enum class DeviceType { Cpu, Gpu, Accelerator };
std::string_view device_type_name(DeviceType type);

struct ApiVersion {
    int major = 0;
    int minor = 0;
    static ApiVersion parse(std::string_view text);  // throws InvalidFilter
    std::string str() const { return std::to_string(major) + "." + std::to_string(minor); }
    auto operator<=>(const ApiVersion&) const = default;
};

struct DeviceDescriptor {
    std::string backend_id;
    std::uint32_t device_index = 0;
    DeviceType device_type = DeviceType::Cpu;
    std::string vendor;
    std::string name;
    std::string api_version;
    std::uint64_t global_memory_bytes = 0;
    std::uint64_t base_alignment_bytes = 1;
    bool supports_source_kernels = false;
    std::string label() const { return backend_id + ":" + name; }
};

class DeviceFilter {
public:
    DeviceFilter() = default;
    DeviceFilter& with_type(DeviceType type);
    DeviceFilter& with_vendor(std::string substring);
    DeviceFilter& with_name(std::string substring);
    DeviceFilter& with_min_api_version(std::string_view version);
    static DeviceFilter parse(std::string_view text);

    bool matches(const DeviceDescriptor& device) const;
    bool is_any() const;
    std::string describe() const;

    const std::optional<DeviceType>& device_type() const { return type_; }
    const std::optional<std::string>& vendor_substring() const { return vendor_; }
    const std::optional<std::string>& name_substring() const { return name_; }
    const std::optional<ApiVersion>& min_api_version() const { return min_version_; }

private:
    std::optional<DeviceType> type_;
    std::optional<std::string> vendor_;
    std::optional<std::string> name_;
    std::optional<ApiVersion> min_version_;
};

std::vector<DeviceDescriptor> enumerate_devices();
DeviceDescriptor select_device(const DeviceFilter& filter = {});
const DeviceDescriptor& select_from(std::span<const DeviceDescriptor> candidates,
                                    const DeviceFilter& filter);

// ---- kernels (kernels.hpp:15-54) ---------------------------------------------------

struct ProgramSource {
    std::string unit_name;
    std::string source_text;
};

struct CompiledKernel {
    std::string name;
    std::string unit_name;
    hetreco_kernel_fn fn = nullptr;  // host stub: device-only kernels refuse host calls
};

class KernelRegistry {
public:
    void add(std::vector<CompiledKernel> kernels);  // all-or-nothing
    const CompiledKernel& find(std::string_view name) const;
    bool contains(std::string_view name) const;
    std::vector<std::string> names() const;
    std::size_t size() const { return table_.size(); }

private:
    std::map<std::string, CompiledKernel, std::less<>> table_;
};

std::span<const ProgramSource> builtin_kernel_sources();

// ---- backend contract (backend.hpp:16-102) -------------------------------------------

using BufferId = std::uint64_t;

enum class TransferPath { Mapped, Staged };

struct KernelBinding {
    BufferId input = 0;
    BufferId input_header = 0;
    BufferId output = 0;
    BufferId output_header = 0;
    std::span<const std::byte> params;
};

class Backend {
public:
    virtual ~Backend() = default;
    virtual std::string_view id() const = 0;
    virtual std::vector<DeviceDescriptor> devices() const = 0;
    virtual TransferPath transfer_path() const = 0;
    virtual bool supports_source_kernels() const = 0;
    virtual BufferId allocate(std::uint64_t bytes) = 0;
    virtual void release(BufferId buffer) = 0;
    virtual void upload(BufferId buffer, std::uint64_t offset, std::span<const std::byte> bytes) = 0;
    virtual void download(BufferId buffer, std::uint64_t offset, std::span<std::byte> into) const = 0;
    virtual void copy(BufferId src, std::uint64_t src_offset, BufferId dst, std::uint64_t dst_offset,
                      std::uint64_t bytes) = 0;
    virtual std::vector<CompiledKernel> intrinsic_kernels() = 0;
    virtual std::vector<CompiledKernel> compile(std::span<const ProgramSource> units) = 0;
    virtual void execute(const CompiledKernel& kernel, const KernelBinding& binding,
                         std::uint64_t global_size) = 0;
    virtual void synchronize() = 0;
};

std::span<Backend* const> backend_snapshot();
Backend& backend_by_id(std::string_view id);

// ---- the CUDA backend -----------------------------------------------------------------

/**
 * One GPU.  Buffers are device allocations (cudaMalloc, 256-B aligned);
 * transfers are cudaMemcpyAsync on the backend's copy streams, ordered after
 * the compute stream by events; kernels launch asynchronously on the compute
 * stream and errors surface as DeviceError at the next synchronize().  Every
 * Backend entry point keeps the reference's synchronous contract for host
 * memory it is handed (upload/download return once the host span is no longer
 * needed); execute() stages a device copy of the borrowed params span.
 */
class CudaBackend final : public Backend {
public:
    explicit CudaBackend(int device_ordinal, std::uint64_t capacity_bytes = 0);
    ~CudaBackend() override;

    std::string_view id() const override { return id_; }
    std::vector<DeviceDescriptor> devices() const override { return {desc_}; }
    TransferPath transfer_path() const override { return TransferPath::Staged; }
    // true when NVRTC is available: compile() builds kernel-source units for
    // sm_100a at run time (the reference's cpujit role)
    bool supports_source_kernels() const override;

    BufferId allocate(std::uint64_t bytes) override;
    void release(BufferId buffer) override;
    void upload(BufferId buffer, std::uint64_t offset, std::span<const std::byte> bytes) override;
    void download(BufferId buffer, std::uint64_t offset, std::span<std::byte> into) const override;
    void copy(BufferId src, std::uint64_t src_offset, BufferId dst, std::uint64_t dst_offset,
              std::uint64_t bytes) override;
    std::vector<CompiledKernel> intrinsic_kernels() override;
    std::vector<CompiledKernel> compile(std::span<const ProgramSource> units) override;
    void execute(const CompiledKernel& kernel, const KernelBinding& binding,
                 std::uint64_t global_size) override;
    void synchronize() override;

    // ---- B200 extensions used by processes and the streaming pipeline ----
    int ordinal() const { return ordinal_; }
    void* device_pointer(BufferId buffer) const;       // base of the allocation
    std::uint64_t buffer_size(BufferId buffer) const;
    std::uint64_t live_bytes() const;
    cudaStream_t compute_stream() const { ensure(); return compute_; }
    cudaStream_t h2d_stream() const { ensure(); return h2d_; }
    cudaStream_t d2h_stream() const { ensure(); return d2h_; }
    void make_current() const;                         // ensure() + cudaSetDevice(ordinal)
    // Creates the device state (context, streams, params ring) on first use.
    void ensure() const;
    bool initialized() const { return ready_.load(std::memory_order_acquire); }
    // Raises DeviceError(last kernel) if the device reported a fault.
    void check(const char* what) const;
    // Sequence number of work enqueued on the compute stream: every enqueue
    // (backend entry points, process launches, streaming, phantom) bumps it,
    // so LaunchStats can tell whether a launch was queued directly behind the
    // same process' previous launch.
    std::uint64_t work_seq() const { return work_seq_.load(std::memory_order_relaxed); }
    void note_work() const { work_seq_.fetch_add(1, std::memory_order_relaxed); }

private:
    struct Buf {
        void* ptr = nullptr;
        std::uint64_t size = 0;
    };
    const Buf& lookup(BufferId id) const;
    void* stage_params(std::span<const std::byte> params);

    int ordinal_;
    std::string id_;
    DeviceDescriptor desc_;
    std::uint64_t capacity_;
    std::uint64_t used_ = 0;
    mutable std::mutex mu_;
    std::unordered_map<BufferId, Buf> bufs_;
    BufferId next_ = 1;
    mutable std::mutex init_mu_;
    mutable std::atomic<bool> ready_{false};
    cudaStream_t compute_ = nullptr, h2d_ = nullptr, d2h_ = nullptr;
    // params staging ring (pinned host -> device), recycled after a sync
    std::byte* ring_host_ = nullptr;
    std::byte* ring_dev_ = nullptr;
    std::uint64_t ring_size_ = 0, ring_head_ = 0;
    mutable std::string last_kernel_;
    mutable std::atomic<std::uint64_t> work_seq_{0};
    // pageable host <-> device transfers through a pinned ring (lazily built)
    mutable std::unique_ptr<detail::HostStager> stager_;
    detail::HostStager& stager() const;
    // host copies of small buffers uploaded whole (layout headers): execute()
    // of the fused kernels reads the shapes without a device round trip
    std::unordered_map<BufferId, std::vector<std::byte>> shadow_;
    // buffers whose device bytes may have been written by device work (kernel
    // outputs, D2D copy targets, raw pointers handed out): a partial upload
    // cannot start a host shadow of them, only a whole-buffer upload can
    mutable std::unordered_set<BufferId> device_written_;
    LayoutDescriptor header_layout(BufferId header) const;
    std::unique_ptr<detail::FusedReconKernels> fused_;
    // run-time compiled (NVRTC) kernels: "<unit tag>/<name>" -> entry point
    std::unordered_map<std::string, cudaKernel_t> jit_;
    std::vector<cudaLibrary_t> jit_libs_;
    std::uint64_t jit_units_ = 0;
};

// Number of CUDA devices visible to this process (0 when no driver/GPU).
int cuda_device_count();

// The intrinsic kernel bundle of CudaBackend: the six reference-ABI builtins
// (kernels/*.cl.src semantics) then the fused "sens_recon" / "rss_recon"
// chains (csrc/host/fused_recon.hpp).  nullptr past the end.
int intrinsic_kernel_count();
const char* intrinsic_kernel_name(int index);

}  // namespace hetreco
