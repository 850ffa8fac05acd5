// session.hpp -- ComputeSession, the CLapp role: one selected device, the
// device-resident Data registry, the kernel registry and an in-order queue.
// API-compatible with the reference's include/hetreco/session.hpp:18-137.
//
// B200 specifics: the queue is the CudaBackend compute stream (kernels run
// asynchronously; fetch_data / synchronize surface device faults as
// DeviceError); each Data set is one cudaMalloc'd buffer laid out by pack()
// plus a device copy of its layout header; pinned NDArrays move by DMA.
#pragma once

#include <cstdint>
#include <span>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "hetreco_b200/data.hpp"
#include "hetreco_b200/runtime.hpp"

namespace hetreco {

struct DataHandle {
    std::uint64_t session_uid = 0;
    std::uint64_t id = 0;
    bool valid() const { return id != 0; }
    bool operator==(const DataHandle&) const = default;
};

struct TransferCounters {
    std::uint64_t host_to_device = 0;
    std::uint64_t device_to_host = 0;
    bool operator==(const TransferCounters&) const = default;
};

class ComputeSession {
public:
    explicit ComputeSession(const DeviceFilter& filter = {});
    explicit ComputeSession(const DeviceDescriptor& device);
    explicit ComputeSession(Backend& backend, std::uint32_t device_index = 0);
    ~ComputeSession();
    ComputeSession(const ComputeSession&) = delete;
    ComputeSession& operator=(const ComputeSession&) = delete;

    const DeviceDescriptor& device() const { return selected_; }
    Backend& backend() { return backend_; }
    std::uint64_t uid() const { return session_uid_; }

    // ---- data (session.hpp:73-90) ----
    DataHandle register_data(const Data& data);
    // register_data from borrowed host buffers (no intermediate NDArray copy;
    // the C-ABI path): one logical transfer, same packing and counters.
    struct HostArrayRef {
        ArrayShape shape;
        const void* data = nullptr;
    };
    DataHandle register_host(std::span<const HostArrayRef> arrays, DataKind kind = DataKind::Generic);
    Data fetch_data(DataHandle handle, HostMemory memory = HostMemory::Pageable);
    void release_data(DataHandle handle);
    const LayoutDescriptor& layout_of(DataHandle handle) const;
    DataKind kind_of(DataHandle handle) const;
    std::size_t live_data_count() const { return slots_.size(); }
    std::vector<std::byte> fetch_header_bytes(DataHandle handle);
    void copy_array(DataHandle src, std::size_t src_index, DataHandle dst, std::size_t dst_index);

    // B200 extensions: device-side allocation without a host payload (zero
    // filled; no transfer is counted), and raw access for processes.
    DataHandle allocate_data(std::span<const ArrayShape> arrays, DataKind kind = DataKind::Generic);
    // Fetch into caller-provided host buffers (one per array, sized per layout);
    // counts one device-to-host transfer.
    void fetch_into(DataHandle handle, std::span<void* const> host_arrays);
    void* device_array(DataHandle handle, std::size_t index) const;
    const std::uint64_t* device_header(DataHandle handle) const;
    CudaBackend& cuda() const;  // throws InvalidArgument when not a CUDA backend

    // ---- kernels (session.hpp:94-124) ----
    void load_builtin_kernels();
    void load_kernels(std::span<const ProgramSource> units);
    const KernelRegistry& kernels() const { return kernel_table_; }
    void launch_kernel(std::string_view name, DataHandle input, DataHandle output,
                       std::span<const std::byte> params, std::uint64_t global_size);
    void synchronize();

    // ---- accounting ----
    TransferCounters counters() const { return transfers_; }
    void reset_counters() { transfers_ = {}; }

private:
    struct Slot {
        BufferId payload = 0;
        BufferId header_buf = 0;
        LayoutDescriptor layout;
        DataKind kind = DataKind::Generic;
    };
    const Slot& resolve(DataHandle handle) const;
    // record `index` of a live entry, with `role` naming the side in errors
    const LayoutRecord& record_of(const Slot& e, std::size_t index, const char* role) const;
    DataHandle insert(const LayoutDescriptor& layout, DataKind kind, std::span<const void* const> host_src);
    void drop_buffers(const Slot& e) noexcept;

    Backend& backend_;
    DeviceDescriptor selected_;
    std::uint64_t session_uid_ = 0;
    std::uint64_t pack_alignment_ = 256;
    std::uint64_t next_handle_id_ = 1;
    std::unordered_map<std::uint64_t, Slot> slots_;
    KernelRegistry kernel_table_;
    TransferCounters transfers_;
    bool have_builtins_ = false;
};

}  // namespace hetreco
