// host_stager.hpp -- pageable <-> device transfers through a pinned ring.
//
// cudaMemcpy from pageable memory makes the driver bounce every byte through
// its own small pinned buffer on one thread (measured ~1.5-5 GB/s for the
// register/fetch path on the B200 box, vs ~55 GB/s for page-locked memory).
// The stager keeps K page-locked slots of `slot_bytes` per backend and
// pipelines: host threads copy chunk i+1 into a free slot while the copy
// engine DMAs chunk i (H2D), or DMA chunk i+1 while the threads drain chunk i
// (D2H).  Page-locked sources/destinations (cudaHostAlloc / registered) skip
// the ring and DMA directly.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace hetreco::detail {

// Tiny fork-join pool for parallel memcpy.
class CopyPool {
public:
    explicit CopyPool(unsigned threads);
    ~CopyPool();
    CopyPool(const CopyPool&) = delete;
    CopyPool& operator=(const CopyPool&) = delete;
    unsigned size() const { return unsigned(workers_.size()) + 1; }
    // memcpy(dst, src, n) split over the pool (the caller's thread takes a part)
    void copy(void* dst, const void* src, std::size_t n);

private:
    void run(unsigned index);
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable go_, done_;
    std::uint64_t generation_ = 0;
    unsigned pending_ = 0;
    bool stop_ = false;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    std::size_t n_ = 0;
};

class HostStager {
public:
    HostStager(int device, std::size_t slot_bytes = std::size_t(16) << 20, int slots = 3);
    ~HostStager();
    HostStager(const HostStager&) = delete;
    HostStager& operator=(const HostStager&) = delete;

    static bool is_pinned(const void* p);
    // Blocking transfers on `stream` (returns when the bytes have landed).
    void upload(void* dev, const void* host, std::size_t n, cudaStream_t stream);
    void download(void* host, const void* dev, std::size_t n, cudaStream_t stream);

private:
    int device_;
    std::size_t slot_;
    std::vector<std::byte*> bufs_;
    std::vector<cudaEvent_t> events_;
    CopyPool pool_;
};

}  // namespace hetreco::detail
