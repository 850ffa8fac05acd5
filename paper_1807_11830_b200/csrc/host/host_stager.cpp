// host_stager.cpp -- see host_stager.hpp.
#include "host_stager.hpp"

#include <emmintrin.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

#include "hetreco_b200/error_types.hpp"

namespace hetreco::detail {

namespace {
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw DeviceError(what, cudaGetErrorString(e));
    }
}
}  // namespace

// ---- CopyPool -----------------------------------------------------------------------------

namespace {
// Bytes per part, rounded up to a cache line; parts * result >= n for every n.
std::size_t part_bytes(std::size_t n, unsigned parts) {
    return ((n + parts - 1) / parts + 63) & ~std::size_t(63);
}

// Streaming (non-temporal) stores for the staging copies: the destination is
// consumed by the copy engine or by the caller much later, so write-allocating
// it in the cache only adds a read-for-ownership per line to a copy that is
// host-memory-bandwidth bound next to the concurrent DMA.  HETRECO_STAGER_NT=0
// falls back to memcpy (A/B runs).
bool nt_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("HETRECO_STAGER_NT");
        return !(v && *v == '0');
    }();
    return on;
}

void copy_part(char* d, const char* s, std::size_t n) {
    if (!nt_enabled() || n < 4096 || (reinterpret_cast<std::uintptr_t>(d) & 15)) {
        std::memcpy(d, s, n);
        return;
    }
    std::size_t i = 0;
    for (; i + 64 <= n; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
        const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
    }
    if (i < n) std::memcpy(d + i, s + i, n - i);
    _mm_sfence();  // the stores are globally visible before the DMA is enqueued
}
}  // namespace

CopyPool::CopyPool(unsigned threads) {
    for (unsigned i = 1; i < std::max(1u, threads); ++i) workers_.emplace_back([this, i] { run(i); });
}

CopyPool::~CopyPool() {
    {
        std::lock_guard lk(mu_);
        stop_ = true;
        ++generation_;
    }
    go_.notify_all();
    for (auto& t : workers_) t.join();
}

void CopyPool::run(unsigned index) {
    std::uint64_t seen = 0;
    for (;;) {
        char* d;
        const char* s;
        std::size_t n;
        {
            std::unique_lock lk(mu_);
            go_.wait(lk, [&] { return generation_ != seen; });
            seen = generation_;
            if (stop_) return;
            d = dst_;
            s = src_;
            n = n_;
        }
        const unsigned parts = size();
        const std::size_t per = part_bytes(n, parts);
        const std::size_t b = std::min(n, per * index), e = std::min(n, b + per);
        if (e > b) copy_part(d + b, s + b, e - b);
        {
            std::lock_guard lk(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
}

void CopyPool::copy(void* dst, const void* src, std::size_t n) {
    if (workers_.empty() || n < (std::size_t(1) << 20)) {
        copy_part(static_cast<char*>(dst), static_cast<const char*>(src), n);
        return;
    }
    {
        std::lock_guard lk(mu_);
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        n_ = n;
        pending_ = unsigned(workers_.size());
        ++generation_;
    }
    go_.notify_all();
    const unsigned parts = size();
    const std::size_t per = part_bytes(n, parts);
    copy_part(static_cast<char*>(dst), static_cast<const char*>(src), std::min(n, per));  // the caller's share (part 0)
    std::unique_lock lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
}

// ---- HostStager ---------------------------------------------------------------------------

// memcpy threads of the staging pool: half the host's hardware threads, at
// most 8 (HETRECO_STAGER_THREADS overrides, for A/B runs).
unsigned copy_threads() {
    if (const char* v = std::getenv("HETRECO_STAGER_THREADS"); v && *v) return unsigned(std::max(1, std::atoi(v)));
    return std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2));
}

HostStager::HostStager(int device, std::size_t slot_bytes, int slots)
    : device_(device), slot_(slot_bytes),
      pool_(copy_threads()) {
    cudaSetDevice(device_);
    for (int i = 0; i < slots; ++i) {
        std::byte* p = nullptr;
        ck(cudaHostAlloc(reinterpret_cast<void**>(&p), slot_, cudaHostAllocPortable), "cudaHostAlloc(stager)");
        bufs_.push_back(p);
        cudaEvent_t e = nullptr;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate(stager)");
        events_.push_back(e);
    }
}

HostStager::~HostStager() {
    for (auto e : events_) cudaEventDestroy(e);
    for (auto p : bufs_) cudaFreeHost(p);
}

bool HostStager::is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void HostStager::upload(void* dev, const void* host, std::size_t n, cudaStream_t st) {
    const int K = int(bufs_.size());
    std::size_t done = 0;
    for (std::size_t i = 0; done < n; ++i) {
        const int k = int(i % std::size_t(K));
        const std::size_t len = std::min(slot_, n - done);
        // the slot's previous DMA (K chunks ago) must have drained
        ck(cudaEventSynchronize(events_[std::size_t(k)]), "stager upload wait");
        pool_.copy(bufs_[std::size_t(k)], static_cast<const char*>(host) + done, len);
        ck(cudaMemcpyAsync(static_cast<char*>(dev) + done, bufs_[std::size_t(k)], len, cudaMemcpyHostToDevice, st),
           "cudaMemcpyAsync(staged H2D)");
        ck(cudaEventRecord(events_[std::size_t(k)], st), "stager upload record");
        done += len;
    }
    ck(cudaStreamSynchronize(st), "stager upload");
}

void HostStager::download(void* host, const void* dev, std::size_t n, cudaStream_t st) {
    const int K = int(bufs_.size());
    const std::size_t chunks = (n + slot_ - 1) / slot_;
    auto issue = [&](std::size_t i) {
        const int k = int(i % std::size_t(K));
        const std::size_t off = i * slot_, len = std::min(slot_, n - off);
        ck(cudaMemcpyAsync(bufs_[std::size_t(k)], static_cast<const char*>(dev) + off, len, cudaMemcpyDeviceToHost, st),
           "cudaMemcpyAsync(staged D2H)");
        ck(cudaEventRecord(events_[std::size_t(k)], st), "stager download record");
    };
    // K-1 chunks in flight ahead of the host drain
    for (std::size_t i = 0; i < std::min<std::size_t>(chunks, std::size_t(K - 1)); ++i) issue(i);
    for (std::size_t i = 0; i < chunks; ++i) {
        const int k = int(i % std::size_t(K));
        ck(cudaEventSynchronize(events_[std::size_t(k)]), "stager download wait");
        const std::size_t off = i * slot_, len = std::min(slot_, n - off);
        pool_.copy(static_cast<char*>(host) + off, bufs_[std::size_t(k)], len);
        if (i + std::size_t(K - 1) < chunks) issue(i + std::size_t(K - 1));
    }
}

}  // namespace hetreco::detail
