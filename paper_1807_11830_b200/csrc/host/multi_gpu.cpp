// multi_gpu.cpp -- MultiGpuRecon: frame slabs of one host volume on several
// GPUs, one persistent host worker per slab (SURVEY.md §8 e).  Nothing
// crosses devices: each worker streams its own contiguous byte range of the
// caller's k-space buffer and writes its own range of the output.
#include "hetreco_b200/multi_gpu.hpp"

#include <chrono>
#include <condition_variable>
#include <exception>
#include <future>
#include <mutex>
#include <thread>

#include "hetreco_b200/numa.hpp"

namespace hetreco {

std::pair<std::uint64_t, std::uint64_t> frame_slab(std::uint64_t index, std::uint64_t count, std::uint64_t frames) {
    if (count == 0 || index >= count)
        throw InvalidArgument("frame slab " + std::to_string(index) + " of " + std::to_string(count) +
                              " does not exist");
    // 128-bit-safe for any realistic frame count: frames * count < 2^64
    return {index * frames / count, (index + 1) * frames / count};
}

struct MultiGpuRecon::Worker {
    std::string backend_id;
    std::thread thread;
    std::mutex mu;
    std::condition_variable cv;
    bool stop = false;
    bool has_job = false;
    bool done = false;
    // job
    const char* src = nullptr;
    char* dst = nullptr;
    std::uint64_t frames = 0;
    double seconds = 0.0;
    std::exception_ptr error;

    void loop(StreamingRecon::Method method, std::uint64_t nx, std::uint64_t ny, std::uint64_t coils,
              std::uint64_t chunk, const void* smaps, bool shift, bool bind_numa, std::promise<void>& ready) {
        std::unique_ptr<ComputeSession> session;
        std::unique_ptr<StreamingRecon> stream;
        try {
            auto* cb = dynamic_cast<CudaBackend*>(&backend_by_id(backend_id));
            if (!cb) throw InvalidArgument("backend '" + backend_id + "' is not a CUDA backend");
            if (bind_numa) bind_thread_to_numa_node(device_numa_node(cb->ordinal()));
            session = std::make_unique<ComputeSession>(*cb);
            stream = std::make_unique<StreamingRecon>(*session, method, nx, ny, coils, chunk, smaps, shift);
            ready.set_value();
        } catch (...) {
            ready.set_exception(std::current_exception());
            return;
        }
        for (;;) {
            std::unique_lock lk(mu);
            cv.wait(lk, [&] { return stop || has_job; });
            if (stop) break;
            lk.unlock();
            std::exception_ptr err;
            const auto t0 = std::chrono::steady_clock::now();
            try {
                if (frames) stream->run(src, frames, dst);
            } catch (...) {
                err = std::current_exception();
            }
            const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            lk.lock();
            error = err;
            seconds = secs;
            has_job = false;
            done = true;
            cv.notify_all();
        }
        // stream and session are destroyed on the thread that made them
        stream.reset();
        session.reset();
    }
};

MultiGpuRecon::MultiGpuRecon(const std::vector<std::string>& ids, StreamingRecon::Method method, std::uint64_t nx,
                             std::uint64_t ny, std::uint64_t coils, std::uint64_t chunk, const void* smaps, bool shift,
                             bool bind_numa) {
    if (ids.empty()) throw InvalidArgument("multi-GPU recon needs at least one device");
    in_frame_bytes_ = nx * ny * coils * 8;
    out_frame_bytes_ = nx * ny * (method == StreamingRecon::Method::Sense ? 8 : 4);
    std::vector<std::future<void>> ready;
    std::vector<std::unique_ptr<std::promise<void>>> promises;
    for (const std::string& id : ids) {
        auto w = std::make_unique<Worker>();
        w->backend_id = id;
        promises.push_back(std::make_unique<std::promise<void>>());
        ready.push_back(promises.back()->get_future());
        Worker* wp = w.get();
        std::promise<void>* pp = promises.back().get();
        w->thread = std::thread([=] { wp->loop(method, nx, ny, coils, chunk, smaps, shift, bind_numa, *pp); });
        workers_.push_back(std::move(w));
    }
    std::exception_ptr first;
    for (auto& f : ready) {
        try {
            f.get();
        } catch (...) {
            if (!first) first = std::current_exception();
        }
    }
    if (first) {
        shutdown();  // joins every worker (a failed one has already returned)
        std::rethrow_exception(first);
    }
}

MultiGpuRecon::~MultiGpuRecon() { shutdown(); }

void MultiGpuRecon::shutdown() {
    for (auto& w : workers_) {
        {
            std::lock_guard lk(w->mu);
            w->stop = true;
        }
        w->cv.notify_all();
    }
    for (auto& w : workers_)
        if (w->thread.joinable()) w->thread.join();
    workers_.clear();
}

std::size_t MultiGpuRecon::device_count() const { return workers_.size(); }

void MultiGpuRecon::run(const void* host_in, std::uint64_t frames, void* host_out) {
    if (frames && (!host_in || !host_out)) throw InvalidArgument("multi-GPU recon: null host buffer");
    const std::uint64_t G = workers_.size();
    last_.assign(G, {});
    for (std::uint64_t g = 0; g < G; ++g) {
        const auto [b, e] = frame_slab(g, G, frames);
        Worker& w = *workers_[g];
        last_[g].backend_id = w.backend_id;
        last_[g].first_frame = b;
        last_[g].frames = e - b;
        std::lock_guard lk(w.mu);
        w.src = static_cast<const char*>(host_in) + b * in_frame_bytes_;
        w.dst = static_cast<char*>(host_out) + b * out_frame_bytes_;
        w.frames = e - b;
        w.error = nullptr;
        w.done = false;
        w.has_job = true;
        w.cv.notify_all();
    }
    std::exception_ptr first;
    for (std::uint64_t g = 0; g < G; ++g) {
        Worker& w = *workers_[g];
        std::unique_lock lk(w.mu);
        w.cv.wait(lk, [&] { return w.done; });
        last_[g].seconds = w.seconds;
        if (w.error && !first) first = w.error;
    }
    if (first) std::rethrow_exception(first);
}

}  // namespace hetreco
