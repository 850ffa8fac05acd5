// multi_gpu.hpp -- one host volume reconstructed over several GPUs by frame
// slab (SURVEY.md §8 e).
//
// The reference has one device per session and no multi-device path
// (SPEC.md:79); frames are independent (Eq. 1 is per frame),
// so the k-space volume [nx, ny, C, F] (column-major: each frame one
// contiguous nx*ny*C*8-byte slab) is split into contiguous frame slabs, slab
// g = frames [floor(g F / G), floor((g + 1) F / G)).  Each device gets one
// host worker thread (bound to the device's NUMA node), its own
// ComputeSession and its own StreamingRecon that moves its slab from the
// caller's (pinned) host buffer and writes its slab of the output in place:
// no gather, no collective, no host copy.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "hetreco_b200/processes.hpp"

namespace hetreco {

// [begin, end) frames of slab `index` out of `count` (floor partition: slab
// sizes differ by at most one frame).  InvalidArgument when index >= count.
std::pair<std::uint64_t, std::uint64_t> frame_slab(std::uint64_t index, std::uint64_t count, std::uint64_t frames);

class MultiGpuRecon {
public:
    struct SlabRun {
        std::string backend_id;
        std::uint64_t first_frame = 0;
        std::uint64_t frames = 0;
        double seconds = 0.0;  // host wall time of this slab's stream, last run()
    };

    // backend_ids: one entry per slab ("cuda0", "cuda1", ...; an id may repeat
    // to split a volume over streams of one GPU).  bind_numa: pin each worker
    // to its GPU's NUMA node.  host_smaps: [nx, ny, C] COMPLEX64 (Sense).
    MultiGpuRecon(const std::vector<std::string>& backend_ids, StreamingRecon::Method method, std::uint64_t nx,
                  std::uint64_t ny, std::uint64_t coils, std::uint64_t chunk_frames, const void* host_smaps,
                  bool shift = false, bool bind_numa = true);
    ~MultiGpuRecon();
    MultiGpuRecon(const MultiGpuRecon&) = delete;
    MultiGpuRecon& operator=(const MultiGpuRecon&) = delete;

    // Reconstructs `frames` frames: host_kspace [nx, ny, C, frames] COMPLEX64,
    // host_out [nx, ny, frames] (COMPLEX64 Sense / FLOAT32 Rss).  Blocks until
    // every slab is written; a failing slab's error is rethrown (lowest slab
    // first) after all workers stopped.
    void run(const void* host_kspace, std::uint64_t frames, void* host_out);

    std::size_t device_count() const;
    const std::vector<SlabRun>& last_run() const { return last_; }

private:
    struct Worker;
    void shutdown();
    std::vector<std::unique_ptr<Worker>> workers_;
    std::vector<SlabRun> last_;
    std::uint64_t in_frame_bytes_ = 0, out_frame_bytes_ = 0;
};

}  // namespace hetreco
