// processes.hpp -- the Process layer: typed parameters, the init()/launch()
// split, chains, and the builtin MRI-reconstruction processes.
//
// The reference declares Process, CompositeProcess, chain, ProcessParams and
// LaunchStats (include/hetreco/process.hpp:21-140) but ships no
// implementation; semantics here follow that header and SPEC.md:293-477.
//
// B200 design: every builtin process is a GraphProcess.  init() validates
// shapes/params, bakes plans (twiddle tables, launch shapes, scratch) and
// captures the device work into a CUDA graph; launch() is one
// cudaGraphLaunch on the session's compute stream, so a chain or a 100x loop
// pays no per-iteration host setup.  A CompositeProcess of GraphProcess
// stages captures all stages into ONE graph.  Re-pointing input/output
// handles after init (same shapes) re-captures on the next launch.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <map>
#include <memory>
#include <string>
#include <string_view>
#include <variant>
#include <vector>

#include "hetreco_b200/compute_session.hpp"

typedef struct CUgraph_st* cudaGraph_t;
typedef struct CUgraphExec_st* cudaGraphExec_t;

namespace hetreco {

// process.hpp:21-52
class ProcessParams {
public:
    using Value = std::variant<bool, std::int64_t, double, std::string>;

    ProcessParams& set(std::string key, bool value);
    ProcessParams& set(std::string key, std::int64_t value);
    ProcessParams& set(std::string key, int value) { return set(std::move(key), std::int64_t(value)); }
    ProcessParams& set(std::string key, double value);
    ProcessParams& set(std::string key, std::string value);
    ProcessParams& set(std::string key, const char* value) { return set(std::move(key), std::string(value)); }

    bool has(std::string_view key) const;
    bool get_bool(std::string_view key, bool fallback) const;
    std::int64_t get_int(std::string_view key, std::int64_t fallback) const;
    double get_real(std::string_view key, double fallback) const;
    std::string get_string(std::string_view key, std::string_view fallback) const;
    void require_known(std::initializer_list<std::string_view> known) const;
    std::size_t size() const { return values_.size(); }
    // copy without `key` (generic keys consumed by Process::init)
    ProcessParams without(std::string_view key) const;

private:
    const Value* find(std::string_view key) const;
    std::map<std::string, Value, std::less<>> values_;
};

// process.hpp:55-64.  Launch times are device time between CUDA events
// recorded around timed launches on the compute stream; they are resolved when
// stats() is read (which waits for the last launch).  Process::init param
// "launch_timing": "sampled" (default: every 16th launch timed, totals
// extrapolated from the sampled mean), "every" or "off".
struct LaunchStats {
    std::uint64_t init_calls = 0;
    std::uint64_t launches = 0;
    double last_launch_seconds = 0.0;
    double total_launch_seconds = 0.0;
    double init_seconds = 0.0;  // host wall time of init() (plan baking + capture)
    double mean_launch_seconds() const {
        return launches == 0 ? 0.0 : total_launch_seconds / double(launches);
    }
};

enum class ProcessState { Created, Initialized };

class Process {
public:
    Process(ComputeSession& session, std::string name);
    virtual ~Process();
    Process(const Process&) = delete;
    Process& operator=(const Process&) = delete;

    const std::string& name() const { return name_; }
    ComputeSession& session() { return session_; }
    ProcessState state() const { return state_; }
    const LaunchStats& stats() const;

    void set_input(DataHandle handle);
    void set_output(DataHandle handle);
    DataHandle input() const { return input_; }
    DataHandle output() const { return output_; }

    void init(const ProcessParams& params = {});
    void launch();

protected:
    virtual void on_init(const ProcessParams& params) = 0;
    virtual void on_launch() = 0;
    // Called by launch() when a handle was re-pointed after init.
    virtual void on_rebind() {}

    DataHandle require_input() const;
    DataHandle require_output() const;
    const LayoutDescriptor& input_layout() const { return session_.layout_of(require_input()); }
    const LayoutDescriptor& output_layout() const { return session_.layout_of(require_output()); }

private:
    void resolve_timings() const;

    ComputeSession& session_;
    std::string name_;
    ProcessState state_ = ProcessState::Created;
    DataHandle input_;
    DataHandle output_;
    bool rebound_ = false;
    mutable LaunchStats stats_;
    struct Timing;
    std::unique_ptr<Timing> timing_;
    int timing_mode_ = 1;  // "launch_timing": 0 every, 1 sampled (default), 2 off
};

// A process whose device work is recorded once into a CUDA graph.
class GraphProcess : public Process {
public:
    using Process::Process;
    ~GraphProcess() override;
    // Enqueue this process' device work on `stream` (used for capture).
    virtual void record(cudaStream_t stream) = 0;
    // Launches the recorded work `reps` times WITHOUT the graph, with CUDA
    // events between kernels on the compute stream; returns the mean device
    // seconds of each kernel in record order (used by bench.py's roofline).
    std::vector<double> profile(int reps);

protected:
    void on_init(const ProcessParams& params) final;
    void on_launch() override;
    void on_rebind() override;
    // Validate params/shapes and bake plans; record() must work afterwards.
    virtual void bake(const ProcessParams& params) = 0;
    // Re-validate after a handle change (default: bake with the same params).
    virtual void rebake() { bake(params_); }
    // Re-read the device pointers after a handle change that kept every array
    // shape and type (SPEC "re-point between launches"): plans, twiddles and
    // scratch stay, the graph is re-recorded and patched in place with
    // cudaGraphExecUpdate instead of re-instantiated.  Default: rebake().
    virtual void repoint() { rebake(); }
    // update: try cudaGraphExecUpdate of the existing executable first.
    void capture(bool update = false);
    // Processes call mark(s) after each kernel they enqueue in record().
    void mark(cudaStream_t s);
    // true while profile() replays record() kernel by kernel (no graph)
    bool profiling() const { return profiling_; }
    // Whether the captured graph's kernel -> kernel edges become programmatic
    // (PDL) edges.  Per-process measured default (HETRECO_PDL=0|1 overrides).
    virtual bool programmatic_edges() const { return false; }

private:
    void snapshot_layouts();
    ProcessParams params_;
    LayoutDescriptor in_snap_, out_snap_;  // layouts the current plans were baked for
    bool profiling_ = false;
    std::vector<cudaEvent_t> marks_;
    cudaGraph_t graph_ = nullptr;
    cudaGraphExec_t exec_ = nullptr;
};

// process.hpp:122-140
class CompositeProcess : public GraphProcess {
public:
    CompositeProcess(ComputeSession& session, std::string name, std::vector<std::unique_ptr<Process>>&& stages);
    std::size_t stage_count() const { return stages_.size(); }
    Process& stage(std::size_t i) { return *stages_.at(i); }
    void record(cudaStream_t stream) override;

protected:
    void bake(const ProcessParams& params) override;
    void rebake() override {}
    void repoint() override {}
    void on_launch() override;

private:
    std::vector<std::unique_ptr<Process>> stages_;
    bool all_graph_ = true;
};

// On failure (ChainMismatch, InvalidArgument) the stages stay in `stages`.
std::unique_ptr<CompositeProcess> chain(ComputeSession& session, std::string name,
                                        std::vector<std::unique_ptr<Process>>&& stages);

// ---- builtin processes ------------------------------------------------

// negate: out = max_value - in over array 0 (UINT8 / FLOAT32).  Params:
// "max_value" (real; default 255 for UINT8, 1.0 for FLOAT32).  In-place allowed.
std::unique_ptr<GraphProcess> make_negate(ComputeSession& s, std::string name = "negate");

// fft2d over array 0 (COMPLEX64 [nx, ny, batch...]) into array 0 of the output.
// Params: "direction" = "forward" | "inverse" (default "forward"; inverse is
// scaled by 1/(nx*ny)), "shift" (bool; ifftshift before / fftshift after,
// both spatial axes).  nx, ny powers of two (else ShapeMismatch).
std::unique_ptr<GraphProcess> make_fft2d(ComputeSession& s, std::string name = "fft2d");

// complex_element_prod: input [x, s] -> out = x * (conj?) s (s repeats
// cyclically).  Params: "conjugate_s" (bool, default true).
std::unique_ptr<GraphProcess> make_complex_element_prod(ComputeSession& s, std::string name = "complex_element_prod");

// ximage_sum: [nx,ny,C,F...] -> [nx,ny,F...] sum over coils.
std::unique_ptr<GraphProcess> make_ximage_sum(ComputeSession& s, std::string name = "ximage_sum");

// rss_combine: COMPLEX64 [nx,ny,C,F...] -> FLOAT32 sqrt(sum_c |x|^2).
std::unique_ptr<GraphProcess> make_rss_combine(ComputeSession& s, std::string name = "rss_combine");

// sens_recon (Eq. 1): input [Y [nx,ny,C,F], S [nx,ny,C]] -> M [nx,ny,F]
// COMPLEX64, fused: axis-1 IFFT pass, then axis-0 IFFT + conj(S) multiply +
// coil sum in one pass.  Params: "shift" (bool).
std::unique_ptr<GraphProcess> make_sens_recon(ComputeSession& s, std::string name = "sens_recon");

// rss_recon: input [Y] -> FLOAT32 [nx,ny,F] = sqrt(sum_c |IFFT(Y_c)|^2), fused
// the same way.  Params: "shift" (bool).
std::unique_ptr<GraphProcess> make_rss_recon(ComputeSession& s, std::string name = "rss_recon");

// Factory by kind name ("negate", "fft2d", "complex_element_prod",
// "ximage_sum", "rss_combine", "sens_recon", "rss_recon", and the SENSE model
// "sense_forward" (E m = P F (S m), input [M, S(, mask)] -> k-space
// [nx,ny,C,F]) / "sense_normal" (E^H E m -> [nx,ny,F]); square images).
std::unique_ptr<GraphProcess> make_process(ComputeSession& s, std::string_view kind, std::string name = {});

// ---- host-streamed reconstruction (paper's pinned/mapped streaming) ------------------------

// Reconstructs F frames of k-space that live in HOST memory (pinned for
// full-rate DMA) chunk by chunk: H2D of chunk k+1 on the H2D copy stream,
// the fused recon of chunk k on the compute stream and D2H of chunk k-1 on
// the D2H copy stream overlap (double-buffered device slabs).  Sensitivity
// maps are uploaded once at construction.
class StreamingRecon {
public:
    enum class Method { Sense, Rss };
    StreamingRecon(ComputeSession& session, Method method, std::uint64_t nx, std::uint64_t ny,
                   std::uint64_t coils, std::uint64_t chunk_frames, const void* host_smaps, bool shift = false);
    ~StreamingRecon();
    StreamingRecon(const StreamingRecon&) = delete;
    StreamingRecon& operator=(const StreamingRecon&) = delete;

    // host_kspace: [nx,ny,C,frames] COMPLEX64; host_out: [nx,ny,frames]
    // (COMPLEX64 for Sense, FLOAT32 for Rss).  Blocks until host_out is filled.
    void run(const void* host_kspace, std::uint64_t frames, void* host_out);

    std::uint64_t chunk_frames() const { return chunk_; }
    std::uint64_t bytes_in_per_frame() const { return in_frame_bytes_; }
    std::uint64_t bytes_out_per_frame() const { return out_frame_bytes_; }

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
    std::uint64_t chunk_ = 0, in_frame_bytes_ = 0, out_frame_bytes_ = 0;
};

}  // namespace hetreco
