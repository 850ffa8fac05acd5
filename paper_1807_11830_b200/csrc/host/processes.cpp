// processes.cpp -- Process / GraphProcess / CompositeProcess and the builtin
// reconstruction processes (reference include/hetreco/process.hpp:21-140,
// SPEC.md:293-477).
#include "hetreco_b200/processes.hpp"

#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "../kernels/launch.hpp"
#include "fused_recon.hpp"

namespace hetreco {

namespace {

void ck(cudaError_t e, const std::string& what) {
    if (e == cudaSuccess) return;
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) throw AllocationFailure(what + ": " + cudaGetErrorString(e));
    throw DeviceError(what, cudaGetErrorString(e));
}

bool is_pow2(std::uint64_t v) { return v && !(v & (v - 1)); }

long env_or(const char* name, long fallback) {
    const char* v = std::getenv(name);
    return v && *v ? std::atol(v) : fallback;
}

// The staged-map SENSE combine (fft_combine_ss.cu) where it measured faster
// (256^2 C3: 131 -> 114 us; 512^2 x 8: 162 -> 159 us; 160^2: even), unless
// HETRECO_COMBINE_SS=0 (off) / =1 (every supported size).
bool combine_ss_enabled(std::uint64_t nx) {
    const char* e = std::getenv("HETRECO_COMBINE_SS");
    if (e && *e == '0') return false;
    if (!dev::combine_ss_supported(nx)) return false;
    return (e && *e == '1') || (nx >= 64 && nx <= 512 && is_pow2(nx));
}

// The measured default axis-0 + combine kernel for a fp32 SENSE/RSS chunk of
// `frames` frames: coil-parallel when the coil-serial kernel would leave the
// SMs short of lines (few frames), the staged-map SENSE kernel where it
// measured faster, else the register-prefetch kernel (variant 11: fp32,
// prefetch, register copy; ping-pong at 512).
dev::LaunchShape plan_combine_fp32(std::uint64_t nx, std::uint64_t ny, std::uint64_t nc, std::uint64_t frames,
                                   dev::Combine mode, int sms) {
    if (dev::combine_cp_preferred(nx, ny * frames, nc, sms)) return dev::plan_combine_cp(nx, mode, ny * frames, sms);
    if (mode == dev::Combine::Sense && combine_ss_enabled(nx)) return dev::plan_combine_ss(nx, ny, frames, sms);
    return dev::plan_contig(nx, mode, ny * frames, sms);
}

// Owning device allocation on the session's GPU.
class DevMem {
public:
    DevMem() = default;
    DevMem(std::uint64_t bytes) : size_(bytes) {
        ck(cudaMalloc(&p_, bytes ? bytes : 1), "cudaMalloc(process scratch)");
    }
    ~DevMem() {
        if (p_) cudaFree(p_);
    }
    DevMem(DevMem&& o) noexcept : p_(o.p_), size_(o.size_) { o.p_ = nullptr; }
    DevMem& operator=(DevMem&& o) noexcept {
        if (this != &o) {
            if (p_) cudaFree(p_);
            p_ = o.p_;
            size_ = o.size_;
            o.p_ = nullptr;
        }
        return *this;
    }
    void* get() const { return p_; }
    template <class T>
    T* as() const { return static_cast<T*>(p_); }
    std::uint64_t size() const { return size_; }

private:
    void* p_ = nullptr;
    std::uint64_t size_ = 0;
};

DevMem upload_bytes(const void* src, std::uint64_t n) {
    DevMem m(n);
    ck(cudaMemcpy(m.get(), src, n, cudaMemcpyHostToDevice), "cudaMemcpy(process constants)");
    return m;
}

// W_N^t = exp(dir * 2 pi i t / N), t < N, computed in double, stored as float
// (the reference bakes its pass payloads the same way, fft_radix2_pass.cl.src:15-16).
DevMem twiddle_table(std::uint64_t N, int dir) {
    std::vector<float> w(2 * std::max<std::uint64_t>(N, 1));
    for (std::uint64_t t = 0; t < N; ++t) {
        const double th = double(dir) * 2.0 * M_PI * double(t) / double(N);
        w[2 * t] = float(std::cos(th));
        w[2 * t + 1] = float(std::sin(th));
    }
    return upload_bytes(w.data(), w.size() * sizeof(float));
}

int sm_count(int ordinal) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, ordinal) != cudaSuccess) n = 148;
    return n;
}

std::uint64_t prod(const LayoutRecord& r, std::uint32_t from, std::uint32_t to) {
    std::uint64_t n = 1;
    for (std::uint32_t d = from; d < to && d < r.rank; ++d) n *= r.dims[d];
    return n;
}

std::string dims_str(const LayoutRecord& r) {
    std::string s = "[";
    for (std::uint32_t d = 0; d < r.rank; ++d) s += (d ? "," : "") + std::to_string(r.dims[d]);
    return s + "]";
}

const LayoutRecord& array_of(const LayoutDescriptor& l, std::size_t i, const std::string& who) {
    if (i >= l.records.size())
        throw ShapeMismatch(who + ": data set has " + std::to_string(l.records.size()) + " array(s), needs array " +
                            std::to_string(i));
    return l.records[i];
}

void require_type(const LayoutRecord& r, ElementType t, const std::string& who) {
    if (r.element_type != t)
        throw UnsupportedElementType(who + ": expected " + std::string(element_type_name(t)) + ", got " +
                                     std::string(element_type_name(r.element_type)));
}

}  // namespace

// ---- ProcessParams ----------------------------------------------------------------------

ProcessParams& ProcessParams::set(std::string k, bool v) { values_[std::move(k)] = v; return *this; }
ProcessParams& ProcessParams::set(std::string k, std::int64_t v) { values_[std::move(k)] = v; return *this; }
ProcessParams& ProcessParams::set(std::string k, double v) { values_[std::move(k)] = v; return *this; }
ProcessParams& ProcessParams::set(std::string k, std::string v) { values_[std::move(k)] = std::move(v); return *this; }

const ProcessParams::Value* ProcessParams::find(std::string_view k) const {
    auto it = values_.find(k);
    return it == values_.end() ? nullptr : &it->second;
}

bool ProcessParams::has(std::string_view k) const { return find(k) != nullptr; }

bool ProcessParams::get_bool(std::string_view k, bool fb) const {
    const Value* v = find(k);
    if (!v) return fb;
    if (auto* b = std::get_if<bool>(v)) return *b;
    throw InvalidParams("parameter '" + std::string(k) + "' is not a boolean");
}

std::int64_t ProcessParams::get_int(std::string_view k, std::int64_t fb) const {
    const Value* v = find(k);
    if (!v) return fb;
    if (auto* i = std::get_if<std::int64_t>(v)) return *i;
    throw InvalidParams("parameter '" + std::string(k) + "' is not an integer");
}

double ProcessParams::get_real(std::string_view k, double fb) const {
    const Value* v = find(k);
    if (!v) return fb;
    if (auto* d = std::get_if<double>(v)) return *d;
    if (auto* i = std::get_if<std::int64_t>(v)) return double(*i);  // integers promote
    throw InvalidParams("parameter '" + std::string(k) + "' is not a real");
}

std::string ProcessParams::get_string(std::string_view k, std::string_view fb) const {
    const Value* v = find(k);
    if (!v) return std::string(fb);
    if (auto* s = std::get_if<std::string>(v)) return *s;
    throw InvalidParams("parameter '" + std::string(k) + "' is not a string");
}

ProcessParams ProcessParams::without(std::string_view key) const {
    ProcessParams p = *this;
    if (auto it = p.values_.find(key); it != p.values_.end()) p.values_.erase(it);
    return p;
}

void ProcessParams::require_known(std::initializer_list<std::string_view> known) const {
    for (const auto& [k, v] : values_) {
        bool ok = false;
        for (auto q : known) ok = ok || q == k;
        if (!ok) {
            std::string allowed;
            for (auto q : known) allowed += (allowed.empty() ? "" : ", ") + std::string(q);
            throw InvalidParams("unknown parameter '" + k + "' (accepted: " + (allowed.empty() ? "none" : allowed) +
                                ")");
        }
    }
}

// ---- Process ----------------------------------------------------------------------------

// Device-side launch timing (LaunchStats, process.hpp:55-64).  A launch that
// is queued behind the previous one on the same stream starts exactly when
// that one stops, so back-to-back launches record only a stop event and chain
// to the previous stop (one cudaEventRecord per launch instead of two: the
// event records were 3/4 of the host cost of a tiny process launch); a launch
// onto an idle stream records its own start.
struct Process::Timing {
    static constexpr int kRing = 128;
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaEvent_t start[kRing]{}, stop[kRing]{};
    bool chained[kRing]{};
    int head = 0, pending = 0;
    int last = -1;  // slot of the most recent launch (its stop event stays valid until resolved + reused)
    std::uint64_t seq_after = ~std::uint64_t(0);  // backend work_seq() right after that launch
    // "launch_timing": 0 = every launch, 1 = every kSample-th launch (default)
    // (totals extrapolated from the sampled mean), 2 = off
    int mode = 1;
    static constexpr std::uint64_t kSample = 16;
    double sampled_seconds = 0.0;
    std::uint64_t sampled = 0;
};

Process::Process(ComputeSession& s, std::string name) : session_(s), name_(std::move(name)) {}

Process::~Process() {
    if (timing_) {
        cudaSetDevice(timing_->device);
        for (int i = 0; i < Timing::kRing; ++i) {
            if (timing_->start[i]) cudaEventDestroy(timing_->start[i]);
            if (timing_->stop[i]) cudaEventDestroy(timing_->stop[i]);
        }
    }
}

void Process::set_input(DataHandle h) {
    session_.layout_of(h);  // UnknownHandle for foreign/stale handles
    if (state_ == ProcessState::Initialized && !(h == input_)) rebound_ = true;
    input_ = h;
}

void Process::set_output(DataHandle h) {
    session_.layout_of(h);
    if (state_ == ProcessState::Initialized && !(h == output_)) rebound_ = true;
    output_ = h;
}

DataHandle Process::require_input() const {
    if (!input_.valid()) throw InvalidArgument("process '" + name_ + "' has no input handle");
    return input_;
}

DataHandle Process::require_output() const {
    if (!output_.valid()) throw InvalidArgument("process '" + name_ + "' has no output handle");
    return output_;
}

void Process::init(const ProcessParams& params) {
    if (state_ != ProcessState::Created) throw AlreadyInitialized("process '" + name_ + "' is already initialized");
    const auto t0 = std::chrono::steady_clock::now();
    // generic key: "launch_timing" = "every" | "sampled" | "off" (LaunchStats cost:
    // a timed CUDA event record is ~3 us of host time per launch on B200)
    // default "sampled": a timed launch costs two event records of host time,
    // which doubles the launch cost of a small process in a tight loop (C1, C4)
    const std::string lt = params.get_string("launch_timing", "sampled");
    if (lt != "every" && lt != "sampled" && lt != "off")
        throw InvalidParams("launch_timing must be \"every\", \"sampled\" or \"off\"");
    timing_mode_ = lt == "every" ? 0 : lt == "sampled" ? 1 : 2;
    on_init(params.without("launch_timing"));
    state_ = ProcessState::Initialized;
    rebound_ = false;
    stats_.init_calls += 1;
    stats_.init_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void Process::launch() {
    if (state_ != ProcessState::Initialized) throw NotInitialized("process '" + name_ + "' launched before init()");
    if (rebound_) {
        on_rebind();
        rebound_ = false;
    }
    if (!timing_) {
        timing_ = std::make_unique<Timing>();
        CudaBackend& cb = session_.cuda();
        timing_->device = cb.ordinal();
        timing_->stream = cb.compute_stream();
        cb.make_current();
        for (int i = 0; i < Timing::kRing; ++i) {
            ck(cudaEventCreate(&timing_->start[i]), "cudaEventCreate");
            ck(cudaEventCreate(&timing_->stop[i]), "cudaEventCreate");
        }
    }
    Timing& t = *timing_;
    t.mode = timing_mode_;
    if (t.mode == 2 || (t.mode == 1 && stats_.launches % Timing::kSample != 0)) {
        on_launch();
        stats_.launches += 1;
        if (t.mode == 1 && t.sampled) stats_.total_launch_seconds = t.sampled_seconds / double(t.sampled) * double(stats_.launches);
        t.last = -1;  // an untimed launch breaks the chain
        return;
    }
    if (t.pending == Timing::kRing) resolve_timings();
    const int slot = (t.head + t.pending) % Timing::kRing;
    cudaSetDevice(t.device);
    // chain to the previous launch only while it is still queued/running AND
    // nothing else was enqueued on the compute stream since (other processes,
    // kernels, copies): otherwise that work would be counted as this launch's
    CudaBackend& cb = session_.cuda();
    const bool chain = t.pending > 0 && t.last >= 0 && cb.work_seq() == t.seq_after &&
                       cudaEventQuery(t.stop[t.last]) == cudaErrorNotReady;
    if (!chain) {
        cudaGetLastError();  // a completed query is not an error
        cudaEventRecord(t.start[slot], t.stream);
    }
    t.chained[slot] = chain;
    on_launch();
    cudaEventRecord(t.stop[slot], t.stream);
    t.seq_after = cb.work_seq();
    t.last = slot;
    t.pending += 1;
    stats_.launches += 1;
}

void Process::resolve_timings() const {
    if (!timing_) return;
    Timing& t = *timing_;
    cudaSetDevice(t.device);
    while (t.pending > 0) {
        const int s = t.head;
        float ms = 0.f;
        const cudaError_t e = cudaEventSynchronize(t.stop[s]);
        if (e != cudaSuccess) {
            t.pending = 0;
            throw DeviceError(name_, cudaGetErrorString(e));
        }
        const cudaEvent_t from = t.chained[s] ? t.stop[(s + Timing::kRing - 1) % Timing::kRing] : t.start[s];
        cudaEventElapsedTime(&ms, from, t.stop[s]);
        stats_.last_launch_seconds = double(ms) * 1e-3;
        if (t.mode == 1) {
            t.sampled_seconds += stats_.last_launch_seconds;
            t.sampled += 1;
            stats_.total_launch_seconds = t.sampled_seconds / double(t.sampled) * double(stats_.launches);
        } else {
            stats_.total_launch_seconds += stats_.last_launch_seconds;
        }
        t.head = (t.head + 1) % Timing::kRing;
        t.pending -= 1;
    }
}

const LaunchStats& Process::stats() const {
    resolve_timings();
    return stats_;
}

// ---- GraphProcess -----------------------------------------------------------------------

GraphProcess::~GraphProcess() {
    if (exec_) cudaGraphExecDestroy(exec_);
    if (graph_) cudaGraphDestroy(graph_);
}

void GraphProcess::snapshot_layouts() {
    in_snap_ = input().valid() ? session().layout_of(input()) : LayoutDescriptor{};
    out_snap_ = output().valid() ? session().layout_of(output()) : LayoutDescriptor{};
}

void GraphProcess::on_init(const ProcessParams& params) {
    params_ = params;
    session().cuda().make_current();
    bake(params);
    capture();
    snapshot_layouts();
}

void GraphProcess::on_rebind() {
    session().cuda().make_current();
    const bool same = (!input().valid() || session().layout_of(input()) == in_snap_) &&
                      (!output().valid() || session().layout_of(output()) == out_snap_);
    if (same)
        repoint();
    else
        rebake();
    capture(same);
    snapshot_layouts();
}

namespace {

// Programmatic dependent launch inside process graphs: every kernel ->
// kernel edge of a captured graph becomes a programmatic edge (kernels/pdl.cuh:
// the upstream kernel triggers at entry, the downstream one waits before it
// touches data), so the launch of kernel i+1 and its prologue overlap the tail
// of kernel i.  Measured on B200 (profiles/round2_small_configs.md): C4 (the
// three-kernel normal operator) 12.76 -> 12.56 us, C2 unchanged, C3 263 ->
// 324 us (early-launched combine CTAs hold SM slots through the axis-1 tail).
// So it is on only where it wins (GraphProcess::programmatic_edges(): the
// SENSE model processes); HETRECO_PDL=1 / 0 forces it on / off everywhere.
int pdl_override() {
    static const int v = [] {
        const char* e = std::getenv("HETRECO_PDL");
        return (e && *e == '1') ? 1 : (e && *e == '0') ? 0 : -1;
    }();
    return v;
}

void make_kernel_edges_programmatic(cudaGraph_t g, bool wanted) {
    const int o = pdl_override();
    if (!(o == 1 || (o < 0 && wanted))) return;
    size_t n = 0;
    if (cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return;
    }
    std::vector<cudaGraphNode_t> from(n), to(n);
    std::vector<cudaGraphEdgeData> data(n);
    ck(cudaGraphGetEdges_v2(g, from.data(), to.data(), data.data(), &n), "cudaGraphGetEdges");
    for (size_t i = 0; i < n; ++i) {
        cudaGraphNodeType a{}, b{};
        ck(cudaGraphNodeGetType(from[i], &a), "cudaGraphNodeGetType");
        ck(cudaGraphNodeGetType(to[i], &b), "cudaGraphNodeGetType");
        if (a != cudaGraphNodeTypeKernel || b != cudaGraphNodeTypeKernel) continue;
        if (data[i].type == cudaGraphDependencyTypeProgrammatic) continue;
        ck(cudaGraphRemoveDependencies_v2(g, &from[i], &to[i], &data[i], 1), "cudaGraphRemoveDependencies");
        cudaGraphEdgeData e{};
        e.from_port = cudaGraphKernelNodePortProgrammatic;
        e.to_port = 0;
        e.type = cudaGraphDependencyTypeProgrammatic;
        ck(cudaGraphAddDependencies_v2(g, &from[i], &to[i], &e, 1), "cudaGraphAddDependencies(programmatic)");
    }
}

}  // namespace

void GraphProcess::capture(bool update) {
    CudaBackend& cb = session().cuda();
    cb.make_current();
    cudaStream_t cs = nullptr;
    ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "cudaStreamCreate");
    cudaGraph_t g = nullptr;
    ck(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    try {
        record(cs);
    } catch (...) {
        cudaStreamEndCapture(cs, &g);
        if (g) cudaGraphDestroy(g);
        cudaStreamDestroy(cs);
        cudaGetLastError();  // an invalidated capture must not poison later calls
        throw;
    }
    const cudaError_t e = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    ck(e, "capture of process '" + name() + "'");
    try {
        make_kernel_edges_programmatic(g, programmatic_edges());
    } catch (...) {
        cudaGraphDestroy(g);
        throw;
    }
    if (update && exec_) {
        // same topology, new pointers: patch the kernel node params in place
        cudaGraphExecUpdateResultInfo info{};
        if (cudaGraphExecUpdate(exec_, g, &info) == cudaSuccess) {
            if (graph_) cudaGraphDestroy(graph_);
            graph_ = g;
            return;
        }
        cudaGetLastError();  // topology changed: instantiate afresh below
    }
    cudaGraphExec_t x = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&x, g, 0);
    if (ei != cudaSuccess) {
        cudaGraphDestroy(g);
        ck(ei, "cudaGraphInstantiate('" + name() + "')");
    }
    if (exec_) cudaGraphExecDestroy(exec_);
    if (graph_) cudaGraphDestroy(graph_);
    graph_ = g;
    exec_ = x;
    cb.note_work();
    ck(cudaGraphUpload(exec_, cb.compute_stream()), "cudaGraphUpload");
}

void GraphProcess::mark(cudaStream_t s) {
    if (!profiling_) return;
    cudaEvent_t e = nullptr;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    cudaEventRecord(e, s);
    marks_.push_back(e);
}

std::vector<double> GraphProcess::profile(int reps) {
    if (state() != ProcessState::Initialized) throw NotInitialized("process '" + name() + "' profiled before init()");
    CudaBackend& cb = session().cuda();
    cb.make_current();
    cudaStream_t s = cb.compute_stream();
    cb.note_work();
    std::vector<double> acc;
    profiling_ = true;
    try {
        for (int r = 0; r < reps; ++r) {
            marks_.clear();
            mark(s);
            record(s);
            ck(cudaStreamSynchronize(s), "profile(" + name() + ")");
            if (acc.empty()) acc.assign(marks_.size() > 1 ? marks_.size() - 1 : 0, 0.0);
            for (std::size_t i = 1; i < marks_.size() && i - 1 < acc.size(); ++i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, marks_[i - 1], marks_[i]);
                acc[i - 1] += double(ms) * 1e-3;
            }
            for (cudaEvent_t e : marks_) cudaEventDestroy(e);
            marks_.clear();
        }
    } catch (...) {
        profiling_ = false;
        for (cudaEvent_t e : marks_) cudaEventDestroy(e);
        marks_.clear();
        throw;
    }
    profiling_ = false;
    for (double& a : acc) a /= std::max(1, reps);
    return acc;
}

void GraphProcess::on_launch() {
    CudaBackend& cb = session().cuda();
    cb.note_work();
    const cudaError_t e = cudaGraphLaunch(exec_, cb.compute_stream());
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw DeviceError(name(), cudaGetErrorString(e));
    }
}

// ---- CompositeProcess -------------------------------------------------------------------------

// The stages are validated in the caller's vector and only taken over once
// nothing can fail any more: a throwing constructor leaves them with the caller.
CompositeProcess::CompositeProcess(ComputeSession& s, std::string name, std::vector<std::unique_ptr<Process>>&& stages)
    : GraphProcess(s, std::move(name)) {
    if (stages.empty()) throw InvalidArgument("chain '" + this->name() + "' has no stages");
    for (std::size_t i = 0; i < stages.size(); ++i) {
        if (!stages[i]) throw InvalidArgument("chain stage " + std::to_string(i) + " is null");
        if (&stages[i]->session() != &s)
            throw ChainMismatch("stage " + std::to_string(i) + " belongs to another session");
        for (std::size_t k = 0; k < i; ++k)
            if (stages[k].get() == stages[i].get())
                throw InvalidArgument("chain stage " + std::to_string(i) + " repeats stage " + std::to_string(k));
        if (!dynamic_cast<GraphProcess*>(stages[i].get())) all_graph_ = false;
    }
    for (std::size_t i = 0; i + 1 < stages.size(); ++i) {
        if (!(stages[i]->output() == stages[i + 1]->input()) || !stages[i]->output().valid())
            throw ChainMismatch("stage " + std::to_string(i) + " ('" + stages[i]->name() +
                                "') output is not the input of stage " + std::to_string(i + 1) + " ('" +
                                stages[i + 1]->name() + "')");
    }
    if (stages.front()->input().valid()) set_input(stages.front()->input());
    if (stages.back()->output().valid()) set_output(stages.back()->output());
    stages_ = std::move(stages);
}

void CompositeProcess::bake(const ProcessParams& params) {
    params.require_known({});
    for (std::size_t i = 0; i < stages_.size(); ++i) {
        try {
            if (stages_[i]->state() == ProcessState::Created) stages_[i]->init();
        } catch (const std::exception& e) {
            throw ChainStageError(i, stages_[i]->name(), e.what());
        }
    }
}

void CompositeProcess::record(cudaStream_t s) {
    for (std::size_t i = 0; i < stages_.size(); ++i) {
        auto* g = dynamic_cast<GraphProcess*>(stages_[i].get());
        if (!g) continue;  // non-graph stages launch one by one (on_launch)
        try {
            g->record(s);
        } catch (const std::exception& e) {
            throw ChainStageError(i, stages_[i]->name(), e.what());
        }
    }
}

void CompositeProcess::on_launch() {
    if (all_graph_) {
        GraphProcess::on_launch();
        return;
    }
    for (std::size_t i = 0; i < stages_.size(); ++i) {
        try {
            stages_[i]->launch();
        } catch (const std::exception& e) {
            throw ChainStageError(i, stages_[i]->name(), e.what());
        }
    }
}

std::unique_ptr<CompositeProcess> chain(ComputeSession& s, std::string name, std::vector<std::unique_ptr<Process>>&& stages) {
    return std::make_unique<CompositeProcess>(s, std::move(name), std::move(stages));
}

// ---- builtin processes ------------------------------------------------------------------------

namespace {

class NegateProcess final : public GraphProcess {
public:
    using GraphProcess::GraphProcess;
    void bake(const ProcessParams& p) override {
        p.require_known({"max_value"});
        const LayoutRecord& ri = array_of(input_layout(), 0, name());
        const LayoutRecord& ro = array_of(output_layout(), 0, name());
        if (ri.element_type != ElementType::UInt8 && ri.element_type != ElementType::Float32)
            throw UnsupportedElementType(name() + ": negate supports uint8 and float32, got " +
                                         std::string(element_type_name(ri.element_type)));
        if (ri.element_type != ro.element_type || ri.dims != ro.dims)
            throw ShapeMismatch(name() + ": output " + dims_str(ro) + " does not match input " + dims_str(ri));
        type_ = int(ri.element_type);
        n_ = ri.element_count();
        mv_ = p.get_real("max_value", ri.element_type == ElementType::UInt8 ? 255.0 : 1.0);
        in_ = session().device_array(require_input(), 0);
        out_ = session().device_array(require_output(), 0);
    }
    void repoint() override {
        in_ = session().device_array(require_input(), 0);
        out_ = session().device_array(require_output(), 0);
    }
    void record(cudaStream_t s) override {
        ck(dev::launch_negate(type_, in_, out_, n_, mv_, s), name());
        mark(s);
    }

private:
    int type_ = 0;
    std::uint64_t n_ = 0;
    double mv_ = 0;
    const void* in_ = nullptr;
    void* out_ = nullptr;
};

// Shared plan for the two-pass FFT (axis 1 strided, then axis 0 contiguous).
struct FftPlan {
    std::uint64_t nx = 0, ny = 0;
    int dir = 1;
    bool shift = false;
    DevMem tw_x, tw_y;
    dev::LaunchShape s1, s2;
    void make(std::uint64_t nx_, std::uint64_t ny_, int dir_, std::uint64_t planes, dev::Combine mode,
              std::uint64_t items, int ordinal) {
        nx = nx_;
        ny = ny_;
        dir = dir_;
        tw_y = twiddle_table(ny, dir);
        tw_x = twiddle_table(nx, dir);
        const int sms = sm_count(ordinal);
        s1 = dev::plan_strided(ny, nx, planes, sms);
        s2 = dev::plan_contig(nx, mode, items, sms);
    }
};

class Fft2dProcess final : public GraphProcess {
public:
    using GraphProcess::GraphProcess;
    void bake(const ProcessParams& p) override {
        p.require_known({"direction", "shift", "algorithm"});
        const std::string d = p.get_string("direction", "forward");
        if (d != "forward" && d != "inverse")
            throw InvalidParams(name() + ": direction must be \"forward\" or \"inverse\", got \"" + d + "\"");
        const std::string algo = p.get_string("algorithm", "stockham");
        if (algo != "stockham" && algo != "radix2")
            throw InvalidParams(name() + ": algorithm must be \"stockham\" or \"radix2\"");
        inverse_ = d == "inverse";
        shift_ = p.get_bool("shift", false);
        const LayoutRecord& ri = array_of(input_layout(), 0, name());
        const LayoutRecord& ro = array_of(output_layout(), 0, name());
        require_type(ri, ElementType::Complex64, name());
        if (ro.element_type != ri.element_type || ro.dims != ri.dims)
            throw ShapeMismatch(name() + ": output " + dims_str(ro) + " does not match input " + dims_str(ri));
        if (require_input() == require_output())
            throw InvalidArgument(name() + ": fft2d does not run in place (use distinct input/output data)");
        nx_ = ri.dims[0];
        ny_ = ri.rank > 1 ? ri.dims[1] : 1;
        batch_ = prod(ri, 2, ri.rank);
        const bool p2 = is_pow2(nx_) && is_pow2(ny_);
        const bool stockham_ok = dev::fft_size_supported(nx_) && dev::fft_size_supported(ny_);
        if (!p2 && !stockham_ok)
            throw ShapeMismatch(name() + ": spatial dims must be powers of two or mixed-radix sides (96, 160, 192, "
                                         "320, 384), got " + dims_str(ri));
        radix2_ = algo == "radix2" || !stockham_ok;
        if (radix2_ && !p2)
            throw ShapeMismatch(name() + ": the radix2 algorithm needs power-of-two dims, got " + dims_str(ri));
        if (radix2_ && shift_) throw InvalidParams(name() + ": shift requires the stockham algorithm");
        in_ = static_cast<const float2*>(session().device_array(require_input(), 0));
        out_ = static_cast<float2*>(session().device_array(require_output(), 0));
        if (radix2_)
            bake_radix2();
        else
            plan_.make(nx_, ny_, inverse_ ? 1 : -1, batch_, dev::Combine::None, ny_ * batch_,
                       session().cuda().ordinal());
    }
    void repoint() override {
        in_ = static_cast<const float2*>(session().device_array(require_input(), 0));
        out_ = static_cast<float2*>(session().device_array(require_output(), 0));
    }
    void record(cudaStream_t s) override {
        if (radix2_) {
            record_radix2(s);
            return;
        }
        const float scale = inverse_ ? float(1.0 / (double(nx_) * double(ny_))) : 1.0f;
        dev::StridedArgs a1{in_, out_, nx_, batch_, shift_, shift_, 1.0f, plan_.tw_y.as<float2>()};
        ck(dev::launch_strided(ny_, plan_.dir, a1, plan_.s1, s), name() + "/axis1");
        mark(s);
        dev::ContigArgs a2{out_, out_, nullptr, ny_, 0, batch_, shift_, shift_, scale, plan_.tw_x.as<float2>()};
        ck(dev::launch_contig(nx_, plan_.dir, dev::Combine::None, a2, plan_.s2, s), name() + "/axis0");
        mark(s);
    }

private:
    // The reference's own pass sequence on the GPU:
    // bit-exact with the CPU reference, used for sizes beyond the fused
    // kernels and on request ("algorithm": "radix2").
    void bake_radix2() {
        passes_.clear();
        const std::uint64_t n = nx_ * ny_ * batch_;
        const float fs = inverse_ ? float(1.0 / (double(nx_) * double(ny_))) : 1.0f;
        auto bits = [](std::uint64_t v) { unsigned b = 0; while ((std::uint64_t(1) << b) < v) ++b; return b; };
        const unsigned bx = bits(nx_), by = bits(ny_);
        std::vector<std::vector<std::byte>> blocks;
        for (int axis = 0; axis < 2; ++axis) {
            const std::uint64_t L = axis == 0 ? nx_ : ny_, S = axis == 0 ? 1 : nx_;
            const unsigned nb = bits(L);
            auto header = [&](std::uint32_t mode, std::uint64_t m, float scale, std::size_t payload) {
                std::vector<std::byte> b(40 + payload);
                std::memcpy(b.data(), &mode, 4);
                std::memcpy(b.data() + 8, &L, 8);
                std::memcpy(b.data() + 16, &S, 8);
                std::memcpy(b.data() + 24, &m, 8);
                std::memcpy(b.data() + 32, &scale, 4);
                return b;
            };
            std::vector<std::byte> rb = header(axis == 0 ? 0u : 1u, 0, 1.0f, 4 * L);
            for (std::uint64_t k = 0; k < L; ++k) {
                std::uint32_t r = 0;
                for (unsigned b = 0; b < nb; ++b)
                    if (k & (std::uint64_t(1) << b)) r |= 1u << (nb - 1 - b);
                std::memcpy(rb.data() + 40 + 4 * k, &r, 4);
            }
            passes_.push_back({blocks.size(), n, axis == 0});
            blocks.push_back(std::move(rb));
            for (unsigned pp = 0; pp < nb; ++pp) {
                const bool last = axis == 0 ? (by == 0 && pp + 1 == bx) : (pp + 1 == by);
                std::vector<std::byte> tb = header(2u, std::uint64_t(1) << pp, last ? fs : 1.0f, 4 * L);
                for (std::uint64_t t = 0; t < L / 2; ++t) {
                    const double th = (inverse_ ? 1.0 : -1.0) * 2.0 * M_PI * double(t) / double(L);
                    const float c = float(std::cos(th)), sn = float(std::sin(th));
                    std::memcpy(tb.data() + 40 + 8 * t, &c, 4);
                    std::memcpy(tb.data() + 44 + 8 * t, &sn, 4);
                }
                passes_.push_back({blocks.size(), n / 2, false});
                blocks.push_back(std::move(tb));
            }
        }
        std::uint64_t total = 0;
        offsets_.clear();
        for (auto& b : blocks) {
            offsets_.push_back(total);
            total += (b.size() + 255) & ~std::uint64_t(255);
        }
        std::vector<std::byte> all(total);
        for (std::size_t i = 0; i < blocks.size(); ++i) std::memcpy(all.data() + offsets_[i], blocks[i].data(), blocks[i].size());
        pblock_ = upload_bytes(all.data(), all.size());
        // array pointers passed to the kernel already include the offsets
        const std::uint64_t h[12] = {1, 0, 4, 1, 1, 1, 1, 1, 1, 1, 1, 1};
        hdr0_ = upload_bytes(h, sizeof h);
    }
    void record_radix2(cudaStream_t s) {
        hetreco_kernel_args a{};
        a.in = session().device_array(require_input(), 0);
        a.out = session().device_array(require_output(), 0);
        // array 0 pointers already include offsets: use a zero-offset header
        a.in_layout = hdr0_.as<std::uint64_t>();
        a.out_layout = hdr0_.as<std::uint64_t>();
        for (const Pass& p : passes_) {
            hetreco_kernel_args b = a;
            if (!p.gather) b.in = b.out;
            b.params = pblock_.as<char>() + offsets_[p.block];
            ck(dev::launch_builtin(dev::Builtin::FftRadix2Pass, b, p.gsize, s), name() + "/radix2");
            mark(s);
        }
    }

    struct Pass {
        std::size_t block;
        std::uint64_t gsize;
        bool gather;
    };
    bool inverse_ = false, shift_ = false, radix2_ = false;
    std::uint64_t nx_ = 0, ny_ = 0, batch_ = 0;
    const float2* in_ = nullptr;
    float2* out_ = nullptr;
    FftPlan plan_;
    std::vector<Pass> passes_;
    std::vector<std::uint64_t> offsets_;
    DevMem pblock_, hdr0_;
};

// Wraps one reference-ABI builtin kernel with baked device params.
class BuiltinProcess final : public GraphProcess {
public:
    BuiltinProcess(ComputeSession& s, std::string name, dev::Builtin which)
        : GraphProcess(s, std::move(name)), which_(which) {}
    void bake(const ProcessParams& p) override {
        const LayoutDescriptor& li = input_layout();
        const LayoutDescriptor& lo = output_layout();
        const LayoutRecord& x = array_of(li, 0, name());
        const LayoutRecord& o = array_of(lo, 0, name());
        std::uint32_t param_word = 0;
        if (which_ == dev::Builtin::ComplexElementProd) {
            p.require_known({"conjugate_s"});
            const LayoutRecord& sm = array_of(li, 1, name());
            require_type(x, ElementType::Complex64, name());
            require_type(sm, ElementType::Complex64, name());
            if (o.element_type != x.element_type || o.dims != x.dims)
                throw ShapeMismatch(name() + ": output " + dims_str(o) + " does not match x " + dims_str(x));
            if (x.element_count() % sm.element_count() != 0)
                throw ShapeMismatch(name() + ": s " + dims_str(sm) + " does not tile x " + dims_str(x));
            param_word = p.get_bool("conjugate_s", true) ? 1u : 0u;
            gsize_ = x.element_count();
        } else if (which_ == dev::Builtin::MatrixAdd) {
            // matrix_add(a, b) -> a + b (matrix_add.cl.src:5-24)
            p.require_known({});
            const LayoutRecord& b = array_of(li, 1, name());
            if (x.element_type != ElementType::Float32 && x.element_type != ElementType::Float64 &&
                x.element_type != ElementType::Int32)
                throw UnsupportedElementType(name() + ": matrix_add takes FLOAT32, FLOAT64 or INT32 arrays");
            require_type(b, x.element_type, name());
            require_type(o, x.element_type, name());
            if (b.dims != x.dims || o.dims != x.dims)
                throw ShapeMismatch(name() + ": a " + dims_str(x) + ", b " + dims_str(b) + " and output " +
                                    dims_str(o) + " must have equal shapes");
            gsize_ = x.element_count();
        } else {
            p.require_known({});
            require_type(x, ElementType::Complex64, name());
            if (x.rank < 3) throw ShapeMismatch(name() + ": input must be [nx, ny, coils, ...], got " + dims_str(x));
            const ElementType ot = which_ == dev::Builtin::RssCombine ? ElementType::Float32 : ElementType::Complex64;
            require_type(o, ot, name());
            std::vector<std::uint64_t> want{x.dims[0], x.dims[1]};
            for (std::uint32_t d = 3; d < x.rank; ++d) want.push_back(x.dims[d]);
            std::uint64_t frames = prod(x, 3, x.rank);
            const bool ok = o.dims[0] == x.dims[0] && o.dims[1] == x.dims[1] &&
                            o.element_count() == x.dims[0] * x.dims[1] * frames;
            if (!ok) throw ShapeMismatch(name() + ": output " + dims_str(o) + " does not match the coil-reduced input");
            gsize_ = x.dims[0] * x.dims[1] * frames;
        }
        params_ = upload_bytes(&param_word, sizeof param_word);
    }
    void repoint() override {}  // record() reads the pointers and headers itself
    void record(cudaStream_t s) override {
        hetreco_kernel_args a{};
        a.in = session().device_array(require_input(), 0);
        a.out = session().device_array(require_output(), 0);
        // device_array includes array 0's offset; the headers carry offsets
        // relative to the buffer base, so pass the base pointers instead.
        a.in = static_cast<const char*>(a.in) - input_layout().records[0].offset_bytes;
        a.out = static_cast<char*>(a.out) - output_layout().records[0].offset_bytes;
        a.in_layout = session().device_header(require_input());
        a.out_layout = session().device_header(require_output());
        a.params = params_.get();
        a.params_size = 4;
        ck(dev::launch_builtin(which_, a, gsize_, s), name());
        mark(s);
    }

private:
    dev::Builtin which_;
    std::uint64_t gsize_ = 0;
    DevMem params_;
};

// Fused reconstruction: SENSE (Eq. 1) or RSS.
class ReconProcess final : public GraphProcess {
public:
    ReconProcess(ComputeSession& s, std::string name, dev::Combine mode)
        : GraphProcess(s, std::move(name)), mode_(mode) {}
    void bake(const ProcessParams& p) override {
        p.require_known({"shift", "chunk_frames", "accumulate", "prefetch", "algorithm", "max_clusters", "cluster_size",
                         "overlap"});
        shift_ = p.get_bool("shift", false);
        const std::string acc = p.get_string("accumulate", "fp32");
        if (acc != "fp32" && acc != "fp64")
            throw InvalidParams(name() + ": accumulate must be \"fp32\" or \"fp64\"");
        std::string algo = p.get_string("algorithm", "auto");
        if (algo != "auto" && algo != "cluster" && algo != "two_pass")
            throw InvalidParams(name() + ": algorithm must be \"auto\", \"cluster\" or \"two_pass\"");
        if (const char* v = std::getenv("HETRECO_RECON_ALGO"); v && *v && algo == "auto") algo = v;
        variant_ = (acc == "fp32" ? 1 : 0) | (p.get_bool("prefetch", true) ? 2 : 0);
        if (const char* v = std::getenv("HETRECO_COMBINE_VARIANT")) variant_ = std::atoi(v);
        const LayoutDescriptor& li = input_layout();
        const LayoutRecord& y = array_of(li, 0, name());
        require_type(y, ElementType::Complex64, name());
        if (y.rank < 3) throw ShapeMismatch(name() + ": k-space must be [nx, ny, coils(, frames)], got " + dims_str(y));
        nx_ = y.dims[0];
        ny_ = y.dims[1];
        nc_ = y.dims[2];
        nf_ = prod(y, 3, y.rank);
        if (!dev::fft_size_supported(nx_) || !dev::fft_size_supported(ny_))
            throw ShapeMismatch(name() + ": spatial dims must be powers of two <= 4096 or mixed-radix sides (96, 160, 192, 320, 384), got " + dims_str(y));
        const LayoutRecord& o = array_of(output_layout(), 0, name());
        require_type(o, mode_ == dev::Combine::Sense ? ElementType::Complex64 : ElementType::Float32, name());
        if (o.dims[0] != nx_ || (o.rank > 1 ? o.dims[1] : 1) != ny_ || o.element_count() != nx_ * ny_ * nf_)
            throw ShapeMismatch(name() + ": output " + dims_str(o) + " must be [nx, ny, frames] for k-space " + dims_str(y));
        smap_ = nullptr;
        if (mode_ == dev::Combine::Sense) {
            const LayoutRecord& sm = array_of(li, 1, name());
            require_type(sm, ElementType::Complex64, name());
            if (sm.dims[0] != nx_ || sm.dims[1] != ny_ || sm.element_count() != nx_ * ny_ * nc_)
                throw ShapeMismatch(name() + ": sensitivity maps " + dims_str(sm) + " must be [nx, ny, coils]");
            smap_ = static_cast<const float2*>(session().device_array(require_input(), 1));
        }
        y_ = static_cast<const float2*>(session().device_array(require_input(), 0));
        out_ = session().device_array(require_output(), 0);
        const int ord = session().cuda().ordinal();
        // Single-pass cluster kernel (fft_cluster.cu), 256x256 with fp32
        // accumulation, on request.  "auto" keeps the two-pass chain: measured
        // faster on B200 (profiles/round1_cluster.md -- the cluster kernel
        // reaches only 120 of 148 SMs and is bound by per-SM shared-memory
        // traffic, not HBM).
        cluster_ = false;
        if (algo == "cluster") {
            const bool ok = dev::cluster_supported(nx_, ny_, mode_) && acc == "fp32";
            if (!ok && algo == "cluster")
                throw InvalidParams(name() + ": algorithm \"cluster\" needs 256x256 images and fp32 accumulation, got " +
                                    dims_str(y) + " / " + acc);
            if (ok) {
                const std::int64_t mc = p.get_int("max_clusters", 0);
                if (mc < 0) throw InvalidParams(name() + ": max_clusters must be >= 0");
                const std::int64_t cs = p.get_int("cluster_size", 0);
                if (cs != 0 && cs != 8 && cs != 16) throw InvalidParams(name() + ": cluster_size must be 8 or 16");
                cplan_ = dev::plan_cluster(mode_, nc_, nf_, int(mc), int(cs));
                if (cplan_.clusters <= 0) {
                    if (algo == "cluster") throw DeviceError(name(), "cluster kernel does not fit on this device");
                } else {
                    cluster_ = true;
                    if (cws_.size() != cplan_.ws_bytes) cws_ = DevMem(cplan_.ws_bytes);
                    ccnt_ = DevMem(cplan_.cnt_bytes);
                    ck(cudaMemset(ccnt_.get(), 0, cplan_.cnt_bytes), "cudaMemset(cluster counters)");
                    ck(cudaDeviceSynchronize(), "cluster counters");
                    ctw_ = twiddle_table(nx_, +1);
                    ck(dev::make_cluster_map(cmap_, y_, ny_ * nc_ * nf_, cplan_.cl), name() + ": TMA descriptor");
                    scratch_ = DevMem();
                    return;
                }
            }
        }
        // Frames may be processed in chunks to bound the axis-1 intermediate
        // (scratch = chunk_frames * nx*ny*coils*8 bytes).  Default: one chunk
        // of all frames -- measured fastest on B200, because the combine pass
        // parallelises over (y, frame) lines and small chunks starve the SMs.
        const std::uint64_t frame_bytes = nx_ * ny_ * nc_ * 8;
        std::int64_t chunk = p.get_int("chunk_frames", 0);
        if (const char* v = std::getenv("HETRECO_CHUNK")) chunk = std::atoll(v);
        if (chunk < 0) throw InvalidParams(name() + ": chunk_frames must be >= 0");
        if (chunk == 0) chunk = std::int64_t(nf_);
        chunk_ = std::min<std::uint64_t>(std::uint64_t(chunk), nf_);
        const std::uint64_t scratch_bytes = frame_bytes * chunk_;
        if (scratch_.size() != scratch_bytes) scratch_ = DevMem(scratch_bytes);
        plan_.make(nx_, ny_, +1, nc_ * chunk_, mode_, ny_ * chunk_, ord);
        // prefetch form measured per size on B200: register copy at 256,
        // ping-pong (two-way unrolled) at 512 (profiles/round1_summary.md)
        if ((variant_ & 2) && !std::getenv("HETRECO_COMBINE_VARIANT") && nx_ != 512) variant_ |= 8;
        // HETRECO_COMBINE_TMA=1: the TMA bulk-copy ring combine
        // (fft_combine_tma.cu), fp32 only.  Measured slower than the register
        // prefetch on B200 (profiles/round1_combine.md), so opt-in.
        const char* tma_env = std::getenv("HETRECO_COMBINE_TMA");
        tma_ = (variant_ & 1) && dev::combine_tma_supported(nx_) && tma_env && *tma_env == '1';
        if (tma_) {
            plan_.s2 = dev::plan_combine_tma(nx_, mode_, ny_, chunk_, sm_count(ord));
            const std::uint64_t tail_f = nf_ % chunk_;
            if (tail_f) tail_tma_ = dev::plan_combine_tma(nx_, mode_, ny_, tail_f, sm_count(ord));
        }
        // small problems (few frames): coil-parallel combine, fp32 only
        auto plan2 = [&](std::uint64_t frames) {
            if ((variant_ & 1) && !std::getenv("HETRECO_COMBINE_VARIANT")) {
                if (dev::combine_cp_preferred(nx_, ny_ * frames, nc_, sm_count(ord)))
                    return dev::plan_combine_cp(nx_, mode_, ny_ * frames, sm_count(ord));
                if (mode_ == dev::Combine::Sense && combine_ss_enabled(nx_))
                    return dev::plan_combine_ss(nx_, ny_, frames, sm_count(ord));
            }
            return dev::plan_contig(nx_, mode_, ny_ * frames, sm_count(ord), variant_);
        };
        if (!tma_) plan_.s2 = plan2(chunk_);
        const std::uint64_t tail = nf_ % chunk_;
        if (tail) {
            tail_s1_ = dev::plan_strided(ny_, nx_, nc_ * tail, sm_count(ord));
            tail_s2_ = plan2(tail);
        }
        // "overlap": true -- pipeline over 8-frame chunks (one full-size
        // intermediate): the axis-1 pass of chunk k+1 runs as a graph branch
        // concurrent with the combine of chunk k (HBM-bound next to
        // issue-bound).  Measured slower on B200 (C3: 337 vs 298 us; both
        // kernels size their grids to fill every SM, so the branches contend
        // instead of overlapping), hence off by default.
        overlap_ = false;
        std::int64_t oc = std::int64_t(env_or("HETRECO_OVERLAP_CHUNK", 8));
        if (p.get_bool("overlap", false) && chunk_ == nf_ && !tma_ && oc > 0 && nf_ >= 2 * std::uint64_t(oc)) {
            overlap_ = true;
            ovl_chunk_ = std::uint64_t(oc);
            const std::uint64_t ot = nf_ % ovl_chunk_;
            ovl_s1_ = dev::plan_strided(ny_, nx_, nc_ * ovl_chunk_, sm_count(ord));
            ovl_s2_ = plan2(ovl_chunk_);
            if (ot) {
                ovl_tail_s1_ = dev::plan_strided(ny_, nx_, nc_ * ot, sm_count(ord));
                ovl_tail_s2_ = plan2(ot);
            }
            const std::size_t nchunks = std::size_t((nf_ + ovl_chunk_ - 1) / ovl_chunk_);
            if (!side_) ck(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking), "cudaStreamCreate(overlap)");
            while (ovl_events_.size() < nchunks + 2) {
                cudaEvent_t e = nullptr;
                ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate(overlap)");
                ovl_events_.push_back(e);
            }
        }
    }
    void repoint() override {
        y_ = static_cast<const float2*>(session().device_array(require_input(), 0));
        if (mode_ == dev::Combine::Sense) smap_ = static_cast<const float2*>(session().device_array(require_input(), 1));
        out_ = session().device_array(require_output(), 0);
        if (cluster_)
            ck(dev::make_cluster_map(cmap_, y_, ny_ * nc_ * nf_, cplan_.cl), name() + ": TMA descriptor");
    }
    void record(cudaStream_t s) override {
        const float scale = float(1.0 / (double(nx_) * double(ny_)));
        if (cluster_) {
            dev::ClusterLaunch a{smap_, out_, cws_.as<float2>(), ccnt_.as<unsigned>(), ctw_.as<float2>(), nc_, nf_,
                                 shift_, scale};
            ck(dev::launch_cluster(mode_, cmap_, a, cplan_, s), name() + "/cluster ifft2+combine");
            mark(s);
            return;
        }
        const std::uint64_t plane = nx_ * ny_;
        const std::uint64_t out_elem = mode_ == dev::Combine::Sense ? 8 : 4;
        if (overlap_ && !profiling()) {
            // fork: the side stream joins the capture, runs the combines
            cudaEvent_t* ev = ovl_events_.data();
            ck(cudaEventRecord(ev[0], s), "overlap fork");
            ck(cudaStreamWaitEvent(side_, ev[0], 0), "overlap fork");
            std::size_t k = 0;
            for (std::uint64_t f0 = 0; f0 < nf_; f0 += ovl_chunk_, ++k) {
                const std::uint64_t fc = std::min(ovl_chunk_, nf_ - f0);
                const bool full = fc == ovl_chunk_;
                float2* x = scratch_.as<float2>() + f0 * plane * nc_;
                dev::StridedArgs a1{y_ + f0 * plane * nc_, x, nx_, nc_ * fc, shift_, shift_, 1.0f,
                                    plan_.tw_y.as<float2>()};
                ck(dev::launch_strided(ny_, +1, a1, full ? ovl_s1_ : ovl_tail_s1_, s), name() + "/axis1");
                ck(cudaEventRecord(ev[k + 1], s), "overlap edge");
                ck(cudaStreamWaitEvent(side_, ev[k + 1], 0), "overlap edge");
                dev::ContigArgs a2{x, static_cast<char*>(out_) + f0 * plane * out_elem, smap_, ny_, nc_, fc, shift_,
                                   shift_, scale, plan_.tw_x.as<float2>()};
                ck(dev::launch_contig(nx_, +1, mode_, a2, full ? ovl_s2_ : ovl_tail_s2_, side_),
                   name() + "/axis0+combine");
            }
            // join
            ck(cudaEventRecord(ev[k + 1], side_), "overlap join");
            ck(cudaStreamWaitEvent(s, ev[k + 1], 0), "overlap join");
            mark(s);
            return;
        }
        for (std::uint64_t f0 = 0; f0 < nf_; f0 += chunk_) {
            const std::uint64_t fc = std::min(chunk_, nf_ - f0);
            const bool full = fc == chunk_;
            dev::StridedArgs a1{y_ + f0 * plane * nc_, scratch_.as<float2>(), nx_, nc_ * fc, shift_, shift_, 1.0f,
                                plan_.tw_y.as<float2>()};
            ck(dev::launch_strided(ny_, +1, a1, full ? plan_.s1 : tail_s1_, s), name() + "/axis1");
            mark(s);
            dev::ContigArgs a2{scratch_.as<float2>(), static_cast<char*>(out_) + f0 * plane * out_elem, smap_, ny_,
                               nc_, fc, shift_, shift_, scale, plan_.tw_x.as<float2>()};
            if (tma_)
                ck(dev::launch_combine_tma(nx_, mode_, a2, full ? plan_.s2 : tail_tma_, s), name() + "/axis0+combine");
            else
                ck(dev::launch_contig(nx_, +1, mode_, a2, full ? plan_.s2 : tail_s2_, s), name() + "/axis0+combine");
            mark(s);
        }
    }

private:
    dev::Combine mode_;
    bool shift_ = false;
    int variant_ = 1;
    std::uint64_t nx_ = 0, ny_ = 0, nc_ = 0, nf_ = 0, chunk_ = 1;
    const float2* y_ = nullptr;
    const float2* smap_ = nullptr;
    void* out_ = nullptr;
    DevMem scratch_;
    FftPlan plan_;
    dev::LaunchShape tail_s1_, tail_s2_;
    bool tma_ = false;
    dev::LaunchShape tail_tma_;
    bool overlap_ = false;
    std::uint64_t ovl_chunk_ = 8;
    dev::LaunchShape ovl_s1_, ovl_s2_, ovl_tail_s1_, ovl_tail_s2_;
    cudaStream_t side_ = nullptr;
    std::vector<cudaEvent_t> ovl_events_;

public:
    ~ReconProcess() override {
        if (side_) {
            cudaStreamSynchronize(side_);
            cudaStreamDestroy(side_);
        }
        for (cudaEvent_t e : ovl_events_) cudaEventDestroy(e);
    }

private:
    bool cluster_ = false;
    dev::ClusterPlan cplan_;
    dev::ClusterMap cmap_{};
    DevMem cws_, ccnt_, ctw_;
};

// SENSE forward model E m = P F (S m) ("sense_forward") and the normal
// operator E^H E m ("sense_normal", the iterative-reconstruction kernel of
// expand + forward x-FFT, y-FFT / mask / inverse y-FFT in
// registers, inverse x-FFT + conj(S) coil combine).  Input Data:
// [M [nx,ny,F], S [nx,ny,C] (, mask FLOAT32 [nx,ny])].
class SenseModelProcess final : public GraphProcess {
public:
    SenseModelProcess(ComputeSession& s, std::string name, bool normal)
        : GraphProcess(s, std::move(name)), normal_(normal) {}
    void bake(const ProcessParams& p) override {
        p.require_known({"shift"});
        shift_ = p.get_bool("shift", false);
        const LayoutDescriptor& li = input_layout();
        const LayoutRecord& m = array_of(li, 0, name());
        const LayoutRecord& sm = array_of(li, 1, name());
        require_type(m, ElementType::Complex64, name());
        require_type(sm, ElementType::Complex64, name());
        nx_ = m.dims[0];
        ny_ = m.rank > 1 ? m.dims[1] : 1;
        nf_ = prod(m, 2, m.rank);
        if (!dev::fft_size_supported(nx_) || !dev::fft_size_supported(ny_))
            throw ShapeMismatch(name() + ": image sides must be powers of two <= 4096 or mixed-radix sides (96, 160, 192, 320, 384), got " + dims_str(m));
        // the masked / round-trip column kernels are square-only; the plain
        // forward model of a rectangular image uses the generic column pass
        const bool masked = li.records.size() > 2;
        generic_cols_ = nx_ != ny_;
        if (generic_cols_ && (normal_ || masked))
            throw ShapeMismatch(name() + ": masked and normal-operator models need square images, got " + dims_str(m));
        if (sm.dims[0] != nx_ || sm.dims[1] != ny_)
            throw ShapeMismatch(name() + ": sensitivity maps " + dims_str(sm) + " do not match image " + dims_str(m));
        nc_ = prod(sm, 2, sm.rank);
        mask_ = nullptr;
        if (li.records.size() > 2) {
            const LayoutRecord& mk = li.records[2];
            require_type(mk, ElementType::Float32, name());
            if (mk.element_count() != nx_ * ny_)
                throw ShapeMismatch(name() + ": mask " + dims_str(mk) + " must be [nx, ny]");
            mask_ = static_cast<const float*>(session().device_array(require_input(), 2));
        }
        const LayoutRecord& o = array_of(output_layout(), 0, name());
        require_type(o, ElementType::Complex64, name());
        const std::uint64_t want = normal_ ? nx_ * ny_ * nf_ : nx_ * ny_ * nc_ * nf_;
        if (o.dims[0] != nx_ || o.element_count() != want)
            throw ShapeMismatch(name() + ": output " + dims_str(o) + (normal_ ? " must be [nx, ny, frames]"
                                                                             : " must be [nx, ny, coils, frames]"));
        m_ = static_cast<const float2*>(session().device_array(require_input(), 0));
        s_ = static_cast<const float2*>(session().device_array(require_input(), 1));
        out_ = static_cast<float2*>(session().device_array(require_output(), 0));
        const int ord = session().cuda().ordinal(), sms = sm_count(ord);
        tw_fwd_ = twiddle_table(nx_, -1);
        s_exp_ = dev::plan_expand(nx_, ny_ * nc_ * nf_, sms);
        if (generic_cols_) {
            tw_fwd_y_ = twiddle_table(ny_, -1);
            s_col_ = dev::plan_strided(ny_, nx_, nc_ * nf_, sms);
        } else {
            s_col_ = dev::plan_strided_masked(ny_, normal_, nc_ * nf_, sms);
        }
        fused_ = dev::LaunchShape{};
        front_clusters_ = 0;
        if (normal_) {
            tw_inv_ = twiddle_table(nx_, +1);
            fused_ = dev::plan_sense_normal_fused(nx_, nc_ * nf_, sms);
            // expand + x-FFT + y-FFT/mask/y-IFFT as one 16-CTA-cluster kernel at
            // 256^2 (fft_sense_cluster.cu; opt-in HETRECO_NORMAL_CLUSTER=1, measured slower)
            front_clusters_ = fused_.block ? 0 : dev::plan_sense_front(nx_, ny_, nc_ * nf_);
            if (scratch_.size() != nx_ * ny_ * nc_ * nf_ * 8) scratch_ = DevMem(nx_ * ny_ * nc_ * nf_ * 8);
            s_comb_ = dev::combine_cp_preferred(nx_, ny_ * nf_, nc_, sms)
                          ? dev::plan_combine_cp(nx_, dev::Combine::Sense, ny_ * nf_, sms)
                          : combine_ss_enabled(nx_) ? dev::plan_combine_ss(nx_, ny_, nf_, sms)
                                                    : dev::plan_contig(nx_, dev::Combine::Sense, ny_ * nf_, sms);
        }
    }
    // chain of 2-3 small dependent kernels: PDL edges measured faster (C4)
    bool programmatic_edges() const override { return true; }
    void repoint() override {
        m_ = static_cast<const float2*>(session().device_array(require_input(), 0));
        s_ = static_cast<const float2*>(session().device_array(require_input(), 1));
        if (mask_) mask_ = static_cast<const float*>(session().device_array(require_input(), 2));
        out_ = static_cast<float2*>(session().device_array(require_output(), 0));
    }
    void record(cudaStream_t s) override {
        float2* z = normal_ ? scratch_.as<float2>() : out_;
        if (normal_ && fused_.block) {  // one cooperative kernel, three grid-barrier phases
            dev::SenseNormalArgs an{m_, s_, mask_, z, out_, tw_fwd_.as<float2>(), tw_inv_.as<float2>(),
                                    std::uint32_t(nc_), std::uint32_t(nf_), shift_,
                                    float(1.0 / (double(nx_) * double(ny_)))};
            an.phases = int(env_or("HETRECO_NORMAL_PHASES", 7));
            ck(dev::launch_sense_normal_fused(nx_, an, fused_, s), name() + "/normal-fused");
            mark(s);
            return;
        }
        if (normal_ && front_clusters_ > 0) {
            dev::SenseFrontArgs af{m_, s_, mask_, z, tw_fwd_.as<float2>(), std::uint32_t(nc_), std::uint32_t(nf_),
                                   shift_, 1.0f};
            ck(dev::launch_sense_front(af, front_clusters_, s), name() + "/expand.x-fft.y-fft.mask.y-ifft (cluster)");
            mark(s);
            dev::ContigArgs ar{z, out_, s_, ny_, nc_, nf_, shift_, shift_, float(1.0 / (double(nx_) * double(ny_))),
                               tw_inv_.as<float2>()};
            ck(dev::launch_contig(nx_, +1, dev::Combine::Sense, ar, s_comb_, s), name() + "/x-ifft+combine");
            mark(s);
            return;
        }
        dev::ContigArgs ae{m_, z, s_, ny_, nc_, nf_, shift_, shift_, 1.0f, tw_fwd_.as<float2>()};
        ck(dev::launch_expand(nx_, ae, s_exp_, s), name() + "/expand+x-fft");
        mark(s);
        if (generic_cols_) {
            dev::StridedArgs ag{z, z, nx_, nc_ * nf_, shift_, shift_, 1.0f, tw_fwd_y_.as<float2>()};
            ck(dev::launch_strided(ny_, -1, ag, s_col_, s), name() + "/y-fft");
            mark(s);
            return;
        }
        dev::StridedArgs ac{z, z, nx_, nc_ * nf_, shift_, shift_, 1.0f, tw_fwd_.as<float2>(), mask_};
        ck(dev::launch_strided_masked(ny_, normal_, ac, s_col_, s), name() + (normal_ ? "/y-fft.mask.y-ifft" : "/y-fft.mask"));
        mark(s);
        if (normal_) {
            dev::ContigArgs ar{z, out_, s_, ny_, nc_, nf_, shift_, shift_, float(1.0 / (double(nx_) * double(ny_))),
                               tw_inv_.as<float2>()};
            ck(dev::launch_contig(nx_, +1, dev::Combine::Sense, ar, s_comb_, s), name() + "/x-ifft+combine");
            mark(s);
        }
    }

private:
    bool normal_;
    bool shift_ = false;
    std::uint64_t nx_ = 0, ny_ = 0, nc_ = 0, nf_ = 0;
    const float2* m_ = nullptr;
    const float2* s_ = nullptr;
    const float* mask_ = nullptr;
    float2* out_ = nullptr;
    DevMem tw_fwd_, tw_fwd_y_, tw_inv_, scratch_;
    dev::LaunchShape s_exp_, s_col_, s_comb_, fused_;
    int front_clusters_ = 0;
    bool generic_cols_ = false;
};

}  // namespace

std::unique_ptr<GraphProcess> make_negate(ComputeSession& s, std::string n) {
    return std::make_unique<NegateProcess>(s, std::move(n));
}
std::unique_ptr<GraphProcess> make_fft2d(ComputeSession& s, std::string n) {
    return std::make_unique<Fft2dProcess>(s, std::move(n));
}
std::unique_ptr<GraphProcess> make_complex_element_prod(ComputeSession& s, std::string n) {
    return std::make_unique<BuiltinProcess>(s, std::move(n), dev::Builtin::ComplexElementProd);
}
std::unique_ptr<GraphProcess> make_matrix_add(ComputeSession& s, std::string n) {
    return std::make_unique<BuiltinProcess>(s, std::move(n), dev::Builtin::MatrixAdd);
}
std::unique_ptr<GraphProcess> make_ximage_sum(ComputeSession& s, std::string n) {
    return std::make_unique<BuiltinProcess>(s, std::move(n), dev::Builtin::XImageSum);
}
std::unique_ptr<GraphProcess> make_rss_combine(ComputeSession& s, std::string n) {
    return std::make_unique<BuiltinProcess>(s, std::move(n), dev::Builtin::RssCombine);
}
std::unique_ptr<GraphProcess> make_sens_recon(ComputeSession& s, std::string n) {
    return std::make_unique<ReconProcess>(s, std::move(n), dev::Combine::Sense);
}
std::unique_ptr<GraphProcess> make_rss_recon(ComputeSession& s, std::string n) {
    return std::make_unique<ReconProcess>(s, std::move(n), dev::Combine::Rss);
}

std::unique_ptr<GraphProcess> make_process(ComputeSession& s, std::string_view kind, std::string name) {
    const std::string n = name.empty() ? std::string(kind) : name;
    if (kind == "negate") return make_negate(s, n);
    if (kind == "fft2d") return make_fft2d(s, n);
    if (kind == "complex_element_prod") return make_complex_element_prod(s, n);
    if (kind == "ximage_sum") return make_ximage_sum(s, n);
    if (kind == "matrix_add") return make_matrix_add(s, n);
    if (kind == "rss_combine") return make_rss_combine(s, n);
    if (kind == "sens_recon") return make_sens_recon(s, n);
    if (kind == "rss_recon") return make_rss_recon(s, n);
    if (kind == "sense_forward") return std::make_unique<SenseModelProcess>(s, n, false);
    if (kind == "sense_normal") return std::make_unique<SenseModelProcess>(s, n, true);
    throw InvalidArgument("unknown process kind '" + std::string(kind) + "'");
}

// ---- StreamingRecon ---------------------------------------------------------------------------

struct StreamingRecon::Impl {
    ComputeSession* session = nullptr;
    dev::Combine mode = dev::Combine::Sense;
    bool shift = false;
    std::uint64_t nx = 0, ny = 0, nc = 0;
    DevMem smaps, ybuf[2], obuf[2], scratch;
    FftPlan plan;
    cudaEvent_t h2d_done[2]{}, y_free[2]{}, comp_done[2]{}, o_free[2]{};
    ~Impl() {
        for (int b = 0; b < 2; ++b)
            for (cudaEvent_t e : {h2d_done[b], y_free[b], comp_done[b], o_free[b]})
                if (e) cudaEventDestroy(e);
    }
};

StreamingRecon::StreamingRecon(ComputeSession& s, Method method, std::uint64_t nx, std::uint64_t ny,
                               std::uint64_t coils, std::uint64_t chunk, const void* host_smaps, bool shift)
    : impl_(std::make_unique<Impl>()) {
    if (!dev::fft_size_supported(nx) || !dev::fft_size_supported(ny))
        throw ShapeMismatch("streaming recon: nx, ny must be powers of two <= 4096 or mixed-radix sides (96, 160, 192, 320, 384)");
    if (coils == 0 || chunk == 0) throw InvalidArgument("streaming recon: coils and chunk_frames must be >= 1");
    Impl& m = *impl_;
    m.session = &s;
    m.mode = method == Method::Sense ? dev::Combine::Sense : dev::Combine::Rss;
    m.shift = shift;
    m.nx = nx;
    m.ny = ny;
    m.nc = coils;
    chunk_ = chunk;
    in_frame_bytes_ = nx * ny * coils * 8;
    out_frame_bytes_ = nx * ny * (method == Method::Sense ? 8 : 4);
    CudaBackend& cb = s.cuda();
    cb.make_current();
    if (method == Method::Sense) {
        if (!host_smaps) throw InvalidArgument("streaming recon: SENSE needs sensitivity maps");
        m.smaps = upload_bytes(host_smaps, nx * ny * coils * 8);
    }
    for (int b = 0; b < 2; ++b) {
        m.ybuf[b] = DevMem(in_frame_bytes_ * chunk);
        m.obuf[b] = DevMem(out_frame_bytes_ * chunk);
        for (cudaEvent_t* e : {&m.h2d_done[b], &m.y_free[b], &m.comp_done[b], &m.o_free[b]})
            ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
    }
    m.scratch = DevMem(in_frame_bytes_ * chunk);
    m.plan.make(nx, ny, +1, coils * chunk, m.mode, ny * chunk, cb.ordinal());
    if (dev::combine_cp_preferred(nx, ny * chunk, coils, sm_count(cb.ordinal())))
        m.plan.s2 = dev::plan_combine_cp(nx, m.mode, ny * chunk, sm_count(cb.ordinal()));
    else if (m.mode == dev::Combine::Sense && combine_ss_enabled(nx))
        m.plan.s2 = dev::plan_combine_ss(nx, ny, chunk, sm_count(cb.ordinal()));
}

StreamingRecon::~StreamingRecon() = default;

void StreamingRecon::run(const void* host_in, std::uint64_t frames, void* host_out) {
    Impl& m = *impl_;
    CudaBackend& cb = m.session->cuda();
    cb.make_current();
    cudaStream_t cs = cb.compute_stream(), hs = cb.h2d_stream(), ds = cb.d2h_stream();
    cb.note_work();
    const int sms = sm_count(cb.ordinal());
    const auto* src = static_cast<const char*>(host_in);
    auto* dst = static_cast<char*>(host_out);
    const float scale = float(1.0 / (double(m.nx) * double(m.ny)));
    // the compute stream may still hold earlier session work
    ck(cudaEventRecord(m.comp_done[0], cs), "cudaEventRecord");
    ck(cudaStreamWaitEvent(hs, m.comp_done[0], 0), "cudaStreamWaitEvent");
    for (std::uint64_t k = 0, f0 = 0; f0 < frames; ++k, f0 += chunk_) {
        const int b = int(k & 1);
        const std::uint64_t nf = std::min(chunk_, frames - f0);
        // H2D of this chunk once the compute pass of chunk k-2 released the slab
        if (k >= 2) ck(cudaStreamWaitEvent(hs, m.y_free[b], 0), "wait y_free");
        ck(cudaMemcpyAsync(m.ybuf[b].get(), src + f0 * in_frame_bytes_, nf * in_frame_bytes_, cudaMemcpyHostToDevice, hs),
           "H2D chunk");
        ck(cudaEventRecord(m.h2d_done[b], hs), "record h2d_done");
        // compute
        ck(cudaStreamWaitEvent(cs, m.h2d_done[b], 0), "wait h2d_done");
        if (k >= 2) ck(cudaStreamWaitEvent(cs, m.o_free[b], 0), "wait o_free");
        dev::LaunchShape s1 = m.plan.s1, s2 = m.plan.s2;
        if (nf != chunk_) {
            s1 = dev::plan_strided(m.ny, m.nx, m.nc * nf, sms);
            s2 = dev::combine_cp_preferred(m.nx, m.ny * nf, m.nc, sms) ? dev::plan_combine_cp(m.nx, m.mode, m.ny * nf, sms)
                 : (m.mode == dev::Combine::Sense && combine_ss_enabled(m.nx)) ? dev::plan_combine_ss(m.nx, m.ny, nf, sms)
                                                                              : dev::plan_contig(m.nx, m.mode, m.ny * nf, sms);
        }
        dev::StridedArgs a1{m.ybuf[b].as<float2>(), m.scratch.as<float2>(), m.nx, m.nc * nf, m.shift, m.shift, 1.0f,
                            m.plan.tw_y.as<float2>()};
        ck(dev::launch_strided(m.ny, +1, a1, s1, cs), "streaming axis1");
        ck(cudaEventRecord(m.y_free[b], cs), "record y_free");
        dev::ContigArgs a2{m.scratch.as<float2>(), m.obuf[b].get(), m.smaps.as<float2>(), m.ny, m.nc, nf,
                           m.shift, m.shift, scale, m.plan.tw_x.as<float2>()};
        ck(dev::launch_contig(m.nx, +1, m.mode, a2, s2, cs), "streaming axis0+combine");
        ck(cudaEventRecord(m.comp_done[b], cs), "record comp_done");
        // D2H
        ck(cudaStreamWaitEvent(ds, m.comp_done[b], 0), "wait comp_done");
        ck(cudaMemcpyAsync(dst + f0 * out_frame_bytes_, m.obuf[b].get(), nf * out_frame_bytes_, cudaMemcpyDeviceToHost, ds),
           "D2H chunk");
        ck(cudaEventRecord(m.o_free[b], ds), "record o_free");
    }
    // join: later work on the compute stream (and events recorded there, e.g.
    // a device timer around run()) is ordered after the last D2H
    if (frames) {
        const int last_b = int(((frames + chunk_ - 1) / chunk_ - 1) & 1);
        ck(cudaStreamWaitEvent(cs, m.o_free[last_b], 0), "join D2H");
    }
    const cudaError_t e = cudaStreamSynchronize(ds);
    if (e != cudaSuccess) throw DeviceError("streaming_recon", cudaGetErrorString(e));
    ck(cudaStreamSynchronize(cs), "streaming recon (compute)");
}

// ---- fused recon as layer-1 kernels (detail::FusedReconKernels) -----------------------------

struct detail::FusedReconKernels::Plan {
    DevMem tw_x, tw_y;
    dev::LaunchShape s1, s2;
};

detail::FusedReconKernels::FusedReconKernels(int ordinal) : ordinal_(ordinal) {}

detail::FusedReconKernels::~FusedReconKernels() {
    if (scratch_) cudaFree(scratch_);
}

bool detail::FusedReconKernels::is_fused(std::string_view name) { return name == kSense || name == kRss; }

void detail::FusedReconKernels::launch(std::string_view name, const LayoutDescriptor& li, const LayoutDescriptor& lo,
                                       const void* in_base, void* out_base, std::span<const std::byte> params,
                                       std::uint64_t gsize, cudaStream_t stream) {
    const bool sense = name == kSense;
    const std::string who(name);
    const dev::Combine mode = sense ? dev::Combine::Sense : dev::Combine::Rss;
    std::uint32_t flags = 0;
    if (!params.empty()) {
        if (params.size() != 4) throw InvalidArgument(who + ": params are empty or one u32 flag word (bit 0 = shift)");
        std::memcpy(&flags, params.data(), 4);
        if (flags & ~1u) throw InvalidArgument(who + ": unknown flag bits in params");
    }
    const LayoutRecord& y = array_of(li, 0, who);
    require_type(y, ElementType::Complex64, who);
    if (y.rank < 3) throw ShapeMismatch(who + ": k-space must be [nx, ny, coils(, frames)], got " + dims_str(y));
    const std::uint64_t nx = y.dims[0], ny = y.dims[1], nc = y.dims[2], nf = prod(y, 3, y.rank);
    if (!dev::fft_size_supported(nx) || !dev::fft_size_supported(ny))
        throw ShapeMismatch(who + ": spatial dims must be powers of two <= 4096 or mixed-radix sides, got " + dims_str(y));
    const LayoutRecord& o = array_of(lo, 0, who);
    require_type(o, sense ? ElementType::Complex64 : ElementType::Float32, who);
    if (o.dims[0] != nx || (o.rank > 1 ? o.dims[1] : 1) != ny || o.element_count() != nx * ny * nf)
        throw ShapeMismatch(who + ": output " + dims_str(o) + " must be [nx, ny, frames] for k-space " + dims_str(y));
    // one work item per output pixel, as the reference's combine kernels
    if (gsize != nx * ny * nf)
        throw InvalidArgument(who + ": global size must be nx*ny*frames = " + std::to_string(nx * ny * nf) + ", got " +
                              std::to_string(gsize));
    const float2* smap = nullptr;
    if (sense) {
        const LayoutRecord& sm = array_of(li, 1, who);
        require_type(sm, ElementType::Complex64, who);
        if (sm.dims[0] != nx || sm.dims[1] != ny || sm.element_count() != nx * ny * nc)
            throw ShapeMismatch(who + ": sensitivity maps " + dims_str(sm) + " must be [nx, ny, coils]");
        smap = reinterpret_cast<const float2*>(static_cast<const char*>(in_base) + sm.offset_bytes);
    }
    const auto* ydev = reinterpret_cast<const float2*>(static_cast<const char*>(in_base) + y.offset_bytes);
    void* out = static_cast<char*>(out_base) + o.offset_bytes;
    const std::string key = who + ":" + std::to_string(nx) + "x" + std::to_string(ny) + "x" + std::to_string(nc) + "x" +
                            std::to_string(nf);
    auto it = plans_.find(key);
    if (it == plans_.end()) {
        auto pl = std::make_unique<Plan>();
        const int sms = sm_count(ordinal_);
        pl->tw_y = twiddle_table(ny, +1);
        pl->tw_x = twiddle_table(nx, +1);
        pl->s1 = dev::plan_strided(ny, nx, nc * nf, sms);
        pl->s2 = plan_combine_fp32(nx, ny, nc, nf, mode, sms);
        it = plans_.emplace(key, std::move(pl)).first;
    }
    const Plan& pl = *it->second;
    const std::uint64_t need = nx * ny * nc * nf * 8;
    if (need > scratch_bytes_) {
        // earlier launches on this stream may still read the old scratch
        ck(cudaStreamSynchronize(stream), who + ": scratch resize");
        if (scratch_) cudaFree(scratch_);
        scratch_ = nullptr;
        scratch_bytes_ = 0;
        ck(cudaMalloc(&scratch_, need), who + ": scratch");
        scratch_bytes_ = need;
    }
    const bool shift = flags & 1u;
    auto* x = static_cast<float2*>(scratch_);
    dev::StridedArgs a1{ydev, x, nx, nc * nf, shift, shift, 1.0f, pl.tw_y.as<float2>()};
    ck(dev::launch_strided(ny, +1, a1, pl.s1, stream), who + "/axis1");
    dev::ContigArgs a2{x, out, smap, ny, nc, nf, shift, shift, float(1.0 / (double(nx) * double(ny))),
                       pl.tw_x.as<float2>()};
    ck(dev::launch_contig(nx, +1, mode, a2, pl.s2, stream), who + "/axis0+combine");
}

}  // namespace hetreco
