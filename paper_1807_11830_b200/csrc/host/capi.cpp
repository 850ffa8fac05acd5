// capi.cpp -- extern "C" boundary over the C++ host library
// (include/hetreco_b200.h).  Exceptions never cross it: each entry point
// returns the hetreco::ErrorCode of what was thrown and records the message.
#include "hetreco_b200.h"

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "../kernels/launch.hpp"
#include "hetreco_b200/io.hpp"
#include "hetreco_b200/multi_gpu.hpp"
#include "hetreco_b200/numa.hpp"
#include "hetreco_b200/phantom.hpp"
#include "nvrtc_compiler.hpp"
#include "hetreco_b200/processes.hpp"

using namespace hetreco;

struct hetreco_session_t {
    std::unique_ptr<ComputeSession> s;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    ~hetreco_session_t() {
        if (t0) cudaEventDestroy(t0);
        if (t1) cudaEventDestroy(t1);
    }
};
struct hetreco_params_t {
    ProcessParams p;
};
struct hetreco_process_t {
    std::unique_ptr<Process> owned;  // null when borrowed (chain stage view)
    Process* p = nullptr;
    std::vector<hetreco_process_t*> stage_views;
    ~hetreco_process_t() {
        for (auto* v : stage_views) delete v;
    }
};
struct hetreco_stream_t {
    std::unique_ptr<StreamingRecon> r;
};
struct hetreco_multi_t {
    std::unique_ptr<MultiGpuRecon> m;
};
struct hetreco_cuda_backend_t {
    std::unique_ptr<CudaBackend> b;
};
struct hetreco_mat_t {
    std::vector<io::MatVariable> vars;
};

namespace {

thread_local std::string g_error;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_error.clear();
        return HETRECO_OK;
    } catch (const Error& e) {
        g_error = e.what();
        return int(e.code());
    } catch (const std::exception& e) {
        g_error = e.what();
        return int(ErrorCode::Error);
    } catch (...) {
        g_error = "unknown exception";
        return int(ErrorCode::Error);
    }
}

void need(const void* p, const char* what) {
    if (!p) throw InvalidArgument(std::string(what) + " is NULL");
}

void copy_str(char* dst, std::size_t cap, const std::string& s) {
    std::size_t n = std::min(cap - 1, s.size());
    std::memcpy(dst, s.data(), n);
    dst[n] = 0;
}

void to_c(const DeviceDescriptor& d, hetreco_device_desc* o) {
    std::memset(o, 0, sizeof *o);
    copy_str(o->backend_id, sizeof o->backend_id, d.backend_id);
    o->device_index = d.device_index;
    o->device_type = d.device_type == DeviceType::Cpu ? 0 : d.device_type == DeviceType::Gpu ? 1 : 2;
    copy_str(o->vendor, sizeof o->vendor, d.vendor);
    copy_str(o->name, sizeof o->name, d.name);
    copy_str(o->api_version, sizeof o->api_version, d.api_version);
    o->global_memory_bytes = d.global_memory_bytes;
    o->base_alignment_bytes = d.base_alignment_bytes;
    o->supports_source_kernels = d.supports_source_kernels;
}

DeviceDescriptor from_c(const hetreco_device_desc& c) {
    DeviceDescriptor d;
    d.backend_id = c.backend_id;
    d.device_index = c.device_index;
    d.device_type = c.device_type == 0 ? DeviceType::Cpu : c.device_type == 1 ? DeviceType::Gpu : DeviceType::Accelerator;
    d.vendor = c.vendor;
    d.name = c.name;
    d.api_version = c.api_version;
    d.global_memory_bytes = c.global_memory_bytes;
    d.base_alignment_bytes = c.base_alignment_bytes;
    d.supports_source_kernels = c.supports_source_kernels != 0;
    return d;
}

DataKind kind_of(int k) {
    if (k == HETRECO_XDATA) return DataKind::XData;
    if (k == HETRECO_KDATA) return DataKind::KData;
    if (k == HETRECO_GENERIC) return DataKind::Generic;
    throw InvalidArgument("unknown data kind " + std::to_string(k));
}

int kind_code(DataKind k) {
    return k == DataKind::XData ? HETRECO_XDATA : k == DataKind::KData ? HETRECO_KDATA : HETRECO_GENERIC;
}

ArrayShape shape_of(const hetreco_array_desc& a) {
    if (!is_valid_element_type(a.element_type))
        throw InvalidArgument("unknown element type code " + std::to_string(a.element_type));
    if (a.rank == 0 || a.rank > kMaxRank) throw InvalidArgument("array rank must be between 1 and 8");
    return {ElementType(a.element_type), std::vector<std::uint64_t>(a.dims, a.dims + a.rank)};
}

DataHandle H(hetreco_handle h) { return {h.session_uid, h.id}; }
hetreco_handle C(DataHandle h) { return {h.session_uid, h.id}; }

ComputeSession& S(hetreco_session s) {
    need(s, "session");
    return *s->s;
}
Process& P(hetreco_process p) {
    need(p, "process");
    return *p->p;
}
CudaBackend& B(hetreco_cuda_backend b) {
    need(b, "backend");
    return *b->b;
}

}  // namespace

extern "C" {

const char* hetreco_last_error(void) { return g_error.c_str(); }
const char* hetreco_version(void) { return "hetreco-b200 0.1 (sm_100a)"; }

// ---- devices ----

int hetreco_enumerate_devices(hetreco_device_desc* out, int cap, int* count) {
    return guard([&] {
        need(count, "count");
        auto ds = enumerate_devices();
        *count = int(ds.size());
        for (int i = 0; i < cap && i < int(ds.size()); ++i) to_c(ds[i], out + i);
    });
}

int hetreco_select_device(const char* text, hetreco_device_desc* out) {
    return guard([&] {
        need(out, "out");
        to_c(select_device(DeviceFilter::parse(text ? text : "")), out);
    });
}

int hetreco_select_from(const hetreco_device_desc* cands, int n, const char* text, int* index) {
    return guard([&] {
        need(index, "index");
        std::vector<DeviceDescriptor> v;
        for (int i = 0; i < n; ++i) v.push_back(from_c(cands[i]));
        const DeviceDescriptor& w = select_from(v, DeviceFilter::parse(text ? text : ""));
        *index = int(&w - v.data());
    });
}

int hetreco_filter_describe(const char* text, char* buf, uint64_t cap) {
    return guard([&] {
        need(buf, "buf");
        copy_str(buf, cap, DeviceFilter::parse(text ? text : "").describe());
    });
}

// ---- layer 1: backend contract ----

int hetreco_cuda_device_count(int* count) {
    return guard([&] {
        need(count, "count");
        *count = cuda_device_count();
    });
}

int hetreco_cuda_backend_create(int ordinal, uint64_t cap, hetreco_cuda_backend* out) {
    return guard([&] {
        need(out, "out");
        if (ordinal < 0 || ordinal >= cuda_device_count())
            throw NoMatchingDevice("no CUDA device with ordinal " + std::to_string(ordinal));
        auto* h = new hetreco_cuda_backend_t;
        h->b = std::make_unique<CudaBackend>(ordinal, cap);
        *out = h;
    });
}

int hetreco_cuda_backend_destroy(hetreco_cuda_backend b) {
    return guard([&] { delete b; });
}

int hetreco_cuda_backend_device(hetreco_cuda_backend b, hetreco_device_desc* out) {
    return guard([&] { to_c(B(b).devices().at(0), out); });
}

int hetreco_cuda_allocate(hetreco_cuda_backend b, uint64_t bytes, uint64_t* id) {
    return guard([&] {
        need(id, "buffer_id");
        *id = B(b).allocate(bytes);
    });
}

int hetreco_cuda_release(hetreco_cuda_backend b, uint64_t id) {
    return guard([&] { B(b).release(id); });
}

int hetreco_cuda_upload(hetreco_cuda_backend b, uint64_t id, uint64_t off, const void* src, uint64_t n) {
    return guard([&] { B(b).upload(id, off, std::span<const std::byte>(static_cast<const std::byte*>(src), n)); });
}

int hetreco_cuda_download(hetreco_cuda_backend b, uint64_t id, uint64_t off, void* dst, uint64_t n) {
    return guard([&] { B(b).download(id, off, std::span<std::byte>(static_cast<std::byte*>(dst), n)); });
}

int hetreco_cuda_copy(hetreco_cuda_backend b, uint64_t src, uint64_t so, uint64_t dst, uint64_t doff, uint64_t n) {
    return guard([&] { B(b).copy(src, so, dst, doff, n); });
}

int hetreco_cuda_kernel_count(int* count) {
    return guard([&] {
        need(count, "count");
        *count = intrinsic_kernel_count();
    });
}

const char* hetreco_cuda_kernel_name(int i) {
    return intrinsic_kernel_name(i);
}

int hetreco_cuda_execute(hetreco_cuda_backend b, const char* name, uint64_t in, uint64_t inh, uint64_t out,
                         uint64_t outh, const void* params, uint64_t psize, uint64_t gsize) {
    return guard([&] {
        need(name, "kernel_name");
        if (gsize == 0) throw InvalidArgument(std::string("launch of kernel '") + name + "' with empty index space");
        CompiledKernel k{name, std::string("sm_100a:") + name, nullptr};
        KernelBinding bind{in, inh, out, outh,
                           std::span<const std::byte>(static_cast<const std::byte*>(params), psize)};
        B(b).execute(k, bind, gsize);
    });
}

int hetreco_cuda_supports_source(hetreco_cuda_backend b, int* yes) {
    return guard([&] {
        need(yes, "yes");
        *yes = B(b).supports_source_kernels() ? 1 : 0;
    });
}

int hetreco_cuda_compile(hetreco_cuda_backend b, int count, const char* const* unit_names, const char* const* sources,
                         char* out, uint64_t cap) {
    return guard([&] {
        if (count < 0) throw InvalidArgument("count must be >= 0");
        std::vector<ProgramSource> units;
        for (int i = 0; i < count; ++i) {
            need(unit_names, "unit_names");
            need(unit_names[i], "unit name");
            need(sources, "sources");
            need(sources[i], "unit source");
            units.push_back({unit_names[i], sources[i]});
        }
        std::string listing;
        for (const CompiledKernel& k : B(b).compile(units)) listing += k.unit_name + "\t" + k.name + "\n";
        if (out && cap) {
            if (listing.size() + 1 > cap) throw InvalidArgument("kernel listing needs " + std::to_string(listing.size() + 1) + " bytes");
            copy_str(out, cap, listing);
        }
    });
}

int hetreco_cuda_execute_unit(hetreco_cuda_backend b, const char* unit_tag, const char* name, uint64_t in,
                              uint64_t inh, uint64_t out, uint64_t outh, const void* params, uint64_t psize,
                              uint64_t gsize) {
    return guard([&] {
        need(unit_tag, "unit_tag");
        need(name, "kernel_name");
        if (gsize == 0) throw InvalidArgument(std::string("launch of kernel '") + name + "' with empty index space");
        CompiledKernel k{name, unit_tag, nullptr};
        KernelBinding bind{in, inh, out, outh,
                           std::span<const std::byte>(static_cast<const std::byte*>(params), psize)};
        B(b).execute(k, bind, gsize);
    });
}

int hetreco_cuda_synchronize(hetreco_cuda_backend b) {
    return guard([&] { B(b).synchronize(); });
}

int hetreco_host_alloc(uint64_t bytes, void** out) {
    return guard([&] {
        need(out, "out");
        const cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw AllocationFailure(std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
        }
    });
}

int hetreco_host_free(void* p) {
    return guard([&] {
        if (p && cudaFreeHost(p) != cudaSuccess) {
            cudaGetLastError();
            throw InvalidArgument("cudaFreeHost failed");
        }
    });
}

// ---- sessions ----

int hetreco_session_create(const char* text, hetreco_session* out) {
    return guard([&] {
        need(out, "out");
        auto* h = new hetreco_session_t;
        try {
            h->s = std::make_unique<ComputeSession>(DeviceFilter::parse(text ? text : ""));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int hetreco_session_create_on(const char* backend_id, hetreco_session* out) {
    return guard([&] {
        need(out, "out");
        need(backend_id, "backend_id");
        Backend& b = backend_by_id(backend_id);
        auto* h = new hetreco_session_t;
        h->s = std::make_unique<ComputeSession>(b.devices().at(0));
        *out = h;
    });
}

int hetreco_session_destroy(hetreco_session s) {
    return guard([&] { delete s; });
}

int hetreco_session_device(hetreco_session s, hetreco_device_desc* out) {
    return guard([&] { to_c(S(s).device(), out); });
}

int hetreco_register_data(hetreco_session s, int kind, int count, const hetreco_array_desc* arrays,
                          hetreco_handle* out) {
    return guard([&] {
        need(out, "out");
        if (count < 0) throw InvalidArgument("count must be >= 0");
        // borrowed host buffers straight to the device (no intermediate copy)
        std::vector<ComputeSession::HostArrayRef> refs;
        for (int i = 0; i < count; ++i) refs.push_back({shape_of(arrays[i]), arrays[i].host});
        *out = C(S(s).register_host(refs, kind_of(kind)));
    });
}

int hetreco_allocate_data(hetreco_session s, int kind, int count, const hetreco_array_desc* arrays,
                          hetreco_handle* out) {
    return guard([&] {
        need(out, "out");
        std::vector<ArrayShape> shapes;
        for (int i = 0; i < count; ++i) shapes.push_back(shape_of(arrays[i]));
        *out = C(S(s).allocate_data(shapes, kind_of(kind)));
    });
}

int hetreco_session_layout(hetreco_session s, hetreco_handle h, hetreco_array_desc* out, int cap, int* count,
                           uint64_t* total, int* kind) {
    return guard([&] {
        const LayoutDescriptor& l = S(s).layout_of(H(h));
        if (count) *count = int(l.records.size());
        if (total) *total = l.total_bytes;
        if (kind) *kind = kind_code(S(s).kind_of(H(h)));
        for (int i = 0; i < cap && i < int(l.records.size()); ++i) {
            const LayoutRecord& r = l.records[i];
            std::memset(&out[i], 0, sizeof out[i]);
            out[i].element_type = std::uint64_t(r.element_type);
            out[i].rank = r.rank;
            for (int d = 0; d < 8; ++d) out[i].dims[d] = r.dims[d];
            out[i].offset_bytes = r.offset_bytes;
        }
    });
}

int hetreco_fetch_data(hetreco_session s, hetreco_handle h, int count, void* const* dst) {
    return guard([&] {
        need(dst, "dst");
        S(s).fetch_into(H(h), std::span<void* const>(dst, std::size_t(count)));
    });
}

int hetreco_release_data(hetreco_session s, hetreco_handle h) {
    return guard([&] { S(s).release_data(H(h)); });
}

int hetreco_fetch_header_bytes(hetreco_session s, hetreco_handle h, void* dst, uint64_t cap, uint64_t* n) {
    return guard([&] {
        auto bytes = S(s).fetch_header_bytes(H(h));
        if (n) *n = bytes.size();
        if (dst) std::memcpy(dst, bytes.data(), std::min<std::uint64_t>(cap, bytes.size()));
    });
}

int hetreco_copy_array(hetreco_session s, hetreco_handle src, uint64_t si, hetreco_handle dst, uint64_t di) {
    return guard([&] { S(s).copy_array(H(src), si, H(dst), di); });
}

int hetreco_load_builtin_kernels(hetreco_session s) {
    return guard([&] { S(s).load_builtin_kernels(); });
}

int hetreco_kernel_names(hetreco_session s, char* buf, uint64_t cap) {
    return guard([&] {
        std::string all;
        for (const auto& n : S(s).kernels().names()) all += (all.empty() ? "" : "\n") + n;
        need(buf, "buf");
        copy_str(buf, cap, all);
    });
}

int hetreco_load_kernels(hetreco_session s, int count, const char* const* names, const char* const* sources) {
    return guard([&] {
        std::vector<ProgramSource> units;
        for (int i = 0; i < count; ++i) units.push_back({names[i], sources[i]});
        S(s).load_kernels(units);
    });
}

int hetreco_launch_kernel(hetreco_session s, const char* name, hetreco_handle in, hetreco_handle out,
                          const void* params, uint64_t psize, uint64_t gsize) {
    return guard([&] {
        need(name, "name");
        S(s).launch_kernel(name, H(in), H(out),
                           std::span<const std::byte>(static_cast<const std::byte*>(params), psize), gsize);
    });
}

int hetreco_synchronize(hetreco_session s) {
    return guard([&] { S(s).synchronize(); });
}

int hetreco_counters(hetreco_session s, uint64_t* h2d, uint64_t* d2h) {
    return guard([&] {
        const TransferCounters c = S(s).counters();
        if (h2d) *h2d = c.host_to_device;
        if (d2h) *d2h = c.device_to_host;
    });
}

int hetreco_reset_counters(hetreco_session s) {
    return guard([&] { S(s).reset_counters(); });
}

int hetreco_live_data_count(hetreco_session s, uint64_t* n) {
    return guard([&] { *n = S(s).live_data_count(); });
}

// ---- params / processes ----

int hetreco_params_create(hetreco_params* out) {
    return guard([&] { *out = new hetreco_params_t; });
}
int hetreco_params_destroy(hetreco_params p) {
    return guard([&] { delete p; });
}
int hetreco_params_set_bool(hetreco_params p, const char* k, int v) {
    return guard([&] { p->p.set(k, bool(v != 0)); });
}
int hetreco_params_set_int(hetreco_params p, const char* k, int64_t v) {
    return guard([&] { p->p.set(k, std::int64_t(v)); });
}
int hetreco_params_set_real(hetreco_params p, const char* k, double v) {
    return guard([&] { p->p.set(k, v); });
}
int hetreco_params_set_string(hetreco_params p, const char* k, const char* v) {
    return guard([&] { p->p.set(k, std::string(v)); });
}

int hetreco_process_create(hetreco_session s, const char* kind, const char* name, hetreco_process* out) {
    return guard([&] {
        need(kind, "kind");
        need(out, "out");
        auto* h = new hetreco_process_t;
        try {
            h->owned = make_process(S(s), kind, name ? name : "");
        } catch (...) {
            delete h;
            throw;
        }
        h->p = h->owned.get();
        *out = h;
    });
}

int hetreco_chain_create(hetreco_session s, const char* name, hetreco_process* stages, int n, hetreco_process* out) {
    return guard([&] {
        need(out, "out");
        need(s, "session");
        if (n <= 0) throw InvalidArgument("chain needs at least one stage");
        need(stages, "stages");
        // Validate everything before ownership moves, so any failure leaves
        // the caller's stage handles intact: owned stages of this session,
        // each handle once, and stage i's output feeding stage i + 1.
        for (int i = 0; i < n; ++i) {
            need(stages[i], "stage");
            if (!stages[i]->owned) throw InvalidArgument("chain stage " + std::to_string(i) + " is not owned");
            if (&stages[i]->p->session() != s->s.get())
                throw ChainMismatch("stage " + std::to_string(i) + " belongs to another session");
            for (int k = 0; k < i; ++k)
                if (stages[k] == stages[i])
                    throw InvalidArgument("chain stage handle " + std::to_string(i) + " repeats stage " +
                                          std::to_string(k));
        }
        for (int i = 0; i + 1 < n; ++i)
            if (!(stages[i]->p->output() == stages[i + 1]->p->input()) || !stages[i]->p->output().valid())
                throw ChainMismatch("stage " + std::to_string(i) + " ('" + stages[i]->p->name() +
                                    "') output is not the input of stage " + std::to_string(i + 1) + " ('" +
                                    stages[i + 1]->p->name() + "')");
        auto h = std::make_unique<hetreco_process_t>();
        std::vector<std::unique_ptr<Process>> v;
        for (int i = 0; i < n; ++i) v.push_back(std::move(stages[i]->owned));
        std::unique_ptr<CompositeProcess> comp;
        try {
            comp = chain(S(s), name ? name : "chain", std::move(v));
        } catch (...) {
            // chain() leaves the stages in `v` when it throws: hand them back
            for (int i = 0; i < n && i < int(v.size()); ++i)
                if (v[i]) stages[i]->owned = std::move(v[i]);
            throw;
        }
        for (int i = 0; i < n; ++i) stages[i]->p = &comp->stage(i);  // caller's handles become views
        h->p = comp.get();
        h->owned = std::move(comp);
        for (int i = 0; i < n; ++i) h->stage_views.push_back(stages[i]);
        *out = h.release();
    });
}

int hetreco_process_destroy(hetreco_process p) {
    return guard([&] {
        if (p && !p->owned && p->p) return;  // a chain stage view: owned by the chain
        delete p;
    });
}

int hetreco_process_set_input(hetreco_process p, hetreco_handle h) {
    return guard([&] { P(p).set_input(H(h)); });
}
int hetreco_process_set_output(hetreco_process p, hetreco_handle h) {
    return guard([&] { P(p).set_output(H(h)); });
}
int hetreco_process_init(hetreco_process p, hetreco_params params) {
    return guard([&] { P(p).init(params ? params->p : ProcessParams{}); });
}
int hetreco_process_launch(hetreco_process p) {
    return guard([&] { P(p).launch(); });
}
int hetreco_process_state(hetreco_process p, int* state) {
    return guard([&] { *state = P(p).state() == ProcessState::Created ? 0 : 1; });
}
int hetreco_process_stats(hetreco_process p, uint64_t* ic, uint64_t* nl, double* last, double* total, double* init) {
    return guard([&] {
        const LaunchStats& st = P(p).stats();
        if (ic) *ic = st.init_calls;
        if (nl) *nl = st.launches;
        if (last) *last = st.last_launch_seconds;
        if (total) *total = st.total_launch_seconds;
        if (init) *init = st.init_seconds;
    });
}
int hetreco_process_profile(hetreco_process p, int reps, double* secs, int cap, int* n) {
    return guard([&] {
        auto* g = dynamic_cast<GraphProcess*>(&P(p));
        if (!g) throw InvalidArgument("process is not a graph process");
        const auto v = g->profile(reps);
        if (n) *n = int(v.size());
        for (int i = 0; i < cap && i < int(v.size()); ++i) secs[i] = v[i];
    });
}

int hetreco_session_timer_start(hetreco_session s) {
    return guard([&] {
        CudaBackend& cb = S(s).cuda();
        cb.make_current();
        if (!s->t0) {
            cudaEventCreate(&s->t0);
            cudaEventCreate(&s->t1);
        }
        if (cudaEventRecord(s->t0, cb.compute_stream()) != cudaSuccess) throw DeviceError("timer", "cudaEventRecord");
    });
}

int hetreco_session_timer_stop(hetreco_session s, double* seconds) {
    return guard([&] {
        CudaBackend& cb = S(s).cuda();
        cb.make_current();
        if (!s->t0) throw InvalidArgument("timer was not started");
        cudaEventRecord(s->t1, cb.compute_stream());
        const cudaError_t e = cudaEventSynchronize(s->t1);
        if (e != cudaSuccess) throw DeviceError("timer", cudaGetErrorString(e));
        float ms = 0;
        cudaEventElapsedTime(&ms, s->t0, s->t1);
        *seconds = double(ms) * 1e-3;
    });
}

int hetreco_chain_stage(hetreco_process c, int index, hetreco_process* out) {
    return guard([&] {
        need(c, "chain");
        if (index < 0 || index >= int(c->stage_views.size())) throw InvalidArgument("stage index out of range");
        *out = c->stage_views[index];
    });
}

// ---- streaming ----

int hetreco_stream_create(hetreco_session s, int method, uint64_t nx, uint64_t ny, uint64_t coils, uint64_t chunk,
                          const void* smaps, int shift, hetreco_stream* out) {
    return guard([&] {
        need(out, "out");
        auto* h = new hetreco_stream_t;
        try {
            h->r = std::make_unique<StreamingRecon>(
                S(s), method == HETRECO_METHOD_SENSE ? StreamingRecon::Method::Sense : StreamingRecon::Method::Rss,
                nx, ny, coils, chunk, smaps, shift != 0);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int hetreco_stream_run(hetreco_stream st, const void* in, uint64_t frames, void* out) {
    return guard([&] {
        need(st, "stream");
        st->r->run(in, frames, out);
    });
}

int hetreco_stream_destroy(hetreco_stream st) {
    return guard([&] { delete st; });
}

int hetreco_frame_slab(uint64_t index, uint64_t count, uint64_t frames, uint64_t* begin, uint64_t* end) {
    return guard([&] {
        const auto [b, e] = frame_slab(index, count, frames);
        if (begin) *begin = b;
        if (end) *end = e;
    });
}

int hetreco_multi_create(int n, const char* const* ids, int method, uint64_t nx, uint64_t ny, uint64_t coils,
                         uint64_t chunk, const void* smaps, int shift, int bind_numa, hetreco_multi* out) {
    return guard([&] {
        need(out, "out");
        if (n <= 0) throw InvalidArgument("multi-GPU recon needs at least one backend id");
        need(ids, "backend_ids");
        std::vector<std::string> v;
        for (int i = 0; i < n; ++i) {
            need(ids[i], "backend id");
            v.emplace_back(ids[i]);
        }
        auto h = std::make_unique<hetreco_multi_t>();
        h->m = std::make_unique<MultiGpuRecon>(
            v, method == HETRECO_METHOD_SENSE ? StreamingRecon::Method::Sense : StreamingRecon::Method::Rss, nx, ny,
            coils, chunk, smaps, shift != 0, bind_numa != 0);
        *out = h.release();
    });
}

int hetreco_multi_run(hetreco_multi m, const void* in, uint64_t frames, void* out) {
    return guard([&] {
        need(m, "multi");
        m->m->run(in, frames, out);
    });
}

int hetreco_multi_slab(hetreco_multi m, int index, uint64_t* first, uint64_t* frames, double* seconds) {
    return guard([&] {
        need(m, "multi");
        const auto& r = m->m->last_run();
        if (index < 0 || std::size_t(index) >= r.size())
            throw InvalidArgument("slab " + std::to_string(index) + " out of range (last run had " +
                                  std::to_string(r.size()) + ")");
        if (first) *first = r[index].first_frame;
        if (frames) *frames = r[index].frames;
        if (seconds) *seconds = r[index].seconds;
    });
}

int hetreco_multi_device_count(hetreco_multi m, int* n) {
    return guard([&] {
        need(m, "multi");
        need(n, "n");
        *n = int(m->m->device_count());
    });
}

int hetreco_multi_destroy(hetreco_multi m) {
    return guard([&] { delete m; });
}

// ---- host-only layout helpers ----

int hetreco_pack_layout(int count, hetreco_array_desc* arrays, uint64_t alignment, uint64_t* words, uint64_t cap,
                        uint64_t* total) {
    return guard([&] {
        std::vector<ArrayShape> shapes;
        for (int i = 0; i < count; ++i) shapes.push_back(shape_of(arrays[i]));
        const LayoutDescriptor l = pack_shapes(shapes, alignment);
        for (int i = 0; i < count; ++i) arrays[i].offset_bytes = l.records[i].offset_bytes;
        const auto bytes = serialize_layout_header(l);
        if (words) std::memcpy(words, bytes.data(), std::min<std::uint64_t>(cap * 8, bytes.size()));
        if (total) *total = l.total_bytes;
    });
}

int hetreco_parse_layout_header(const void* bytes, uint64_t n, hetreco_array_desc* out, int cap, int* count,
                                uint64_t* alignment, uint64_t* total) {
    return guard([&] {
        const LayoutDescriptor l = parse_layout_header(std::span<const std::byte>(static_cast<const std::byte*>(bytes), n));
        if (count) *count = int(l.records.size());
        if (alignment) *alignment = l.alignment_bytes;
        if (total) *total = l.total_bytes;
        for (int i = 0; i < cap && i < int(l.records.size()); ++i) {
            std::memset(&out[i], 0, sizeof out[i]);
            out[i].element_type = std::uint64_t(l.records[i].element_type);
            out[i].rank = l.records[i].rank;
            for (int d = 0; d < 8; ++d) out[i].dims[d] = l.records[i].dims[d];
            out[i].offset_bytes = l.records[i].offset_bytes;
        }
    });
}

}  // extern "C"

// ---- io (SPEC.md io module :470-533; include/hetreco_b200/io.hpp) --------------------

namespace {
NDArray array_of_desc(const hetreco_array_desc& d) {
    ArrayShape sh = shape_of(d);
    NDArray a(sh.element_type, sh.dims);
    if (a.byte_size()) {
        need(d.host, "array payload");
        std::memcpy(a.bytes().data(), d.host, a.byte_size());
    }
    return a;
}
HostMemory mem_of(int pinned) { return pinned ? HostMemory::Pinned : HostMemory::Pageable; }
}  // namespace

extern "C" {

int hetreco_mat_read(const char* path, int pinned, hetreco_mat* out) {
    return guard([&] {
        need(path, "path");
        need(out, "out");
        auto m = std::make_unique<hetreco_mat_t>();
        m->vars = io::read_mat(path, mem_of(pinned));
        *out = m.release();
    });
}

int hetreco_mat_parse(const void* bytes, uint64_t size, int pinned, hetreco_mat* out) {
    return guard([&] {
        need(bytes, "bytes");
        need(out, "out");
        auto m = std::make_unique<hetreco_mat_t>();
        m->vars = io::parse_mat(static_cast<const std::byte*>(bytes), size, mem_of(pinned));
        *out = m.release();
    });
}

int hetreco_image_read(const char* path, int pinned, hetreco_mat* out) {
    return guard([&] {
        need(path, "path");
        need(out, "out");
        auto m = std::make_unique<hetreco_mat_t>();
        m->vars.push_back({"image", io::read_image(path, mem_of(pinned))});
        *out = m.release();
    });
}

int hetreco_raw_read(const char* path, const char* sidecar_path, int pinned, hetreco_mat* out) {
    return guard([&] {
        need(path, "path");
        need(sidecar_path, "sidecar_path");
        need(out, "out");
        auto m = std::make_unique<hetreco_mat_t>();
        m->vars.push_back({"raw", io::read_raw(path, sidecar_path, mem_of(pinned))});
        *out = m.release();
    });
}

int hetreco_mat_count(hetreco_mat m, int* count) {
    return guard([&] {
        need(m, "mat");
        need(count, "count");
        *count = int(m->vars.size());
    });
}

int hetreco_mat_variable(hetreco_mat m, int index, char* name, uint64_t cap, hetreco_array_desc* desc) {
    return guard([&] {
        need(m, "mat");
        need(desc, "desc");
        if (index < 0 || std::size_t(index) >= m->vars.size())
            throw InvalidArgument("variable index " + std::to_string(index) + " out of range");
        io::MatVariable& v = m->vars[std::size_t(index)];
        if (name && cap) copy_str(name, cap, v.name);
        std::memset(desc, 0, sizeof *desc);
        desc->element_type = std::uint64_t(v.array.element_type());
        desc->rank = std::uint32_t(v.array.rank());
        for (std::size_t i = 0; i < v.array.rank(); ++i) desc->dims[i] = v.array.dims()[i];
        desc->host = v.array.bytes().data();
        desc->offset_bytes = v.array.pinned() ? 1 : 0;  // io: 1 = payload is page-locked
    });
}

int hetreco_mat_free(hetreco_mat m) {
    return guard([&] { delete m; });
}

int hetreco_mat_write(const char* path, int count, const char* const* names, const hetreco_array_desc* arrays) {
    return guard([&] {
        need(path, "path");
        if (count < 0) throw InvalidArgument("count must be >= 0");
        std::vector<io::MatVariable> vars;
        for (int i = 0; i < count; ++i) {
            need(names, "names");
            need(arrays, "arrays");
            need(names[i], "variable name");
            vars.push_back({names[i], array_of_desc(arrays[i])});
        }
        io::write_mat(path, vars);
    });
}

int hetreco_image_write(const char* path, const hetreco_array_desc* image) {
    return guard([&] {
        need(path, "path");
        need(image, "image");
        io::write_image(path, array_of_desc(*image));
    });
}

int hetreco_raw_write(const char* path, const char* sidecar_path, const hetreco_array_desc* array) {
    return guard([&] {
        need(path, "path");
        need(sidecar_path, "sidecar_path");
        need(array, "array");
        io::write_raw(path, sidecar_path, array_of_desc(*array));
    });
}

}  // extern "C"

// ---- gen_phantom (include/hetreco_b200/phantom.hpp) ------------------

extern "C" int hetreco_gen_phantom(hetreco_session s, uint64_t nx, uint64_t ny, uint64_t frames, uint64_t coils,
                                   uint64_t seed, void* kdata, void* smaps, void* truth) {
    return guard([&] {
        need(s, "session");
        Phantom ph = gen_phantom(*s->s, PhantomSpec{nx, ny, frames, coils, seed});
        auto put = [](void* dst, const Data& d) {
            if (dst) std::memcpy(dst, d.arrays[0].bytes().data(), d.arrays[0].byte_size());
        };
        put(kdata, ph.kdata);
        put(smaps, ph.smaps);
        put(truth, ph.truth);
    });
}

extern "C" int hetreco_phantom_blobs(uint64_t nx, uint64_t ny, uint64_t seed, double* out12) {
    return guard([&] {
        need(out12, "out");
        const auto b = phantom_blobs(PhantomSpec{nx, ny, 1, 1, seed});
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 4; ++j) out12[4 * i + j] = b[i][j];
    });
}

// ---- source kernels: compile-only check (no device needed) ---------------------------

extern "C" int hetreco_nvrtc_compile_check(const char* unit_name, const char* source, char* names, uint64_t names_cap,
                                           char* log, uint64_t log_cap) {
    return guard([&] {
        need(unit_name, "unit_name");
        need(source, "source");
        nvrtc::Unit u;
        try {
            u = nvrtc::compile(unit_name, source, "sm_100a");
        } catch (const CompileError& e) {
            if (log && log_cap) copy_str(log, log_cap, e.diagnostics().empty() ? e.what() : e.diagnostics()[0].log);
            throw;
        }
        std::string joined;
        for (const auto& k : u.kernels) joined += (joined.empty() ? "" : "\n") + k;
        if (names && names_cap) copy_str(names, names_cap, joined);
        if (log && log_cap) copy_str(log, log_cap, u.log);
    });
}

extern "C" int hetreco_nvrtc_available(int* available) {
    return guard([&] {
        need(available, "available");
        *available = nvrtc::available() ? 1 : 0;
    });
}

// ---- NUMA placement (SURVEY.md §8 e) ---------------------------------------------------

extern "C" int hetreco_device_numa_node(int ordinal, int* node) {
    return guard([&] {
        need(node, "node");
        *node = device_numa_node(ordinal);
    });
}

extern "C" int hetreco_bind_numa_node(int node, int* cpus) {
    return guard([&] {
        const int n = bind_thread_to_numa_node(node);
        if (cpus) *cpus = n;
    });
}

extern "C" int hetreco_parse_cpulist(const char* text, int* cpus, int cap, int* count) {
    return guard([&] {
        need(text, "text");
        need(count, "count");
        const std::vector<int> v = parse_cpulist(text);
        *count = int(v.size());
        for (int i = 0; i < int(v.size()) && i < cap && cpus; ++i) cpus[i] = v[std::size_t(i)];
    });
}
