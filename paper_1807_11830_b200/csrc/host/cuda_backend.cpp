// cuda_backend.cpp -- the Backend contract (reference include/hetreco/
// backend.hpp:44-79) implemented on one B200, plus the process-wide backend
// list (backend.cpp:294-323 role) and the kernel registry (kernels.cpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <set>

#include "../kernels/launch.hpp"
#include "hetreco_b200/runtime.hpp"

#include "fused_recon.hpp"
#include "host_stager.hpp"
#include "nvrtc_compiler.hpp"

namespace hetreco {

namespace {

[[noreturn]] void raise_cuda(cudaError_t e, const std::string& what) {
    if (e == cudaErrorMemoryAllocation) throw AllocationFailure(what + ": " + cudaGetErrorString(e));
    throw Error(what + ": " + cudaGetErrorString(e));
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise_cuda(e, what);
}

// Host entry point stored in CompiledKernel::fn for device kernels: the
// registry requires a non-null fn (kernels.cpp:13), but these kernels only
// run on the GPU, so a host call is an error, never a silent CPU fallback.
void device_only_entry(const hetreco_kernel_args*, std::uint64_t, std::uint64_t) {
    throw DeviceError("<device kernel>", "sm_100a kernels cannot be invoked on the host");
}

void check_window(const char* what, std::uint64_t off, std::uint64_t len, std::uint64_t size) {
    if (off > size || len > size - off)
        throw InvalidArgument(std::string(what) + " window [" + std::to_string(off) + ", " +
                              std::to_string(off + len) + ") exceeds buffer size " + std::to_string(size));
}

}  // namespace

int cuda_device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// ---- CudaBackend ------------------------------------------------------------------------

// Construction only reads the device properties (no context): the backend
// list holds one CudaBackend per visible GPU, and a process that uses one GPU
// (one rank per GPU under torchrun) must not open contexts, streams and
// pinned rings on the others.  The device state is created on first use
// (ensure()), like the reference's lazily populated backend list
// (backend.cpp:294-313) but per device.
CudaBackend::CudaBackend(int ordinal, std::uint64_t capacity) : ordinal_(ordinal), capacity_(capacity) {
    id_ = "cuda" + std::to_string(ordinal);
    cudaDeviceProp p{};
    ck(cudaGetDeviceProperties(&p, ordinal), "cudaGetDeviceProperties");
    desc_.backend_id = id_;
    desc_.device_index = 0;
    desc_.device_type = DeviceType::Gpu;
    desc_.vendor = "NVIDIA";
    desc_.name = p.name;
    desc_.api_version = std::to_string(p.major) + "." + std::to_string(p.minor);
    desc_.global_memory_bytes = capacity ? capacity : std::uint64_t(p.totalGlobalMem);
    desc_.base_alignment_bytes = 256;
    desc_.supports_source_kernels = nvrtc::available();
}

void CudaBackend::ensure() const {
    if (ready_.load(std::memory_order_acquire)) return;
    std::lock_guard lk(init_mu_);
    if (ready_.load(std::memory_order_relaxed)) return;
    auto* self = const_cast<CudaBackend*>(this);
    ck(cudaSetDevice(ordinal_), "cudaSetDevice");
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, ordinal_) == cudaSuccess) {
        std::uint64_t keep = ~std::uint64_t(0);
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    } else {
        cudaGetLastError();
    }
    ck(cudaStreamCreateWithFlags(&self->compute_, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&self->h2d_, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&self->d2h_, cudaStreamNonBlocking), "cudaStreamCreate");
    self->ring_size_ = 1u << 20;
    ck(cudaHostAlloc(reinterpret_cast<void**>(&self->ring_host_), ring_size_, cudaHostAllocDefault), "cudaHostAlloc");
    ck(cudaMalloc(reinterpret_cast<void**>(&self->ring_dev_), ring_size_), "cudaMalloc");
    ready_.store(true, std::memory_order_release);
}

CudaBackend::~CudaBackend() {
    if (!ready_.load()) return;
    cudaSetDevice(ordinal_);
    cudaStreamSynchronize(compute_);
    for (auto& [id, b] : bufs_) cudaFreeAsync(b.ptr, compute_);
    cudaStreamSynchronize(compute_);
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, ordinal_) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    cudaFree(ring_dev_);
    cudaFreeHost(ring_host_);
    cudaStreamDestroy(compute_);
    cudaStreamDestroy(h2d_);
    cudaStreamDestroy(d2h_);
    for (cudaLibrary_t l : jit_libs_) cudaLibraryUnload(l);
    fused_.reset();
    stager_.reset();
}

void CudaBackend::make_current() const {
    ensure();
    ck(cudaSetDevice(ordinal_), "cudaSetDevice");
}

const CudaBackend::Buf& CudaBackend::lookup(BufferId id) const {
    auto it = bufs_.find(id);
    if (it == bufs_.end()) throw UnknownHandle("unknown buffer " + std::to_string(id));
    return it->second;
}

BufferId CudaBackend::allocate(std::uint64_t bytes) {
    std::lock_guard lk(mu_);
    if (capacity_ && (bytes > capacity_ || used_ > capacity_ - bytes))
        throw AllocationFailure("allocation of " + std::to_string(bytes) + " bytes exceeds device capacity (" +
                                std::to_string(capacity_ - used_) + " of " + std::to_string(capacity_) +
                                " bytes free)");
    make_current();
    // stream-ordered allocation from the device pool (kept warm: the release
    // threshold is unlimited), so register/release cycles do not pay a
    // cudaMalloc/cudaFree (and its device-wide sync) each time
    void* p = nullptr;
    const cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 1, compute_);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw AllocationFailure("cudaMallocAsync of " + std::to_string(bytes) + " bytes failed: " +
                                cudaGetErrorString(e));
    }
    // zero-filled like the reference's buffers (backend.cpp:137-141), in queue order
    ck(cudaMemsetAsync(p, 0, bytes ? bytes : 1, compute_), "cudaMemsetAsync");
    note_work();
    const BufferId id = next_++;
    bufs_.emplace(id, Buf{p, bytes});
    used_ += bytes;
    return id;
}

void CudaBackend::release(BufferId id) {
    std::lock_guard lk(mu_);
    auto it = bufs_.find(id);
    if (it == bufs_.end()) throw UnknownHandle("release of unknown buffer " + std::to_string(id));
    make_current();
    // stream-ordered: in-flight work on the compute stream finishes first
    cudaFreeAsync(it->second.ptr, compute_);
    note_work();
    shadow_.erase(id);
    device_written_.erase(id);
    used_ -= it->second.size;
    bufs_.erase(it);
}

// Transfers of at least this many bytes from/to pageable memory go through
// the pinned staging ring (host_stager.hpp); smaller ones and page-locked
// buffers use a direct cudaMemcpyAsync.
constexpr std::size_t kStageMin = std::size_t(4) << 20;

detail::HostStager& CudaBackend::stager() const {
    if (!stager_) {
        // experiment knobs: HETRECO_STAGER_SLOT_MB (16), HETRECO_STAGER_SLOTS (3)
        const char* mb = std::getenv("HETRECO_STAGER_SLOT_MB");
        const char* k = std::getenv("HETRECO_STAGER_SLOTS");
        const std::size_t slot = std::size_t(mb && *mb ? std::max(1, std::atoi(mb)) : 16) << 20;
        stager_ = std::make_unique<detail::HostStager>(ordinal_, slot, k && *k ? std::max(2, std::atoi(k)) : 3);
    }
    return *stager_;
}

void CudaBackend::upload(BufferId id, std::uint64_t off, std::span<const std::byte> bytes) {
    std::lock_guard lk(mu_);
    const Buf& b = lookup(id);
    check_window("upload", off, bytes.size(), b.size);
    if (bytes.empty()) return;
    constexpr std::uint64_t kShadowMax = 4096;  // layout headers are (1 + 11 A) * 8 bytes
    if (b.size <= kShadowMax) {
        const bool whole = off == 0 && bytes.size() == b.size;
        auto it = shadow_.find(id);
        if (it == shadow_.end() && (whole || !device_written_.count(id)))
            it = shadow_.emplace(id, std::vector<std::byte>(b.size)).first;  // fresh buffers are zero-filled
        if (it != shadow_.end()) std::memcpy(it->second.data() + off, bytes.data(), bytes.size());
    }
    make_current();
    note_work();
    if (bytes.size() >= kStageMin && !detail::HostStager::is_pinned(bytes.data())) {
        try {
            stager().upload(static_cast<char*>(b.ptr) + off, bytes.data(), bytes.size(), compute_);
        } catch (const DeviceError& e) {
            throw DeviceError(last_kernel_.empty() ? "<upload>" : last_kernel_, e.what());
        }
        return;
    }
    ck(cudaMemcpyAsync(static_cast<char*>(b.ptr) + off, bytes.data(), bytes.size(), cudaMemcpyHostToDevice,
                       compute_),
       "cudaMemcpyAsync(H2D)");
    const cudaError_t e = cudaStreamSynchronize(compute_);  // host span is borrowed
    if (e != cudaSuccess) throw DeviceError(last_kernel_.empty() ? "<upload>" : last_kernel_, cudaGetErrorString(e));
}

void CudaBackend::download(BufferId id, std::uint64_t off, std::span<std::byte> into) const {
    std::lock_guard lk(mu_);
    const Buf& b = lookup(id);
    check_window("download", off, into.size(), b.size);
    if (into.empty()) return;
    make_current();
    note_work();
    if (into.size() >= kStageMin && !detail::HostStager::is_pinned(into.data())) {
        try {
            stager().download(into.data(), static_cast<const char*>(b.ptr) + off, into.size(), compute_);
        } catch (const DeviceError& e) {
            throw DeviceError(last_kernel_.empty() ? "<download>" : last_kernel_, e.what());
        }
        return;
    }
    ck(cudaMemcpyAsync(into.data(), static_cast<const char*>(b.ptr) + off, into.size(), cudaMemcpyDeviceToHost,
                       compute_),
       "cudaMemcpyAsync(D2H)");
    const cudaError_t e = cudaStreamSynchronize(compute_);
    if (e != cudaSuccess) throw DeviceError(last_kernel_.empty() ? "<download>" : last_kernel_, cudaGetErrorString(e));
}

void CudaBackend::copy(BufferId src, std::uint64_t so, BufferId dst, std::uint64_t doff, std::uint64_t n) {
    std::lock_guard lk(mu_);
    const Buf& s = lookup(src);
    const Buf& d = lookup(dst);
    check_window("copy source", so, n, s.size);
    check_window("copy destination", doff, n, d.size);
    if (src == dst && so < doff + n && doff < so + n)
        throw InvalidArgument("overlapping copy within buffer " + std::to_string(src));
    if (n == 0) return;
    make_current();
    note_work();
    shadow_.erase(dst);
    device_written_.insert(dst);
    ck(cudaMemcpyAsync(static_cast<char*>(d.ptr) + doff, static_cast<const char*>(s.ptr) + so, n,
                       cudaMemcpyDeviceToDevice, compute_),
       "cudaMemcpyAsync(D2D)");
}

std::vector<CompiledKernel> CudaBackend::intrinsic_kernels() {
    std::vector<CompiledKernel> ks;
    for (int i = 0; i < intrinsic_kernel_count(); ++i) {
        const char* n = intrinsic_kernel_name(i);
        ks.push_back({n, std::string("sm_100a:") + n, &device_only_entry});
    }
    return ks;
}

int intrinsic_kernel_count() { return int(dev::Builtin::Count) + 2; }

const char* intrinsic_kernel_name(int i) {
    if (i >= 0 && i < int(dev::Builtin::Count)) return dev::builtin_name(dev::Builtin(i));
    if (i == int(dev::Builtin::Count)) return detail::FusedReconKernels::kSense;
    if (i == int(dev::Builtin::Count) + 1) return detail::FusedReconKernels::kRss;
    return nullptr;
}

LayoutDescriptor CudaBackend::header_layout(BufferId header) const {
    auto it = shadow_.find(header);
    if (it != shadow_.end()) return parse_layout_header(it->second);
    const Buf& b = lookup(header);  // not uploaded whole from the host: read it back
    std::vector<std::byte> bytes(b.size);
    ck(cudaMemcpyAsync(bytes.data(), b.ptr, b.size, cudaMemcpyDeviceToHost, compute_), "cudaMemcpyAsync(header)");
    ck(cudaStreamSynchronize(compute_), "cudaStreamSynchronize(header)");
    return parse_layout_header(bytes);
}

bool CudaBackend::supports_source_kernels() const { return nvrtc::available(); }

// Kernel-source units -> NVRTC sm_100a cubins -> loaded libraries.  All units
// compile before any loads (a failure anywhere throws CompileError carrying
// every failing unit's log, and nothing is registered: the registry's
// all-or-nothing rule, kernels.hpp:27-32).
std::vector<CompiledKernel> CudaBackend::compile(std::span<const ProgramSource> units) {
    if (!nvrtc::available())
        throw UnsupportedSource("backend '" + id_ + "': NVRTC is not available, kernel source cannot be compiled");
    std::vector<nvrtc::Unit> built;
    std::vector<BuildDiagnostic> failures;
    for (const ProgramSource& u : units) {
        try {
            built.push_back(nvrtc::compile(u.unit_name, u.source_text, "sm_100a"));
        } catch (const CompileError& e) {
            for (const auto& d : e.diagnostics()) failures.push_back(d);
        }
    }
    if (!failures.empty()) throw CompileError(std::move(failures));
    std::lock_guard lk(mu_);
    make_current();
    std::vector<CompiledKernel> out;
    for (const nvrtc::Unit& u : built) {
        cudaLibrary_t lib = nullptr;
        cudaError_t e = cudaLibraryLoadData(&lib, u.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw CompileError({{u.unit_name, std::string("cubin load failed: ") + cudaGetErrorString(e)}});
        }
        jit_libs_.push_back(lib);
        const std::string tag = "nvrtc#" + std::to_string(++jit_units_) + ":" + u.unit_name;
        for (const std::string& name : u.kernels) {
            cudaKernel_t k = nullptr;
            e = cudaLibraryGetKernel(&k, lib, ("hetreco_entry_" + name).c_str());
            if (e != cudaSuccess) {
                cudaGetLastError();
                throw CompileError({{u.unit_name, "entry point for kernel '" + name + "' missing from the cubin"}});
            }
            jit_[tag + "/" + name] = k;
            out.push_back({name, tag, &device_only_entry});
        }
    }
    return out;
}

void* CudaBackend::stage_params(std::span<const std::byte> params) {
    const std::uint64_t need = std::max<std::uint64_t>(256, (params.size() + 255) & ~std::uint64_t(255));
    if (need > ring_size_) {
        ck(cudaStreamSynchronize(compute_), "cudaStreamSynchronize");
        cudaFree(ring_dev_);
        cudaFreeHost(ring_host_);
        ring_size_ = need * 2;
        ck(cudaHostAlloc(reinterpret_cast<void**>(&ring_host_), ring_size_, cudaHostAllocDefault), "cudaHostAlloc");
        ck(cudaMalloc(reinterpret_cast<void**>(&ring_dev_), ring_size_), "cudaMalloc");
        ring_head_ = 0;
    }
    if (ring_head_ + need > ring_size_) {
        // every earlier staging copy is consumed once the queue drains
        ck(cudaStreamSynchronize(compute_), "cudaStreamSynchronize");
        ring_head_ = 0;
    }
    std::byte* h = ring_host_ + ring_head_;
    std::byte* d = ring_dev_ + ring_head_;
    if (!params.empty()) std::memcpy(h, params.data(), params.size());
    ck(cudaMemcpyAsync(d, h, need, cudaMemcpyHostToDevice, compute_), "cudaMemcpyAsync(params)");
    ring_head_ += need;
    return d;
}

void CudaBackend::execute(const CompiledKernel& kernel, const KernelBinding& bind, std::uint64_t gsize) {
    std::lock_guard lk(mu_);
    // kernels write their output data buffer (the ABI hands them const headers)
    shadow_.erase(bind.output);
    device_written_.insert(bind.output);
    cudaKernel_t jit = nullptr;
    if (kernel.unit_name.rfind("nvrtc#", 0) == 0) {
        auto it = jit_.find(kernel.unit_name + "/" + kernel.name);
        if (it == jit_.end()) throw DeviceError(kernel.name, "kernel was compiled by another backend");
        jit = it->second;
    }
    if (!jit && detail::FusedReconKernels::is_fused(kernel.name)) {
        // fused IFFT2 + coil combine (fused_recon.hpp): shapes from the headers
        const Buf& in = lookup(bind.input);
        const Buf& out = lookup(bind.output);
        const LayoutDescriptor li = header_layout(bind.input_header);
        const LayoutDescriptor lo = header_layout(bind.output_header);
        for (const LayoutRecord& r : li.records) check_window("sens/rss_recon input array", r.offset_bytes, r.byte_size(), in.size);
        for (const LayoutRecord& r : lo.records) check_window("sens/rss_recon output array", r.offset_bytes, r.byte_size(), out.size);
        make_current();
        if (!fused_) fused_ = std::make_unique<detail::FusedReconKernels>(ordinal_);
        last_kernel_ = kernel.name;
        note_work();
        fused_->launch(kernel.name, li, lo, in.ptr, out.ptr, bind.params, gsize, compute_);
        return;
    }
    const int which = jit ? -1 : dev::builtin_from_name(kernel.name.c_str());
    if (!jit && which < 0) throw DeviceError(kernel.name, "no sm_100a implementation registered under this name");
    hetreco_kernel_args args{};
    args.in = lookup(bind.input).ptr;
    args.in_layout = static_cast<const std::uint64_t*>(lookup(bind.input_header).ptr);
    args.out = lookup(bind.output).ptr;
    args.out_layout = static_cast<const std::uint64_t*>(lookup(bind.output_header).ptr);
    make_current();
    args.params = stage_params(bind.params);
    args.params_size = bind.params.size();
    last_kernel_ = kernel.name;
    note_work();
    cudaError_t e;
    if (jit) {
        // grid-stride entry: enough CTAs to fill the GPU, never more than needed
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ordinal_);
        const std::uint64_t blocks = std::min<std::uint64_t>((gsize + 255) / 256, std::uint64_t(sms) * 16);
        void* kargs[] = {&args, &gsize};
        e = cudaLaunchKernel(reinterpret_cast<const void*>(jit), dim3(unsigned(blocks ? blocks : 1)), dim3(256), kargs, 0,
                             compute_);
    } else {
        e = dev::launch_builtin(dev::Builtin(which), args, gsize, compute_);
    }
    if (e != cudaSuccess) throw DeviceError(kernel.name, cudaGetErrorString(e));
}

void CudaBackend::synchronize() {
    make_current();
    const cudaError_t e = cudaStreamSynchronize(compute_);
    if (e != cudaSuccess) throw DeviceError(last_kernel_.empty() ? "<none>" : last_kernel_, cudaGetErrorString(e));
}

void CudaBackend::check(const char* what) const {
    ensure();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamQuery(compute_);
    if (e != cudaSuccess && e != cudaErrorNotReady) throw DeviceError(what, cudaGetErrorString(e));
}

void* CudaBackend::device_pointer(BufferId id) const {
    std::lock_guard lk(mu_);
    void* p = lookup(id).ptr;
    device_written_.insert(id);  // raw device access may write (process outputs)
    return p;
}

std::uint64_t CudaBackend::buffer_size(BufferId id) const {
    std::lock_guard lk(mu_);
    return lookup(id).size;
}

std::uint64_t CudaBackend::live_bytes() const {
    std::lock_guard lk(mu_);
    return used_;
}

// ---- backend list ----------------------------------------------------------------------

namespace {

// Backends live for the process lifetime (backend.hpp:81-85).  They are
// intentionally never destroyed: at exit the CUDA runtime tears itself down
// and stream/memory releases from static destructors would race with it.
std::vector<CudaBackend*>& owned() {
    static std::vector<CudaBackend*>* list = [] {
        auto* v = new std::vector<CudaBackend*>;
        const int n = cuda_device_count();
        for (int i = 0; i < n; ++i) v->push_back(new CudaBackend(i));
        return v;
    }();
    return *list;
}

}  // namespace

std::span<Backend* const> backend_snapshot() {
    static const std::vector<Backend*> ptrs = [] {
        std::vector<Backend*> v;
        for (CudaBackend* b : owned()) v.push_back(b);
        return v;
    }();
    return ptrs;
}

Backend& backend_by_id(std::string_view id) {
    std::string known;
    for (Backend* b : backend_snapshot()) {
        if (b->id() == id) return *b;
        known += (known.empty() ? "" : ", ") + std::string(b->id());
    }
    throw InvalidArgument("unknown backend '" + std::string(id) + "'; known backends: " +
                          (known.empty() ? "(none)" : known));
}

// ---- kernel registry (kernels.cpp:8-50 semantics) ------------------------------------------

void KernelRegistry::add(std::vector<CompiledKernel> ks) {
    std::set<std::string> batch;
    for (const CompiledKernel& k : ks) {
        if (k.name.empty()) throw InvalidArgument("kernel with empty name in unit '" + k.unit_name + "'");
        if (!k.fn) throw InvalidArgument("kernel '" + k.name + "' has no entry point");
        if (!batch.insert(k.name).second)
            throw DuplicateKernel("kernel '" + k.name + "' appears twice in one batch (unit '" + k.unit_name + "')");
        if (auto it = table_.find(k.name); it != table_.end())
            throw DuplicateKernel("kernel '" + k.name + "' from unit '" + k.unit_name +
                                  "' is already registered (unit '" + it->second.unit_name + "')");
    }
    for (CompiledKernel& k : ks) {
        std::string key = k.name;
        table_.emplace(std::move(key), std::move(k));
    }
}

const CompiledKernel& KernelRegistry::find(std::string_view name) const {
    if (auto it = table_.find(name); it != table_.end()) return it->second;
    std::string msg = "unknown kernel '" + std::string(name) + "'; registered:";
    if (table_.empty()) msg += " (none)";
    for (const auto& [k, v] : table_) msg += " " + k;
    throw UnknownKernel(msg);
}

bool KernelRegistry::contains(std::string_view name) const { return table_.find(name) != table_.end(); }

std::vector<std::string> KernelRegistry::names() const {
    std::vector<std::string> v;
    for (const auto& [k, x] : table_) v.push_back(k);
    return v;
}

std::span<const ProgramSource> builtin_kernel_sources() {
    // The builtins ship as precompiled sm_100a code (no source text to JIT);
    // the units are listed by name so callers can enumerate them.
    static const std::vector<ProgramSource> units = [] {
        std::vector<ProgramSource> v;
        for (int i = 0; i < int(dev::Builtin::Count); ++i) {
            const std::string n = dev::builtin_name(dev::Builtin(i));
            v.push_back({n + ".cu", "// precompiled sm_100a builtin '" + n + "'"});
        }
        return v;
    }();
    return units;
}

}  // namespace hetreco
