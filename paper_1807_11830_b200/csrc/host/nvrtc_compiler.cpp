// nvrtc_compiler.cpp -- the source-kernel path: kernel
// units written against the reference's kernel-source API (HETRECO_KERNEL,
// hetreco_array_in, hetreco_param_*, hetreco_cfloat ..., the role the
// reference's cpujit backend plays with the host compiler,
// src/cpujit_backend.cpp:121-177) are compiled at run time by NVRTC into
// sm_100a cubins.
//
// Each HETRECO_KERNEL(name) body becomes a __device__ function called from a
// grid-stride __global__ entry `hetreco_entry_<name>(args, gsize)`, so one
// launch covers the whole index space the reference iterates work item by
// work item.  Compiled with --fmad=false: the reference's arithmetic is
// uncontracted, so source kernels stay bit-exact with it.
//
// libnvrtc is dlopen'ed on first use; without it the backend reports
// supports_source_kernels() == false and load_kernels throws UnsupportedSource.
#include "nvrtc_compiler.hpp"

#include <dlfcn.h>

#include <mutex>
#include <regex>

namespace hetreco::nvrtc {

namespace {

// nvrtc.h signatures (CUDA 12), resolved at run time.
using nvrtcResult = int;
using nvrtcProgram = struct _nvrtcProgram*;
struct Api {
    nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult (*destroy)(nvrtcProgram*);
    nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
    nvrtcResult (*log_size)(nvrtcProgram, std::size_t*);
    nvrtcResult (*log)(nvrtcProgram, char*);
    nvrtcResult (*cubin_size)(nvrtcProgram, std::size_t*);
    nvrtcResult (*cubin)(nvrtcProgram, char*);
    const char* (*error_string)(nvrtcResult);
    void (*version)(int*, int*);
    bool ok = false;
};

const Api& api() {
    static Api a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        for (const char* n : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                              "/usr/local/cuda/lib64/libnvrtc.so"}) {
            h = ::dlopen(n, RTLD_NOW | RTLD_LOCAL);
            if (h) break;
        }
        if (!h) return;
        auto sym = [&](const char* s) { return ::dlsym(h, s); };
        a.create = reinterpret_cast<decltype(a.create)>(sym("nvrtcCreateProgram"));
        a.destroy = reinterpret_cast<decltype(a.destroy)>(sym("nvrtcDestroyProgram"));
        a.compile = reinterpret_cast<decltype(a.compile)>(sym("nvrtcCompileProgram"));
        a.log_size = reinterpret_cast<decltype(a.log_size)>(sym("nvrtcGetProgramLogSize"));
        a.log = reinterpret_cast<decltype(a.log)>(sym("nvrtcGetProgramLog"));
        a.cubin_size = reinterpret_cast<decltype(a.cubin_size)>(sym("nvrtcGetCUBINSize"));
        a.cubin = reinterpret_cast<decltype(a.cubin)>(sym("nvrtcGetCUBIN"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("nvrtcGetErrorString"));
        a.version = reinterpret_cast<decltype(a.version)>(sym("nvrtcVersion"));
        a.ok = a.create && a.destroy && a.compile && a.log_size && a.log && a.cubin_size && a.cubin &&
               a.error_string;
    });
    return a;
}

// The kernel-source API on the device.  Same names and argument meaning as
// the reference's kernel_abi.h helpers; the header decoders follow the wire
// format of include/hetreco_b200/device_abi.h (u64 words [A, {offset, type,
// rank, d0..d7} x A]).
const char* kPreamble = R"PRE(
typedef unsigned char uint8_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
#define HETRECO_UINT8 1
#define HETRECO_INT32 2
#define HETRECO_FLOAT32 3
#define HETRECO_COMPLEX64 4
#define HETRECO_FLOAT64 5
#define HETRECO_COMPLEX128 6
typedef struct hetreco_kernel_args {
    const void* in;
    const uint64_t* in_layout;
    void* out;
    const uint64_t* out_layout;
    const void* params;
    uint64_t params_size;
} hetreco_kernel_args;
#define HETRECO_DEV static __device__ __forceinline__
HETRECO_DEV uint64_t hetreco_element_size(uint64_t t) {
    return t == 1 ? 1 : (t == 2 || t == 3) ? 4 : (t == 4 || t == 5) ? 8 : t == 6 ? 16 : 0;
}
HETRECO_DEV uint64_t hetreco_layout_count(const uint64_t* h) { return h[0]; }
HETRECO_DEV uint64_t hetreco_layout_offset(const uint64_t* h, uint64_t i) { return h[1 + 11 * i]; }
HETRECO_DEV uint64_t hetreco_layout_type(const uint64_t* h, uint64_t i) { return h[2 + 11 * i]; }
HETRECO_DEV uint64_t hetreco_layout_rank(const uint64_t* h, uint64_t i) { return h[3 + 11 * i]; }
HETRECO_DEV uint64_t hetreco_layout_dim(const uint64_t* h, uint64_t i, uint64_t d) { return h[4 + 11 * i + d]; }
HETRECO_DEV uint64_t hetreco_layout_elements(const uint64_t* h, uint64_t i) {
    uint64_t n = 1;
    for (uint64_t d = 0; d < 8; ++d) n *= hetreco_layout_dim(h, i, d);
    return n;
}
HETRECO_DEV const void* hetreco_array_in(const hetreco_kernel_args* a, uint64_t i) {
    return (const char*)a->in + hetreco_layout_offset(a->in_layout, i);
}
HETRECO_DEV void* hetreco_array_out(const hetreco_kernel_args* a, uint64_t i) {
    return (char*)a->out + hetreco_layout_offset(a->out_layout, i);
}
template <class T>
HETRECO_DEV T hetreco_param_(const hetreco_kernel_args* a, uint64_t off) {
    T v;
    unsigned char* d = (unsigned char*)&v;
    const unsigned char* s = (const unsigned char*)a->params + off;
    for (unsigned k = 0; k < sizeof(T); ++k) d[k] = s[k];
    return v;
}
HETRECO_DEV uint32_t hetreco_param_u32(const hetreco_kernel_args* a, uint64_t off) { return hetreco_param_<uint32_t>(a, off); }
HETRECO_DEV uint64_t hetreco_param_u64(const hetreco_kernel_args* a, uint64_t off) { return hetreco_param_<uint64_t>(a, off); }
HETRECO_DEV float hetreco_param_f32(const hetreco_kernel_args* a, uint64_t off) { return hetreco_param_<float>(a, off); }
HETRECO_DEV double hetreco_param_f64(const hetreco_kernel_args* a, uint64_t off) { return hetreco_param_<double>(a, off); }
typedef struct hetreco_cfloat { float re; float im; } hetreco_cfloat;
HETRECO_DEV hetreco_cfloat hetreco_cmake(float re, float im) { hetreco_cfloat c; c.re = re; c.im = im; return c; }
HETRECO_DEV hetreco_cfloat hetreco_cadd(hetreco_cfloat a, hetreco_cfloat b) { return hetreco_cmake(a.re + b.re, a.im + b.im); }
HETRECO_DEV hetreco_cfloat hetreco_csub(hetreco_cfloat a, hetreco_cfloat b) { return hetreco_cmake(a.re - b.re, a.im - b.im); }
HETRECO_DEV hetreco_cfloat hetreco_cmul(hetreco_cfloat a, hetreco_cfloat b) {
    return hetreco_cmake(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
HETRECO_DEV hetreco_cfloat hetreco_conjf(hetreco_cfloat a) { return hetreco_cmake(a.re, -a.im); }
HETRECO_DEV float hetreco_cabs2(hetreco_cfloat a) { return a.re * a.re + a.im * a.im; }
#define HETRECO_KERNEL(kname)                                                                      \
    static __device__ void hetreco_kernel_##kname(const hetreco_kernel_args* args, uint64_t gid,   \
                                                  uint64_t gsize);                                 \
    extern "C" __global__ void hetreco_entry_##kname(hetreco_kernel_args a, uint64_t gsize) {      \
        for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < gsize;               \
             g += (uint64_t)gridDim.x * blockDim.x)                                                 \
            hetreco_kernel_##kname(&a, g, gsize);                                                   \
    }                                                                                              \
    static __device__ void hetreco_kernel_##kname(const hetreco_kernel_args* args, uint64_t gid,   \
                                                  uint64_t gsize)
)PRE";

std::string strip_comments(const std::string& s) {
    std::string o;
    o.reserve(s.size());
    for (std::size_t i = 0; i < s.size();) {
        if (s.compare(i, 2, "//") == 0) {
            while (i < s.size() && s[i] != '\n') ++i;
        } else if (s.compare(i, 2, "/*") == 0) {
            const std::size_t e = s.find("*/", i + 2);
            i = e == std::string::npos ? s.size() : e + 2;
            o += ' ';
        } else if (s[i] == '"') {  // keep string literals intact
            o += s[i++];
            while (i < s.size() && s[i] != '"') {
                if (s[i] == '\\' && i + 1 < s.size()) o += s[i++];
                o += s[i++];
            }
            if (i < s.size()) o += s[i++];
        } else {
            o += s[i++];
        }
    }
    return o;
}

std::string sanitize(std::string n) {
    for (char& c : n)
        if (c == '"' || c == '\\' || c == '\n' || c == '\r') c = '_';
    return n;
}

}  // namespace

bool available() { return api().ok; }

std::string version() {
    if (!api().ok || !api().version) return {};
    int a = 0, b = 0;
    api().version(&a, &b);
    return std::to_string(a) + "." + std::to_string(b);
}

std::vector<std::string> kernel_names(const std::string& source) {
    static const std::regex re(R"(HETRECO_KERNEL\s*\(\s*([A-Za-z_][A-Za-z0-9_]*)\s*\))");
    const std::string s = strip_comments(source);
    std::vector<std::string> v;
    for (auto it = std::sregex_iterator(s.begin(), s.end(), re); it != std::sregex_iterator(); ++it) {
        // skip the macro's own definition if a unit carries one
        const std::size_t at = std::size_t(it->position(0));
        const std::size_t ls = s.rfind('\n', at);
        const std::string line = s.substr(ls == std::string::npos ? 0 : ls + 1, at - (ls == std::string::npos ? 0 : ls + 1));
        if (line.find("#define") != std::string::npos) continue;
        v.push_back((*it)[1].str());
    }
    return v;
}

Unit compile(const std::string& unit_name, const std::string& source, const std::string& arch) {
    const Api& a = api();
    if (!a.ok) throw UnsupportedSource("NVRTC (libnvrtc.so.12) is not available: cannot compile unit '" + unit_name + "'");
    Unit u;
    u.unit_name = unit_name;
    u.kernels = kernel_names(source);
    const std::string text = std::string(kPreamble) + "#line 1 \"" + sanitize(unit_name) + "\"\n" + source + "\n";
    nvrtcProgram prog = nullptr;
    if (a.create(&prog, text.c_str(), unit_name.c_str(), 0, nullptr, nullptr) != 0)
        throw CompileError({{unit_name, "nvrtcCreateProgram failed"}});
    const std::string arch_opt = "--gpu-architecture=" + arch;
    // 177: unused preamble helpers
    const char* opts[] = {arch_opt.c_str(), "--fmad=false", "-default-device", "--diag-suppress=177"};
    const nvrtcResult rc = a.compile(prog, 4, opts);
    std::size_t n = 0;
    a.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) a.log(prog, log.data());
    while (!log.empty() && (log.back() == '\0' || log.back() == '\n')) log.pop_back();
    u.log = log;
    if (rc != 0) {
        a.destroy(&prog);
        if (log.empty()) log = a.error_string(rc);
        throw CompileError({{unit_name, log}});
    }
    std::size_t cb = 0;
    a.cubin_size(prog, &cb);
    u.cubin.resize(cb);
    if (cb) a.cubin(prog, u.cubin.data());
    a.destroy(&prog);
    if (u.kernels.empty()) throw CompileError({{unit_name, "no HETRECO_KERNEL(name) definition in unit"}});
    return u;
}

}  // namespace hetreco::nvrtc
