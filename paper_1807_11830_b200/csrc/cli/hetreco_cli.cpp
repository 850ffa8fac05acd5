// hetreco -- command-line front-end (SPEC.md cli module :535-579; SURVEY.md
// §8 f.3): the paper's §III-C protocol (device setup -> data -> process
// init -> launch -> fetch) over files, plus the §IV benchmark harness.
//
//   hetreco devices [--json]
//   hetreco negate --input in.pgm --output out.pgm [--device F]
//   hetreco gen-phantom [--nx 128 --ny 128 --frames 16 --coils 8 --seed 1]
//                       --out-kdata k.mat --out-smaps s.mat --out-truth t.mat [--device F]
//   hetreco reconstruct --kdata k.mat [--smaps s.mat] --method sens|rss --output o.mat
//                       [--shift] [--device F]
//   hetreco bench --op fft|rss|sens|negate|matadd --sizes L --repeats N [--device F]
//                 [--csv path] [--deterministic-timing]
//   hetreco compile --source unit.cl.src [--source ...]
//
// Built against the exported C-ABI only (include/hetreco_b200.h), like any
// reference-side binding.  Every command exits 0 on success, nonzero with a
// one-line diagnostic on failure.  --device defaults to $HETRECO_DEVICE.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "hetreco_b200.h"

namespace {

struct Fail : std::runtime_error {
    int code;
    Fail(const std::string& m, int c = 1) : std::runtime_error(m), code(c) {}
};

void ck(int rc, const char* what) {
    if (rc != HETRECO_OK) throw Fail(std::string(what) + ": " + hetreco_last_error(), rc);
}

// ---- arguments ------------------------------------------------------------------------------

struct Args {
    std::map<std::string, std::string> kv;
    std::map<std::string, bool> flags;
    bool has(const std::string& k) const { return kv.count(k) || flags.count(k); }
    std::string get(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    std::string need(const std::string& k) const {
        auto it = kv.find(k);
        if (it == kv.end() || it->second.empty()) throw Fail("missing required option --" + k, 2);
        return it->second;
    }
    std::uint64_t num(const std::string& k, std::uint64_t def) const {
        auto it = kv.find(k);
        if (it == kv.end()) return def;
        char* end = nullptr;
        const unsigned long long v = std::strtoull(it->second.c_str(), &end, 10);
        if (!end || *end) throw Fail("--" + k + " expects an integer, got '" + it->second + "'", 2);
        return v;
    }
};

Args parse(int argc, char** argv, const std::vector<std::string>& flag_names) {
    Args a;
    for (int i = 2; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) != 0) throw Fail("unexpected argument '" + s + "'", 2);
        s = s.substr(2);
        const auto eq = s.find('=');
        if (eq != std::string::npos) {
            a.kv[s.substr(0, eq)] = s.substr(eq + 1);
        } else if (std::find(flag_names.begin(), flag_names.end(), s) != flag_names.end()) {
            a.flags[s] = true;
        } else {
            if (i + 1 >= argc) throw Fail("option --" + s + " needs a value", 2);
            a.kv[s] = argv[++i];
        }
    }
    return a;
}

std::string device_filter(const Args& a) {
    if (a.has("device")) return a.get("device");
    const char* e = std::getenv("HETRECO_DEVICE");
    return e ? e : "";
}

// ---- RAII over the C-ABI ---------------------------------------------------------------------

struct Session {
    hetreco_session s = nullptr;
    explicit Session(const std::string& filter) { ck(hetreco_session_create(filter.c_str(), &s), "session"); }
    ~Session() {
        if (s) hetreco_session_destroy(s);
    }
    std::string label() const {
        hetreco_device_desc d{};
        ck(hetreco_session_device(s, &d), "device");
        return std::string(d.backend_id) + ":" + d.name;
    }
};

struct Params {
    hetreco_params p = nullptr;
    Params() { ck(hetreco_params_create(&p), "params"); }
    ~Params() { hetreco_params_destroy(p); }
};

struct Proc {
    hetreco_process p = nullptr;
    Proc(hetreco_session s, const char* kind) { ck(hetreco_process_create(s, kind, kind, &p), kind); }
    ~Proc() { hetreco_process_destroy(p); }
};

struct Mat {
    hetreco_mat m = nullptr;
    ~Mat() {
        if (m) hetreco_mat_free(m);
    }
    int count() const {
        int n = 0;
        ck(hetreco_mat_count(m, &n), "mat");
        return n;
    }
    std::pair<std::string, hetreco_array_desc> var(int i) const {
        char name[128];
        hetreco_array_desc d{};
        ck(hetreco_mat_variable(m, i, name, sizeof name, &d), "mat variable");
        return {name, d};
    }
};

hetreco_array_desc desc(std::uint64_t type, std::vector<std::uint64_t> dims, void* host) {
    hetreco_array_desc d{};
    d.element_type = type;
    d.rank = std::uint32_t(dims.size());
    for (std::size_t i = 0; i < dims.size(); ++i) d.dims[i] = dims[i];
    d.host = host;
    return d;
}

std::uint64_t count_of(const hetreco_array_desc& d) {
    std::uint64_t n = 1;
    for (std::uint32_t i = 0; i < d.rank; ++i) n *= d.dims[i];
    return n;
}

constexpr std::uint64_t U8 = 1, I32 = 2, F32 = 3, C64 = 4, F64 = 5;

// picks a variable: by preferred names, else the first of the wanted type
std::pair<std::string, hetreco_array_desc> pick(const Mat& m, std::uint64_t type, std::vector<std::string> names,
                                                const std::string& file) {
    for (int i = 0; i < m.count(); ++i) {
        auto v = m.var(i);
        for (auto& n : names)
            if (v.first == n && v.second.element_type == type) return v;
    }
    for (int i = 0; i < m.count(); ++i) {
        auto v = m.var(i);
        if (v.second.element_type == type) return v;
    }
    throw Fail(file + ": no COMPLEX64 variable found (save k-space/maps as complex single)", 3);
}

// ---- commands ----------------------------------------------------------------------------------

int cmd_devices(const Args& a) {
    std::vector<hetreco_device_desc> d(64);
    int n = 0;
    ck(hetreco_enumerate_devices(d.data(), int(d.size()), &n), "enumerate_devices");
    if (a.has("json")) {
        std::printf("[");
        for (int i = 0; i < n; ++i)
            std::printf("%s{\"backend_id\": \"%s\", \"type\": \"%s\", \"vendor\": \"%s\", \"name\": \"%s\", "
                        "\"api_version\": \"%s\", \"global_memory_bytes\": %llu, \"base_alignment_bytes\": %llu}",
                        i ? ", " : "", d[i].backend_id, d[i].device_type == 1 ? "GPU" : "CPU", d[i].vendor,
                        d[i].name, d[i].api_version, (unsigned long long)d[i].global_memory_bytes,
                        (unsigned long long)d[i].base_alignment_bytes);
        std::printf("]\n");
    } else {
        std::printf("%-8s %-4s %-8s %-28s %-6s %12s\n", "backend", "type", "vendor", "name", "cc", "memory_GiB");
        for (int i = 0; i < n; ++i)
            std::printf("%-8s %-4s %-8s %-28s %-6s %12.1f\n", d[i].backend_id, d[i].device_type == 1 ? "GPU" : "CPU",
                        d[i].vendor, d[i].name, d[i].api_version, double(d[i].global_memory_bytes) / (1ull << 30));
        if (n == 0) std::printf("(no CUDA device on this host; the B200 build has no CPU backend)\n");
    }
    return 0;
}

// §III-C steps 0-10 over a PGM image: app/session, load, register, process init, launch, fetch, save.
int cmd_negate(const Args& a) {
    const std::string in = a.need("input"), out = a.need("output");
    Mat img;
    ck(hetreco_image_read(in.c_str(), 1, &img.m), in.c_str());
    auto [name, d] = img.var(0);
    if (d.rank != 2) throw Fail(in + ": negate takes a grayscale (P5) image", 3);
    Session s(device_filter(a));
    hetreco_handle hin{}, hout{};
    ck(hetreco_register_data(s.s, HETRECO_XDATA, 1, &d, &hin), "register_data");
    hetreco_array_desc o = desc(U8, {d.dims[0], d.dims[1]}, nullptr);
    ck(hetreco_allocate_data(s.s, HETRECO_XDATA, 1, &o, &hout), "allocate_data");
    Proc p(s.s, "negate");
    Params prm;
    ck(hetreco_params_set_real(prm.p, "max_value", 255.0), "params");
    ck(hetreco_process_set_input(p.p, hin), "set_input");
    ck(hetreco_process_set_output(p.p, hout), "set_output");
    ck(hetreco_process_init(p.p, prm.p), "init");
    ck(hetreco_process_launch(p.p), "launch");
    std::vector<std::uint8_t> px(count_of(d));
    void* dst[1] = {px.data()};
    ck(hetreco_fetch_data(s.s, hout, 1, dst), "fetch_data");
    hetreco_array_desc w = desc(U8, {d.dims[0], d.dims[1]}, px.data());
    ck(hetreco_image_write(out.c_str(), &w), out.c_str());
    return 0;
}

int cmd_gen_phantom(const Args& a) {
    const std::uint64_t nx = a.num("nx", 128), ny = a.num("ny", 128), nf = a.num("frames", 16),
                        nc = a.num("coils", 8), seed = a.num("seed", 1);
    const std::string ok = a.need("out-kdata"), os_ = a.need("out-smaps"), ot = a.need("out-truth");
    Session s(device_filter(a));
    std::vector<std::complex<float>> Y(nx * ny * nc * nf), S(nx * ny * nc), M(nx * ny * nf);
    ck(hetreco_gen_phantom(s.s, nx, ny, nf, nc, seed, Y.data(), S.data(), M.data()), "gen_phantom");
    auto write1 = [](const std::string& path, const char* name, hetreco_array_desc d) {
        const char* names[1] = {name};
        ck(hetreco_mat_write(path.c_str(), 1, names, &d), path.c_str());
    };
    write1(ok, "kdata", desc(C64, {nx, ny, nc, nf}, Y.data()));
    write1(os_, "smaps", desc(C64, {nx, ny, nc}, S.data()));
    write1(ot, "truth", desc(C64, {nx, ny, nf}, M.data()));
    return 0;
}

int cmd_reconstruct(const Args& a) {
    const std::string method = a.get("method", "sens");
    if (method != "sens" && method != "rss") throw Fail("--method must be sens or rss", 2);
    const std::string kpath = a.need("kdata"), out = a.need("output");
    if (method == "sens" && !a.has("smaps")) throw Fail("--method sens needs --smaps", 2);
    Mat km, sm;
    ck(hetreco_mat_read(kpath.c_str(), 1, &km.m), kpath.c_str());  // pinned: DMA straight from the file buffer
    auto [kn, kd] = pick(km, C64, {"kdata", "Y", "k"}, kpath);
    if (kd.rank < 3) throw Fail(kpath + ": k-space must be [nx, ny, coils(, frames)]", 3);
    const std::uint64_t nx = kd.dims[0], ny = kd.dims[1], nc = kd.dims[2];
    const std::uint64_t nf = count_of(kd) / (nx * ny * nc);
    std::vector<hetreco_array_desc> ins{kd};
    if (method == "sens") {
        const std::string spath = a.get("smaps");
        ck(hetreco_mat_read(spath.c_str(), 1, &sm.m), spath.c_str());
        auto [sn, sd] = pick(sm, C64, {"smaps", "S", "maps"}, spath);
        if (count_of(sd) != nx * ny * nc || sd.dims[0] != nx || sd.dims[1] != ny)
            throw Fail(spath + ": sensitivity maps must be [nx, ny, coils] matching the k-space", 3);
        ins.push_back(sd);
    }
    Session s(device_filter(a));
    hetreco_handle hin{}, hout{};
    ck(hetreco_register_data(s.s, HETRECO_KDATA, int(ins.size()), ins.data(), &hin), "register_data");
    const std::uint64_t ot = method == "sens" ? C64 : F32;
    hetreco_array_desc od = desc(ot, {nx, ny, nf}, nullptr);
    ck(hetreco_allocate_data(s.s, HETRECO_XDATA, 1, &od, &hout), "allocate_data");
    Proc p(s.s, method == "sens" ? "sens_recon" : "rss_recon");
    Params prm;
    if (a.has("shift")) ck(hetreco_params_set_bool(prm.p, "shift", 1), "params");
    ck(hetreco_process_set_input(p.p, hin), "set_input");
    ck(hetreco_process_set_output(p.p, hout), "set_output");
    ck(hetreco_process_init(p.p, prm.p), "init");
    ck(hetreco_process_launch(p.p), "launch");
    std::vector<std::byte> buf(nx * ny * nf * (ot == C64 ? 8 : 4));
    void* dst[1] = {buf.data()};
    ck(hetreco_fetch_data(s.s, hout, 1, dst), "fetch_data");
    hetreco_array_desc w = desc(ot, {nx, ny, nf}, buf.data());
    const char* names[1] = {"image"};
    ck(hetreco_mat_write(out.c_str(), 1, names, &w), out.c_str());
    return 0;
}

// ---- bench ---------------------------------------------------------------

std::vector<std::uint64_t> dims_of(const std::string& size) {
    std::vector<std::uint64_t> d;
    std::stringstream ss(size);
    std::string t;
    while (std::getline(ss, t, 'x')) {
        char* end = nullptr;
        const unsigned long long v = std::strtoull(t.c_str(), &end, 10);
        if (t.empty() || !end || *end || v == 0) throw Fail("bad size '" + size + "'", 2);
        d.push_back(v);
    }
    return d;
}

struct Row {
    std::string op, device, size;
    std::uint64_t repeats;
    double init_s, mean_s, stddev_s, speedup;  // speedup < 0: column empty
};

int cmd_bench(const Args& a) {
    const std::string op = a.need("op");
    const std::uint64_t repeats = a.num("repeats", 100);
    if (repeats < 1) throw Fail("--repeats must be >= 1", 2);
    const bool det = a.has("deterministic-timing");
    std::vector<std::string> sizes;
    {
        std::stringstream ss(a.need("sizes"));
        std::string t;
        while (std::getline(ss, t, ',')) sizes.push_back(t);
    }
    Session s(device_filter(a));
    const std::string dev = s.label();
    std::vector<Row> rows;
    std::uint64_t seed = 12345;
    auto rnd = [&seed]() {  // deterministic LCG inputs
        seed = seed * 6364136223846793005ull + 1442695040888963407ull;
        return float(double(seed >> 11) * (1.0 / 9007199254740992.0)) * 2.0f - 1.0f;
    };
    for (const std::string& size : sizes) {
        const std::vector<std::uint64_t> d = dims_of(size);
        std::vector<hetreco_array_desc> ins;
        std::vector<std::vector<std::byte>> bufs;
        hetreco_array_desc od{};
        const char* kind = nullptr;
        Params prm;
        auto host = [&](std::uint64_t type, std::vector<std::uint64_t> dims) {
            std::uint64_t n = 1;
            for (auto v : dims) n *= v;
            const std::size_t es = type == C64 ? 8 : type == F32 ? 4 : type == U8 ? 1 : 8;
            bufs.emplace_back(n * es);
            auto& b = bufs.back();
            if (type == U8) {
                for (std::size_t i = 0; i < b.size(); ++i) b[i] = std::byte(std::uint8_t(rnd() * 127 + 128));
            } else {
                float* f = reinterpret_cast<float*>(b.data());
                for (std::size_t i = 0; i < b.size() / 4; ++i) f[i] = rnd();
            }
            ins.push_back(desc(type, dims, b.data()));
        };
        if (op == "fft") {
            if (d.size() < 2 || d.size() > 3) throw Fail("fft sizes are NXxNY[xBATCH]", 2);
            host(C64, d);
            od = desc(C64, d, nullptr);
            kind = "fft2d";
            ck(hetreco_params_set_string(prm.p, "direction", "inverse"), "params");
        } else if (op == "rss" || op == "sens") {
            // NXxNYxFRAMESxCOILS (gen_phantom order)
            if (d.size() != 4) throw Fail(op + " sizes are NXxNYxFRAMESxCOILS", 2);
            host(C64, {d[0], d[1], d[3], d[2]});
            if (op == "sens") host(C64, {d[0], d[1], d[3]});
            od = desc(op == "sens" ? C64 : F32, {d[0], d[1], d[2]}, nullptr);
            kind = op == "sens" ? "sens_recon" : "rss_recon";
        } else if (op == "negate") {
            const std::vector<std::uint64_t> nn = d.size() == 1 ? std::vector<std::uint64_t>{d[0], d[0]} : d;
            host(F32, nn);
            od = desc(F32, nn, nullptr);
            kind = "negate";
            ck(hetreco_params_set_real(prm.p, "max_value", 1.0), "params");
        } else if (op == "matadd") {
            const std::vector<std::uint64_t> nn = d.size() == 1 ? std::vector<std::uint64_t>{d[0], d[0]} : d;
            host(F32, nn);
            host(F32, nn);
            od = desc(F32, nn, nullptr);
            kind = "matrix_add";
        } else {
            throw Fail("--op must be fft, rss, sens, negate or matadd", 2);
        }
        hetreco_handle hin{}, hout{};
        ck(hetreco_register_data(s.s, HETRECO_KDATA, int(ins.size()), ins.data(), &hin), "register_data");
        ck(hetreco_allocate_data(s.s, HETRECO_XDATA, 1, &od, &hout), "allocate_data");
        Proc p(s.s, kind);
        ck(hetreco_process_set_input(p.p, hin), "set_input");
        ck(hetreco_process_set_output(p.p, hout), "set_output");
        const auto t0 = std::chrono::steady_clock::now();
        ck(hetreco_process_init(p.p, prm.p), "init");
        ck(hetreco_synchronize(s.s), "synchronize");
        const double init_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::vector<double> t(repeats);
        for (std::uint64_t r = 0; r < repeats; ++r) {  // launch + synchronize, as the paper times (§IV-B)
            const auto a0 = std::chrono::steady_clock::now();
            ck(hetreco_process_launch(p.p), "launch");
            ck(hetreco_synchronize(s.s), "synchronize");
            t[r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - a0).count();
        }
        const double mean = std::accumulate(t.begin(), t.end(), 0.0) / double(repeats);
        double var = 0;
        for (double v : t) var += (v - mean) * (v - mean);
        const double sd = repeats > 1 ? std::sqrt(var / double(repeats - 1)) : 0.0;
        double speedup = -1;
        if (op == "matadd") {
            // single-thread host baseline + bitwise correctness check
            const float* x = reinterpret_cast<const float*>(bufs[0].data());
            const float* y = reinterpret_cast<const float*>(bufs[1].data());
            const std::size_t n = bufs[0].size() / 4;
            std::vector<float> ref(n), got(n);
            double best = 1e30, sum = 0;
            for (std::uint64_t r = 0; r < repeats; ++r) {
                const auto a0 = std::chrono::steady_clock::now();
                for (std::size_t i = 0; i < n; ++i) ref[i] = x[i] + y[i];
                const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - a0).count();
                sum += dt;
                best = std::min(best, dt);
            }
            void* dst[1] = {got.data()};
            ck(hetreco_fetch_data(s.s, hout, 1, dst), "fetch_data");
            if (std::memcmp(ref.data(), got.data(), n * 4) != 0)
                throw Fail("matadd: device result differs from the host baseline", 4);
            speedup = (sum / double(repeats)) / mean;
        }
        ck(hetreco_release_data(s.s, hin), "release");
        ck(hetreco_release_data(s.s, hout), "release");
        if (det) {
            rows.push_back({op, dev, size, repeats, 0, 0, 0, speedup < 0 ? -1.0 : 0.0});
        } else {
            rows.push_back({op, dev, size, repeats, init_s, mean, sd, speedup});
        }
    }
    std::string csv = "op,device,size,repeats,init_s,mean_s,stddev_s,speedup\n";
    for (const Row& r : rows) {
        char line[512];
        std::snprintf(line, sizeof line, "%s,%s,%s,%llu,%.9g,%.9g,%.9g,", r.op.c_str(), r.device.c_str(),
                      r.size.c_str(), (unsigned long long)r.repeats, r.init_s, r.mean_s, r.stddev_s);
        csv += line;
        if (r.speedup >= 0) {
            std::snprintf(line, sizeof line, "%.6g", r.speedup);
            csv += line;
        }
        csv += "\n";
    }
    if (a.has("csv")) {
        FILE* f = std::fopen(a.get("csv").c_str(), "wb");
        if (!f) throw Fail("cannot write " + a.get("csv"), 5);
        std::fwrite(csv.data(), 1, csv.size(), f);
        std::fclose(f);
    } else {
        std::fputs(csv.c_str(), stdout);
    }
    return 0;
}

// Compiles kernel-source units for sm_100a (NVRTC; no device needed) and lists
// their kernels.  A failing unit's compiler log is printed verbatim and the
// command exits nonzero ("error log is immediately available").
int cmd_compile(int argc, char** argv) {
    std::vector<std::string> files;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--source" && i + 1 < argc) {
            files.push_back(argv[++i]);
        } else {
            throw Fail("usage: hetreco compile --source unit.cl.src [--source ...]", 2);
        }
    }
    if (files.empty()) throw Fail("missing required option --source", 2);
    int failed = 0;
    for (const std::string& f : files) {
        FILE* fp = std::fopen(f.c_str(), "rb");
        if (!fp) throw Fail("cannot read " + f, 3);
        std::string src;
        char buf[4096];
        std::size_t n;
        while ((n = std::fread(buf, 1, sizeof buf, fp)) > 0) src.append(buf, n);
        std::fclose(fp);
        std::vector<char> names(8192), log(1 << 20);
        const std::string unit = f.substr(f.find_last_of('/') == std::string::npos ? 0 : f.find_last_of('/') + 1);
        const int rc = hetreco_nvrtc_compile_check(unit.c_str(), src.c_str(), names.data(), names.size(), log.data(),
                                                   log.size());
        if (rc != HETRECO_OK) {
            std::fprintf(stderr, "hetreco compile: %s: %s\n", unit.c_str(), hetreco_last_error());
            ++failed;
            continue;
        }
        std::string ns = names.data();
        for (char& c : ns)
            if (c == '\n') c = ' ';
        std::printf("%s: %s\n", unit.c_str(), ns.c_str());
    }
    return failed ? 4 : 0;
}

void usage() {
    std::fprintf(stderr,
                 "usage: hetreco <command> [options]\n"
                 "  devices [--json]\n"
                 "  negate --input in.pgm --output out.pgm [--device F]\n"
                 "  gen-phantom [--nx --ny --frames --coils --seed] --out-kdata k.mat --out-smaps s.mat "
                 "--out-truth t.mat\n"
                 "  reconstruct --kdata k.mat [--smaps s.mat] --method sens|rss --output o.mat [--shift]\n"
                 "  bench --op fft|rss|sens|negate|matadd --sizes L --repeats N [--csv path] "
                 "[--deterministic-timing]\n"
                 "  compile --source unit.cl.src [--source ...]   (NVRTC, sm_100a)\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "devices") return cmd_devices(parse(argc, argv, {"json"}));
        if (cmd == "negate") return cmd_negate(parse(argc, argv, {}));
        if (cmd == "gen-phantom") return cmd_gen_phantom(parse(argc, argv, {}));
        if (cmd == "reconstruct") return cmd_reconstruct(parse(argc, argv, {"shift"}));
        if (cmd == "bench") return cmd_bench(parse(argc, argv, {"deterministic-timing"}));
        if (cmd == "compile") return cmd_compile(argc, argv);
        if (cmd == "--help" || cmd == "-h" || cmd == "help") {
            usage();
            return 0;
        }
        std::fprintf(stderr, "hetreco: unknown command '%s'\n", cmd.c_str());
        usage();
        return 2;
    } catch (const Fail& e) {
        std::fprintf(stderr, "hetreco %s: %s\n", cmd.c_str(), e.what());
        return e.code ? (e.code > 125 ? 1 : e.code) : 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "hetreco %s: %s\n", cmd.c_str(), e.what());
        return 1;
    }
}
