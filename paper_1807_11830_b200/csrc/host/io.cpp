// io.cpp -- MAT-file Level 5, PGM/PPM and raw+sidecar readers/writers
// (SPEC.md io module, :470-533).  The reference repository
// specifies these formats but ships no implementation, so this file follows
// the public byte-level layouts:
//
//   MAT v5: 128-byte header (116 text + 8 subsystem offset + u16 version
//   0x0100 + "IM" endian tag), then data elements, each an 8-byte tag (u32
//   type, u32 byte count) or a 4-byte "small element" tag (u16 count in the
//   high half), payload padded to 8 bytes.  A variable is one miMATRIX
//   element holding: array flags (miUINT32 x2: class | flag bits, nzmax),
//   dimensions (miINT32), name (miINT8), real part, optional imaginary part.
//
// Complex data is stored split (real block, imaginary block) in the file and
// interleaved in a COMPLEX64/COMPLEX128 NDArray; everything else is a
// straight column-major copy, so a k-space variable lands in (pinned) host
// memory with one pass over the bytes.
#include "hetreco_b200/io.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>

namespace hetreco::io {

namespace {

// data element types (miXXX) and array classes (mxXXX_CLASS)
enum : std::uint32_t {
    miINT8 = 1, miUINT8 = 2, miINT16 = 3, miUINT16 = 4, miINT32 = 5, miUINT32 = 6, miSINGLE = 7, miDOUBLE = 9,
    miINT64 = 12, miUINT64 = 13, miMATRIX = 14, miCOMPRESSED = 15, miUTF8 = 16, miUTF16 = 17, miUTF32 = 18,
};
enum : std::uint32_t {
    mxCELL = 1, mxSTRUCT = 2, mxOBJECT = 3, mxCHAR = 4, mxSPARSE = 5, mxDOUBLE = 6, mxSINGLE = 7, mxINT8 = 8,
    mxUINT8 = 9, mxINT16 = 10, mxUINT16 = 11, mxINT32 = 12, mxUINT32 = 13, mxINT64 = 14, mxUINT64 = 15,
};
constexpr std::uint32_t kFlagComplex = 0x0800;

std::size_t mi_size(std::uint32_t t) {
    switch (t) {
        case miINT8: case miUINT8: return 1;
        case miINT16: case miUINT16: return 2;
        case miINT32: case miUINT32: case miSINGLE: return 4;
        case miDOUBLE: case miINT64: case miUINT64: return 8;
        default: return 0;
    }
}

const char* class_name(std::uint32_t c) {
    switch (c) {
        case mxCELL: return "cell";
        case mxSTRUCT: return "struct";
        case mxOBJECT: return "object";
        case mxCHAR: return "char";
        case mxSPARSE: return "sparse";
        case mxINT8: return "int8";
        case mxINT16: return "int16";
        case mxUINT16: return "uint16";
        case mxUINT32: return "uint32";
        case mxINT64: return "int64";
        case mxUINT64: return "uint64";
        default: return "unknown class";
    }
}

std::uint32_t rd32(const std::byte* p) {
    std::uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}

struct Element {
    std::uint32_t type = 0;
    const std::byte* data = nullptr;
    std::size_t size = 0;
};

// Bounds-checked cursor over a byte range.
class Cursor {
public:
    Cursor(const std::byte* p, std::size_t n) : p_(p), end_(p + n) {}
    bool done() const { return p_ >= end_; }
    std::size_t left() const { return std::size_t(end_ - p_); }
    Element next(const char* what) {
        if (left() < 8) throw MalformedFile(std::string("truncated data element tag (") + what + ")");
        const std::uint32_t w0 = rd32(p_);
        Element e;
        if (w0 >> 16) {  // small data element: 4-byte tag, <= 4 payload bytes
            e.type = w0 & 0xffff;
            e.size = w0 >> 16;
            if (e.size > 4) throw MalformedFile(std::string("small data element longer than 4 bytes (") + what + ")");
            e.data = p_ + 4;
            p_ += 8;
            return e;
        }
        e.type = w0;
        const std::uint64_t n = rd32(p_ + 4);
        p_ += 8;
        if (n > left()) throw MalformedFile(std::string("data element overruns the file (") + what + ")");
        e.data = p_;
        e.size = std::size_t(n);
        const std::uint64_t padded = e.type == miCOMPRESSED ? n : (n + 7) & ~std::uint64_t(7);
        p_ += std::min<std::uint64_t>(padded, left());
        return e;
    }

private:
    const std::byte* p_;
    const std::byte* end_;
};

// Converts `count` stored values of storage type `mi` to the class's
// element type (T) at dst with stride `stride` (elements of T).
template <class T>
void widen(const Element& e, std::uint64_t count, T* dst, std::size_t stride, const char* part) {
    const std::size_t es = mi_size(e.type);
    if (es == 0) throw MalformedFile(std::string("unsupported storage type ") + std::to_string(e.type) + " for " + part);
    if (e.size != count * es)
        throw MalformedFile(std::string(part) + " holds " + std::to_string(e.size) + " bytes, dimensions require " +
                            std::to_string(count * es));
    auto conv = [&](auto tag) {
        using S = decltype(tag);
        if constexpr (std::is_same_v<S, T>) {
            if (stride == 1) {
                std::memcpy(dst, e.data, count * sizeof(T));
                return;
            }
        }
        for (std::uint64_t i = 0; i < count; ++i) {
            S v;
            std::memcpy(&v, e.data + i * sizeof(S), sizeof(S));
            dst[i * stride] = static_cast<T>(v);
        }
    };
    switch (e.type) {
        case miINT8: conv(std::int8_t{}); break;
        case miUINT8: conv(std::uint8_t{}); break;
        case miINT16: conv(std::int16_t{}); break;
        case miUINT16: conv(std::uint16_t{}); break;
        case miINT32: conv(std::int32_t{}); break;
        case miUINT32: conv(std::uint32_t{}); break;
        case miSINGLE: conv(float{}); break;
        case miDOUBLE: conv(double{}); break;
        case miINT64: conv(std::int64_t{}); break;
        case miUINT64: conv(std::uint64_t{}); break;
        default: throw MalformedFile("bad storage type");
    }
}

MatVariable parse_matrix(const std::byte* p, std::size_t n, HostMemory memory) {
    Cursor c(p, n);
    const Element flags = c.next("array flags");
    if (flags.type != miUINT32 || flags.size != 8) throw MalformedFile("array flags sub-element must be 2 x miUINT32");
    const std::uint32_t fw = rd32(flags.data);
    const std::uint32_t cls = fw & 0xff;
    const bool cplx = (fw & kFlagComplex) != 0;
    if (cls == mxCELL || cls == mxSTRUCT || cls == mxOBJECT || cls == mxSPARSE || cls == mxCHAR)
        throw UnsupportedFeature(class_name(cls));
    const Element dim = c.next("dimensions");
    if (dim.type != miINT32 || dim.size % 4 || dim.size < 8) throw MalformedFile("dimensions sub-element must be >= 2 x miINT32");
    std::vector<std::uint64_t> dims;
    std::uint64_t count = 1;
    for (std::size_t i = 0; i < dim.size / 4; ++i) {
        const std::int32_t d = std::int32_t(rd32(dim.data + 4 * i));
        if (d < 0) throw MalformedFile("negative dimension");
        if (d == 0) throw UnsupportedFeature("empty array");
        dims.push_back(std::uint64_t(d));
        if (__builtin_mul_overflow(count, std::uint64_t(d), &count)) throw MalformedFile("dimension product overflows");
    }
    // trailing singleton dimensions beyond rank 8 cannot be represented
    while (dims.size() > kMaxRank && dims.back() == 1) dims.pop_back();
    if (dims.size() > kMaxRank) throw UnsupportedFeature("rank > 8");
    const Element name = c.next("array name");
    if (name.type != miINT8 && name.type != miUINT8 && name.type != miUTF8) throw MalformedFile("array name must be miINT8");
    MatVariable v{std::string(reinterpret_cast<const char*>(name.data), name.size), NDArray(ElementType::UInt8, {1})};
    ElementType et;
    switch (cls) {
        case mxDOUBLE: et = cplx ? ElementType::Complex128 : ElementType::Float64; break;
        case mxSINGLE: et = cplx ? ElementType::Complex64 : ElementType::Float32; break;
        case mxUINT8: et = ElementType::UInt8; break;
        case mxINT32: et = ElementType::Int32; break;
        default: throw UnsupportedFeature(class_name(cls));
    }
    if (cplx && (cls == mxUINT8 || cls == mxINT32)) throw UnsupportedFeature(std::string("complex ") + (cls == mxUINT8 ? "uint8" : "int32"));
    const Element re = c.next("real part");
    if (re.type == miCOMPRESSED) throw UnsupportedFeature("compression");
    Element im;
    const bool is_cplx = et == ElementType::Complex64 || et == ElementType::Complex128;
    if (is_cplx) im = c.next("imaginary part");
    // validate the stored sizes before allocating (a corrupt header must not
    // trigger a huge allocation)
    for (const Element* e : {&re, is_cplx ? &im : &re}) {
        const std::size_t es = mi_size(e->type);
        if (es == 0) throw MalformedFile("unsupported storage type " + std::to_string(e->type));
        if (count > e->size / es || count * es != e->size)
            throw MalformedFile("data block holds " + std::to_string(e->size) + " bytes, dimensions require " +
                                std::to_string(count) + " elements");
    }
    NDArray a(et, dims, memory);
    std::byte* out = a.bytes().data();
    switch (et) {
        case ElementType::Float64: widen(re, count, reinterpret_cast<double*>(out), 1, "real part"); break;
        case ElementType::Float32: widen(re, count, reinterpret_cast<float*>(out), 1, "real part"); break;
        case ElementType::UInt8: widen(re, count, reinterpret_cast<std::uint8_t*>(out), 1, "real part"); break;
        case ElementType::Int32: widen(re, count, reinterpret_cast<std::int32_t*>(out), 1, "real part"); break;
        case ElementType::Complex64:
        case ElementType::Complex128: {
            if (et == ElementType::Complex64) {
                widen(re, count, reinterpret_cast<float*>(out), 2, "real part");
                widen(im, count, reinterpret_cast<float*>(out) + 1, 2, "imaginary part");
            } else {
                widen(re, count, reinterpret_cast<double*>(out), 2, "real part");
                widen(im, count, reinterpret_cast<double*>(out) + 1, 2, "imaginary part");
            }
            break;
        }
    }
    v.array = std::move(a);
    return v;
}

void append(std::vector<std::byte>& b, const void* p, std::size_t n) {
    const std::byte* s = static_cast<const std::byte*>(p);
    b.insert(b.end(), s, s + n);
}
void pad8(std::vector<std::byte>& b) { b.resize((b.size() + 7) & ~std::size_t(7), std::byte{0}); }
void tag(std::vector<std::byte>& b, std::uint32_t type, std::uint64_t bytes) {
    if (bytes > std::numeric_limits<std::uint32_t>::max())
        throw InvalidParams("MAT v5 data element larger than 4 GiB (use raw format)");
    const std::uint32_t t[2] = {type, std::uint32_t(bytes)};
    append(b, t, 8);
}

void check_name(const std::string& name) {
    if (name.empty() || name.size() > 63) throw InvalidParams("MAT variable name must be 1..63 bytes, got \"" + name + "\"");
}

std::vector<std::byte> slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open " + path + " for reading");
    f.seekg(0, std::ios::end);
    const std::streamoff n = f.tellg();
    if (n < 0) throw IoError("cannot size " + path);
    f.seekg(0);
    std::vector<std::byte> b(static_cast<std::size_t>(n));
    if (n && !f.read(reinterpret_cast<char*>(b.data()), n)) throw IoError("read failed: " + path);
    return b;
}

void spit(const std::string& path, const void* p, std::size_t n) {
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw IoError("cannot open " + path + " for writing");
    if (n && !f.write(static_cast<const char*>(p), std::streamsize(n))) throw IoError("write failed: " + path);
    f.close();
    if (!f) throw IoError("close failed: " + path);
}

}  // namespace

std::vector<MatVariable> parse_mat(const std::byte* data, std::size_t size, HostMemory memory) {
    if (size < 128) throw MalformedFile("MAT file shorter than its 128-byte header");
    const char e0 = char(data[126]), e1 = char(data[127]);
    if (e0 == 'M' && e1 == 'I') throw UnsupportedFeature("big-endian");
    if (e0 != 'I' || e1 != 'M') throw MalformedFile("missing MAT v5 endian indicator");
    std::uint16_t version;
    std::memcpy(&version, data + 124, 2);
    if (version != 0x0100) throw UnsupportedFeature("MAT version " + std::to_string(version) + " (v7.3/HDF5?)");
    std::vector<MatVariable> out;
    Cursor c(data + 128, size - 128);
    while (!c.done()) {
        if (c.left() < 8) break;  // trailing pad bytes
        const Element e = c.next("variable");
        if (e.type == miCOMPRESSED) throw UnsupportedFeature("compression");
        if (e.type != miMATRIX) throw MalformedFile("top-level element of type " + std::to_string(e.type) + " is not miMATRIX");
        out.push_back(parse_matrix(e.data, e.size, memory));
    }
    return out;
}

std::vector<MatVariable> read_mat(const std::string& path, HostMemory memory) {
    const std::vector<std::byte> b = slurp(path);
    return parse_mat(b.data(), b.size(), memory);
}

std::vector<std::byte> serialize_mat(const std::vector<MatVariable>& variables) {
    std::vector<std::byte> b;
    char hdr[128];
    std::memset(hdr, ' ', 116);
    const char* text = "MATLAB 5.0 MAT-file, created by hetreco";
    std::memcpy(hdr, text, std::strlen(text));
    std::memset(hdr + 116, 0, 8);
    const std::uint16_t version = 0x0100;
    std::memcpy(hdr + 124, &version, 2);
    hdr[126] = 'I';
    hdr[127] = 'M';
    append(b, hdr, 128);
    for (const MatVariable& v : variables) {
        check_name(v.name);
        const NDArray& a = v.array;
        std::uint32_t cls, mi;
        bool cplx = false;
        switch (a.element_type()) {
            case ElementType::UInt8: cls = mxUINT8; mi = miUINT8; break;
            case ElementType::Int32: cls = mxINT32; mi = miINT32; break;
            case ElementType::Float32: cls = mxSINGLE; mi = miSINGLE; break;
            case ElementType::Float64: cls = mxDOUBLE; mi = miDOUBLE; break;
            case ElementType::Complex64: cls = mxSINGLE; mi = miSINGLE; cplx = true; break;
            case ElementType::Complex128: cls = mxDOUBLE; mi = miDOUBLE; cplx = true; break;
            default: throw InvalidParams("unsupported element type for MAT output");
        }
        std::vector<std::int32_t> dims;
        for (auto d : a.dims()) {
            if (d > std::uint64_t(std::numeric_limits<std::int32_t>::max()))
                throw InvalidParams("dimension too large for MAT v5: " + std::to_string(d));
            dims.push_back(std::int32_t(d));
        }
        if (dims.size() == 1) dims.push_back(1);
        const std::uint64_t count = a.element_count();
        const std::size_t es = mi_size(mi);
        std::vector<std::byte> m;
        tag(m, miUINT32, 8);
        const std::uint32_t fl[2] = {cls | (cplx ? kFlagComplex : 0u), 0u};
        append(m, fl, 8);
        tag(m, miINT32, dims.size() * 4);
        append(m, dims.data(), dims.size() * 4);
        pad8(m);
        tag(m, miINT8, v.name.size());
        append(m, v.name.data(), v.name.size());
        pad8(m);
        const std::byte* src = a.bytes().data();
        if (!cplx) {
            tag(m, mi, count * es);
            append(m, src, count * es);
            pad8(m);
        } else {
            for (int part = 0; part < 2; ++part) {
                tag(m, mi, count * es);
                const std::size_t at = m.size();
                m.resize(at + count * es);
                for (std::uint64_t i = 0; i < count; ++i)
                    std::memcpy(m.data() + at + i * es, src + (2 * i + part) * es, es);
                pad8(m);
            }
        }
        tag(b, miMATRIX, m.size());
        append(b, m.data(), m.size());
    }
    return b;
}

void write_mat(const std::string& path, const std::vector<MatVariable>& variables) {
    const std::vector<std::byte> b = serialize_mat(variables);
    spit(path, b.data(), b.size());
}

// ---- PGM / PPM ---------------------------------------------------------------------------

NDArray read_image(const std::string& path, HostMemory memory) {
    const std::vector<std::byte> b = slurp(path);
    std::size_t i = 0;
    auto skip_ws = [&] {
        for (;;) {
            while (i < b.size() && std::isspace(int(b[i]))) ++i;
            if (i < b.size() && char(b[i]) == '#') {
                while (i < b.size() && char(b[i]) != '\n') ++i;
                continue;
            }
            return;
        }
    };
    auto number = [&](const char* what) {
        skip_ws();
        if (i >= b.size() || !std::isdigit(int(b[i]))) throw MalformedFile(std::string("PNM header: missing ") + what);
        std::uint64_t v = 0;
        while (i < b.size() && std::isdigit(int(b[i]))) {
            v = v * 10 + std::uint64_t(char(b[i]) - '0');
            if (v > (1u << 24)) throw MalformedFile(std::string("PNM header: ") + what + " too large");
            ++i;
        }
        return v;
    };
    if (b.size() < 2 || char(b[0]) != 'P') throw MalformedFile("not a PNM file");
    const char kind = char(b[1]);
    if (kind == '2' || kind == '3' || kind == '1' || kind == '4')
        throw UnsupportedFeature(std::string("ASCII/bitmap PNM variant P") + kind);
    if (kind != '5' && kind != '6') throw MalformedFile(std::string("unknown PNM variant P") + kind);
    i = 2;
    const std::uint64_t w = number("width"), h = number("height"), maxval = number("maxval");
    if (w == 0 || h == 0) throw MalformedFile("PNM image with zero size");
    if (maxval != 255) throw UnsupportedFeature("maxval " + std::to_string(maxval) + " (only 255)");
    if (i >= b.size() || !std::isspace(int(b[i]))) throw MalformedFile("PNM header not terminated by whitespace");
    ++i;
    const std::uint64_t ch = kind == '6' ? 3 : 1;
    const std::uint64_t n = w * h * ch;
    if (b.size() - i < n) throw MalformedFile("PNM payload truncated");
    NDArray a(ElementType::UInt8, ch == 1 ? std::vector<std::uint64_t>{w, h} : std::vector<std::uint64_t>{3, w, h},
              memory);
    std::memcpy(a.bytes().data(), b.data() + i, n);
    return a;
}

void write_image(const std::string& path, const NDArray& image) {
    const auto& d = image.dims();
    const bool color = d.size() == 3 && d[0] == 3;
    if (!(d.size() == 2 || color)) throw InvalidParams("image must be [w, h] or [3, w, h]");
    const std::uint64_t w = color ? d[1] : d[0], h = color ? d[2] : d[1];
    std::vector<std::uint8_t> px(image.element_count());
    if (image.element_type() == ElementType::UInt8) {
        std::memcpy(px.data(), image.bytes().data(), px.size());
    } else if (image.element_type() == ElementType::Float32) {
        auto v = image.view<float>();
        for (std::size_t k = 0; k < px.size(); ++k) {
            const float c = std::clamp(v[k], 0.0f, 1.0f);
            px[k] = std::uint8_t(std::lround(double(c) * 255.0));
        }
    } else {
        throw InvalidParams("write_image takes UINT8 or FLOAT32 arrays");
    }
    std::string hdr = std::string(color ? "P6\n" : "P5\n") + std::to_string(w) + " " + std::to_string(h) + "\n255\n";
    std::vector<std::byte> b(hdr.size() + px.size());
    std::memcpy(b.data(), hdr.data(), hdr.size());
    std::memcpy(b.data() + hdr.size(), px.data(), px.size());
    spit(path, b.data(), b.size());
}

// ---- raw + sidecar ---------------------------------------------------------------------------

void write_raw(const std::string& path, const std::string& sidecar_path, const NDArray& array) {
    std::ostringstream s;
    s << "hetreco-raw 1\nelement_type " << std::uint64_t(array.element_type()) << "\nrank " << array.rank() << "\ndims";
    for (auto d : array.dims()) s << ' ' << d;
    s << "\nbyte_order little\n";
    const std::string t = s.str();
    spit(sidecar_path, t.data(), t.size());
    spit(path, array.bytes().data(), array.byte_size());
}

NDArray read_raw(const std::string& path, const std::string& sidecar_path, HostMemory memory) {
    const std::vector<std::byte> sb = slurp(sidecar_path);
    std::istringstream s(std::string(reinterpret_cast<const char*>(sb.data()), sb.size()));
    std::string magic, key, order;
    int ver = 0;
    std::uint64_t code = 0, rank = 0;
    if (!(s >> magic >> ver) || magic != "hetreco-raw" || ver != 1) throw MalformedSidecar("missing 'hetreco-raw 1' line");
    if (!(s >> key >> code) || key != "element_type" || !is_valid_element_type(code))
        throw MalformedSidecar("bad element_type line");
    if (!(s >> key >> rank) || key != "rank" || rank < 1 || rank > kMaxRank)
        throw MalformedSidecar("rank must be 1..8");
    if (!(s >> key) || key != "dims") throw MalformedSidecar("missing dims line");
    std::vector<std::uint64_t> dims(rank);
    for (auto& d : dims)
        if (!(s >> d) || d == 0) throw MalformedSidecar("dims must be rank positive integers");
    if (!(s >> key >> order) || key != "byte_order" || order != "little")
        throw MalformedSidecar("byte_order must be 'little'");
    NDArray a(ElementType(code), dims, memory);
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open " + path + " for reading");
    f.seekg(0, std::ios::end);
    const std::uint64_t n = std::uint64_t(f.tellg());
    if (n != a.byte_size())
        throw SizeMismatch(path + " holds " + std::to_string(n) + " bytes, sidecar describes " +
                           std::to_string(a.byte_size()));
    f.seekg(0);
    if (n && !f.read(reinterpret_cast<char*>(a.bytes().data()), std::streamsize(n))) throw IoError("read failed: " + path);
    return a;
}

}  // namespace hetreco::io
