// data.cpp -- NDArray/Data storage and the packing rules.
// Behaviour follows the reference's src/ndarray.cpp:1-107 and
// src/layout.cpp:57-152 (alignment rounding, overflow checks, the u64 LE
// header words, validation on parse); the code is written for this build.
#include "hetreco_b200/data.hpp"

#include <cuda_runtime.h>

#include <limits>
#include <new>

namespace hetreco {

// ---- element types -------------------------------------------------------------

std::size_t element_size(ElementType t) {
    static constexpr std::size_t sizes[] = {0, 1, 4, 4, 8, 8, 16};
    const auto code = static_cast<std::uint64_t>(t);
    if (!is_valid_element_type(code))
        throw InvalidArgument("unknown element type code " + std::to_string(code));
    return sizes[code];
}

bool is_valid_element_type(std::uint64_t code) { return code >= 1 && code <= 6; }

std::string_view element_type_name(ElementType t) {
    static constexpr std::string_view names[] = {"unknown", "uint8",   "int32",     "float32",
                                                 "complex64", "float64", "complex128"};
    const auto code = static_cast<std::uint64_t>(t);
    return is_valid_element_type(code) ? names[code] : names[0];
}

std::string_view data_kind_name(DataKind k) {
    switch (k) {
        case DataKind::XData: return "xdata";
        case DataKind::KData: return "kdata";
        case DataKind::Generic: return "generic";
    }
    return "unknown";
}

// ---- host storage ----------------------------------------------------------------

void detail::HostFree::operator()(std::byte* p) const {
    if (!p) return;
    if (pinned)
        cudaFreeHost(p);
    else
        ::operator delete[](p, std::align_val_t(256));
}

HostBuffer::HostBuffer(std::size_t bytes, HostMemory kind) : size_(bytes) {
    const std::size_t n = bytes ? bytes : 1;
    std::byte* p = nullptr;
    if (kind == HostMemory::Pinned) {
        void* raw = nullptr;
        if (cudaHostAlloc(&raw, n, cudaHostAllocPortable) == cudaSuccess) {
            p = static_cast<std::byte*>(raw);
            pinned_ = true;
        } else {
            cudaGetLastError();  // no driver here: keep a pageable payload
        }
    }
    if (!p) {
        try {
            p = static_cast<std::byte*>(::operator new[](n, std::align_val_t(256)));
        } catch (const std::bad_alloc&) {
            throw AllocationFailure("host allocation of " + std::to_string(bytes) + " bytes failed");
        }
    }
    std::memset(p, 0, n);
    ptr_ = std::unique_ptr<std::byte, detail::HostFree>(p, detail::HostFree{pinned_});
}

HostBuffer::HostBuffer(const HostBuffer& o)
    : HostBuffer(o.size_, o.pinned_ ? HostMemory::Pinned : HostMemory::Pageable) {
    if (size_) std::memcpy(ptr_.get(), o.ptr_.get(), size_);
}

HostBuffer& HostBuffer::operator=(const HostBuffer& o) {
    if (this != &o) {
        HostBuffer tmp(o);
        *this = std::move(tmp);
    }
    return *this;
}

// ---- NDArray -----------------------------------------------------------------------

namespace {

std::uint64_t count_of(const std::vector<std::uint64_t>& dims) {
    if (dims.empty() || dims.size() > kMaxRank)
        throw InvalidArgument("array rank must be between 1 and " + std::to_string(kMaxRank) +
                              ", got " + std::to_string(dims.size()));
    std::uint64_t n = 1;
    for (auto d : dims) {
        if (d == 0) throw InvalidArgument("array dimensions must be >= 1");
        if (__builtin_mul_overflow(n, d, &n)) throw Overflow("element count overflows 64 bits");
    }
    return n;
}

std::uint64_t bytes_of(std::uint64_t count, ElementType t) {
    std::uint64_t b = 0;
    if (__builtin_mul_overflow(count, std::uint64_t(element_size(t)), &b))
        throw Overflow("payload byte size overflows 64 bits");
    return b;
}

}  // namespace

NDArray::NDArray(ElementType type, std::vector<std::uint64_t> dims, HostMemory memory)
    : type_(type), dims_(std::move(dims)), count_(count_of(dims_)),
      storage_(bytes_of(count_, type_), memory) {}

NDArray::NDArray(ElementType type, std::vector<std::uint64_t> dims, std::vector<std::byte> payload)
    : type_(type), dims_(std::move(dims)), count_(count_of(dims_)) {
    const std::uint64_t need = bytes_of(count_, type_);
    if (payload.size() != need)
        throw InvalidArgument("payload is " + std::to_string(payload.size()) +
                              " bytes, shape requires " + std::to_string(need));
    storage_ = HostBuffer(need, HostMemory::Pageable);
    if (need) std::memcpy(storage_.data(), payload.data(), need);
}

bool NDArray::operator==(const NDArray& o) const {
    return type_ == o.type_ && dims_ == o.dims_ && byte_size() == o.byte_size() &&
           std::memcmp(storage_.data(), o.storage_.data(), byte_size()) == 0;
}

void NDArray::require_type(ElementType t) const {
    if (t != type_)
        throw InvalidArgument("typed view of " + std::string(element_type_name(type_)) +
                              " array requested as " + std::string(element_type_name(t)));
}

std::uint64_t Data::payload_byte_size() const {
    std::uint64_t s = 0;
    for (const auto& a : arrays) s += a.byte_size();
    return s;
}

// ---- layout ------------------------------------------------------------------------

std::uint64_t LayoutRecord::element_count() const {
    std::uint64_t n = 1;
    for (std::uint32_t d = 0; d < rank; ++d) n *= dims[d];
    return n;
}

std::uint64_t LayoutRecord::byte_size() const { return element_count() * element_size(element_type); }

namespace {

std::uint64_t align_up(std::uint64_t v, std::uint64_t a) {
    const std::uint64_t r = v % a;
    if (r == 0) return v;
    if (v > std::numeric_limits<std::uint64_t>::max() - (a - r))
        throw Overflow("packed size overflows 64 bits");
    return v + (a - r);
}

constexpr std::size_t kWords = 11;  // words per header record

}  // namespace

LayoutDescriptor pack_shapes(std::span<const ArrayShape> arrays, std::uint64_t alignment) {
    if (arrays.empty()) throw EmptyData("cannot pack a data set with no arrays");
    if (alignment == 0 || (alignment & (alignment - 1)) != 0)
        throw InvalidArgument("alignment must be a power of two, got " + std::to_string(alignment));
    LayoutDescriptor out;
    out.alignment_bytes = alignment;
    std::uint64_t end = 0;
    for (const ArrayShape& a : arrays) {
        LayoutRecord r;
        r.offset_bytes = align_up(end, alignment);
        r.element_type = a.element_type;
        const std::uint64_t bytes = bytes_of(count_of(a.dims), a.element_type);
        r.rank = static_cast<std::uint32_t>(a.dims.size());
        for (std::size_t d = 0; d < a.dims.size(); ++d) r.dims[d] = a.dims[d];
        if (r.offset_bytes > std::numeric_limits<std::uint64_t>::max() - bytes)
            throw Overflow("packed size overflows 64 bits");
        end = r.offset_bytes + bytes;
        out.records.push_back(r);
    }
    out.total_bytes = align_up(end, alignment);
    return out;
}

LayoutDescriptor pack(const Data& data, std::uint64_t alignment) {
    std::vector<ArrayShape> shapes;
    shapes.reserve(data.arrays.size());
    for (const NDArray& a : data.arrays) shapes.push_back({a.element_type(), a.dims()});
    return pack_shapes(shapes, alignment);
}

std::vector<std::byte> serialize_layout_header(const LayoutDescriptor& layout) {
    std::vector<std::uint64_t> words;
    words.reserve(1 + kWords * layout.records.size());
    words.push_back(layout.records.size());
    for (const LayoutRecord& r : layout.records) {
        words.push_back(r.offset_bytes);
        words.push_back(static_cast<std::uint64_t>(r.element_type));
        words.push_back(r.rank);
        words.insert(words.end(), r.dims.begin(), r.dims.end());
    }
    std::vector<std::byte> bytes(words.size() * 8);
    for (std::size_t w = 0; w < words.size(); ++w)
        for (int b = 0; b < 8; ++b) bytes[8 * w + b] = std::byte((words[w] >> (8 * b)) & 0xffu);
    return bytes;
}

LayoutDescriptor parse_layout_header(std::span<const std::byte> bytes) {
    if (bytes.size() < 8 || bytes.size() % 8 != 0)
        throw MalformedHeader("header length " + std::to_string(bytes.size()) +
                              " is not a whole number of 64-bit words");
    auto word = [&](std::size_t i) {
        std::uint64_t v = 0;
        for (int b = 7; b >= 0; --b) v = (v << 8) | std::uint64_t(bytes[8 * i + b]);
        return v;
    };
    const std::uint64_t n = word(0);
    if (n > (bytes.size() / 8) || bytes.size() != (1 + kWords * n) * 8)
        throw MalformedHeader("header declares " + std::to_string(n) + " arrays but is " +
                              std::to_string(bytes.size()) + " bytes long");
    LayoutDescriptor out;
    std::uint64_t offsets_or = 0;
    for (std::uint64_t i = 0; i < n; ++i) {
        const std::size_t b = 1 + kWords * i;
        LayoutRecord r;
        r.offset_bytes = word(b);
        const std::uint64_t code = word(b + 1);
        if (!is_valid_element_type(code))
            throw MalformedHeader("record " + std::to_string(i) + " has unknown element type code " +
                                  std::to_string(code));
        r.element_type = ElementType(code);
        const std::uint64_t rank = word(b + 2);
        if (rank == 0 || rank > kMaxRank)
            throw MalformedHeader("record " + std::to_string(i) + " has rank " + std::to_string(rank));
        r.rank = std::uint32_t(rank);
        for (std::size_t d = 0; d < kMaxRank; ++d) {
            r.dims[d] = word(b + 3 + d);
            if (r.dims[d] == 0 || (d >= rank && r.dims[d] != 1))
                throw MalformedHeader("record " + std::to_string(i) + " has invalid dim " +
                                      std::to_string(r.dims[d]) + " at axis " + std::to_string(d));
        }
        offsets_or |= r.offset_bytes;
        out.records.push_back(r);
    }
    out.alignment_bytes = offsets_or == 0 ? 1 : (offsets_or & (~offsets_or + 1));
    out.total_bytes = out.records.empty() ? 0 : out.records.back().end_offset();
    return out;
}

}  // namespace hetreco
