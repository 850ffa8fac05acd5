// data.hpp -- the data model: typed n-d arrays, heterogeneous Data sets with
// the XData/KData role tags, and the packed layout + kernel-visible header.
//
// API-compatible with the reference's include/hetreco/ndarray.hpp:17-152 and
// include/hetreco/layout.hpp:14-65 (same names, argument meaning, errors and
// the bit-exact header wire format).  B200 difference: an NDArray payload can
// live in page-locked host memory (HostMemory::Pinned, cudaHostAlloc), so
// register/fetch and the streaming pipeline DMA straight from/to it over the
// copy engines instead of staging through a pageable bounce buffer.
#pragma once

#include <array>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "hetreco_b200/error_types.hpp"

namespace hetreco {

// ndarray.hpp:17-24 -- codes are wire format.
enum class ElementType : std::uint64_t {
    UInt8 = 1,
    Int32 = 2,
    Float32 = 3,
    Complex64 = 4,
    Float64 = 5,
    Complex128 = 6,
};

std::size_t element_size(ElementType type);
bool is_valid_element_type(std::uint64_t code);
std::string_view element_type_name(ElementType type);

template <typename T> struct element_type_of;
template <> struct element_type_of<std::uint8_t> { static constexpr ElementType value = ElementType::UInt8; };
template <> struct element_type_of<std::int32_t> { static constexpr ElementType value = ElementType::Int32; };
template <> struct element_type_of<float> { static constexpr ElementType value = ElementType::Float32; };
template <> struct element_type_of<std::complex<float>> { static constexpr ElementType value = ElementType::Complex64; };
template <> struct element_type_of<double> { static constexpr ElementType value = ElementType::Float64; };
template <> struct element_type_of<std::complex<double>> { static constexpr ElementType value = ElementType::Complex128; };

inline constexpr std::size_t kMaxRank = 8;

enum class HostMemory { Pageable, Pinned };

namespace detail {
struct HostFree {
    bool pinned = false;
    void operator()(std::byte* p) const;
};
}  // namespace detail

// Owning host byte buffer: pageable (operator new) or page-locked
// (cudaHostAlloc).  Zero-filled on construction.
class HostBuffer {
public:
    HostBuffer() = default;
    HostBuffer(std::size_t bytes, HostMemory kind);
    HostBuffer(const HostBuffer& other);
    HostBuffer& operator=(const HostBuffer& other);
    HostBuffer(HostBuffer&&) noexcept = default;
    HostBuffer& operator=(HostBuffer&&) noexcept = default;

    std::byte* data() { return ptr_.get(); }
    const std::byte* data() const { return ptr_.get(); }
    std::size_t size() const { return size_; }
    bool pinned() const { return pinned_; }

private:
    std::unique_ptr<std::byte, detail::HostFree> ptr_;
    std::size_t size_ = 0;
    bool pinned_ = false;
};

// One typed n-d array, column-major (dims fastest first), interleaved complex
// (ndarray.hpp:61-122).
class NDArray {
public:
    NDArray(ElementType type, std::vector<std::uint64_t> dims,
            HostMemory memory = HostMemory::Pageable);
    NDArray(ElementType type, std::vector<std::uint64_t> dims, std::vector<std::byte> payload);

    template <typename T>
    static NDArray from_values(std::vector<std::uint64_t> dims, std::span<const T> values,
                               HostMemory memory = HostMemory::Pageable) {
        NDArray a(element_type_of<T>::value, std::move(dims), memory);
        if (values.size() != a.element_count())
            throw InvalidArgument("from_values: " + std::to_string(values.size()) +
                                  " values supplied for " + std::to_string(a.element_count()) +
                                  " elements");
        std::memcpy(a.bytes().data(), values.data(), a.byte_size());
        return a;
    }

    ElementType element_type() const { return type_; }
    const std::vector<std::uint64_t>& dims() const { return dims_; }
    std::size_t rank() const { return dims_.size(); }
    std::uint64_t element_count() const { return count_; }
    std::size_t byte_size() const { return storage_.size(); }
    bool pinned() const { return storage_.pinned(); }

    std::span<const std::byte> bytes() const { return {storage_.data(), storage_.size()}; }
    std::span<std::byte> bytes() { return {storage_.data(), storage_.size()}; }

    template <typename T>
    std::span<const T> view() const {
        require_type(element_type_of<T>::value);
        return {reinterpret_cast<const T*>(storage_.data()), count_};
    }
    template <typename T>
    std::span<T> view() {
        require_type(element_type_of<T>::value);
        return {reinterpret_cast<T*>(storage_.data()), count_};
    }

    bool operator==(const NDArray& other) const;

private:
    void require_type(ElementType t) const;

    ElementType type_;
    std::vector<std::uint64_t> dims_;
    std::uint64_t count_ = 0;
    HostBuffer storage_;
};

// ndarray.hpp:125-129 -- the paper's XData / KData roles.
enum class DataKind { XData, KData, Generic };
std::string_view data_kind_name(DataKind kind);

// ndarray.hpp:139-152 -- ordered heterogeneous arrays moved as one unit.
struct Data {
    std::vector<NDArray> arrays;
    DataKind kind = DataKind::Generic;

    Data() = default;
    explicit Data(std::vector<NDArray> arrays_, DataKind kind_ = DataKind::Generic)
        : arrays(std::move(arrays_)), kind(kind_) {}

    std::size_t array_count() const { return arrays.size(); }
    bool empty() const { return arrays.empty(); }
    std::uint64_t payload_byte_size() const;
};

// ---- packed layout (layout.hpp:14-65) ---------------------------------------

struct LayoutRecord {
    std::uint64_t offset_bytes = 0;
    ElementType element_type = ElementType::UInt8;
    std::uint32_t rank = 1;
    std::array<std::uint64_t, kMaxRank> dims{1, 1, 1, 1, 1, 1, 1, 1};

    std::uint64_t element_count() const;
    std::uint64_t byte_size() const;
    std::uint64_t end_offset() const { return offset_bytes + byte_size(); }
    bool operator==(const LayoutRecord&) const = default;
};

struct LayoutDescriptor {
    std::vector<LayoutRecord> records;
    std::uint64_t total_bytes = 0;
    std::uint64_t alignment_bytes = 1;

    std::size_t array_count() const { return records.size(); }
    bool operator==(const LayoutDescriptor& o) const { return records == o.records; }
};

// Shape-only description of one array (used to pack without payloads).
struct ArrayShape {
    ElementType element_type = ElementType::UInt8;
    std::vector<std::uint64_t> dims;
};

LayoutDescriptor pack(const Data& data, std::uint64_t alignment_bytes);
LayoutDescriptor pack_shapes(std::span<const ArrayShape> arrays, std::uint64_t alignment_bytes);
std::vector<std::byte> serialize_layout_header(const LayoutDescriptor& layout);
LayoutDescriptor parse_layout_header(std::span<const std::byte> bytes);

}  // namespace hetreco
