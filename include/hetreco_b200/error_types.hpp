// error_types.hpp -- exception taxonomy of the hetreco API
// (reference: include/hetreco/errors.hpp:12-219).  Same class names and
// meanings so code written against the reference catches the same types;
// each class also carries a stable numeric code that the C-ABI returns.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace hetreco {

// Numeric status codes used by the C-ABI (include/hetreco_b200.h).
enum class ErrorCode : int {
    Ok = 0,
    Error = 1,
    InvalidFilter,
    NoMatchingDevice,
    InvalidArgument,
    EmptyData,
    Overflow,
    MalformedHeader,
    AllocationFailure,
    UnknownHandle,
    DeviceError,
    CompileError,
    DuplicateKernel,
    UnsupportedSource,
    UnknownKernel,
    InvalidParams,
    ShapeMismatch,
    AlreadyInitialized,
    NotInitialized,
    ChainMismatch,
    ChainStageError,
    UnsupportedElementType,
    // io (SPEC.md io module)
    MalformedFile,
    UnsupportedFeature,
    IoError,
    SizeMismatch,
    MalformedSidecar,
};

class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what, ErrorCode code = ErrorCode::Error)
        : std::runtime_error(what), code_(code) {}
    ErrorCode code() const { return code_; }

private:
    ErrorCode code_;
};

#define HETRECO_SIMPLE_ERROR(Name)                                             \
    class Name : public Error {                                                \
    public:                                                                    \
        explicit Name(const std::string& what) : Error(what, ErrorCode::Name) {} \
    }

HETRECO_SIMPLE_ERROR(InvalidFilter);          // errors.hpp:21
HETRECO_SIMPLE_ERROR(NoMatchingDevice);       // errors.hpp:29
HETRECO_SIMPLE_ERROR(InvalidArgument);        // errors.hpp:37
HETRECO_SIMPLE_ERROR(EmptyData);              // errors.hpp:43
HETRECO_SIMPLE_ERROR(Overflow);               // errors.hpp:49
HETRECO_SIMPLE_ERROR(MalformedHeader);        // errors.hpp:55
HETRECO_SIMPLE_ERROR(AllocationFailure);      // errors.hpp:61
HETRECO_SIMPLE_ERROR(UnknownHandle);          // errors.hpp:67
HETRECO_SIMPLE_ERROR(DuplicateKernel);        // errors.hpp:117
HETRECO_SIMPLE_ERROR(UnsupportedSource);      // errors.hpp:124
HETRECO_SIMPLE_ERROR(UnknownKernel);          // errors.hpp:130
HETRECO_SIMPLE_ERROR(InvalidParams);          // errors.hpp:138
HETRECO_SIMPLE_ERROR(ShapeMismatch);          // errors.hpp:142
HETRECO_SIMPLE_ERROR(AlreadyInitialized);     // errors.hpp:147
HETRECO_SIMPLE_ERROR(NotInitialized);         // errors.hpp:152
HETRECO_SIMPLE_ERROR(ChainMismatch);          // errors.hpp:158
HETRECO_SIMPLE_ERROR(UnsupportedElementType); // errors.hpp:179
HETRECO_SIMPLE_ERROR(MalformedFile);          // SPEC.md:494 (io)
HETRECO_SIMPLE_ERROR(UnsupportedFeature);     // message names the feature
HETRECO_SIMPLE_ERROR(IoError);
HETRECO_SIMPLE_ERROR(SizeMismatch);
HETRECO_SIMPLE_ERROR(MalformedSidecar);
#undef HETRECO_SIMPLE_ERROR

// A kernel failed on the device; names the kernel (errors.hpp:73-83).
class DeviceError : public Error {
public:
    DeviceError(std::string kernel, const std::string& detail)
        : Error("device error in kernel '" + kernel + "': " + detail, ErrorCode::DeviceError),
          kernel_(std::move(kernel)) {}
    const std::string& kernel_name() const { return kernel_; }

private:
    std::string kernel_;
};

// errors.hpp:88-112.  Source kernels are not compiled by this backend (the
// NVRTC path is future work); the type exists so callers
// that catch it keep compiling.
struct BuildDiagnostic {
    std::string unit_name;
    std::string log;
};

class CompileError : public Error {
public:
    explicit CompileError(std::vector<BuildDiagnostic> diags)
        : Error(render(diags), ErrorCode::CompileError), diags_(std::move(diags)) {}
    const std::vector<BuildDiagnostic>& diagnostics() const { return diags_; }

private:
    static std::string render(const std::vector<BuildDiagnostic>& d) {
        std::string s = "kernel compilation failed";
        for (const auto& x : d) s += "\n--- unit '" + x.unit_name + "' ---\n" + x.log;
        return s;
    }
    std::vector<BuildDiagnostic> diags_;
};

// A stage of a composite process failed (errors.hpp:164-175).
class ChainStageError : public Error {
public:
    ChainStageError(std::size_t index, const std::string& stage, const std::string& detail)
        : Error("stage " + std::to_string(index) + " (" + stage + "): " + detail,
                ErrorCode::ChainStageError),
          index_(index) {}
    std::size_t stage_index() const { return index_; }

private:
    std::size_t index_;
};

}  // namespace hetreco
