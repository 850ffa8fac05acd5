// nvrtc_compiler.hpp -- run-time compilation of kernel-source units for
// sm_100a (see nvrtc_compiler.cpp).
#pragma once

#include <string>
#include <vector>

#include "hetreco_b200/error_types.hpp"

namespace hetreco::nvrtc {

struct Unit {
    std::string unit_name;
    std::vector<std::string> kernels;  // HETRECO_KERNEL names, source order
    std::vector<char> cubin;           // sm_100a code; entry per kernel: hetreco_entry_<name>
    std::string log;                   // compiler log (warnings)
};

bool available();
std::string version();
// HETRECO_KERNEL(name) definitions in a unit (comments ignored).
std::vector<std::string> kernel_names(const std::string& source);
// Throws CompileError({unit, log}) on failure, UnsupportedSource without NVRTC.
Unit compile(const std::string& unit_name, const std::string& source, const std::string& arch = "sm_100a");

}  // namespace hetreco::nvrtc
