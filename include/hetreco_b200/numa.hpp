// numa.hpp -- bind a host thread to the NUMA node of its GPU (multi-GPU
// streaming placement, SURVEY.md §8 e).  Linux sysfs based; no-op without NUMA
// information.
#pragma once

#include <string>
#include <vector>

namespace hetreco {

// "0-3,8,10-11" -> {0,1,2,3,8,10,11}; InvalidArgument on malformed text.
std::vector<int> parse_cpulist(const std::string& text);
// NUMA node of CUDA device `ordinal` (-1 when the platform reports none).
int device_numa_node(int ordinal);
// Restricts the calling thread (and threads it creates later) to the CPUs of
// `node`; returns the CPU count (0 = nothing done, node < 0).
int bind_thread_to_numa_node(int node);

}  // namespace hetreco
