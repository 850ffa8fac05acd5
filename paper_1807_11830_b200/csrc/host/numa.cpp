// numa.cpp -- host-side placement for multi-GPU streaming (SURVEY.md §8 e:
// "one ComputeSession plus host thread per GPU, NUMA-pinned to the GPU's
// socket, with pinned buffers allocated on that node").  On an 8-GPU box each
// rank binds to the NUMA node its GPU hangs off before allocating its pinned
// k-space slab, so the slab's pages are local to the root complex that DMAs
// them (the H2D stream then never crosses the inter-socket link).
#include "hetreco_b200/numa.hpp"

#include <cuda_runtime.h>
#include <sched.h>

#include <cctype>
#include <fstream>
#include <sstream>
#include <string>

#include "hetreco_b200/error_types.hpp"

namespace hetreco {

std::vector<int> parse_cpulist(const std::string& text) {
    std::vector<int> cpus;
    std::stringstream ss(text);
    std::string part;
    while (std::getline(ss, part, ',')) {
        while (!part.empty() && std::isspace(static_cast<unsigned char>(part.back()))) part.pop_back();
        while (!part.empty() && std::isspace(static_cast<unsigned char>(part.front()))) part.erase(part.begin());
        if (part.empty()) continue;
        const std::size_t dash = part.find('-');
        try {
            if (dash == std::string::npos) {
                cpus.push_back(std::stoi(part));
            } else {
                const int a = std::stoi(part.substr(0, dash)), b = std::stoi(part.substr(dash + 1));
                if (b < a || b - a > 65535) throw InvalidArgument("bad cpulist range '" + part + "'");
                for (int c = a; c <= b; ++c) cpus.push_back(c);
            }
        } catch (const std::logic_error&) {
            throw InvalidArgument("bad cpulist entry '" + part + "'");
        }
    }
    return cpus;
}

int device_numa_node(int ordinal) {
    char bus[64] = {0};
    const cudaError_t e = cudaDeviceGetPCIBusId(bus, sizeof bus, ordinal);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw InvalidArgument("no CUDA device " + std::to_string(ordinal));
    }
    std::string id(bus);
    for (char& c : id) c = char(std::tolower(static_cast<unsigned char>(c)));
    std::ifstream f("/sys/bus/pci/devices/" + id + "/numa_node");
    int node = -1;
    if (!(f >> node)) return -1;
    return node;
}

int bind_thread_to_numa_node(int node) {
    if (node < 0) return 0;  // no NUMA information: leave the thread alone
    std::ifstream f("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist");
    std::string text;
    if (!std::getline(f, text)) throw InvalidArgument("NUMA node " + std::to_string(node) + " has no cpulist");
    const std::vector<int> cpus = parse_cpulist(text);
    cpu_set_t set;
    CPU_ZERO(&set);
    int n = 0;
    for (int c : cpus)
        if (c >= 0 && c < CPU_SETSIZE) {
            CPU_SET(c, &set);
            ++n;
        }
    if (n == 0) return 0;
    if (sched_setaffinity(0, sizeof set, &set) != 0)
        throw InvalidArgument("sched_setaffinity to NUMA node " + std::to_string(node) + " failed");
    return n;
}

}  // namespace hetreco
