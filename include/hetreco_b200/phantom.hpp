// phantom.hpp -- gen_phantom: a seeded
// synthetic cardiac-cine experiment -- ground truth M_true (three Gaussian
// blobs rotating 2 pi f / F per frame), normalised complex coil maps S
// (sum_i |S_i|^2 = 1) and the multi-coil k-space Y_i = F(S_i . M_true) --
// generated on the device (phantom.cu + the sense_forward process) and
// returned as host Data.  The forward-model identity makes
// sens_recon(Y, S) == M_true an exact reconstruction target.
#pragma once

#include <array>
#include <cstdint>

#include "hetreco_b200/compute_session.hpp"
#include "hetreco_b200/data.hpp"

namespace hetreco {

struct PhantomSpec {
    std::uint64_t nx = 128, ny = 128, frames = 16, coils = 8;  // SPEC.md:531 defaults
    std::uint64_t seed = 1;
};

struct Phantom {
    Data kdata;  // KData [Y [nx, ny, coils, frames] COMPLEX64]
    Data smaps;  // [S [nx, ny, coils] COMPLEX64]
    Data truth;  // XData [M_true [nx, ny, frames] COMPLEX64]
};

// Blob parameters drawn from `seed`: amp, radius, angle, sigma per blob
// (mt19937_64, 53-bit uniforms; identical on every platform).
std::array<std::array<double, 4>, 3> phantom_blobs(const PhantomSpec& spec);

// Throws InvalidParams unless nx, ny are powers of two in [2, 4096] and
// frames, coils >= 1.
Phantom gen_phantom(ComputeSession& session, const PhantomSpec& spec, HostMemory memory = HostMemory::Pageable);

}  // namespace hetreco
