// launch.hpp -- host-side entry points of the sm_100a kernels.
// Everything here enqueues asynchronously on the given stream and returns the
// launch status; nothing synchronises.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "hetreco_b200/device_abi.h"

namespace hetreco::dev {

// ---- reference-ABI builtins (kernels/*.cl.src semantics, bit-exact) ---------------

enum class Builtin : int {
    Negate = 0,
    FftRadix2Pass,
    ComplexElementProd,
    XImageSum,
    RssCombine,
    MatrixAdd,
    Count
};
const char* builtin_name(Builtin b);
int builtin_from_name(const char* name);  // -1 when unknown

// `args` holds device pointers (params too); gsize as in the reference.
cudaError_t launch_builtin(Builtin which, const hetreco_kernel_args& args, std::uint64_t gsize,
                           cudaStream_t stream);

// ---- fast paths used by the processes ----------------------------------------------

// out[i] = max - in[i] for n elements of type UINT8 or FLOAT32 (negate.cl.src),
// vectorised 16 B per thread.
cudaError_t launch_negate(int type_code, const void* in, void* out, std::uint64_t n, double max_value,
                          cudaStream_t stream);

// Supported FFT line lengths (powers of two 1..4096).
bool fft_size_supported(std::uint64_t n);

// Strided-axis pass: transforms every column (stride nx) of the [nx, N, planes]
// array along axis 1.  `tw` = device table of W_N^t (direction applied).
struct StridedArgs {
    const float2* in;
    float2* out;
    std::uint64_t nx;
    std::uint64_t planes;
    int shift_in;   // ifftshift along the axis on load
    int shift_out;  // fftshift along the axis on store
    float scale;
    const float2* tw;
    const float* mask = nullptr;  // k-space sampling mask [nx, N] (forward-model kernels only)
};

enum class Combine : int { None = 0, Sense = 1, Rss = 2 };

// Contiguous-axis pass (axis 0, lines of N samples) with an optional coil
// combine epilogue.
//   None : `lines` = ny*batch independent lines, out = float2 lines.
//   Sense: in = [N, ny, C, F] lines, smap = [N, ny, C];
//          out[x,y,f] = sum_c conj(smap[x,y,c]) * X[x,y,c,f]   (COMPLEX64)
//   Rss  : out[x,y,f] = sqrt(sum_c |X[x,y,c,f]|^2)            (FLOAT32)
// The combine multiplies in fp32 with the reference's rounding order and
// accumulates in fp64 in coil order (complex_element_prod.cl.src,
// ximage_sum.cl.src, rss_combine.cl.src).
struct ContigArgs {
    const float2* in;
    void* out;
    const float2* smap;
    std::uint64_t ny;
    std::uint64_t coils;   // Sense/Rss only
    std::uint64_t frames;  // Sense/Rss: F; None: batch
    int shift_in;
    int shift_out;
    float scale;
    const float2* tw;
};

struct LaunchShape {
    int block = 0;
    int grid = 0;
    int smem = 0;
    int variant = 0;  // combine kernel variant (bit0 fp32 acc, bit1 prefetch, bit2 8 pts/thread)
    int rq = 0;       // points per thread of the chosen instantiation
};

// Pick block/grid/smem for a given problem (called once at init, baked into
// the process' CUDA graph).
LaunchShape plan_strided(std::uint64_t N, std::uint64_t nx, std::uint64_t planes, int device_sms);
// variant (combine modes only): bit 0 fp32 accumulators, bit 1 register
// prefetch, bit 2 eight points per thread; -1 = HETRECO_COMBINE_VARIANT or 3.
LaunchShape plan_contig(std::uint64_t N, Combine mode, std::uint64_t items, int device_sms, int variant = -1);

cudaError_t launch_strided(std::uint64_t N, int dir, const StridedArgs& a, const LaunchShape& s,
                           cudaStream_t stream);
cudaError_t launch_contig(std::uint64_t N, int dir, Combine mode, const ContigArgs& a,
                          const LaunchShape& s, cudaStream_t stream);

// ---- coil-parallel axis-0 + combine for small problems (fft_combine_cp.cu) -------
// One CTA per output line, G coil groups transform coils in parallel and the
// partials are summed in group order (fp32).  launch_contig dispatches a shape
// from plan_combine_cp (variant bit 128) here.
bool combine_cp_preferred(std::uint64_t N, std::uint64_t items /* ny*F */, std::uint64_t coils, int device_sms);
LaunchShape plan_combine_cp(std::uint64_t N, Combine mode, std::uint64_t items, int device_sms);
cudaError_t launch_combine_cp(std::uint64_t N, Combine mode, const ContigArgs& a, const LaunchShape& s,
                              cudaStream_t stream);

// ---- SENSE combine with the map row staged in shared memory (fft_combine_ss.cu) --
// CTA = one row y of 8 consecutive frames sharing S[:, y, c]; fp32, SENSE only.
// launch_contig dispatches a shape from plan_combine_ss (variant bit 256) here.
bool combine_ss_supported(std::uint64_t N);
LaunchShape plan_combine_ss(std::uint64_t N, std::uint64_t ny, std::uint64_t frames, int device_sms);
cudaError_t launch_combine_ss(std::uint64_t N, const ContigArgs& a, const LaunchShape& s, cudaStream_t stream);

// ---- SENSE combine with the 16 x 16 DFT stages on tcgen05 (fft_combine_tc.cu) ------
// 256-point lines only; HETRECO_COMBINE_TC=1 selects it in place of the
// staged-map kernel (plan_combine_ss returns its shape, variant bit 512).
bool combine_tc_enabled(std::uint64_t N);
LaunchShape plan_combine_tc(std::uint64_t N, std::uint64_t ny, std::uint64_t frames, int device_sms);
cudaError_t launch_combine_tc(std::uint64_t N, const ContigArgs& a, const LaunchShape& s, cudaStream_t stream);

// ---- SENSE normal operator E^H E in one cooperative kernel (fft_sense_normal.cu) --
// Square power-of-two sides 64..256; three phases separated by grid barriers.
// Opt-in (HETRECO_NORMAL_FUSED=1; measured slower than the three-kernel graph);
// plan returns block == 0 otherwise.
struct SenseNormalArgs {
    const float2* m;     // image [N, N, F]
    const float2* s;     // maps [N, N, C]
    const float* mask;   // [N, N] or null
    float2* z;           // scratch [N, N, C, F]
    float2* out;         // [N, N, F]
    const float2* tw_fwd;
    const float2* tw_inv;
    std::uint32_t coils;
    std::uint32_t frames;
    int shift;
    float scale;         // 1 / (N * N)
    int phases = 7;      // timing experiments only (HETRECO_NORMAL_PHASES): bit i runs phase i
};
LaunchShape plan_sense_normal_fused(std::uint64_t N, std::uint64_t planes, int device_sms);
cudaError_t launch_sense_normal_fused(std::uint64_t N, const SenseNormalArgs& a, const LaunchShape& s,
                                      cudaStream_t stream);

// ---- axis-0 + combine fed by a TMA bulk-copy ring (fft_combine_tma.cu) -----------
// Same contract as launch_contig with mode Sense/Rss and fp32 accumulation;
// a.in = X [N, ny, C, F].  HETRECO_TMA_STAGES (2|3|4|6, default 4) = tiles in
// flight per CTA.
bool combine_tma_supported(std::uint64_t N);
LaunchShape plan_combine_tma(std::uint64_t N, Combine mode, std::uint64_t ny, std::uint64_t frames, int device_sms);
cudaError_t launch_combine_tma(std::uint64_t N, Combine mode, const ContigArgs& a, const LaunchShape& s,
                               cudaStream_t stream);

// ---- single-pass cluster reconstruction (fft_cluster.cu) ------------------------
//
// IFFT2 + Sense/Rss combine of [256, 256, C, F] k-space in ONE kernel: an
// 8-CTA cluster holds a coil image across its SMs (TMA tile loads, DSMEM
// transpose), coils accumulate in registers.  fp32 accumulation only.

bool cluster_supported(std::uint64_t nx, std::uint64_t ny, Combine mode);
int cluster_smem_bytes(int cluster_size);

struct ClusterPlan {
    int cl = 0;                   // CTAs per cluster (8 or 16)
    int clusters = 0;             // resident clusters launched (persistent grid)
    std::uint64_t ws_bytes = 0;   // split-frame partials workspace
    std::uint64_t cnt_bytes = 0;  // split-frame arrival counters (zero-initialise once)
};
// max_clusters <= 0: as many as fit on the device; cluster_size 0 = pick
// (HETRECO_CLUSTER_SIZE, else 16 when it launches, else 8).  clusters == 0
// in the result: the kernel cannot run here.
ClusterPlan plan_cluster(Combine mode, std::uint64_t coils, std::uint64_t frames, int max_clusters = 0,
                         int cluster_size = 0);

// Opaque TMA descriptor (CUtensorMap) for the k-space array [256, rows]
// (rows = 256 * C * F), box = one CTA's column tile for cluster size `cl`;
// re-made when the k-space pointer changes.
struct alignas(64) ClusterMap {
    unsigned char bytes[128];
};
cudaError_t make_cluster_map(ClusterMap& m, const float2* y, std::uint64_t rows, int cl);

struct ClusterLaunch {
    const float2* smap;  // Sense: S [256, 256, C]
    void* out;           // [256, 256, F]
    float2* ws;
    unsigned* cnt;
    const float2* tw;  // inverse W_256^t table
    std::uint64_t coils, frames;
    int shift;
    float scale;
};
cudaError_t launch_cluster(Combine mode, const ClusterMap& m, const ClusterLaunch& a, const ClusterPlan& p,
                           cudaStream_t st);

// ---- SENSE forward model E = P F S and normal operator E^H E ----

// Normal-operator front half at 256 x 256 on 16-CTA clusters
// (fft_sense_cluster.cu): out[:, :, c, f] = F_y^-1 P F_y F_x (S_c . M_f), the
// output of launch_expand + launch_strided_masked(roundtrip), bit-identical.
struct SenseFrontArgs {
    const float2* m;     // M [256, 256, F]
    const float2* smap;  // S [256, 256, C]
    const float* mask;   // P [256, 256] or null
    float2* out;         // [256, 256, C, F]
    const float2* tw;    // forward W_256^t
    std::uint32_t coils, frames;
    int shift;
    float scale;  // applied at the store (1 in the normal operator)
};
// Clusters to launch (<= coil images), 0 when the kernel does not apply
// (size; opt-in with HETRECO_NORMAL_CLUSTER=1, measured slower) or cannot run
// on this device.
int plan_sense_front(std::uint64_t nx, std::uint64_t ny, std::uint64_t coil_images);
cudaError_t launch_sense_front(const SenseFrontArgs& a, int clusters, cudaStream_t stream);


// Expand + forward axis-0 FFT: out line (y, c, f) = F_x( S[:, y, c] * M[:, y, f] ).
// a.in = M [N, ny, F], a.smap = S [N, ny, C], a.out = [N, ny, C, F].
LaunchShape plan_expand(std::uint64_t N, std::uint64_t items /* ny*C*F */, int device_sms);
cudaError_t launch_expand(std::uint64_t N, const ContigArgs& a, const LaunchShape& s, cudaStream_t stream);

// Forward axis-1 FFT of every column with the sampling mask applied at the
// store (roundtrip = false), or forward FFT, mask, inverse FFT in registers
// (roundtrip = true: the k-space never leaves the SM).  a.mask may be null.
// Square images only (a.nx == N).
LaunchShape plan_strided_masked(std::uint64_t N, bool roundtrip, std::uint64_t planes, int device_sms);
cudaError_t launch_strided_masked(std::uint64_t N, bool roundtrip, const StridedArgs& a, const LaunchShape& s,
                                  cudaStream_t stream);

// ---- synthetic phantom (phantom.cu) ------------------------------

struct PhantomBlob {
    double amp, radius, angle, sigma;  // pixels / radians, relative to the image centre
};
struct PhantomArgs {
    float2* truth;  // [nx, ny, frames]
    float2* smaps;  // [nx, ny, coils]
    std::uint32_t nx, ny, frames, coils;
    PhantomBlob blob[3];
    double coil_radius, coil_width;
};
cudaError_t launch_phantom(const PhantomArgs& a, int device_sms, cudaStream_t st);

}  // namespace hetreco::dev
