// builtin_kernels.cu -- the reference's six builtin kernels as sm_100a
// kernels behind the same five-argument ABI (device_abi.h), so that
// ComputeSession::launch_kernel("<name>", ...) behaves exactly as on the
// reference backend.  Semantics and rounding are bit-exact with
// kernels/*.cl.src: products/sums use __fmul_rn/__fadd_rn (no FMA
// contraction, as in the reference's ISO C++ build) and reductions
// accumulate in fp64 in coil order.  Work item `gid` is one CUDA thread of a
// grid-stride loop over [0, gsize).
//
// `launch_negate` is the vectorised fast path used by the Negate process
// (16 B per thread per iteration, float4 / 16 x u8).
#include <cstring>

#include "launch.hpp"
#include "pdl.cuh"

namespace hetreco::dev {

namespace {

__device__ __forceinline__ const void* arr_in(const hetreco_kernel_args& a, int i) {
    return static_cast<const char*>(a.in) + hetreco_hdr_offset(a.in_layout, i);
}
__device__ __forceinline__ void* arr_out(const hetreco_kernel_args& a, int i) {
    return static_cast<char*>(a.out) + hetreco_hdr_offset(a.out_layout, i);
}
template <class T>
__device__ __forceinline__ T param(const hetreco_kernel_args& a, int off) {
    T v;
    memcpy(&v, static_cast<const char*>(a.params) + off, sizeof(T));
    return v;
}

// kernel_abi.h:123-125 with explicit rounding
__device__ __forceinline__ float2 cmul_rn(float2 a, float2 b) {
    return make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                       __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
}

#define GRID_STRIDE(g, n) \
    for (std::uint64_t g = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; g < (n); g += std::uint64_t(gridDim.x) * blockDim.x)

// negate.cl.src:6-22
__global__ void k_negate(hetreco_kernel_args a, std::uint64_t n) {
    pdl_launch_dependents();
    pdl_wait();
    const double mv = param<double>(a, 0);
    const std::uint64_t type = hetreco_hdr_type(a.in_layout, 0);
    if (type == HETRECO_UINT8) {
        const unsigned char* in = static_cast<const unsigned char*>(arr_in(a, 0));
        unsigned char* out = static_cast<unsigned char*>(arr_out(a, 0));
        GRID_STRIDE(g, n) {
            double v = mv - double(in[g]);
            v = v < 0.0 ? 0.0 : v;
            v = v > 255.0 ? 255.0 : v;
            out[g] = (unsigned char)(v + 0.5);
        }
    } else if (type == HETRECO_FLOAT32) {
        const float* in = static_cast<const float*>(arr_in(a, 0));
        float* out = static_cast<float*>(arr_out(a, 0));
        const float m = float(mv);
        GRID_STRIDE(g, n) out[g] = __fsub_rn(m, in[g]);
    }
}

// fft_radix2_pass.cl.src:22-69
__global__ void k_fft_radix2_pass(hetreco_kernel_args a, std::uint64_t n) {
    pdl_launch_dependents();
    pdl_wait();
    const std::uint32_t mode = param<std::uint32_t>(a, 0);
    const std::uint64_t L = param<std::uint64_t>(a, 8);
    const std::uint64_t S = param<std::uint64_t>(a, 16);
    float2* out = static_cast<float2*>(arr_out(a, 0));
    if (mode == 2) {
        const std::uint64_t m = param<std::uint64_t>(a, 24);
        const float scale = param<float>(a, 32);
        const float2* tw = reinterpret_cast<const float2*>(static_cast<const char*>(a.params) + 40);
        const std::uint64_t half = L / 2, tstep = L / (2 * m);
        GRID_STRIDE(g, n) {
            const std::uint64_t line = g / half, jj = g % half;
            const std::uint64_t grp = jj / m, k = jj % m;
            const std::uint64_t base = (line % S) + (line / S) * (S * L);
            const std::uint64_t i0 = base + (grp * 2 * m + k) * S, i1 = i0 + m * S;
            const float2 w = tw[k * tstep];
            const float2 x0 = out[i0];
            const float2 b = cmul_rn(out[i1], w);
            out[i0] = make_float2(__fmul_rn(__fadd_rn(x0.x, b.x), scale), __fmul_rn(__fadd_rn(x0.y, b.y), scale));
            out[i1] = make_float2(__fmul_rn(__fsub_rn(x0.x, b.x), scale), __fmul_rn(__fsub_rn(x0.y, b.y), scale));
        }
        return;
    }
    const std::uint32_t* rev = reinterpret_cast<const std::uint32_t*>(static_cast<const char*>(a.params) + 40);
    if (mode == 0) {
        const float2* in = static_cast<const float2*>(arr_in(a, 0));
        GRID_STRIDE(g, n) {
            const std::uint64_t k = g % L, line = g / L;
            const std::uint64_t base = (line % S) + (line / S) * (S * L);
            out[base + k * S] = in[base + std::uint64_t(rev[k]) * S];
        }
    } else {
        GRID_STRIDE(g, n) {
            const std::uint64_t k = g % L, line = g / L;
            const std::uint64_t r = rev[k];
            if (k < r) {
                const std::uint64_t base = (line % S) + (line / S) * (S * L);
                const float2 t = out[base + k * S];
                out[base + k * S] = out[base + r * S];
                out[base + r * S] = t;
            }
        }
    }
}

// complex_element_prod.cl.src:9-19
__global__ void k_complex_element_prod(hetreco_kernel_args a, std::uint64_t n) {
    pdl_launch_dependents();
    pdl_wait();
    const std::uint32_t conj = param<std::uint32_t>(a, 0);
    const float2* x = static_cast<const float2*>(arr_in(a, 0));
    const float2* s = static_cast<const float2*>(arr_in(a, 1));
    float2* out = static_cast<float2*>(arr_out(a, 0));
    const std::uint64_t ns = hetreco_hdr_elements(a.in_layout, 1);
    GRID_STRIDE(g, n) {
        float2 b = s[g % ns];
        if (conj) b.y = -b.y;
        out[g] = cmul_rn(x[g], b);
    }
}

// ximage_sum.cl.src:6-23
__global__ void k_ximage_sum(hetreco_kernel_args a, std::uint64_t n) {
    pdl_launch_dependents();
    pdl_wait();
    const std::uint64_t plane = hetreco_hdr_dim(a.in_layout, 0, 0) * hetreco_hdr_dim(a.in_layout, 0, 1);
    const std::uint64_t nc = hetreco_hdr_dim(a.in_layout, 0, 2);
    const float2* in = static_cast<const float2*>(arr_in(a, 0));
    float2* out = static_cast<float2*>(arr_out(a, 0));
    GRID_STRIDE(g, n) {
        const std::uint64_t f = g / plane, p = g % plane;
        double re = 0.0, im = 0.0;
        for (std::uint64_t c = 0; c < nc; ++c) {
            const float2 v = in[p + plane * (c + nc * f)];
            re = __dadd_rn(re, double(v.x));
            im = __dadd_rn(im, double(v.y));
        }
        out[g] = make_float2(float(re), float(im));
    }
}

// rss_combine.cl.src:5-20
__global__ void k_rss_combine(hetreco_kernel_args a, std::uint64_t n) {
    pdl_launch_dependents();
    pdl_wait();
    const std::uint64_t plane = hetreco_hdr_dim(a.in_layout, 0, 0) * hetreco_hdr_dim(a.in_layout, 0, 1);
    const std::uint64_t nc = hetreco_hdr_dim(a.in_layout, 0, 2);
    const float2* in = static_cast<const float2*>(arr_in(a, 0));
    float* out = static_cast<float*>(arr_out(a, 0));
    GRID_STRIDE(g, n) {
        const std::uint64_t f = g / plane, p = g % plane;
        double acc = 0.0;
        for (std::uint64_t c = 0; c < nc; ++c) {
            const float2 v = in[p + plane * (c + nc * f)];
            const double re = v.x, im = v.y;
            acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
        }
        out[g] = float(sqrt(acc));
    }
}

// matrix_add.cl.src:5-24
__global__ void k_matrix_add(hetreco_kernel_args a, std::uint64_t n) {
    pdl_launch_dependents();
    pdl_wait();
    const std::uint64_t type = hetreco_hdr_type(a.in_layout, 0);
    if (type == HETRECO_FLOAT32) {
        const float* x = static_cast<const float*>(arr_in(a, 0));
        const float* y = static_cast<const float*>(arr_in(a, 1));
        float* o = static_cast<float*>(arr_out(a, 0));
        GRID_STRIDE(g, n) o[g] = __fadd_rn(x[g], y[g]);
    } else if (type == HETRECO_FLOAT64) {
        const double* x = static_cast<const double*>(arr_in(a, 0));
        const double* y = static_cast<const double*>(arr_in(a, 1));
        double* o = static_cast<double*>(arr_out(a, 0));
        GRID_STRIDE(g, n) o[g] = __dadd_rn(x[g], y[g]);
    } else if (type == HETRECO_INT32) {
        const int* x = static_cast<const int*>(arr_in(a, 0));
        const int* y = static_cast<const int*>(arr_in(a, 1));
        int* o = static_cast<int*>(arr_out(a, 0));
        GRID_STRIDE(g, n) o[g] = int(unsigned(x[g]) + unsigned(y[g]));
    }
}

// ---- vectorised negate (process fast path) -------------------------------------------------

__device__ __forceinline__ unsigned char neg_u8(unsigned char x, double mv) {
    double v = mv - double(x);
    v = v < 0.0 ? 0.0 : v;
    v = v > 255.0 ? 255.0 : v;
    return (unsigned char)(v + 0.5);
}

__global__ void k_negate_f32_vec(const float4* __restrict__ in, float4* __restrict__ out, std::uint64_t n4,
                                 const float* __restrict__ tin, float* __restrict__ tout, int tail, float m) {
    pdl_launch_dependents();
    pdl_wait();
    GRID_STRIDE(g, n4) {
        const float4 v = __ldcs(in + g);
        __stcs(out + g, make_float4(__fsub_rn(m, v.x), __fsub_rn(m, v.y), __fsub_rn(m, v.z), __fsub_rn(m, v.w)));
    }
    if (blockIdx.x == 0 && threadIdx.x < tail) tout[threadIdx.x] = __fsub_rn(m, tin[threadIdx.x]);
}

__global__ void k_negate_u8_vec(const uint4* __restrict__ in, uint4* __restrict__ out, std::uint64_t n16,
                                const unsigned char* __restrict__ tin, unsigned char* __restrict__ tout, int tail,
                                double mv) {
    pdl_launch_dependents();
    pdl_wait();
    // u8 results depend only on the byte value: build the 256-entry table once
    // per block with the reference's double formula (bit-exact), then map.
    __shared__ unsigned char lut[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = neg_u8((unsigned char)i, mv);
    __syncthreads();
    GRID_STRIDE(g, n16) {
        uint4 v = __ldcs(in + g);
        unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned x = w[k];
            w[k] = unsigned(lut[x & 0xff]) | unsigned(lut[(x >> 8) & 0xff]) << 8 |
                   unsigned(lut[(x >> 16) & 0xff]) << 16 | unsigned(lut[x >> 24]) << 24;
        }
        __stcs(out + g, make_uint4(w[0], w[1], w[2], w[3]));
    }
    if (blockIdx.x == 0 && threadIdx.x < tail) tout[threadIdx.x] = lut[tin[threadIdx.x]];
}

int grid_for(std::uint64_t n, int block) {
    const std::uint64_t g = (n + block - 1) / block;
    return int(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

const char* const kNames[] = {"negate", "fft_radix2_pass", "complex_element_prod", "ximage_sum",
                              "rss_combine", "matrix_add"};

}  // namespace

const char* builtin_name(Builtin b) {
    const int i = int(b);
    return (i >= 0 && i < int(Builtin::Count)) ? kNames[i] : "";
}

int builtin_from_name(const char* name) {
    for (int i = 0; i < int(Builtin::Count); ++i)
        if (std::strcmp(kNames[i], name) == 0) return i;
    return -1;
}

cudaError_t launch_builtin(Builtin which, const hetreco_kernel_args& a, std::uint64_t gsize, cudaStream_t st) {
    constexpr int B = 256;
    const int G = grid_for(gsize, B);
    switch (which) {
        case Builtin::Negate: k_negate<<<G, B, 0, st>>>(a, gsize); break;
        case Builtin::FftRadix2Pass: k_fft_radix2_pass<<<G, B, 0, st>>>(a, gsize); break;
        case Builtin::ComplexElementProd: k_complex_element_prod<<<G, B, 0, st>>>(a, gsize); break;
        case Builtin::XImageSum: k_ximage_sum<<<G, B, 0, st>>>(a, gsize); break;
        case Builtin::RssCombine: k_rss_combine<<<G, B, 0, st>>>(a, gsize); break;
        case Builtin::MatrixAdd: k_matrix_add<<<G, B, 0, st>>>(a, gsize); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_negate(int type, const void* in, void* out, std::uint64_t n, double mv, cudaStream_t st) {
    constexpr int B = 256;
    if (type == HETRECO_FLOAT32) {
        const std::uint64_t n4 = n / 4;
        const int tail = int(n - n4 * 4);
        k_negate_f32_vec<<<grid_for(n4 ? n4 : 1, B), B, 0, st>>>(
            static_cast<const float4*>(in), static_cast<float4*>(out), n4, static_cast<const float*>(in) + n4 * 4,
            static_cast<float*>(out) + n4 * 4, tail, float(mv));
    } else if (type == HETRECO_UINT8) {
        const std::uint64_t n16 = n / 16;
        const int tail = int(n - n16 * 16);
        k_negate_u8_vec<<<grid_for(n16 ? n16 : 1, B), B, 0, st>>>(
            static_cast<const uint4*>(in), static_cast<uint4*>(out), n16,
            static_cast<const unsigned char*>(in) + n16 * 16, static_cast<unsigned char*>(out) + n16 * 16, tail, mv);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace hetreco::dev
