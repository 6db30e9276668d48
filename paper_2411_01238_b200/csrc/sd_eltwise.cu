// sd_eltwise.cu — the MLP block's activation between the two SparseDrop
// Linears (configs[2]): GELU forward and its backward, each ONE
// HBM pass over bf16 data (16-byte vectors, grid = multiple of the SM count).
// Exact (erf) GELU, fp32 math: act = h * Phi(h);  dh = g * (Phi(h) + h * phi(h)).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <mutex>

#include "sd_internal.h"

namespace sd {
namespace {

constexpr int kThreads = 256;

uint64_t mix64_host_eltwise(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float phi_cdf(float x) { return 0.5f * (1.0f + erff(x * 0.70710678118654752f)); }

__device__ __forceinline__ uint4 ld_nc(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(b[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
    uint4 v;
    __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return v;
}

// Each thread keeps kUnroll 16-byte loads in flight before doing the erf math
// (one load per thread left the kernels at ~50% of HBM bandwidth: latency-bound
// with the ALU work in between).
constexpr int kUnroll = 4;

__global__ void __launch_bounds__(kThreads) gelu_fwd_kernel(const uint4* __restrict__ h, uint4* __restrict__ act,
                                                            int64_t n8) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n8; i += kUnroll * stride) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = ld_nc(h + i + u * stride);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            float x[8];
            unpack8(v[u], x);
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = x[j] * phi_cdf(x[j]);
            act[i + u * stride] = pack8(x);
        }
    }
    for (; i < n8; i += stride) {
        float x[8];
        unpack8(ld_nc(h + i), x);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = x[j] * phi_cdf(x[j]);
        act[i] = pack8(x);
    }
}

// d GELU / dh = Phi(h) + h phi(h), one explicit FMA so the direct kernel and
// the table builder below round identically
__device__ __forceinline__ float gelu_dgrad(float x) {
    const float pdf = 0.3989422804014327f * __expf(-0.5f * x * x);
    return __fmaf_rn(x, pdf, phi_cdf(x));
}

__device__ __forceinline__ uint4 gelu_bwd8(const uint4& hv, const uint4& gv) {
    float x[8], gr[8];
    unpack8(hv, x);
    unpack8(gv, gr);
#pragma unroll
    for (int j = 0; j < 8; ++j) gr[j] = gr[j] * gelu_dgrad(x[j]);
    return pack8(gr);
}

__global__ void __launch_bounds__(kThreads) gelu_bwd_kernel(const uint4* __restrict__ h, const uint4* __restrict__ g,
                                                            uint4* __restrict__ dh, int64_t n8) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n8; i += kUnroll * stride) {
        uint4 hv[kUnroll], gv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            hv[u] = ld_nc(h + i + u * stride);
            gv[u] = ld_nc(g + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) dh[i + u * stride] = gelu_bwd8(hv[u], gv[u]);
    }
    for (; i < n8; i += stride) dh[i] = gelu_bwd8(ld_nc(h + i), ld_nc(g + i));
}

// Forward table: GELU of the bf16 inputs with exponent field in
// [kDE0, kDE0 + kDNE) (2^-31 <= |h| < 2^33), with exactly gelu_fwd_kernel's
// math, as bf16: 16 K entries, 32 KB of shared memory, so three 512-thread
// CTAs fit per SM (the 64 K-entry, 128 KB table held one, 4.9 TB/s). Inputs
// outside the range are evaluated directly: outputs are identical either way.
constexpr int kDE0 = 96, kDNE = 64;
constexpr int kDPerSign = kDNE * 128;
constexpr int kLutThreads = 512;
constexpr int kLutBytes = 2 * kDPerSign * 2;

__device__ __forceinline__ uint32_t gelu_bf16_bits(float x) {
    const __nv_bfloat162 r = __floats2bfloat162_rn(x * phi_cdf(x), 0.0f);
    return *reinterpret_cast<const uint16_t*>(&r);
}

__global__ void __launch_bounds__(kThreads) gelu_lut_build_kernel(uint16_t* lut) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= 2 * kDPerSign) return;
    const uint32_t sign = static_cast<uint32_t>(i / kDPerSign);
    const uint32_t a = static_cast<uint32_t>(i % kDPerSign) + (kDE0 << 7);
    lut[i] = static_cast<uint16_t>(gelu_bf16_bits(__uint_as_float(((sign << 15) | a) << 16)));
}

__global__ void __launch_bounds__(kLutThreads, 3) gelu_fwd_lut_kernel(const uint4* __restrict__ h,
                                                                     uint4* __restrict__ act, int64_t n8,
                                                                     const uint4* __restrict__ lut) {
    extern __shared__ uint4 lut_s4[];
    for (int i = threadIdx.x; i < kLutBytes / 16; i += kLutThreads) lut_s4[i] = __ldg(lut + i);
    __syncthreads();
    const uint16_t* t = reinterpret_cast<const uint16_t*>(lut_s4);
    const auto one = [&](uint32_t v) -> uint32_t {
        const uint32_t off = (v & 0x7FFFu) - (kDE0 << 7);
        return off < static_cast<uint32_t>(kDPerSign) ? t[(v >> 15) * kDPerSign + off]
                                                      : gelu_bf16_bits(__uint_as_float(v << 16));
    };
    auto apply = [&](const uint4& v) {
        uint4 o;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int j = 0; j < 4; ++j) ow[j] = one(w[j] & 0xFFFFu) | (one(w[j] >> 16) << 16);
        return o;
    };
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kLutThreads;
    int64_t i = static_cast<int64_t>(blockIdx.x) * kLutThreads + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n8; i += kUnroll * stride) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = ld_nc(h + i + u * stride);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) act[i + u * stride] = apply(v[u]);
    }
    for (; i < n8; i += stride) act[i] = apply(ld_nc(h + i));
}

// Backward table: d GELU / dh (fp32, exactly gelu_dgrad) of the bf16 inputs
// with exponent field in [kDE0, kDE0 + kDNE), i.e. 2^-31 <= |h| < 2^33 —
// 16 K entries, 64 KB of shared memory, two CTAs per SM. Inputs outside the
// range (tiny, huge, NaN/Inf) are evaluated directly: same bits either way.
constexpr int kDLutBytes = 2 * kDPerSign * 4;
constexpr int kDThreads = 512;

__global__ void __launch_bounds__(kThreads) gelu_dlut_build_kernel(float* lut) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= 2 * kDPerSign) return;
    const uint32_t sign = static_cast<uint32_t>(i / kDPerSign);
    const uint32_t a = static_cast<uint32_t>(i % kDPerSign) + (kDE0 << 7);
    const float x = __uint_as_float(((sign << 15) | a) << 16);
    lut[i] = gelu_dgrad(x);
}

__global__ void __launch_bounds__(kDThreads, 2) gelu_bwd_lut_kernel(const uint4* __restrict__ h,
                                                                    const uint4* __restrict__ g,
                                                                    uint4* __restrict__ dh, int64_t n8,
                                                                    const float4* __restrict__ lut) {
    extern __shared__ float4 dlut_s4[];
    for (int i = threadIdx.x; i < kDLutBytes / 16; i += kDThreads) dlut_s4[i] = __ldg(lut + i);
    __syncthreads();
    const float* t = reinterpret_cast<const float*>(dlut_s4);
    auto apply = [&](const uint4& hv, const uint4& gv) {
        float gr[8];
        unpack8(gv, gr);
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&hv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t v = (w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
            const uint32_t off = (v & 0x7FFFu) - (kDE0 << 7);
            const float d = off < static_cast<uint32_t>(kDPerSign) ? t[(v >> 15) * kDPerSign + off]
                                                                    : gelu_dgrad(__uint_as_float(v << 16));
            gr[j] = gr[j] * d;
        }
        return pack8(gr);
    };
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kDThreads;
    int64_t i = static_cast<int64_t>(blockIdx.x) * kDThreads + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n8; i += kUnroll * stride) {
        uint4 hv[kUnroll], gv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            hv[u] = ld_nc(h + i + u * stride);
            gv[u] = ld_nc(g + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) dh[i + u * stride] = apply(hv[u], gv[u]);
    }
    for (; i < n8; i += stride) dh[i] = apply(ld_nc(h + i), ld_nc(g + i));
}

const float4* gelu_dlut() {
    static float* luts[64] = {nullptr};
    static std::mutex mu;
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= 64) fail(SD_ERUNTIME, "device index out of range");
    std::lock_guard<std::mutex> lock(mu);
    if (!luts[dev]) {
        float* p = nullptr;
        check_cuda(cudaMalloc(&p, kDLutBytes), "cudaMalloc(GELU' table)");
        cudaStream_t s;
        check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        gelu_dlut_build_kernel<<<(2 * kDPerSign + kThreads - 1) / kThreads, kThreads, 0, s>>>(p);
        check_cuda(cudaGetLastError(), "GELU' table build");
        check_cuda(cudaStreamSynchronize(s), "GELU' table build");
        cudaStreamDestroy(s);
        check_cuda(cudaFuncSetAttribute(gelu_bwd_lut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDLutBytes),
                   "GELU' kernel smem");
        luts[dev] = p;
    }
    return reinterpret_cast<const float4*>(luts[dev]);
}

// The table, built once per device (synchronously, before first use).
const uint4* gelu_lut() {
    static uint16_t* luts[64] = {nullptr};
    static std::mutex mu;
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= 64) fail(SD_ERUNTIME, "device index out of range");
    std::lock_guard<std::mutex> lock(mu);
    if (!luts[dev]) {
        uint16_t* p = nullptr;
        check_cuda(cudaMalloc(&p, kLutBytes), "cudaMalloc(GELU table)");
        cudaStream_t s;
        check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        gelu_lut_build_kernel<<<(2 * kDPerSign + kThreads - 1) / kThreads, kThreads, 0, s>>>(p);
        check_cuda(cudaGetLastError(), "GELU table build");
        check_cuda(cudaStreamSynchronize(s), "GELU table build");
        cudaStreamDestroy(s);
        check_cuda(cudaFuncSetAttribute(gelu_fwd_lut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLutBytes),
                   "GELU kernel smem");
        luts[dev] = p;
    }
    return reinterpret_cast<const uint4*>(luts[dev]);
}

int grid_for(int64_t n8) {
    const int64_t blocks = (n8 + kThreads - 1) / kThreads;
    const int cap = num_sms() * 8;
    return static_cast<int>(blocks < cap ? blocks : cap);
}

}  // namespace
}  // namespace sd

using namespace sd;

extern "C" {

SD_API int sd_gelu_forward(const void* h, void* act, int64_t n, void* stream);
SD_API int sd_gelu_backward(const void* h, const void* grad, void* dh, int64_t n, void* stream);

int sd_gelu_forward(const void* h, void* act, int64_t n, void* stream) {
    if (!h || !act || n < 0 || n % 8 || reinterpret_cast<uintptr_t>(h) % 16 || reinterpret_cast<uintptr_t>(act) % 16)
        return SD_EINVAL;
    if (n == 0) return SD_OK;
    try {
        const uint4* lut = gelu_lut();
        const int64_t n8 = n / 8;
        if (n8 >= 65536) {
            // large activations: the table kernel (a 32 KB smem copy per CTA)
            gelu_fwd_lut_kernel<<<3 * num_sms(), kLutThreads, kLutBytes, static_cast<cudaStream_t>(stream)>>>(
                static_cast<const uint4*>(h), static_cast<uint4*>(act), n8, lut);
        } else {
            gelu_fwd_kernel<<<grid_for(n8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
                static_cast<const uint4*>(h), static_cast<uint4*>(act), n8);
        }
    } catch (const Error&) {
        return SD_ERUNTIME;
    }
    note_launch();
    return cudaGetLastError() == cudaSuccess ? SD_OK : SD_ERUNTIME;
}

int sd_gelu_backward(const void* h, const void* grad, void* dh, int64_t n, void* stream) {
    if (!h || !grad || !dh || n < 0 || n % 8 || reinterpret_cast<uintptr_t>(h) % 16 ||
        reinterpret_cast<uintptr_t>(grad) % 16 || reinterpret_cast<uintptr_t>(dh) % 16)
        return SD_EINVAL;
    if (n == 0) return SD_OK;
    const int64_t n8 = n / 8;
    if (n8 >= 65536 && !(tuning() & kTuneNoGeluTable)) {
        // large activations: d GELU / dh from a 64 KB shared-memory table
        const float4* lut = nullptr;
        try {
            lut = gelu_dlut();
        } catch (const Error&) {
            return SD_ERUNTIME;
        }
        gelu_bwd_lut_kernel<<<2 * num_sms(), kDThreads, kDLutBytes, static_cast<cudaStream_t>(stream)>>>(
            static_cast<const uint4*>(h), static_cast<const uint4*>(grad), static_cast<uint4*>(dh), n8, lut);
    } else {
        gelu_bwd_kernel<<<grid_for(n8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
            static_cast<const uint4*>(h), static_cast<const uint4*>(grad), static_cast<uint4*>(dh), n8);
    }
    note_launch();
    return cudaGetLastError() == cudaSuccess ? SD_OK : SD_ERUNTIME;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Dropout-mask application for the paper's comparison baselines (SURVEY §8f2,
// PAPER.md:161,178, layer.hpp:69-76, 105-111, 148-156):
//   element mode: m(i,j) = unit_interval(counter_hash(seed, i, j)) >= p
//                 (sample_element_mask, bit-exact, exact integer threshold)
//   block mode:   m(i,j) = kept(i / m_blk, j / k_blk) of a device BlockMask
//   out = in * m * scale   (bf16; the product keeps the reference's signed
//   zeros: elementwise_mul multiplies, matrix.hpp:80-91)
namespace sd {
namespace {

__device__ __forceinline__ uint64_t mix64_dev(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void __launch_bounds__(kThreads) dropout_apply_kernel(const uint4* __restrict__ in, uint4* __restrict__ out,
                                                                 int rows, int cols, uint64_t seed_mix,
                                                                 uint64_t threshold, float scale,
                                                                 const uint64_t* __restrict__ words, int m_blk,
                                                                 int k_blk, int mask_cols) {
    const int64_t n8 = static_cast<int64_t>(rows) * cols / 8;
    const int c8 = cols / 8;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n8;
         i += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int r = static_cast<int>(i / c8);
        const int c0 = static_cast<int>(i - static_cast<int64_t>(r) * c8) * 8;
        float x[8];
        unpack8(ld_nc(in + i), x);
        if (words) {
            const int64_t b0 = static_cast<int64_t>(r / m_blk) * mask_cols;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int64_t b = b0 + (c0 + j) / k_blk;
                const bool keep = (__ldg(words + (b >> 6)) >> (b & 63)) & 1ull;
                x[j] = x[j] * (keep ? scale : 0.0f);
            }
        } else {
            const uint64_t hr = mix64_dev(seed_mix ^ static_cast<uint64_t>(r));
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint64_t h = mix64_dev(hr ^ static_cast<uint64_t>(c0 + j));
                x[j] = x[j] * (((h >> 11) >= threshold) ? scale : 0.0f);
            }
        }
        out[i] = pack8(x);
    }
}

// A caller-style kernel with Programmatic Dependent Launch (tests only): it
// triggers its dependents FIRST, as PDL-enabled library kernels (CUTLASS,
// cuBLASLt, Triton) may, then spins and writes out = 2 * in. A following
// launch that skipped griddepcontrol.wait would read `out` before it is
// written (the early backward must be opt-in).
__global__ void pdl_early_writer_kernel(const __nv_bfloat16* in, __nv_bfloat16* out, int64_t n, int spin_ns) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (spin_ns > 0) {
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
            __nanosleep(1000);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        } while (t - t0 < static_cast<unsigned long long>(spin_ns));
    }
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16(2.0f * __bfloat162float(in[i]));
}

}  // namespace
}  // namespace sd

extern "C" {

// Development entry (not in the public header): out = 2 * in (bf16), launched
// with programmatic stream serialization and an early trigger (see above).
SD_API int sd_dev_pdl_early_writer(const void* in, void* out, int64_t n, int32_t spin_ns, void* stream) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(sd::num_sms()));
    cfg.blockDim = dim3(256);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, sd::pdl_early_writer_kernel, static_cast<const __nv_bfloat16*>(in),
                                             static_cast<__nv_bfloat16*>(out), n, static_cast<int>(spin_ns));
    return e == cudaSuccess ? SD_OK : SD_ERUNTIME;
}

SD_API int sd_dropout_apply(const void* in, void* out, int32_t rows, int32_t cols, uint64_t seed, double p,
                            float scale, const sd_block_mask* block_mask, void* stream);

int sd_dropout_apply(const void* in, void* out, int32_t rows, int32_t cols, uint64_t seed, double p, float scale,
                     const sd_block_mask* block_mask, void* stream) {
    if (!in || !out || rows <= 0 || cols <= 0 || cols % 8 || reinterpret_cast<uintptr_t>(in) % 16 ||
        reinterpret_cast<uintptr_t>(out) % 16)
        return SD_EINVAL;
    if (block_mask && (block_mask->block_rows * block_mask->m_blk != rows ||
                       block_mask->block_cols * block_mask->k_blk != cols))
        return SD_EINVAL;
    if (!block_mask && !(p >= 0.0 && p < 1.0)) return SD_EINVAL;
    const uint64_t seed_mix = mix64_host_eltwise(seed);
    const uint64_t threshold = static_cast<uint64_t>(std::ceil(std::ldexp(p, 53)));
    const int64_t n8 = static_cast<int64_t>(rows) * cols / 8;
    dropout_apply_kernel<<<grid_for(n8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(in), static_cast<uint4*>(out), rows, cols, seed_mix, threshold, scale,
        block_mask ? block_mask->words : nullptr, block_mask ? block_mask->m_blk : 1,
        block_mask ? block_mask->k_blk : 1, block_mask ? block_mask->block_cols : 1);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? SD_OK : SD_ERUNTIME;
}

}  // extern "C"
