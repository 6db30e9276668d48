// ingress_bench.cu — per-SM global->shared ingress bandwidth by load path (dev tool).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ingress_bench tools/ingress_bench.cu -lcuda
//   ./ingress_bench
//
// Each CTA (1 per SM, 256 threads) streams a private 32 MiB slice of a buffer
// into a 4 x 48 KB shared-memory ring, like the GEMM producer, and reports
// bytes / SM-cycle. Modes:
//   0  TMA (cp.async.bulk.tensor 2D, 64x128 bf16 boxes, 128B swizzle), 1 thread
//   1  cp.async 16 B (LDGSTS) from 4 warps
//   2  both: TMA for 2/3 of each stage, cp.async for 1/3
// Results are for deciding how the GEMM producer should feed the MMA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            std::printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); \
            return 1;                                                              \
        }                                                                          \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load(const void* tmap, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// cp.async completions of this thread arrive (without incrementing the pending count) on the barrier
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int kStages = 4;
constexpr int kStage = 48 * 1024;
constexpr int kRows = 8192;  // rows of 128 B (64 bf16) per CTA slice per "column" of 2D map

// The CTA's slice is rows [blockIdx.x * rows_per_cta, ...) of a (total_rows x 64) bf16 matrix.
__global__ void __launch_bounds__(256, 1) ingress(const __grid_constant__ CUtensorMap tm, const uint8_t* base,
                                                  int rows_per_cta, int stages_total, int mode,
                                                  unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
    const int warp = threadIdx.x / 32;
    // full barrier: 1 arrival (TMA expect_tx) + 128 cp.async threads (noinc arrivals)
    const uint32_t cp_threads = (mode == 0) ? 0 : 128;
    if (threadIdx.x == 0)
        for (int i = 0; i < kStages; ++i) mbar_init(full + i, 1 + cp_threads);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const long long t0 = clock64();
    const int row0 = blockIdx.x * rows_per_cta;
    // bytes per stage by path
    const int tma_bytes = mode == 0 ? kStage : (mode == 1 ? 0 : 32 * 1024);
    const int cp_bytes = kStage - tma_bytes;
    for (int s = 0; s < stages_total; ++s) {
        const int st = s % kStages;
        // wait for the previous fill of this slot (the consumer is instantaneous)
        if (s >= kStages) mbar_wait(full + st, ((s / kStages) - 1) & 1);
        uint8_t* dst = smem + st * kStage;
        const int r = row0 + (s * (kStage / 128)) % (rows_per_cta - kStage / 128);
        if (threadIdx.x == 0) {
            if (tma_bytes) {
                mbar_expect_tx(full + st, tma_bytes);
                for (int b = 0; b < tma_bytes / 16384; ++b) tma_load(&tm, full + st, dst + b * 16384, 0, r + b * 128);
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(full + st)) : "memory");
            }
        }
        if (cp_bytes && warp >= 4) {
            const int t = threadIdx.x - 128;
            const uint8_t* src = base + static_cast<int64_t>(r + tma_bytes / 128) * 128;
            for (int off = t * 16; off < cp_bytes; off += 128 * 16) cp_async16(dst + tma_bytes + off, src + off);
            cp_async_arrive(full + st);
        }
    }
    for (int s = stages_total - kStages; s < stages_total; ++s) mbar_wait(full + s % kStages, (s / kStages) & 1);
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int rows_per_cta = 65536;  // 8 MiB per CTA slice (64 cols bf16 = 128 B rows)
    const size_t bytes = static_cast<size_t>(rows_per_cta) * sms * 128;
    uint8_t* buf = nullptr;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 1, bytes));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(rows_per_cta) * sms};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    reinterpret_cast<EncodeFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = kStages * kStage + 64;
    CK(cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* cyc = nullptr;
    CK(cudaMalloc(&cyc, sms * sizeof(unsigned long long)));
    const int stages_total = 2000;
    for (int mode = 0; mode < 3; ++mode) {
        for (int ctas : {sms, sms / 4}) {
            for (int rep = 0; rep < 2; ++rep)
                ingress<<<ctas, 256, smem>>>(tm, buf, rows_per_cta, stages_total, mode, cyc);
            CK(cudaDeviceSynchronize());
            std::vector<unsigned long long> h(ctas);
            CK(cudaMemcpy(h.data(), cyc, ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            double mean = 0;
            for (auto v : h) mean += v;
            mean /= ctas;
            std::printf("mode %d (%s) ctas %3d: %.1f cycles/stage, %.1f B/clk/SM\n", mode,
                        mode == 0 ? "TMA" : mode == 1 ? "cp.async" : "TMA+cp.async", ctas, mean / stages_total,
                        stages_total * double(kStage) / mean);
        }
    }
    return 0;
}
