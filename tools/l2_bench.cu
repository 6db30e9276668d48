// l2_bench.cu — L2 -> SM TMA throughput when CTAs share tiles in time (dev tool).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bench tools/l2_bench.cu -lcuda
//   ./tools/l2_bench
//
// One CTA per SM streams 48 KB stages (3 x 16 KB TMA boxes, 64 x 128 bf16,
// 128B swizzle) from a 32 MiB L2-resident matrix through a 4-stage ring, like
// the GEMM producer without MMAs. CTAs are split into sharing groups of G:
// the CTAs of one group load the SAME tile sequence (as CTAs working on the
// same operand slab at the same time would); different groups load disjoint
// sequences. Reports the chip-wide delivered bytes per ns and per SM-cycle,
// to tell whether simultaneous reads of a tile by several SMs cost L2
// throughput once or G times.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
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
__device__ __forceinline__ void tma_load(const CUtensorMap* tm, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int kStage = 48 * 1024, kStages = 4;
constexpr int kRows = 4096, kCols = 4096;  // bf16, 32 MiB
constexpr int kTilesK = kCols / 64, kTilesR = kRows / 128;
constexpr int kTiles = kTilesK * kTilesR;  // 16 KB tiles

__global__ void __launch_bounds__(128, 1) l2_stream(const __grid_constant__ CUtensorMap tm, int group, int lag, int stages_total,
                                                   unsigned long long* t_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) mbar_init(full + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int seq = blockIdx.x / group;  // CTAs of one sharing group read the same tiles
    const unsigned long long t0 = gtimer();
    if (threadIdx.x == 0) {
        // disjoint per-group start; within the sequence tiles advance like a K-loop
        // member m of a group runs m * lag stages behind member 0 on the same sequence
        const int m = blockIdx.x % group;
        int tile = ((seq * 97 * 3 - m * lag * 3) % kTiles + kTiles) % kTiles;
        for (int s = 0; s < stages_total; ++s) {
            const int st = s % kStages;
            if (s >= kStages) mbar_wait(full + st, ((s / kStages) - 1) & 1);
            mbar_expect_tx(full + st, kStage);
            for (int j = 0; j < 3; ++j) {
                const int t = (tile + j) % kTiles;
                tma_load(&tm, full + st, smem + st * kStage + j * 16384, (t % kTilesK) * 64, (t / kTilesK) * 128);
            }
            tile = (tile + 3) % kTiles;
        }
        for (int s = stages_total; s < stages_total + kStages; ++s) {
            const int st = s % kStages;
            mbar_wait(full + st, ((s / kStages) - 1) & 1);
        }
        t_out[2 * blockIdx.x] = t0;
        t_out[2 * blockIdx.x + 1] = gtimer();
    }
}

// Cluster-of-2 variant: each CTA loads HALF of every stage (3 of 6 8 KB boxes)
// and multicasts it to both CTAs, so each SM still receives 48 KB per stage
// while L2 serves 24 KB per CTA. Slots are re-armed once both CTAs saw them full.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
    return r;
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    l2_stream_mc(const __grid_constant__ CUtensorMap tm64, int stages_total, unsigned long long* t_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
    uint64_t* empty = full + kStages;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const int seq = blockIdx.x / 2;
    const unsigned long long t0 = gtimer();
    if (threadIdx.x == 0) {
        int tile = (seq * 97 * 6) % (2 * kTiles);  // 8 KB tiles of 64 x 64
        for (int s = 0; s < stages_total; ++s) {
            const int st = s % kStages;
            if (s >= kStages) mbar_wait(empty + st, ((s / kStages) - 1) & 1);
            mbar_expect_tx(full + st, kStage);
            for (int j = rank; j < 6; j += 2) {
                const int t = (tile + j) % (2 * kTiles);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                    " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem + st * kStage + j * 8192)),
                    "l"(reinterpret_cast<uint64_t>(&tm64)), "r"(smem_u32(full + st)), "r"((t % kTilesK) * 64),
                    "r"((t / kTilesK) * 64), "h"((uint16_t)3)
                    : "memory");
            }
            tile = (tile + 6) % (2 * kTiles);
            // retire the oldest outstanding fill (pipelined): once it completed
            // here, release its slot to both CTAs' producers
            const int sc = s - (kStages - 1);
            if (sc >= 0) {
                const int sts = sc % kStages;
                mbar_wait(full + sts, (sc / kStages) & 1);
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + sts)) : "memory");
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 mapa_u32(smem_u32(empty + sts), rank ^ 1))
                             : "memory");
            }
        }
        for (int sc = stages_total - (kStages - 1); sc < stages_total; ++sc) mbar_wait(full + sc % kStages, (sc / kStages) & 1);
        t_out[2 * blockIdx.x] = t0;
        t_out[2 * blockIdx.x + 1] = gtimer();
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Ring-shape variant: `nst` stages of `nbox` 16 KB boxes, distinct streams.
__global__ void __launch_bounds__(128, 1) l2_ring(const __grid_constant__ CUtensorMap tm, int nst, int nbox,
                                                 long long total_bytes, unsigned long long* t_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = nbox * 16384;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stage_bytes);
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) mbar_init(full + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned long long t0 = gtimer();
    if (threadIdx.x == 0) {
        const int stages_total = static_cast<int>(total_bytes / stage_bytes);
        int tile = (blockIdx.x * 97 * 3) % kTiles;
        for (int s = 0; s < stages_total; ++s) {
            const int st = s % nst;
            if (s >= nst) mbar_wait(full + st, ((s / nst) - 1) & 1);
            mbar_expect_tx(full + st, stage_bytes);
            for (int j = 0; j < nbox; ++j) {
                const int t = (tile + j) % kTiles;
                tma_load(&tm, full + st, smem + st * stage_bytes + j * 16384, (t % kTilesK) * 64, (t / kTilesK) * 128);
            }
            tile = (tile + nbox) % kTiles;
        }
        for (int s = stages_total; s < stages_total + nst; ++s) mbar_wait(full + s % nst, ((s / nst) - 1) & 1);
        t_out[2 * blockIdx.x] = t0;
        t_out[2 * blockIdx.x + 1] = gtimer();
    }
}

// GEMM-shaped stages: one 16 KB A box {64,128} + nb 8 KB B boxes {64,64}.
__global__ void __launch_bounds__(128, 1) l2_gemm_ring(const __grid_constant__ CUtensorMap tmA,
                                                      const __grid_constant__ CUtensorMap tmB, int nst, int nb,
                                                      long long total_bytes, unsigned long long* t_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = 16384 + nb * 8192;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stage_bytes);
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) mbar_init(full + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned long long t0 = gtimer();
    if (threadIdx.x == 0) {
        const int stages_total = static_cast<int>(total_bytes / stage_bytes);
        int ta = (blockIdx.x * 97) % kTiles, tb = (blockIdx.x * 193) % (2 * kTiles);
        for (int s = 0; s < stages_total; ++s) {
            const int st = s % nst;
            if (s >= nst) mbar_wait(full + st, ((s / nst) - 1) & 1);
            mbar_expect_tx(full + st, stage_bytes);
            uint8_t* base = smem + st * stage_bytes;
            tma_load(&tmA, full + st, base, (ta % kTilesK) * 64, (ta / kTilesK) * 128);
            for (int j = 0; j < nb; ++j) {
                const int t = (tb + j) % (2 * kTiles);
                tma_load(&tmB, full + st, base + 16384 + j * 8192, (t % kTilesK) * 64, (t / kTilesK) * 64);
            }
            ta = (ta + 1) % kTiles;
            tb = (tb + nb) % (2 * kTiles);
        }
        for (int s = stages_total; s < stages_total + nst; ++s) mbar_wait(full + s % nst, ((s / nst) - 1) & 1);
        t_out[2 * blockIdx.x] = t0;
        t_out[2 * blockIdx.x + 1] = gtimer();
    }
}

__device__ __forceinline__ void tma_load3(const CUtensorMap* tm, uint64_t* bar, void* dst, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// GEMM-shaped stages with ONE 3D box for B: {64 n, 64 k, nb n-atoms} = nb * 8 KB
// laid out atom-major (the MN-major SW128 operand layout), plus the A box.
__global__ void __launch_bounds__(128, 1) l2_gemm3d_ring(const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmB3, int nst, int nb,
                                                        long long total_bytes, unsigned long long* t_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = 16384 + nb * 8192;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stage_bytes);
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) mbar_init(full + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned long long t0 = gtimer();
    if (threadIdx.x == 0) {
        const int stages_total = static_cast<int>(total_bytes / stage_bytes);
        int ta = (blockIdx.x * 97) % kTiles;
        int kb = (blockIdx.x * 13) % (kRows / 64), nt = (blockIdx.x * 7) % (kCols / (64 * nb));
        for (int s = 0; s < stages_total; ++s) {
            const int st = s % nst;
            if (s >= nst) mbar_wait(full + st, ((s / nst) - 1) & 1);
            mbar_expect_tx(full + st, stage_bytes);
            uint8_t* base = smem + st * stage_bytes;
            tma_load(&tmA, full + st, base, (ta % kTilesK) * 64, (ta / kTilesK) * 128);
            tma_load3(&tmB3, full + st, base + 16384, 0, kb * 64, nt * nb);
            ta = (ta + 1) % kTiles;
            kb = (kb + 1) % (kRows / 64);
            if (kb == 0) nt = (nt + 1) % (kCols / (64 * nb));
        }
        for (int s = stages_total; s < stages_total + nst; ++s) mbar_wait(full + s % nst, ((s / nst) - 1) & 1);
        t_out[2 * blockIdx.x] = t0;
        t_out[2 * blockIdx.x + 1] = gtimer();
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const bool quick = argc > 1;
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    void* buf = nullptr;
    CK(cudaMalloc(&buf, size_t(kRows) * kCols * 2));
    CK(cudaMemset(buf, 1, size_t(kRows) * kCols * 2));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {kCols, kRows}, strides[1] = {kCols * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    if (reinterpret_cast<EncodeFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
        std::printf("encode failed\n");
        return 1;
    }
    if (quick) return 0;
    CUtensorMap tm64;
    cuuint32_t box64[2] = {64, 64};
    if (reinterpret_cast<EncodeFn>(fn)(&tm64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box64, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
        std::printf("encode failed\n");
        return 1;
    }
    const int smem = kStages * kStage + 1024 + 256;
    CK(cudaFuncSetAttribute(l2_stream_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(l2_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* t_dev = nullptr;
    CK(cudaMalloc(&t_dev, 2 * 1024 * sizeof(unsigned long long)));
    std::vector<unsigned long long> t(2 * 1024);
    const int stages_total = 400;
    for (int ctas : {sms, sms / 2, 32}) {
        if (quick && ctas != sms) continue;
        for (int group : {1, 2, 4, 8, 16, 148}) {
            if (quick && group > 2) continue;
            if (group > ctas) continue;
            double best = 0;
            for (int rep = 0; rep < (quick ? 1 : 3); ++rep) {
                l2_stream<<<ctas, 128, smem>>>(tm, group, 0, stages_total, t_dev);
                CK(cudaDeviceSynchronize());
                CK(cudaMemcpy(t.data(), t_dev, 2 * ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
                unsigned long long lo = ~0ull, hi = 0;
                for (int c = 0; c < ctas; ++c) {
                    lo = t[2 * c] < lo ? t[2 * c] : lo;
                    hi = t[2 * c + 1] > hi ? t[2 * c + 1] : hi;
                }
                const double bytes = double(ctas) * stages_total * kStage;
                const double gbs = bytes / double(hi - lo);  // bytes per ns = GB/s / 1
                best = gbs > best ? gbs : best;
            }
            std::printf("ctas %3d group %3d: delivered %7.1f GB/s total, %6.1f GB/s per SM\n", ctas, group, best * 1e0 * 1,
                        best / ctas);
        }
    }
    for (int ctas : {sms, 32}) {
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            l2_stream_mc<<<ctas, 128, smem>>>(tm64, stages_total, t_dev);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(t.data(), t_dev, 2 * ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            unsigned long long lo = ~0ull, hi = 0;
            for (int c = 0; c < ctas; ++c) {
                lo = t[2 * c] < lo ? t[2 * c] : lo;
                hi = t[2 * c + 1] > hi ? t[2 * c + 1] : hi;
            }
            const double gbs = double(ctas) * stages_total * kStage / double(hi - lo);
            best = gbs > best ? gbs : best;
        }
        std::printf("ctas %3d cluster-2 multicast halves: delivered %7.1f GB/s total, %6.1f GB/s per SM\n", ctas, best,
                    best / ctas);
    }
    CK(cudaFuncSetAttribute(l2_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    const int shapes[][2] = {{4, 3}, {3, 3}, {2, 3}, {2, 5}, {2, 4}, {3, 4}, {5, 2}, {6, 2}, {4, 2}, {8, 1}, {12, 1}};
    for (auto& sh : shapes) {
        const int smem_r = sh[0] * sh[1] * 16384 + 1024 + 256;
        if (smem_r > 227 * 1024) continue;
        for (int ctas : {sms, 37}) {
            double best = 0;
            for (int rep = 0; rep < 3; ++rep) {
                l2_ring<<<ctas, 128, smem_r>>>(tm, sh[0], sh[1], 400ll * 48 * 1024, t_dev);
                CK(cudaDeviceSynchronize());
                CK(cudaMemcpy(t.data(), t_dev, 2 * ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
                unsigned long long lo = ~0ull, hi = 0;
                for (int c = 0; c < ctas; ++c) {
                    lo = t[2 * c] < lo ? t[2 * c] : lo;
                    hi = t[2 * c + 1] > hi ? t[2 * c + 1] : hi;
                }
                const double gbs = double(ctas) * 400.0 * 48 * 1024 / double(hi - lo);
                best = gbs > best ? gbs : best;
            }
            std::printf("ring %d x %3d KB (%3d KB in flight) ctas %3d: %7.1f GB/s total, %6.1f GB/s per SM\n", sh[0],
                        sh[1] * 16, sh[0] * sh[1] * 16, ctas, best, best / ctas);
        }
    }
    CK(cudaFuncSetAttribute(l2_gemm_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    const int gshapes[][2] = {{4, 4}, {3, 4}, {2, 8}, {3, 6}};
    for (auto& sh : gshapes) {
        const int sb = 16384 + sh[1] * 8192;
        const int smem_r = sh[0] * sb + 1024 + 256;
        if (smem_r > 227 * 1024) continue;
        for (int ctas : {sms, 37}) {
            double best = 0;
            for (int rep = 0; rep < 3; ++rep) {
                l2_gemm_ring<<<ctas, 128, smem_r>>>(tm, tm64, sh[0], sh[1], 400ll * 48 * 1024, t_dev);
                CK(cudaDeviceSynchronize());
                CK(cudaMemcpy(t.data(), t_dev, 2 * ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
                unsigned long long lo = ~0ull, hi = 0;
                for (int c = 0; c < ctas; ++c) {
                    lo = t[2 * c] < lo ? t[2 * c] : lo;
                    hi = t[2 * c + 1] > hi ? t[2 * c + 1] : hi;
                }
                const double gbs = double(ctas) * 400.0 * 48 * 1024 / double(hi - lo);
                best = gbs > best ? gbs : best;
            }
            std::printf("gemm ring %d x (A16 + %d x B8 = %3d KB) ctas %3d: %7.1f GB/s total, %6.1f GB/s per SM\n", sh[0],
                        sh[1], sb / 1024, ctas, best, best / ctas);
        }
    }
    {
        // 3D view of the row-major [kRows][kCols] matrix: (n_in 64, k rows, n_out atoms)
        CUtensorMap tm3;
        cuuint64_t d3[3] = {64, kRows, kCols / 64}, s3[2] = {kCols * 2, 128};
        cuuint32_t es3[3] = {1, 1, 1};
        CK(cudaFuncSetAttribute(l2_gemm3d_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        for (int nb : {4, 8}) {
            cuuint32_t b3[3] = {64, 64, (cuuint32_t)nb};
            CUresult r = reinterpret_cast<EncodeFn>(fn)(&tm3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, es3,
                                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != 0) {
                std::printf("3d encode failed (%d) for nb=%d\n", (int)r, nb);
                continue;
            }
            for (int nst : {2, 3, 4}) {
                const int sb = 16384 + nb * 8192;
                const int smem_r = nst * sb + 1024 + 256;
                if (smem_r > 227 * 1024) continue;
                for (int ctas : {sms, 37}) {
                    double best = 0;
                    for (int rep = 0; rep < 3; ++rep) {
                        l2_gemm3d_ring<<<ctas, 128, smem_r>>>(tm, tm3, nst, nb, 400ll * 48 * 1024, t_dev);
                        CK(cudaDeviceSynchronize());
                        CK(cudaMemcpy(t.data(), t_dev, 2 * ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
                        unsigned long long lo = ~0ull, hi = 0;
                        for (int c = 0; c < ctas; ++c) {
                            lo = t[2 * c] < lo ? t[2 * c] : lo;
                            hi = t[2 * c + 1] > hi ? t[2 * c + 1] : hi;
                        }
                        const double gbs = double(ctas) * 400.0 * 48 * 1024 / double(hi - lo);
                        best = gbs > best ? gbs : best;
                    }
                    std::printf("gemm3d ring %d x (A16 + B3d %d KB = %3d KB, 2 boxes) ctas %3d: %7.1f GB/s total, %6.1f GB/s per SM\n",
                                nst, nb * 8, sb / 1024, ctas, best, best / ctas);
                }
            }
        }
    }
    // how far apart in time may two readers of the same tiles be and still share?
    for (int lag : {0, 1, 2, 4, 8, 16, 32, 64, 128}) {
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            l2_stream<<<sms, 128, smem>>>(tm, 2, lag, stages_total, t_dev);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(t.data(), t_dev, 2 * sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            unsigned long long lo = ~0ull, hi = 0;
            for (int c = 0; c < sms; ++c) {
                lo = t[2 * c] < lo ? t[2 * c] : lo;
                hi = t[2 * c + 1] > hi ? t[2 * c + 1] : hi;
            }
            const double gbs = double(sms) * stages_total * kStage / double(hi - lo);
            best = gbs > best ? gbs : best;
        }
        std::printf("ctas %3d group 2 lag %3d stages: delivered %7.1f GB/s total, %6.1f GB/s per SM\n", sms, lag, best,
                    best / sms);
    }
    return 0;
}
