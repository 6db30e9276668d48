// share_bench.cu — does a PARTIALLY shared operand stream get cheaper when the
// CTAs sharing it run in step? (dev tool, decides the sparse GEMM's cluster mode)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/share_bench tools/share_bench.cu -lcuda
//
// One CTA per SM streams GEMM-shaped 48 KB stages (3 x 16 KB TMA boxes) from a
// 32 MiB L2-resident matrix through a 4-stage ring, no MMAs. Box 0 plays the
// masked operand tile (X), boxes 1-2 the per-CTA W slab. CTAs form groups of G
// consecutive blocks: with `share` set, all CTAs of a group read the SAME box-0
// sequence (as CTAs on one mask row, different column slabs, would); boxes 1-2
// are always distinct per CTA. mode 1 = groups launched as hardware clusters
// (G CTAs co-scheduled in one GPC), mode 2 = clusters + box 0 split in G parts
// multicast to the whole cluster (each SM still receives 48 KB per stage).
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
__device__ __forceinline__ void tma_load_mc(const CUtensorMap* tm, uint64_t* bar, void* dst, int c0, int c1,
                                            uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
    return r;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int kStage = 48 * 1024, kStages = 4;
constexpr int kRows = 4096, kCols = 4096;  // bf16, 32 MiB
constexpr int kTilesK = kCols / 64, kTilesR = kRows / 128;
constexpr int kTiles = kTilesK * kTilesR;  // 16 KB tiles {64, 128}

// mode 0/1: every CTA loads its 3 boxes itself; mode 2: box 0 multicast in G parts
template <int MODE>
__global__ void __launch_bounds__(128, 1) share_stream(const __grid_constant__ CUtensorMap tm,
                                                      const __grid_constant__ CUtensorMap tm_part, int group, int share,
                                                      int stages_total, unsigned long long* t_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
    uint64_t* empty = full + kStages;
    const uint32_t rank = MODE == 0 ? blockIdx.x % group : cluster_rank();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, group);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (MODE != 0) cluster_sync_all(); else __syncthreads();
    const int gid = blockIdx.x / group;
    const unsigned long long t0 = gtimer();
    if (threadIdx.x == 0) {
        int ta = share ? (gid * 97) % kTiles : (blockIdx.x * 97) % kTiles;
        int tb = (blockIdx.x * 389 + 7) % kTiles;
        const int part_rows = 128 / group;
        for (int s = 0; s < stages_total; ++s) {
            const int st = s % kStages;
            if (MODE == 2) {
                if (s >= kStages) mbar_wait(empty + st, ((s / kStages) - 1) & 1);
            } else if (s >= kStages) {
                mbar_wait(full + st, ((s / kStages) - 1) & 1);
            }
            mbar_expect_tx(full + st, kStage);
            uint8_t* base = smem + st * kStage;
            if (MODE == 2) {
                tma_load_mc(&tm_part, full + st, base + rank * part_rows * 128, (ta % kTilesK) * 64,
                            (ta / kTilesK) * 128 + rank * part_rows, static_cast<uint16_t>((1u << group) - 1));
            } else {
                tma_load(&tm, full + st, base, (ta % kTilesK) * 64, (ta / kTilesK) * 128);
            }
            for (int j = 1; j < 3; ++j) {
                const int t = (tb + j) % kTiles;
                tma_load(&tm, full + st, base + j * 16384, (t % kTilesK) * 64, (t / kTilesK) * 128);
            }
            ta = (ta + 1) % kTiles;
            tb = (tb + 2) % kTiles;
            if (MODE == 2) {
                // retire the oldest fill: release its slot to every CTA of the cluster
                const int sc = s - (kStages - 2);
                if (sc >= 0) {
                    const int sts = sc % kStages;
                    mbar_wait(full + sts, (sc / kStages) & 1);
                    for (int c = 0; c < group; ++c)
                        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(
                                         mapa_u32(smem_u32(empty + sts), c))
                                     : "memory");
                }
            }
        }
        if (MODE == 2) {
            for (int sc = stages_total - (kStages - 2); sc < stages_total; ++sc)
                if (sc >= 0) mbar_wait(full + sc % kStages, (sc / kStages) & 1);
        } else {
            for (int s = stages_total; s < stages_total + kStages; ++s)
                mbar_wait(full + s % kStages, ((s / kStages) - 1) & 1);
        }
        t_out[2 * blockIdx.x] = t0;
        t_out[2 * blockIdx.x + 1] = gtimer();
    }
    if (MODE != 0) cluster_sync_all();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    void* buf = nullptr;
    CK(cudaMalloc(&buf, size_t(kRows) * kCols * 2));
    CK(cudaMemset(buf, 1, size_t(kRows) * kCols * 2));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    auto enc = [&](CUtensorMap* tm, uint32_t rows) {
        cuuint64_t dims[2] = {kCols, kRows}, strides[1] = {kCols * 2};
        cuuint32_t box[2] = {64, rows}, es[2] = {1, 1};
        return reinterpret_cast<EncodeFn>(fn)(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap tm, tm64, tm32;
    if (enc(&tm, 128) || enc(&tm64, 64) || enc(&tm32, 32)) {
        std::printf("encode failed\n");
        return 1;
    }
    const int smem = kStages * kStage + 1024 + 256;
    CK(cudaFuncSetAttribute(share_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(share_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(share_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* t_dev = nullptr;
    CK(cudaMalloc(&t_dev, 2 * 1024 * sizeof(unsigned long long)));
    std::vector<unsigned long long> t(2 * 1024);
    const int stages_total = 600;
    struct Case { int mode, group, share; };
    const Case cases[] = {{0, 1, 0}, {1, 2, 0}, {1, 2, 1}, {2, 2, 1}, {1, 4, 1}, {2, 4, 1}};
    for (const Case& c : cases) {
        // cluster 4 fits only 33 clusters (132 CTAs) at this smem size on B200
        for (int ctas : {c.group == 4 ? 132 : sms, 36}) {
            double best = 0;
            for (int rep = 0; rep < 3; ++rep) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(ctas);
                cfg.blockDim = dim3(128);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = c.mode ? c.group : 1;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                const CUtensorMap& tp = c.group == 2 ? tm64 : tm32;
                cudaError_t e;
                if (c.mode == 0) e = cudaLaunchKernelEx(&cfg, share_stream<0>, tm, tp, c.group, c.share, stages_total, t_dev);
                else if (c.mode == 1) e = cudaLaunchKernelEx(&cfg, share_stream<1>, tm, tp, c.group, c.share, stages_total, t_dev);
                else e = cudaLaunchKernelEx(&cfg, share_stream<2>, tm, tp, c.group, c.share, stages_total, t_dev);
                CK(e);
                CK(cudaDeviceSynchronize());
                CK(cudaMemcpy(t.data(), t_dev, 2 * ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
                unsigned long long lo = ~0ull, hi = 0;
                for (int i = 0; i < ctas; ++i) {
                    lo = t[2 * i] < lo ? t[2 * i] : lo;
                    hi = t[2 * i + 1] > hi ? t[2 * i + 1] : hi;
                }
                const double gbs = double(ctas) * stages_total * kStage / double(hi - lo);
                best = gbs > best ? gbs : best;
            }
            std::printf("mode %d group %d share %d ctas %3d: delivered %7.1f GB/s total, %6.1f GB/s per SM, %6.1f ns/stage\n",
                        c.mode, c.group, c.share, ctas, best, best / ctas, kStage / (best / ctas));
        }
    }
    return 0;
}
