// box_bench.cu — per-SM TMA load throughput vs box geometry (dev tool).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/box_bench tools/box_bench.cu -lcuda
//
// One CTA per SM streams stages of `boxes` identical TMA boxes from a 64 MiB
// bf16 matrix (L2-resident after the first pass is NOT guaranteed: 64 MiB < L2
// so it is) through a 4-stage ring, no consumer. Geometries (all 128B swizzle):
//   2d64x128   {64, 128}          16 KB, 128 rows x 128 B  (today's K-major box)
//   2d64x256   {64, 256}          32 KB, 256 rows x 128 B
//   3dk2       {64, 128, 2 atoms} 32 KB, 128 rows x 256 B  (K-major, 128-deep)
//   3dmn2      {64, 64, 2 atoms}  16 KB,  64 rows x 256 B  (today's MN-major box)
//   3dmn4      {64, 64, 4 atoms}  32 KB,  64 rows x 512 B
// Prints delivered GB/s per SM at 148 and 37 CTAs.
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
__device__ __forceinline__ void tma2(const CUtensorMap* tm, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma3(const CUtensorMap* tm, uint64_t* bar, void* dst, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int kRows = 8192, kCols = 4096;  // bf16 64 MiB
constexpr int kStages = 4;

// kind: 0 = 2D box (bw inner elems, bh rows); 1 = 3D K-major (64, bh rows, na atoms): coords (0, row, atom)
//       2 = 3D MN-major (64, bh k-rows, na atoms)
__global__ void __launch_bounds__(128, 1) box_stream(const __grid_constant__ CUtensorMap tm, int kind, int box_bytes,
                                                    int boxes, int bh, int na, int stages_total,
                                                    unsigned long long* t_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = box_bytes * boxes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * stage_bytes);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) mbar_init(full + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned long long t0 = gtimer();
    if (threadIdx.x == 0) {
        // walk boxes along the inner dimension of a per-CTA row band
        const int band_rows = kind == 2 ? 64 : bh;
        const int bands = kRows / band_rows;
        const int inner_boxes = kind == 0 ? kCols / 64 : kCols / (64 * na);
        int row = ((blockIdx.x * 37) % bands) * band_rows;
        int ib = 0;
        for (int s = 0; s < stages_total; ++s) {
            const int st = s % kStages;
            if (s >= kStages) mbar_wait(full + st, ((s / kStages) - 1) & 1);
            mbar_expect_tx(full + st, stage_bytes);
            for (int j = 0; j < boxes; ++j) {
                uint8_t* dst = smem + st * stage_bytes + j * box_bytes;
                if (kind == 0) tma2(&tm, full + st, dst, ib * 64, row);
                else tma3(&tm, full + st, dst, 0, row, ib * na);
                if (++ib == inner_boxes) {
                    ib = 0;
                    row = (row + band_rows) % kRows;
                }
            }
        }
        for (int s = stages_total; s < stages_total + kStages; ++s) mbar_wait(full + s % kStages, ((s / kStages) - 1) & 1);
        t_out[2 * blockIdx.x] = t0;
        t_out[2 * blockIdx.x + 1] = gtimer();
    }
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
    EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
    struct G { const char* name; int kind, bh, na, box_bytes; };
    const G gs[] = {{"2d64x128", 0, 128, 1, 16384}, {"2d64x256", 0, 256, 1, 32768}, {"3dk2 ", 1, 128, 2, 32768},
                    {"3dk4 ", 1, 64, 4, 32768},      {"3dmn2", 2, 64, 2, 16384},     {"3dmn4", 2, 64, 4, 32768},
                    {"3dmn8", 2, 64, 8, 65536}};
    unsigned long long* t_dev = nullptr;
    CK(cudaMalloc(&t_dev, 2 * 1024 * sizeof(unsigned long long)));
    std::vector<unsigned long long> t(2 * 1024);
    CK(cudaFuncSetAttribute(box_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    for (const G& g : gs) {
        CUtensorMap tm;
        CUresult r;
        if (g.kind == 0) {
            cuuint64_t dims[2] = {kCols, kRows}, strides[1] = {kCols * 2};
            cuuint32_t box[2] = {64, (cuuint32_t)g.bh}, es[2] = {1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            // (64 inner, rows, atoms): atom stride 128 B, row stride kCols*2
            cuuint64_t dims[3] = {64, kRows, kCols / 64}, strides[2] = {kCols * 2, 128};
            cuuint32_t box[3] = {64, (cuuint32_t)g.bh, (cuuint32_t)g.na}, es[3] = {1, 1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) {
            std::printf("%s: encode failed %d\n", g.name, (int)r);
            continue;
        }
        for (int stage_kb : {48, 32, 64}) {
            const int boxes = stage_kb * 1024 / g.box_bytes;
            if (boxes < 1 || boxes * g.box_bytes != stage_kb * 1024) continue;
            const int smem = kStages * stage_kb * 1024 + 1024 + 256;
            if (smem > 227 * 1024) continue;
            for (int ctas : {sms, 37}) {
                double best = 0;
                const int stages_total = 300;
                for (int rep = 0; rep < 3; ++rep) {
                    box_stream<<<ctas, 128, smem>>>(tm, g.kind, g.box_bytes, boxes, g.bh, g.na, stages_total, t_dev);
                    CK(cudaGetLastError());
                    CK(cudaDeviceSynchronize());
                    CK(cudaMemcpy(t.data(), t_dev, 2 * ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
                    unsigned long long lo = ~0ull, hi = 0;
                    for (int c = 0; c < ctas; ++c) {
                        lo = t[2 * c] < lo ? t[2 * c] : lo;
                        hi = t[2 * c + 1] > hi ? t[2 * c + 1] : hi;
                    }
                    const double gbs = double(ctas) * stages_total * stage_kb * 1024 / double(hi - lo);
                    best = gbs > best ? gbs : best;
                }
                std::printf("%s stage %2d KB (%d boxes) ctas %3d: %8.1f GB/s total %6.1f GB/s per SM\n", g.name, stage_kb,
                            boxes, ctas, best, best / ctas);
            }
        }
    }
    return 0;
}
