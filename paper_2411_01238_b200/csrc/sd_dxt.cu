// sd_dxt.cu — dX on 2-CTA pairs in the transposed form (development path).
//
// dX = s (dY W^T) (.) m (layer.hpp:158, gemm.hpp:176-213) computed as
// dX^T = W dY^T, one block row r of the mask at a time: a CTA pair (cluster of
// 2) issues tcgen05.mma.cta_group::2 with M = 256 = two KEPT 128-wide column
// blocks of row r (CTA 0's W block c_a, CTA 1's W block c_b: W rows are dX
// columns, read K-major in place) and N = 128 = the 128 dY rows of row block r
// (each CTA loads 64 of them). Unlike a 256-row pair over two mask rows, both
// halves reduce over the full N with no mask on the reduction, so nothing is
// wasted: every pair unit takes the next 2 * kJ kept blocks of one row.
// With kJ = 2 MMAs per 64-deep stage sharing the stage's dY half, a CTA moves
// 2 x 16 KB (W) + 8 KB (dY) per 2M MACs = 20 KB per 1M MACs, against the 1-CTA
// sdd unit's 24 KB, with a double-buffered 2 x 256-column accumulator.
// The epilogue transposes through shared memory (TMEM lane = dX column,
// TMEM column = dX row) into 32 x 32 bf16 boxes; each unit also zero-fills its
// share of the row's dropped blocks (exact +0.0, gemm.hpp:184,193).
// Every kept element is the same 16-deep MMA chain over n in the same order as
// the 1-CTA sdd kernel's (only the operand roles of the products are swapped).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "sd_internal.h"
#include "sd_ptx.cuh"

namespace sd {
namespace {

constexpr int kJ = 2;                        // kept blocks per CTA per unit (MMAs per K=16 step)
constexpr int kABox = 128 * kBK * 2;         // 16 KB: one W block (128 rows) x 64 n
constexpr int kBBox = 64 * kBK * 2;          // 8 KB: this CTA's 64 dY rows x 64 n
constexpr int kStageBytes = kJ * kABox + kBBox;  // 40 KB
constexpr int kStagesT = 5;
constexpr int kEpiWarpsT = 4;
constexpr int kEpiBox = 32 * 32 * 2;         // 2 KB: 32 dX rows x 32 dX columns, bf16
constexpr int kThreadsT = 256;
constexpr int kTmemColsT = 512;              // two accumulator sets of kJ x 128 columns
constexpr int kOffEpiT = kStagesT * kStageBytes;
constexpr int kOffBarT = kOffEpiT + kEpiWarpsT * 2 * kEpiBox;
constexpr int kNumBarsT = 2 * kStagesT + 4;
constexpr int kOffTmemSlotT = kOffBarT + kNumBarsT * 8;
constexpr int kSmemT = kOffTmemSlotT + 16 + 1024;
static_assert(kSmemT <= 232448, "shared memory budget");
static_assert(kStageBytes % 1024 == 0 && kABox % 1024 == 0, "SW128 atoms stay 1024-byte aligned");

struct DxtArgs {
    int rows;         // M (dX rows)
    int cols;         // K_out (dX columns)
    int red;          // N (reduction)
    int R, C;         // mask grid (128 x 128 blocks)
    const int32_t* row_cnt;
    const int32_t* row_idx;  // [R][C]: kept ascending from the front, dropped from the back
    float scale;
    void* out;               // dX, bf16
    int no_wait;
    unsigned int* release;   // mask workspace release counter (+1 per CTA at exit)
};

__device__ __forceinline__ void tma_load_2sm_t(const void* tmap, uint64_t* bar, void* dst, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(ptx::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(ptx::smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void mma2_t(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void commit2_mc_t(uint64_t* bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                     "r"(ptx::smem_u32(bar)),
                 "h"(mask)
                 : "memory");
}
__device__ __forceinline__ void st_shared_u16(uint32_t addr, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}

// Units in order: unit u is group g = u - base of mask row `row`; a row of cnt
// kept blocks has max(1, ceil(cnt / (2 kJ))) units (a fully dropped row still
// gets one, for its zero fill). Walkers only move forward.
struct RowWalk {
    int row = 0, base = 0, n = -1, cnt = 0;
};
__device__ __forceinline__ bool row_walk(RowWalk& w, int u, const DxtArgs& P) {
    while (w.row < P.R) {
        if (w.n < 0) {
            w.cnt = __ldcg(P.row_cnt + w.row);
            w.n = max(1, (w.cnt + 2 * kJ - 1) / (2 * kJ));
        }
        if (u < w.base + w.n) return true;
        w.base += w.n;
        ++w.row;
        w.n = -1;
    }
    return false;
}
// MMAs of group g: slot j runs when CTA 0's block 2 kJ g + 2 j exists
__device__ __forceinline__ int unit_slots(int cnt, int g) { return min(kJ, max(0, (cnt - 2 * kJ * g + 1) / 2)); }

__global__ void __launch_bounds__(kThreadsT, 1) __cluster_dims__(2, 1, 1)
    sd_dxt_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmDy,
                  const __grid_constant__ CUtensorMap tmOut, const DxtArgs P) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    const uint32_t sbase = ptx::smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBarT);
    uint64_t* full_bar = bars;                 // leader only
    uint64_t* empty_bar = bars + kStagesT;     // each CTA
    uint64_t* tfull_bar = bars + 2 * kStagesT; // each CTA
    uint64_t* tempty_bar = tfull_bar + 2;      // leader only
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmemSlotT);

    const uint32_t warp = threadIdx.x / 32;
    const uint32_t lane = ptx::lane_id();
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int cluster_id = blockIdx.x / 2, n_clusters = gridDim.x / 2;
    const int nst = P.red / kBK;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmW);
        ptx::prefetch_tmap(&tmDy);
        ptx::prefetch_tmap(&tmOut);
        for (int i = 0; i < kStagesT; ++i) {
            ptx::mbar_init(full_bar + i, 2);  // leader's expect_tx arrive + peer's remote arrive
            ptx::mbar_init(empty_bar + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(tfull_bar + i, 1);
            ptx::mbar_init(tempty_bar + i, 2 * kEpiWarpsT);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(tmem_slot)),
                     "n"(kTmemColsT)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (!P.no_wait) ptx::pdl_wait();
    ptx::pdl_launch_dependents();

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            RowWalk wk;
            for (int u = cluster_id; row_walk(wk, u, P); u += n_clusters) {
                const int g = u - wk.base;
                const int js = unit_slots(wk.cnt, g);
                if (js == 0) continue;
                const int32_t* lst = P.row_idx + static_cast<int64_t>(wk.row) * P.C;
                int wrow[kJ];
#pragma unroll
                for (int j = 0; j < kJ; ++j) {
                    const int li = 2 * kJ * g + 2 * j + static_cast<int>(rank);
                    // a missing block: a box wholly past W's last row (TMA zero fill, no traffic)
                    wrow[j] = (j < js && li < wk.cnt) ? __ldcg(lst + li) * 128 : P.cols;
                }
                const int yrow = wk.row * 128 + 64 * static_cast<int>(rank);
                for (int s = 0; s < nst; ++s) {
                    ptx::mbar_wait(empty_bar + stage, phase ^ 1);
                    uint8_t* st = smem + stage * kStageBytes;
                    if (leader)
                        ptx::mbar_arrive_expect_tx(full_bar + stage, 2 * (js * kABox + kBBox));
                    else
                        ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(full_bar + stage), 0));
#pragma unroll
                    for (int j = 0; j < kJ; ++j)
                        if (j < js) tma_load_2sm_t(&tmW, full_bar + stage, st + j * kABox, s * kBK, wrow[j]);
                    tma_load_2sm_t(&tmDy, full_bar + stage, st + kJ * kABox, s * kBK, yrow);
                    if (++stage == kStagesT) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader only) =====================
        if (leader && lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t acc_iter = 0;
            const uint32_t idesc = ptx::make_idesc_bf16(256, 128, false, false);
            RowWalk wk;
            for (int u = cluster_id; row_walk(wk, u, P); u += n_clusters) {
                const int js = unit_slots(wk.cnt, u - wk.base);
                if (js == 0) continue;
                const uint32_t acc = acc_iter & 1;
                const uint32_t acc_phase = (acc_iter >> 1) & 1;
                ++acc_iter;
                ptx::mbar_wait(tempty_bar + acc, acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * (kJ * 128);
                for (int s = 0; s < nst; ++s) {
                    ptx::mbar_wait(full_bar + stage, phase);
                    ptx::tc_fence_after();
                    const uint32_t st = sbase + stage * kStageBytes;
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        const uint64_t bd = ptx::make_sw128_desc(st + kJ * kABox + k * 32, 0, 1024);
#pragma unroll
                        for (int j = 0; j < kJ; ++j) {
                            if (j < js) {
                                const uint64_t ad = ptx::make_sw128_desc(st + j * kABox + k * 32, 0, 1024);
                                mma2_t(d_tmem + j * 128, ad, bd, idesc, (s > 0 || k > 0) ? 1u : 0u);
                            }
                        }
                    }
                    commit2_mc_t(empty_bar + stage, 0x3);
                    if (++stage == kStagesT) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                commit2_mc_t(tfull_bar + acc, 0x3);
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (both CTAs) =====================
        // TMEM lane = dX column (this CTA's W block rows), TMEM column = dX row
        const uint32_t q = warp & 3;  // lanes 32q .. 32q+31: dX columns c*128 + 32q + lane
        const uint32_t ebuf_addr = sbase + kOffEpiT + q * 2 * kEpiBox;
        uint8_t* ebuf = smem + kOffEpiT + q * 2 * kEpiBox;
        uint32_t bi = 0, acc_iter = 0;
        RowWalk wk;
        for (int u = cluster_id; row_walk(wk, u, P); u += n_clusters) {
            const int g = u - wk.base;
            const int32_t* lst = P.row_idx + static_cast<int64_t>(wk.row) * P.C;
            // this CTA's share of the row's dropped blocks (from the list tail)
            {
                const int ndrop = P.C - wk.cnt;
                const int per = (ndrop + wk.n - 1) / wk.n;
                const int z0 = g * per, z1 = min(ndrop, z0 + per);
                char* base = static_cast<char*>(P.out);
                for (int li = z0 + static_cast<int>(rank); li < z1; li += 2) {
                    const int cb = __ldcg(lst + P.C - 1 - li);
                    // 32 rows of this warp x 128 columns x 2 B = 256 B per row
                    for (int idx = lane; idx < 32 * 16; idx += 32) {
                        const int r = idx >> 4, ch = idx & 15;
                        ptx::st_global_v4_zero(base + (static_cast<int64_t>(wk.row * 128 + 32 * q + r) * P.cols +
                                                       cb * 128) * 2 + ch * 16);
                    }
                }
            }
            const int js = unit_slots(wk.cnt, g);
            if (js == 0) continue;
            const uint32_t acc = acc_iter & 1;
            const uint32_t acc_phase = (acc_iter >> 1) & 1;
            ++acc_iter;
            ptx::mbar_wait(tfull_bar + acc, acc_phase);
            ptx::tc_fence_after();
            for (int j = 0; j < js; ++j) {
                const int li = 2 * kJ * g + 2 * j + static_cast<int>(rank);
                const bool valid = li < wk.cnt;
                const int cb = valid ? __ldcg(lst + li) : 0;
                for (int i = 0; i < 4; ++i) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(tmem_base + ((32 * q) << 16) + acc * (kJ * 128) + j * 128 + i * 32, v);
                    ptx::tmem_ld_wait();
                    if (j == js - 1 && i == 3) {
                        // accumulator set drained: the leader may reuse it
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(tempty_bar + acc), 0));
                    }
                    if (!valid) continue;
                    if (lane == 0) ptx::bulk_wait_group_read<1>();
                    __syncwarp();
                    // v[t] = dX[row 32 i + t][column 32 q + lane] of this block: transpose
                    // into a 32 x 32 box, row t at t * 64 bytes
                    const uint32_t box = ebuf_addr + bi * kEpiBox;
#pragma unroll
                    for (int t = 0; t < 32; ++t) {
                        const __nv_bfloat16 h = __float2bfloat16_rn(__uint_as_float(v[t]) * P.scale);
                        st_shared_u16(box + t * 64 + lane * 2, *reinterpret_cast<const uint16_t*>(&h));
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_2d(&tmOut, ebuf + bi * kEpiBox, cb * 128 + 32 * static_cast<int>(q),
                                          wk.row * 128 + 32 * i);
                        ptx::bulk_commit_group();
                    }
                    bi ^= 1;
                }
            }
        }
        if (lane == 0) ptx::bulk_wait_group<0>();
        __syncwarp();
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemColsT) : "memory");
    if (P.release && threadIdx.x == 0) {
        __threadfence();
        atomicAdd(P.release, 1u);
    }
}

}  // namespace

bool dxt_supported(const GemmArgs& dx) {
    return (dx.flags & kFlagSDD) && !(dx.flags & (kFlagF32 | kFlagBMN | kFlagPairs)) && dx.out_row_blk == 128 &&
           dx.out_col_blk == 128 && dx.rows_out % 128 == 0 && dx.cols_out % 128 == 0 && dx.red % kBK == 0 &&
           dx.list_cnt && dx.list_idx && dx.list_stride == dx.mask_cols;
}

// dx: a prepared sdd call of the layer's dX (prep_layer_dx: A = dY K-major, B =
// W K-major). The 2-CTA kernel needs its own maps: W rows as the M operand
// (the same 64 x 128 box as tb), dY rows in 64-row halves, and the transposed
// 32 x 32 output box (no swizzle).
void launch_dxt(const GemmCall& dx, const void* dy, const void* w, cudaStream_t s, bool no_wait) {
    const GemmArgs& a = dx.args;
    if (!dxt_supported(a)) fail(SD_ERUNTIME, "launch_dxt: unsupported dX problem");
    configure_once_per_device(3, [] {
        check_cuda(cudaFuncSetAttribute(sd_dxt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemT),
                   "cudaFuncSetAttribute(dxt smem)");
    });
    const CUtensorMap tmW = dx.tb;  // W [cols_out rows][red], box 64 x 128
    const CUtensorMap tmDy = make_tmap_2d(dy, false, static_cast<uint64_t>(a.red), static_cast<uint64_t>(a.rows_out),
                                          64, 64);
    const CUtensorMap tmOut = make_tmap_2d_noswizzle(a.out, false, static_cast<uint64_t>(a.cols_out),
                                                     static_cast<uint64_t>(a.rows_out), 32, 32);
    (void)w;
    DxtArgs P;
    std::memset(&P, 0, sizeof P);
    P.rows = a.rows_out;
    P.cols = a.cols_out;
    P.red = a.red;
    P.R = a.rows_out / 128;
    P.C = a.mask_cols;
    P.row_cnt = a.list_cnt;
    P.row_idx = a.list_idx;
    P.scale = a.scale;
    P.out = a.out;
    P.no_wait = no_wait && !(tuning() & kTuneNoEarlyBackward) ? 1 : 0;
    P.release = dx.release;
    const int max_units = P.R * std::max(1, (P.C + 2 * kJ - 1) / (2 * kJ));
    const int clusters = std::min(max_units, num_sms() / 2);
    if (clusters <= 0) return;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(kThreadsT);
    cfg.dynamicSmemBytes = kSmemT;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    check_cuda(cudaLaunchKernelEx(&cfg, sd_dxt_kernel, tmW, tmDy, tmOut, P), "sd_dxt_kernel launch");
    note_launch();
    if (dx.release) mask_note_readers(dx.release, static_cast<int>(cfg.gridDim.x), s);
}

}  // namespace sd
