// sd_gemm.cu — the SparseDrop tensor-core GEMMs for sm_100a.
//
// One persistent, warp-specialised tcgen05 kernel, templated on operand
// major-ness and on how the block mask enters, serves every GEMM of the path:
//
//   dsd (reduction-block skipping, gemm.hpp:133-170):
//     forward  Y  = s (X (.) m) W      A = X  K-major, B = W  MN-major, row lists
//     dW       dW = s (X (.) m)^T dY   A = X  MN-major, B = dY MN-major, column lists
//     dense    (list == null: every reduction block)
//   sdd (output-block skipping, gemm.hpp:176-213):
//     dX       dX = s (dY W^T) (.) m   A = dY K-major, B = W  K-major, row lists
//              (kept output blocks packed two per 256-wide unit; dropped = +0.0)
//
// Tile: 128 output rows (one tcgen05 M=128 MMA, TMEM lanes = rows) x up to 256
// output columns (MMA N chosen per tile at run time: 256, or 128 for a ragged
// edge / a half-kept sdd pair). Reduction in 64-element stages = one 128-byte
// swizzle atom; a 128-wide mask block is two stages (the paper's retile(1,2),
// PAPER.md:149-151). Only kept reduction blocks are ever loaded by TMA.
//
// Warp roles (256 threads, 1 CTA per SM, grid = min(units, #SMs)):
//   warp 0      TMA producer (one lane): 4-stage smem ring, mbarrier full/empty
//   warp 1      MMA issuer (one lane): tcgen05.mma -> TMEM, tcgen05.commit
//   warp 2      TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warps 4..7  epilogue: tcgen05.ld -> scale -> bf16/fp32 -> swizzled smem
//               -> TMA store; all-dropped tiles written as +0.0 directly.
// Two TMEM accumulators let the epilogue of tile i overlap the MMAs of i+1.
// Scheduling is dynamic: the producer steals units from a global atomic counter
// (units ordered heaviest first, grouped for L2 reuse), decodes them (list
// lookups) and hands the decoded unit to the MMA and epilogue roles through a
// shared-memory ring; zero-work units skip TMEM entirely.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "sd_internal.h"
#include "sd_ptx.cuh"

namespace sd {
namespace {

constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK * 2;  // 16 KB per stage
constexpr int kBBytes = kBN * kBK * 2;  // 32 KB per stage
constexpr int kEpiWarps = 4;
constexpr int kEpiBufBytes = 32 * 128;  // one warp's 32 rows x 128 B store box
constexpr int kThreads = 256;
constexpr int kTmemCols = 512;

constexpr int kOffA = 0;
constexpr int kOffB = kOffA + kStages * kABytes;
constexpr int kOffEpi = kOffB + kStages * kBBytes;
constexpr int kOffBar = kOffEpi + kEpiWarps * 2 * kEpiBufBytes;
constexpr int kGroupRows = 16;  // tile rows per rasterization group
constexpr int kSchedDepth = 4;  // unit-index ring between the producer and the consumers
constexpr int kNumBars = 2 * kStages + 4 + 2 * kSchedDepth;
constexpr int kOffTmemSlot = kOffBar + kNumBars * 8;
constexpr int kOffSched = kOffTmemSlot + 16;
constexpr int kUnitInts = 12;  // sizeof(Unit) / 4
constexpr int kSmemBytes = kOffSched + 4 * kUnitInts * kSchedDepth + 1024;  // + alignment slack

static_assert(kSmemBytes <= 232448, "shared memory budget");
static_assert(kUnitInts * 4 == 48, "Unit layout");

struct Unit {
    int row0;      // first output row; -1 = end of work
    int list_row;  // mask row (list index) of this tile row
    int n0;        // first output column (dsd)
    int n_eff;     // MMA N; 0 => no MMA work
    int nstages;   // reduction stages
    int nslots;    // sdd: kept output blocks in this unit
    int slot_blk[2];
    int nzero;     // sdd: dropped output blocks in this unit
    int zero_blk[2];
};

template <bool SDD>
__device__ __forceinline__ Unit decode_unit(const GemmArgs& a, int u) {
    Unit t;
    // Grouped rasterization: tile rows (sorted heaviest first) are taken in
    // groups of kGroupRows; inside a group units go column-unit-major. The
    // CTAs in flight then share a few operand column/row slabs (L2 reuse), heavy
    // groups still go first, and for sdd the units carrying MMA work (kept
    // blocks are packed into the low column units) precede the zero-fill-only
    // units of their group.
    const int g = u / (kGroupRows * a.n_col_units);
    const int rem_u = u - g * kGroupRows * a.n_col_units;
    const int rows_in_group = min(kGroupRows, a.n_row_tiles - g * kGroupRows);
    const int cu = rem_u / rows_in_group;
    const int i = g * kGroupRows + (rem_u - cu * rows_in_group);
    const int rt = a.row_order ? __ldg(a.row_order + i) : i;
    t.row0 = rt * kBM;
    t.list_row = t.row0 / a.out_row_blk;
    t.nslots = 0;
    t.nzero = 0;
    if constexpr (!SDD) {
        t.n0 = cu * kBN;
        const int rem = a.cols_out - t.n0;
        t.n_eff = rem < kBN ? rem : kBN;
        const int cnt = a.list_cnt ? __ldg(a.list_cnt + t.list_row) : a.red / a.red_blk;
        t.nstages = cnt * (a.red_blk / kBK);
        if (cnt == 0) t.n_eff = 0;
    } else {
        // Pack the row's KEPT output blocks (compacted list, ascending) into
        // 256-wide units, so every unit but the row's last runs a full N=256 MMA;
        // the same unit index also zero-fills the row's DROPPED blocks (kept at
        // the tail of the list by the mask kernel).
        const int per_unit = kBN / a.out_col_blk;
        const int cnt = __ldg(a.list_cnt + t.list_row);
        const int ndrop = a.mask_cols - cnt;
        const int32_t* row = a.list_idx + static_cast<int64_t>(t.list_row) * a.list_stride;
        t.n0 = 0;
        for (int j = 0; j < per_unit; ++j) {
            const int li = cu * per_unit + j;
            if (li < cnt) t.slot_blk[t.nslots++] = __ldg(row + li);
            if (li < ndrop) t.zero_blk[t.nzero++] = __ldg(row + a.mask_cols - 1 - li);
        }
        t.n_eff = t.nslots * a.out_col_blk;
        t.nstages = a.red / kBK;
    }
    return t;
}

// Zero a 32-row x `ncols` slab of the output with coalesced 16-byte stores.
template <bool OUT_F32>
__device__ __forceinline__ void zero_rows(const GemmArgs& a, int row_first, int col0, int ncols,
                                          uint32_t lane) {
    constexpr int kElem = OUT_F32 ? 4 : 2;
    const int chunks_per_row = ncols * kElem / 16;
    const int total = 32 * chunks_per_row;
    char* base = static_cast<char*>(a.out);
    for (int idx = lane; idx < total; idx += 32) {
        const int r = idx / chunks_per_row;
        const int ch = idx - r * chunks_per_row;
        char* p = base + (static_cast<int64_t>(row_first + r) * a.cols_out + col0) * kElem + ch * 16;
        ptx::st_global_v4_zero(p);
    }
}

template <bool A_MN, bool B_MN, bool SDD, bool OUT_F32>
__global__ void __launch_bounds__(kThreads, 1)
    sd_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmOut, const GemmArgs args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    const uint32_t sbase = ptx::smem_u32(smem);

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = bars + kStages;
    uint64_t* tfull_bar = bars + 2 * kStages;
    uint64_t* tempty_bar = bars + 2 * kStages + 2;
    uint64_t* sfull_bar = bars + 2 * kStages + 4;
    uint64_t* sempty_bar = sfull_bar + kSchedDepth;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmemSlot);
    // ring of decoded units: the producer decodes (global loads), the MMA and
    // epilogue roles read the decoded unit from shared memory
    Unit* sched_unit = reinterpret_cast<Unit*>(smem + kOffSched);

    const uint32_t warp = threadIdx.x / 32;
    const uint32_t lane = ptx::lane_id();
    const int num_units = args.n_row_tiles * args.n_col_units;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        ptx::prefetch_tmap(&tmOut);
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(full_bar + i, 1);
            ptx::mbar_init(empty_bar + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(tfull_bar + i, 1);
            ptx::mbar_init(tempty_bar + i, kEpiWarps);
        }
        for (int i = 0; i < kSchedDepth; ++i) {
            ptx::mbar_init(sfull_bar + i, 1);
            ptx::mbar_init(sempty_bar + i, 1 + kEpiWarps);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // Everything above overlapped the previous kernel's tail (PDL); from here on
    // we read its outputs (mask lists, operands), so wait for it to complete.
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_normal();
            int stage = 0;
            uint32_t phase = 0;
            int sslot = 0;
            uint32_t sphase = 0;
            // Dynamic persistent scheduling: first unit = blockIdx.x, then work
            // stealing through a global atomic counter (units are ordered
            // heaviest first, so this is greedy longest-processing-time).
            int u = blockIdx.x;
            int nxt = u < num_units ? static_cast<int>(gridDim.x) + static_cast<int>(atomicAdd(args.sched, 1u))
                                    : num_units;
            Unit t;
            if (u < num_units) t = decode_unit<SDD>(args, u); else t.row0 = -1;
            while (true) {
                ptx::mbar_wait(sempty_bar + sslot, sphase ^ 1);
                sched_unit[sslot] = t;
                ptx::mbar_arrive(sfull_bar + sslot);
                if (++sslot == kSchedDepth) {
                    sslot = 0;
                    sphase ^= 1;
                }
                if (t.row0 < 0) break;
                // decode the next unit now: its global loads (and the atomic
                // for the one after) overlap this unit's TMA stream
                const Unit cur = t;
                u = nxt;
                if (u < num_units) {
                    nxt = static_cast<int>(gridDim.x) + static_cast<int>(atomicAdd(args.sched, 1u));
                    t = decode_unit<SDD>(args, u);
                } else {
                    t.row0 = -1;
                }
                if (cur.n_eff == 0) continue;
                const uint32_t tx_bytes = kABytes + cur.n_eff * kBK * 2;
                const int spb = args.red_blk / kBK;
                const int32_t* lst =
                    args.list_idx ? args.list_idx + static_cast<int64_t>(cur.list_row) * args.list_stride : nullptr;
                // kept-block index prefetched one block ahead (off the TMA issue path)
                int kb_next = (!SDD && lst) ? __ldg(lst) : 0;
                int kb = 0;
                for (int s = 0, li = 0, sub = 0; s < cur.nstages; ++s) {
                    int r0;
                    if constexpr (!SDD) {
                        if (sub == 0) {
                            kb = lst ? kb_next : li;
                            if (lst && li + 1 < cur.nstages / spb) kb_next = __ldg(lst + li + 1);
                        }
                        r0 = kb * args.red_blk + sub * kBK;
                        if (++sub == spb) {
                            sub = 0;
                            ++li;
                        }
                    } else {
                        r0 = s * kBK;
                    }
                    ptx::mbar_wait(empty_bar + stage, phase ^ 1);
                    uint64_t* fb = full_bar + stage;
                    ptx::mbar_arrive_expect_tx(fb, tx_bytes);
                    uint8_t* sA = smem + kOffA + stage * kABytes;
                    uint8_t* sB = smem + kOffB + stage * kBBytes;
                    if constexpr (!A_MN) {
                        ptx::tma_load_2d(&tmA, fb, sA, r0, cur.row0, pol);
                    } else {
                        ptx::tma_load_2d(&tmA, fb, sA, cur.row0, r0, pol);
                        ptx::tma_load_2d(&tmA, fb, sA + 8192, cur.row0 + 64, r0, pol);
                    }
                    if constexpr (!SDD) {
                        if constexpr (!B_MN) {
                            for (int j = 0; j < cur.n_eff / 128; ++j)
                                ptx::tma_load_2d(&tmB, fb, sB + j * 16384, r0, cur.n0 + 128 * j, pol);
                        } else {
                            for (int j = 0; j < cur.n_eff / 64; ++j)
                                ptx::tma_load_2d(&tmB, fb, sB + j * 8192, cur.n0 + 64 * j, r0, pol);
                        }
                    } else {
                        for (int sl = 0; sl < cur.nslots; ++sl) {
                            const int col0 = cur.slot_blk[sl] * args.out_col_blk;
                            if constexpr (!B_MN) {
                                const int per = args.out_col_blk / 128;
                                for (int j = 0; j < per; ++j)
                                    ptx::tma_load_2d(&tmB, fb, sB + (sl * per + j) * 16384, r0,
                                                     col0 + 128 * j, pol);
                            } else {
                                const int per = args.out_col_blk / 64;
                                for (int j = 0; j < per; ++j)
                                    ptx::tma_load_2d(&tmB, fb, sB + (sl * per + j) * 8192,
                                                     col0 + 64 * j, r0, pol);
                            }
                        }
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t acc_iter = 0;
            int sslot = 0;
            uint32_t sphase = 0;
            while (true) {
                ptx::mbar_wait(sfull_bar + sslot, sphase);
                const Unit t = sched_unit[sslot];
                ptx::mbar_arrive(sempty_bar + sslot);
                if (++sslot == kSchedDepth) {
                    sslot = 0;
                    sphase ^= 1;
                }
                if (t.row0 < 0) break;
                if (t.n_eff == 0) continue;
                const uint32_t acc = acc_iter & 1;
                const uint32_t acc_phase = (acc_iter >> 1) & 1;
                ++acc_iter;
                ptx::mbar_wait(tempty_bar + acc, acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * kBN;
                const uint32_t idesc = ptx::make_idesc_bf16(kBM, t.n_eff, A_MN, B_MN);
                for (int s = 0; s < t.nstages; ++s) {
                    ptx::mbar_wait(full_bar + stage, phase);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = sbase + kOffA + stage * kABytes;
                    const uint32_t b_addr = sbase + kOffB + stage * kBBytes;
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        const uint64_t ad = A_MN ? ptx::make_sw128_desc(a_addr + k * 2048, 8192, 1024)
                                                 : ptx::make_sw128_desc(a_addr + k * 32, 0, 1024);
                        const uint64_t bd = B_MN ? ptx::make_sw128_desc(b_addr + k * 2048, 8192, 1024)
                                                 : ptx::make_sw128_desc(b_addr + k * 32, 0, 1024);
                        ptx::mma_bf16_ss(d_tmem, ad, bd, idesc, (s > 0 || k > 0) ? 1u : 0u);
                    }
                    ptx::mma_commit(empty_bar + stage);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit(tfull_bar + acc);
                if (args.counters)
                    atomicAdd(args.counters + t.row0 / kBM,
                              static_cast<unsigned long long>(t.nstages / 2) * (t.n_eff / 128));
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue =====================
        const uint32_t q = warp & 3;  // TMEM lane quarter == output row quarter
        uint8_t* ebuf = smem + kOffEpi + q * 2 * kEpiBufBytes;
        const uint32_t ebuf_addr = sbase + kOffEpi + q * 2 * kEpiBufBytes;
        uint32_t bi = 0;
        uint32_t acc_iter = 0;
        constexpr int kChunkCols = OUT_F32 ? 32 : 64;  // 128 bytes of output per row
        int sslot = 0;
        uint32_t sphase = 0;
        while (true) {
            ptx::mbar_wait(sfull_bar + sslot, sphase);
            const Unit t = sched_unit[sslot];
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(sempty_bar + sslot);
            if (++sslot == kSchedDepth) {
                sslot = 0;
                sphase ^= 1;
            }
            if (t.row0 < 0) break;
            const int row_first = t.row0 + 32 * q;
            if constexpr (SDD) {
                for (int z = 0; z < t.nzero; ++z)
                    zero_rows<OUT_F32>(args, row_first, t.zero_blk[z] * args.out_col_blk,
                                       args.out_col_blk, lane);
            }
            if (t.n_eff == 0) {
                if constexpr (!SDD) {
                    const int rem = args.cols_out - t.n0;
                    zero_rows<OUT_F32>(args, row_first, t.n0, rem < kBN ? rem : kBN, lane);
                }
                continue;
            }
            const uint32_t acc = acc_iter & 1;
            const uint32_t acc_phase = (acc_iter >> 1) & 1;
            ++acc_iter;
            ptx::mbar_wait(tfull_bar + acc, acc_phase);
            ptx::tc_fence_after();
            const int nchunks = t.n_eff / kChunkCols;
            for (int c = 0; c < nchunks; ++c) {
                const uint32_t taddr = tmem_base + ((32 * q) << 16) + acc * kBN + c * kChunkCols;
                uint32_t v[kChunkCols];
                ptx::tmem_ld_32x32b_x32(taddr, v);
                if constexpr (!OUT_F32) ptx::tmem_ld_32x32b_x32(taddr + 32, v + 32);
                ptx::tmem_ld_wait();
                if (c == nchunks - 1) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(tempty_bar + acc);
                }
                // staging buffer bi must no longer be read by the TMA store issued 2 chunks ago
                if (lane == 0) ptx::bulk_wait_group_read<1>();
                __syncwarp();
                const uint32_t row_addr = ebuf_addr + bi * kEpiBufBytes + lane * 128;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    uint32_t w0, w1, w2, w3;
                    if constexpr (OUT_F32) {
                        w0 = __float_as_uint(__uint_as_float(v[4 * j + 0]) * args.scale);
                        w1 = __float_as_uint(__uint_as_float(v[4 * j + 1]) * args.scale);
                        w2 = __float_as_uint(__uint_as_float(v[4 * j + 2]) * args.scale);
                        w3 = __float_as_uint(__uint_as_float(v[4 * j + 3]) * args.scale);
                    } else {
                        const float* f = reinterpret_cast<const float*>(v) + 8 * j;
                        w0 = ptx::pack_bf16x2(f[0] * args.scale, f[1] * args.scale);
                        w1 = ptx::pack_bf16x2(f[2] * args.scale, f[3] * args.scale);
                        w2 = ptx::pack_bf16x2(f[4] * args.scale, f[5] * args.scale);
                        w3 = ptx::pack_bf16x2(f[6] * args.scale, f[7] * args.scale);
                    }
                    ptx::st_shared_v4(row_addr + ((j ^ (lane & 7)) << 4), w0, w1, w2, w3);
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    int col;
                    if constexpr (SDD) {
                        const int tcol = c * kChunkCols;
                        const int sl = tcol / args.out_col_blk;
                        col = t.slot_blk[sl] * args.out_col_blk + (tcol - sl * args.out_col_blk);
                    } else {
                        col = t.n0 + c * kChunkCols;
                    }
                    ptx::tma_store_2d(&tmOut, ebuf + bi * kEpiBufBytes, col, row_first);
                    ptx::bulk_commit_group();
                }
                bi ^= 1;
            }
        }
        if (lane == 0) ptx::bulk_wait_group<0>();
        __syncwarp();
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc<kTmemCols>(tmem_base);
    if (threadIdx.x == 0) {
        // last CTA out re-arms the scheduler slot for the next launch
        __threadfence();
        if (atomicAdd(args.sched + 1, 1u) == gridDim.x - 1) {
            args.sched[0] = 0u;
            args.sched[1] = 0u;
            __threadfence();
        }
    }
}

template <bool A_MN, bool B_MN, bool SDD, bool OUT_F32>
void launch_impl(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tout,
                 const GemmArgs& args, cudaStream_t s) {
    auto kern = sd_gemm_kernel<A_MN, B_MN, SDD, OUT_F32>;
    static bool configured = false;  // per instantiation; attribute is per-function
    if (!configured) {
        check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes),
                   "cudaFuncSetAttribute(max dynamic smem)");
        configured = true;
    }
    const int units = args.n_row_tiles * args.n_col_units;
    const int grid = units < num_sms() ? units : num_sms();
    if (grid <= 0) return;
    GemmArgs a = args;
    a.sched = sched_slot();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    check_cuda(cudaLaunchKernelEx(&cfg, kern, ta, tb, tout, a), "sd_gemm_kernel launch");
    check_cuda(cudaGetLastError(), "sd_gemm_kernel launch");
    note_launch();
}

}  // namespace

void launch_gemm(bool a_mn, bool b_mn, GemmKind kind, bool out_f32, const CUtensorMap& ta,
                 const CUtensorMap& tb, const CUtensorMap& tout, const GemmArgs& args,
                 cudaStream_t s) {
    const bool sdd = kind == GemmKind::sdd;
#define SD_DISPATCH(AM, BM_, SD_, F32)                                                    \
    if (a_mn == AM && b_mn == BM_ && sdd == SD_ && out_f32 == F32)                        \
        return launch_impl<AM, BM_, SD_, F32>(ta, tb, tout, args, s);
    // dsd / dense forward (X K-major, W MN-major)
    SD_DISPATCH(false, true, false, false)
    SD_DISPATCH(false, true, false, true)
    // dsd dW (X^T MN-major, dY MN-major) and dense x^T dy
    SD_DISPATCH(true, true, false, false)
    SD_DISPATCH(true, true, false, true)
    // dense dy W^T (both K-major)
    SD_DISPATCH(false, false, false, false)
    SD_DISPATCH(false, false, false, true)
    // sdd dX in the layer (dY K-major, W K-major)
    SD_DISPATCH(false, false, true, false)
    SD_DISPATCH(false, false, true, true)
    // sdd reference form (a K-major, b row-major = MN-major)
    SD_DISPATCH(false, true, true, false)
    SD_DISPATCH(false, true, true, true)
#undef SD_DISPATCH
    fail(SD_EINVAL, "unsupported GEMM operand layout combination");
}

}  // namespace sd
