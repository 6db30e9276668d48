// sd_gemm2.cu — the 2-CTA (cta_group::2) tcgen05 GEMM for dense-mask work.
//
// A CTA pair (cluster of 2, one TPC) computes a 256 x 256 output tile with
// one M=256 / N=256 tcgen05.mma per K=16 step issued by the leader CTA:
//   CTA r holds A rows [128 r, 128 r + 128) and B columns [128 r, 128 r + 128)
//   of the tile, so each SM ingests 32 KB per 64-deep stage instead of the
//   1-CTA kernel's 48 KB for the same MACs per SM — the per-SM TMA ingress
//   (~80 B/clk, profiles/r01_load_path_diag.txt) stops being the bound.
// Pair protocol:
//   full barrier    leader only; both CTAs' TMAs complete_tx on it (peer bit
//                   cleared), the peer adds a remote arrive
//   empty barrier   each CTA; the leader's commit multicasts to both
//   TMEM full       each CTA; the leader's commit multicasts to both
//   TMEM empty      leader only; all 8 epilogue warps of the pair arrive
// Row-pair (biclique) sdd mode, kFlagPairs (the dX of a layer at mid p): for
// 128-row mask rows 2i and 2i+1, the output column blocks BOTH keep are taken in
// ascending pairs (c_a, c_b); each pair is one 256 x 256 unit — CTA 0 computes
// rows 2i, CTA 1 rows 2i+1, both over B = W rows of blocks c_a (CTA 0's half)
// and c_b (CTA 1's half) — so a fraction (1-p) of dX's kept work runs at the
// pair's 16 KB of operands per 1M MACs instead of the 1-CTA sdd tile's 24 KB.
// The remaining kept blocks (and the zero fill of the dropped ones) are the
// 1-CTA sdd kernel's (sd_gemm.cu, kFlagPairs: remainder lists). Units are
// enumerated from the mask words on the fly (pair_walk below). Every kept
// block is reduced over the same 64-deep stages in the same order as in the
// 1-CTA kernel: bit-identical.
// Union mode (dsd with a list per 128-row block): the pair's two row blocks
// walk the UNION of their kept lists; a CTA whose own row dropped a block
// loads an all-out-of-bounds box instead (TMA zero fill, no memory traffic), so
// the dropped block still contributes exact zeros (no wrong results, only
// redundant MMA work) and the accumulation order of every kept product is the
// 1-CTA kernel's.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "sd_internal.h"
#include "sd_ptx.cuh"

namespace sd {
namespace {

constexpr int kHalfBytes = 128 * kBK * 2;  // 16 KB: one CTA's half of A or B per stage
constexpr int kEpiWarps = 4;
constexpr int kEpiBufBytes = 32 * 128;
constexpr int kThreads = 256;
constexpr int kTmemCols = 512;
constexpr int kTile = 256;  // pair tile rows (and columns of the narrow tile)
constexpr int kMaxOwnUnits = 512;  // static smem: keep bits of a CTA's units (kFlagOutMask)

// Pair-tile shapes.
//   narrow: 256 x 256 per pair, one M=256/N=256 MMA per K=16 step; each CTA
//           ingests 32 KB per 64-deep stage for 2M MACs (16 KB / 1M); two
//           256-column TMEM accumulators (tile i's epilogue overlaps tile i+1).
//   WIDE:   256 x 512 per pair, two N=256 MMAs per K=16 step sharing the A
//           tile; each CTA ingests 48 KB per stage for 4M MACs (12 KB / 1M, the
//           shape cuBLAS uses for large bf16 GEMMs on this part: 256x256 per
//           CTA, 4 x 48 KB stages). One 512-column accumulator whose two halves
//           are released to the next tile one by one as the epilogue drains them.
template <bool W>
struct K2Cfg {
    static constexpr int kStages = W ? 4 : 6;
    static constexpr int kBSlots = W ? 2 : 1;  // 16 KB B boxes per stage per CTA
    static constexpr int kTileN = W ? 512 : 256;
    static constexpr int kOffA = 0;
    static constexpr int kOffB = kOffA + kStages * kHalfBytes;
    static constexpr int kOffEpi = kOffB + kStages * kBSlots * kHalfBytes;
    static constexpr int kOffBar = kOffEpi + kEpiWarps * 2 * kEpiBufBytes;
    static constexpr int kNumBars = 2 * kStages + 4;
    static constexpr int kOffTmemSlot = kOffBar + kNumBars * 8;
    static constexpr int kSmem = kOffTmemSlot + 16 + 1024;
    static_assert(kSmem + kMaxOwnUnits <= 232448, "shared memory budget (dynamic + static own_bits)");
};

__device__ __forceinline__ void tma_load_2sm_3d(const void* tmap, uint64_t* bar, void* dst, int32_t c0, int32_t c1,
                                                int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(ptx::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(ptx::smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// 2-SM TMA load: completes tx on the LEADER's barrier (peer bit cleared)
__device__ __forceinline__ void tma_load_2sm(const void* tmap, uint64_t* bar, void* dst, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(ptx::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(ptx::smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void mma2_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                     "r"(ptx::smem_u32(bar)),
                 "h"(mask)
                 : "memory");
}

// Bits of mask row r (C <= 64 columns, bit c = column c), row-major LSB-first words.
__device__ __forceinline__ uint64_t row_bits(const uint64_t* words, int r, int C) {
    const int64_t b = static_cast<int64_t>(r) * C;
    const int sh = static_cast<int>(b & 63);
    uint64_t v = __ldcg(words + (b >> 6)) >> sh;
    if (sh + C > 64) v |= __ldcg(words + (b >> 6) + 1) << (64 - sh);
    return C == 64 ? v : (v & ((1ull << C) - 1));
}
// index of the n-th (0-based) set bit of v (v has more than n set bits)
__device__ __forceinline__ int nth_set_bit(uint64_t v, int n) {
    for (int i = 0; i < n; ++i) v &= v - 1;
    return __ffsll(static_cast<long long>(v)) - 1;
}

// Enumerates the row-pair units in order: unit u lies in pair row `row`, as its
// (u - base)-th pair of common kept columns. Walkers only move forward.
struct PairWalk {
    int row = 0, base = 0, cnt = -1;
    uint64_t common = 0;
};
__device__ __forceinline__ bool pair_walk(PairWalk& w, int u, const uint64_t* words, int n_pair_rows, int C) {
    while (w.row < n_pair_rows) {
        if (w.cnt < 0) {
            w.common = row_bits(words, 2 * w.row, C) & row_bits(words, 2 * w.row + 1, C);
            w.cnt = __popcll(w.common) / 2;
        }
        if (u < w.base + w.cnt) return true;
        w.base += w.cnt;
        ++w.row;
        w.cnt = -1;
    }
    return false;
}

struct Pair2Args {
    GemmArgs g;         // rows_out, cols_out, red, flags (kFlagAMN/BMN/F32), scale, out, list*, red_blk, out_row_blk
    int n_pair_rows;    // rows_out / 256
    int n_col_tiles;    // cols_out / 256
    // union mode: for each 256-row pair, the merged kept list with an owner mask
    const int32_t* pair_cnt;   // [n_pair_rows]
    const int32_t* pair_idx;   // [n_pair_rows][list_stride]: (block << 2) | owner_mask(bit0 = row 2i, bit1 = 2i+1)
    int pair_stride;
    int no_wait;  // skip griddepcontrol.wait (see launch_gemms)
    unsigned int* release;  // mask workspace read (kFlagOutMask words): +1 per CTA at exit
    int own_cap;            // units whose keep bits are read up front (<= kMaxOwnUnits; 0: per chunk)
};

template <bool W>
__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    sd_gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmOut, const Pair2Args P) {
    using C = K2Cfg<W>;
    constexpr int kStages2 = C::kStages;
    constexpr int kTileN = C::kTileN;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    const uint32_t sbase = ptx::smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* full_bar = bars;               // leader only
    uint64_t* empty_bar = bars + kStages2;   // each CTA
    uint64_t* tfull_bar = bars + 2 * kStages2;
    uint64_t* tempty_bar = bars + 2 * kStages2 + 2;  // leader only
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffTmemSlot);

    const GemmArgs& a = P.g;
    const uint32_t warp = threadIdx.x / 32;
    const uint32_t lane = ptx::lane_id();
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const bool a_mn = a.flags & kFlagAMN, b_mn = a.flags & kFlagBMN, f32 = a.flags & kFlagF32;
    const bool unioned = !W && P.pair_cnt != nullptr;
    const bool pairs = !W && (a.flags & kFlagPairs);  // row-pair sdd units (dX)
    const int num_units = P.n_pair_rows * P.n_col_tiles;
    const int cluster_id = blockIdx.x / 2, n_clusters = gridDim.x / 2;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        ptx::prefetch_tmap(&tmOut);
        for (int i = 0; i < kStages2; ++i) {
            ptx::mbar_init(full_bar + i, 2);  // leader's expect_tx arrive + peer's remote arrive
            ptx::mbar_init(empty_bar + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(tfull_bar + i, 1);
            ptx::mbar_init(tempty_bar + i, 2 * kEpiWarps);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(tmem_slot)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    __syncthreads();  // also a CTA barrier: compute-sanitizer racecheck does not treat barrier.cluster as one
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (!P.no_wait) ptx::pdl_wait();
    ptx::pdl_launch_dependents();

    // static schedule over pair units, heaviest pair rows first (pair rows are
    // ordered by the host/mask planner), column-tile-major within groups of 8
    auto decode = [&](int u, int& prow, int& ct) {
        constexpr int G = 8;
        const int g = u / (G * P.n_col_tiles);
        const int rem = u - g * G * P.n_col_tiles;
        const int rows_in_group = min(G, P.n_pair_rows - g * G);
        ct = rem / rows_in_group;
        prow = g * G + (rem - ct * rows_in_group);
    };

    // kFlagOutMask: this CTA's keep bits (its 128-row block x the tile's two or
    // four 128-column blocks) for every unit it will run, read once up front, so the
    // mask workspace is released now instead of at exit and the next mask
    // generation overlaps this grid (more than kMaxOwnUnits units: at exit)
    __shared__ uint8_t own_bits[kMaxOwnUnits];
    const int own_units = (num_units - cluster_id + n_clusters - 1) / n_clusters;
    const bool bits_up_front = !pairs && (a.flags & kFlagOutMask) && own_units <= P.own_cap;
    if (bits_up_front) {
        for (int k = threadIdx.x; k < own_units; k += kThreads) {
            int prow, ct;
            decode(cluster_id + k * n_clusters, prow, ct);
            constexpr int nb = kTileN / 128;
            const int64_t bit = static_cast<int64_t>(2 * prow + static_cast<int>(rank)) * a.mask_cols + nb * ct;
            uint32_t v = 0;
#pragma unroll
            for (int j = 0; j < nb; ++j) v |= static_cast<uint32_t>((__ldcg(a.words + ((bit + j) >> 6)) >> ((bit + j) & 63)) & 1ull) << j;
            own_bits[k] = static_cast<uint8_t>(v);
        }
        __syncthreads();
        if (P.release && threadIdx.x == 0) {
            __threadfence();
            atomicAdd(P.release, 1u);
        }
    }
    auto unit_stages = [&](int prow) -> int {
        if (unioned) return __ldg(P.pair_cnt + prow) * (a.red_blk / kBK);
        return a.red / kBK;
    };
    // next unit of this cluster: u -> pair row, column tile (dense/union) or the
    // two 128-column output blocks (row-pair mode); false past the last unit
    auto next_unit = [&](PairWalk& wk, int u, int& prow, int& ct, int& ca, int& cb) -> bool {
        if (!pairs) {
            if (u >= num_units) return false;
            decode(u, prow, ct);
            ca = 2 * ct;
            cb = 2 * ct + 1;
            return true;
        }
        if (!pair_walk(wk, u, a.words, P.n_pair_rows, a.mask_cols)) return false;
        prow = wk.row;
        ct = 0;
        const int j = u - wk.base;
        ca = nth_set_bit(wk.common, 2 * j);
        cb = nth_set_bit(wk.common, 2 * j + 1);
        return true;
    };

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            PairWalk wk;
            int prow, ct, ca, cb;
            for (int u = cluster_id; next_unit(wk, u, prow, ct, ca, cb); u += n_clusters) {
                const int nst = unit_stages(prow);
                const int row0 = prow * kTile + 128 * static_cast<int>(rank);  // this CTA's A rows
                // this CTA's B columns (per 256); row-pair mode: its output column block
                const int col0 = pairs ? (rank ? cb : ca) * 128 : ct * kTileN + 128 * static_cast<int>(rank);
                const int spb = a.red_blk / kBK;
                const int32_t* lst = unioned ? P.pair_idx + static_cast<int64_t>(prow) * P.pair_stride : nullptr;
                int entry = 0;
                for (int s = 0; s < nst; ++s) {
                    int r0;
                    bool own = true;
                    if (unioned) {
                        if (s % spb == 0) entry = __ldg(lst + s / spb);
                        r0 = (entry >> 2) * a.red_blk + (s % spb) * kBK;
                        own = (entry >> rank) & 1;
                    } else {
                        r0 = s * kBK;
                    }
                    ptx::mbar_wait(empty_bar + stage, phase ^ 1);
                    uint8_t* sA = smem + C::kOffA + stage * kHalfBytes;
                    uint8_t* sB = smem + C::kOffB + stage * C::kBSlots * kHalfBytes;
                    if (leader) {
                        // both CTAs' A and B halves (a dropped A half is a zero-filled box, same bytes)
                        ptx::mbar_arrive_expect_tx(full_bar + stage, (2 + 2 * C::kBSlots) * kHalfBytes);
                    } else {
                        ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(full_bar + stage), 0));
                    }
                    // own row dropped this block: load a box lying wholly past the last
                    // row instead; TMA fills it with exact zeros without touching memory
                    const int arow = own ? row0 : a.rows_out;
                    if (!a_mn) {
                        tma_load_2sm(&tmA, full_bar + stage, sA, r0, arow);
                    } else {
                        tma_load_2sm_3d(&tmA, full_bar + stage, sA, 0, r0, arow / 64);
                    }
#pragma unroll
                    for (int j = 0; j < C::kBSlots; ++j) {
                        if (!b_mn) {
                            tma_load_2sm(&tmB, full_bar + stage, sB + j * kHalfBytes, r0, col0 + 256 * j);
                        } else {
                            tma_load_2sm_3d(&tmB, full_bar + stage, sB + j * kHalfBytes, 0, r0, (col0 + 256 * j) / 64);
                        }
                    }
                    if (++stage == kStages2) {
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
            const uint32_t idesc = ptx::make_idesc_bf16(256, 256, a_mn, b_mn);
            const uint32_t a_step = a_mn ? 2048u : 32u, b_step = b_mn ? 2048u : 32u;
            const uint32_t a_lbo = a_mn ? 8192u : 0u, b_lbo = b_mn ? 8192u : 0u;
            PairWalk wk;
            int prow, ct, ca, cb;
            for (int u = cluster_id; next_unit(wk, u, prow, ct, ca, cb); u += n_clusters) {
                const int nst = unit_stages(prow);
                if (nst == 0) continue;
                if constexpr (!W) {
                    const uint32_t acc = acc_iter & 1;
                    const uint32_t acc_phase = (acc_iter >> 1) & 1;
                    ++acc_iter;
                    ptx::mbar_wait(tempty_bar + acc, acc_phase ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * kTile;
                    for (int s = 0; s < nst; ++s) {
                        ptx::mbar_wait(full_bar + stage, phase);
                        ptx::tc_fence_after();
                        const uint32_t a_addr = sbase + C::kOffA + stage * kHalfBytes;
                        const uint32_t b_addr = sbase + C::kOffB + stage * kHalfBytes;
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            const uint64_t ad = ptx::make_sw128_desc(a_addr + k * a_step, a_lbo, 1024);
                            const uint64_t bd = ptx::make_sw128_desc(b_addr + k * b_step, b_lbo, 1024);
                            mma2_bf16(d_tmem, ad, bd, idesc, (s > 0 || k > 0) ? 1u : 0u);
                        }
                        commit2_mc(empty_bar + stage, 0x3);
                        if (++stage == kStages2) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    commit2_mc(tfull_bar + acc, 0x3);
                } else {
                    // one 512-column accumulator, half h = TMEM columns [256h, 256h + 256):
                    // half 0 is free once the previous tile's epilogue drained it
                    // (tempty[0]), half 1 likewise (tempty[1]) — waited for only
                    // before the first MMA into it
                    const uint32_t rphase = acc_iter & 1;
                    ++acc_iter;
                    ptx::mbar_wait(tempty_bar + 0, rphase ^ 1);
                    ptx::tc_fence_after();
                    for (int s = 0; s < nst; ++s) {
                        ptx::mbar_wait(full_bar + stage, phase);
                        ptx::tc_fence_after();
                        const uint32_t a_addr = sbase + C::kOffA + stage * kHalfBytes;
                        const uint32_t b_addr = sbase + C::kOffB + stage * 2 * kHalfBytes;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            if (h == 1 && s == 0) {
                                ptx::mbar_wait(tempty_bar + 1, rphase ^ 1);
                                ptx::tc_fence_after();
                            }
#pragma unroll
                            for (int k = 0; k < kBK / 16; ++k) {
                                const uint64_t ad = ptx::make_sw128_desc(a_addr + k * a_step, a_lbo, 1024);
                                const uint64_t bd =
                                    ptx::make_sw128_desc(b_addr + h * kHalfBytes + k * b_step, b_lbo, 1024);
                                mma2_bf16(tmem_base + 256 * h, ad, bd, idesc, (s > 0 || k > 0) ? 1u : 0u);
                            }
                        }
                        commit2_mc(empty_bar + stage, 0x3);
                        if (++stage == kStages2) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    commit2_mc(tfull_bar + 0, 0x3);
                }
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (both CTAs, own 128 rows) =====================
        const uint32_t q = warp & 3;
        uint8_t* ebuf = smem + C::kOffEpi + q * 2 * kEpiBufBytes;
        const uint32_t ebuf_addr = sbase + C::kOffEpi + q * 2 * kEpiBufBytes;
        uint32_t bi = 0, acc_iter = 0;
        const int chunk = f32 ? 32 : 64;
        const int esz = f32 ? 4 : 2;
        PairWalk wk;
        int prow, ct, ca, cb;
        for (int u = cluster_id; next_unit(wk, u, prow, ct, ca, cb); u += n_clusters) {
            const int row_first = prow * kTile + 128 * static_cast<int>(rank) + 32 * q;
            if (unit_stages(prow) == 0) {
                // both rows of the pair fully dropped: exact zeros
                char* base = static_cast<char*>(a.out);
                const int cpr = kTile * esz / 16;
                for (int idx = lane; idx < 32 * cpr; idx += 32) {
                    const int r = idx / cpr, c = idx - r * cpr;
                    ptx::st_global_v4_zero(base + (static_cast<int64_t>(row_first + r) * a.cols_out + ct * kTile) * esz +
                                           c * 16);
                }
                continue;
            }
            // narrow: accumulator (acc_iter & 1); WIDE: the one 512-column accumulator
            const uint32_t acc = W ? 0u : (acc_iter & 1);
            const uint32_t acc_phase = W ? (acc_iter & 1) : ((acc_iter >> 1) & 1);
            ++acc_iter;
            ptx::mbar_wait(tfull_bar + acc, acc_phase);
            ptx::tc_fence_after();
            const int nchunks = kTileN / chunk;
            for (int c = 0; c < nchunks; ++c) {
                const uint32_t taddr = tmem_base + ((32 * q) << 16) + acc * kTile + c * chunk;
                uint32_t v[64];
                ptx::tmem_ld_32x32b_x32(taddr, v);
                if (!f32) ptx::tmem_ld_32x32b_x32(taddr + 32, v + 32);
                ptx::tmem_ld_wait();
                if (a.flags & kFlagOutMask) {
                    // dropped 128x128 output block (dX = s (dY W^T) (.) m): exact +0.0
                    const int cb = (c * chunk) / 128;  // column block within the tile
                    bool kept;
                    if (bits_up_front) {
                        kept = (own_bits[(u - cluster_id) / n_clusters] >> cb) & 1u;
                    } else {
                        const int64_t bit =
                            static_cast<int64_t>(row_first / 128) * a.mask_cols + (kTileN / 128) * ct + cb;
                        kept = (__ldcg(a.words + (bit >> 6)) >> (bit & 63)) & 1ull;
                    }
                    if (!kept) {
#pragma unroll
                        for (int j = 0; j < 64; ++j) v[j] = 0u;
                    }
                }
                if constexpr (!W) {
                    if (c == nchunks - 1) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(tempty_bar + acc), 0));
                    }
                } else {
                    // half 0 drained: the next tile's MMAs may start on it
                    const bool end_h0 = (c + 1) * chunk == 256, end_h1 = c == nchunks - 1;
                    if (end_h0 || end_h1) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0)
                            ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(tempty_bar + (end_h0 ? 0 : 1)), 0));
                    }
                }
                if (lane == 0) ptx::bulk_wait_group_read<1>();
                __syncwarp();
                const uint32_t row_addr = ebuf_addr + bi * kEpiBufBytes + lane * 128;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    uint32_t w0, w1, w2, w3;
                    if (f32) {
                        w0 = __float_as_uint(__uint_as_float(v[4 * j + 0]) * a.scale);
                        w1 = __float_as_uint(__uint_as_float(v[4 * j + 1]) * a.scale);
                        w2 = __float_as_uint(__uint_as_float(v[4 * j + 2]) * a.scale);
                        w3 = __float_as_uint(__uint_as_float(v[4 * j + 3]) * a.scale);
                    } else {
                        const float* f = reinterpret_cast<const float*>(v) + 8 * j;
                        w0 = ptx::pack_bf16x2(f[0] * a.scale, f[1] * a.scale);
                        w1 = ptx::pack_bf16x2(f[2] * a.scale, f[3] * a.scale);
                        w2 = ptx::pack_bf16x2(f[4] * a.scale, f[5] * a.scale);
                        w3 = ptx::pack_bf16x2(f[6] * a.scale, f[7] * a.scale);
                    }
                    ptx::st_shared_v4(row_addr + ((j ^ (lane & 7)) << 4), w0, w1, w2, w3);
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    // row-pair mode: columns [0,128) of the unit are block ca, [128,256) block cb
                    const int col = pairs ? (c * chunk < 128 ? ca * 128 + c * chunk : cb * 128 + c * chunk - 128)
                                          : ct * kTileN + c * chunk;
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
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols) : "memory");
    if (P.release && !bits_up_front && threadIdx.x == 0) {
        __threadfence();
        atomicAdd(P.release, 1u);
    }
}

}  // namespace

bool gemm2_routed(const GemmArgs& a) {
    return !(tuning() & kTuneNoGemm2) && a.list_cnt == nullptr && a.counters == nullptr && gemm2_supported(a) &&
           (a.rows_out / 256) * (a.cols_out / 256) >= num_sms() / 2;
}

bool gemm2_supported(const GemmArgs& a) {
    return !(a.flags & (kFlagSDD | kFlagReduce)) && a.rows_out % 256 == 0 && a.cols_out % 256 == 0 &&
           a.red % kBK == 0;
}

bool gemm2_pairs_supported(const GemmArgs& a) {
    return !(a.flags & (kFlagSDD | kFlagReduce)) && a.rows_out % 256 == 0 && a.red % kBK == 0 &&
           a.out_row_blk == 128 && a.out_col_blk == 128 && a.mask_cols >= 2 && a.mask_cols <= 64 &&
           a.cols_out == 128 * a.mask_cols && a.words != nullptr;
}

void launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tout, const GemmArgs& g,
                  const int32_t* pair_cnt, const int32_t* pair_idx, int pair_stride, cudaStream_t s,
                  bool no_wait, unsigned int* release) {
    configure_once_per_device(1, [] {
        check_cuda(cudaFuncSetAttribute(sd_gemm2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        K2Cfg<false>::kSmem),
                   "cudaFuncSetAttribute(gemm2 smem)");
        check_cuda(cudaFuncSetAttribute(sd_gemm2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        K2Cfg<true>::kSmem),
                   "cudaFuncSetAttribute(gemm2 wide smem)");
    });
    // 256 x 512 pair tiles (12 KB of operands per 1M MACs instead of 16) when
    // the columns allow it and there are at least two waves of them
    const int sms = num_sms();
    const int wide_units = (g.rows_out / 256) * (g.cols_out / 512);
    const bool pairs = g.flags & kFlagPairs;
    bool wide = !pair_cnt && !pairs && g.cols_out % 512 == 0 && wide_units >= sms;
    if (tuning() & kTuneGemm2Narrow) wide = false;
    if ((tuning() & kTuneGemm2Wide) && !pair_cnt && !pairs && g.cols_out % 512 == 0) wide = true;
    Pair2Args P;
    std::memset(&P, 0, sizeof P);
    P.g = g;
    P.n_pair_rows = g.rows_out / 256;
    P.n_col_tiles = g.cols_out / (wide ? 512 : 256);
    P.pair_cnt = pair_cnt;
    P.pair_idx = pair_idx;
    P.pair_stride = pair_stride;
    P.no_wait = no_wait && !(tuning() & kTuneNoEarlyBackward) ? 1 : 0;
    P.release = release;
    P.own_cap = (tuning() & kTuneNoOwnBits) ? 0 : kMaxOwnUnits;
    // row-pair mode: the unit count is data-dependent (on the device); at most
    // one unit per pair of mask columns per pair row
    const int units = pairs ? P.n_pair_rows * (g.mask_cols / 2) : P.n_pair_rows * P.n_col_tiles;
    int clusters = std::min(units, sms / 2);
    if (clusters <= 0) return;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = wide ? K2Cfg<true>::kSmem : K2Cfg<false>::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (wide) check_cuda(cudaLaunchKernelEx(&cfg, sd_gemm2_kernel<true>, ta, tb, tout, P), "sd_gemm2_kernel<wide> launch");
    else check_cuda(cudaLaunchKernelEx(&cfg, sd_gemm2_kernel<false>, ta, tb, tout, P), "sd_gemm2_kernel launch");
    note_launch();
    if (release) mask_note_readers(release, static_cast<int>(cfg.gridDim.x), s);
    // this kernel does not release mask workspaces: a following generation
    // into one it reads waits for the whole grid
    for (const void* q : {static_cast<const void*>(pair_cnt), static_cast<const void*>(pair_idx),
                          static_cast<const void*>(g.list_cnt), static_cast<const void*>(g.list_idx),
                          static_cast<const void*>(g.row_order)})
        mask_note_untracked(q);
}

}  // namespace sd
