// sd_gemm.cu — the SparseDrop tensor-core GEMMs for sm_100a.
//
// One persistent, warp-specialised tcgen05 kernel serves every GEMM of the
// path; operand major-ness and the way the block mask enters are per-problem
// run-time flags, and one launch may carry TWO independent problems sharing one
// work queue (the backward's dW and dX):
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
// edge / an odd kept sdd block), or, in the WIDE instantiation, up to 512
// columns as two N=256 MMAs sharing each stage's A tile: 20 KB of operands per
// 1M MACs instead of 24, which matters because these kernels are bound by the
// chip-wide L2->SM bandwidth (~20 TB/s whatever the TMA box shape,
// tools/box_bench.cu). Reduction in 64-element stages = one 128-byte
// swizzle atom; a 128-wide mask block is two stages (the paper's retile(1,2),
// PAPER.md:149-151). Only kept reduction blocks are ever loaded by TMA.
//
// Warp roles (256 threads, 1 CTA per SM, grid = min(units, #SMs)):
//   warp 0      TMA producer (one lane): 4-stage smem ring, mbarrier full/empty
//   warp 1      MMA issuer (one lane): tcgen05.mma -> TMEM, tcgen05.commit
//   warp 2      TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warp 3      scheduler (one lane): claims + decodes units
//   warps 4..7  epilogue: tcgen05.ld -> scale -> bf16/fp32 -> swizzled smem
//               -> TMA store; all-dropped tiles written as +0.0 directly.
// Two TMEM accumulators let the epilogue of tile i overlap the MMAs of i+1
// (WIDE: one 128x512 accumulator whose halves are released one by one).
// Scheduling is dynamic: the scheduler warp steals units from a global atomic
// counter (units ordered heaviest first, grouped for L2 reuse; problem 0 before
// problem 1) when the producer nears the end of its current unit, decodes them
// (list lookups) and hands the decoded unit to the producer, MMA and epilogue
// roles through a shared-memory ring; zero-work units skip TMEM.
//
// Launch overlap (PDL): every CTA triggers its dependents right after its
// griddepcontrol.wait, which a plan's backward skips when it directly follows
// the plan's forward (LaunchArgs.no_wait: it reads nothing the forward writes).
// Mask lists are only read by the scheduler (ld.global.cg, staged in smem): the
// CTA that decodes the launch's last unit releases the mask workspace for the
// whole grid (LaunchArgs.release), so the next mask generation can overwrite
// it while the grid's last units still compute.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "sd_internal.h"
#include "sd_ptx.cuh"

// Optional instrumentation (build with -DSD_TRACE, `make trace`): per-CTA
// cycle counters of every wait, read back with sd_trace_read().
#ifdef SD_TRACE
constexpr int kTraceSlots = 16;
__device__ unsigned long long g_sd_trace[1024 * kTraceSlots];
#define SD_TWAIT(slot, expr)                          \
    do {                                              \
        const long long t0_ = clock64();              \
        expr;                                         \
        tr[slot] += clock64() - t0_;                  \
    } while (0)
#define SD_TADD(slot, v) tr[slot] += (v)
__device__ unsigned long long g_sd_timeline[256 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#else
#define SD_TWAIT(slot, expr) expr
#define SD_TADD(slot, v) ((void)0)
#endif

namespace sd {
namespace {

#ifndef SD_STAGES
#define SD_STAGES 4
#endif
// Stages before a unit's last load at which the next unit is claimed. The
// claim atomic and the decode's dependent list loads run under the GEMM's own
// L2 traffic and take several microseconds: with 6 the producer ran dry at unit
// boundaries; 12-18 are equally good (4096^3 steps -3..-5%, ViT-B fc2 backward
// -12%, neutral at 8192^3 / cfg4; profiles/r02_claim_lead_ab.txt).
#ifndef SD_CLAIM_LEAD
#define SD_CLAIM_LEAD 14
#endif
// wide (128 x 512) tiles: separate A / B rings (a 64-deep stage = one A slot +
// one or two 256-column B slots)
#ifndef SD_WSTAGES_A
#define SD_WSTAGES_A 3
#endif
#ifndef SD_WSTAGES_B
#define SD_WSTAGES_B 4
#endif
#ifndef SD_CLAIM_LEAD_W
#define SD_CLAIM_LEAD_W 4
#endif
#ifndef SD_WEPIBUFS
#define SD_WEPIBUFS 2  // wide: store boxes per epilogue warp (1 frees 16 KB for a 5th B slot)
#endif
constexpr int kABytes = kBM * kBK * 2;  // 16 KB: one A slot (128 rows x 64)
constexpr int kBBytes = kBN * kBK * 2;  // 32 KB: one B slot (256 columns x 64)
constexpr int kEpiWarps = 4;
constexpr int kEpiBufBytes = 32 * 128;  // one warp's 32 rows x 128 B store box
constexpr int kThreads = 256;
constexpr int kTmemCols = 512;
constexpr int kMaxProblems = 2;
constexpr int kGroupRows = 16;  // tile rows per rasterization group
constexpr int kSchedDepth = 4;  // decoded-unit ring between the scheduler and the other roles
constexpr int kListCap = 64;    // kept-block list entries staged per ring slot (longer lists: __ldg)

struct Unit {
    int prob;      // problem index; -1 = end of work
    int row0;      // first output row
    int list_row;  // mask row (list index) of this tile row
    int n0;        // first output column (dsd)
    int n_eff;     // output columns (MMA N; wide: two 256-column halves); 0 => no MMA work
    int nstages;   // reduction stages
    int nslots;    // sdd: kept output blocks in this unit
    int nzero;     // sdd: dropped output blocks in this unit
    int slot_blk[4];
    int zero_blk[4];
    int first_entry;  // dsd: first list entry (split-K)
    int width;        // unit width in columns (zero fill of an all-dropped dsd unit)
    int split;        // dsd split-K: this unit's split index (0 = stores, > 0 = ordered reduce-add)
    int tile;         // dsd split-K: output tile index within the split (turnstile index)
    int pad[4];
};
static_assert(sizeof(Unit) == 96, "Unit layout");

// Per-mode kernel configuration.
//   narrow: 128 x 256 units, a 4-stage ring of {A 16 KB, B 32 KB}, two 128x256
//           fp32 TMEM accumulators (tile i's epilogue overlaps tile i+1's MMAs)
//   WIDE:   128 x 512 units: 20 KB of operands per 1M MACs instead of 24 (the
//           kernels are bound by chip-wide L2->SM bandwidth, tools/box_bench.cu).
//           An A ring and a B ring of 256-column slots; ONE 128x512 accumulator
//           whose halves are released to the next unit as the epilogue drains
//           them. Narrower units (ragged edges) use half 0 only.
template <bool WIDE>
struct KCfg {
    static constexpr int kSA = WIDE ? SD_WSTAGES_A : SD_STAGES;
    static constexpr int kSB = WIDE ? SD_WSTAGES_B : SD_STAGES;
    static constexpr int kWidth = WIDE ? 2 * kBN : kBN;
    static constexpr int kClaimLead = WIDE ? SD_CLAIM_LEAD_W : SD_CLAIM_LEAD;
    static constexpr int kEpiBufs = WIDE ? SD_WEPIBUFS : 2;
    static constexpr int kOffA = 0;
    static constexpr int kOffB = kOffA + kSA * kABytes;
    static constexpr int kOffEpi = kOffB + kSB * kBBytes;
    static constexpr int kOffBar = kOffEpi + kEpiWarps * kEpiBufs * kEpiBufBytes;
    // full[kSB] empty[kSB] aempty[kSA] tfull[2] tempty[2] sfull[D] sempty[D] claim
    static constexpr int kNumBars = 2 * kSB + kSA + 4 + 2 * kSchedDepth + 1;
    static constexpr int kOffTmemSlot = kOffBar + kNumBars * 8;
    static constexpr int kOffSched = kOffTmemSlot + 16;
    static constexpr int kOffList = kOffSched + static_cast<int>(sizeof(Unit)) * kSchedDepth;
    static constexpr int kSmem = kOffList + kListCap * 4 * kSchedDepth + 1024;  // + align slack
    static_assert(kSmem <= 232448, "shared memory budget");
};

struct LaunchArgs {
    GemmArgs p[kMaxProblems];
    int nprob;
    int total_units;
    int trace_id;  // launch sequence number (SD_TRACE timeline)
    unsigned int* sched;  // {next-unit counter, CTAs-done counter, units-decoded counter, -}
    // release counters of the bound mask workspaces this launch reads lists
    // from (sd_internal.h, reader tracking); null = none
    unsigned int* release[2];
    int no_wait;  // skip griddepcontrol.wait (launch_gemms)
    // 1: no unit's list can exceed the smem staging, so the mask workspaces are
    // free once every unit is decoded: the CTA that decodes the last unit
    // releases for the whole grid. 0: each CTA releases when it stops reading.
    int release_all;
};

struct TensorMaps {
    CUtensorMap m[3 * kMaxProblems];  // A, B, Out per problem
};

// Bits of mask row r (C <= 64 columns), row-major LSB-first words.
__device__ __forceinline__ uint64_t pair_row_bits(const uint64_t* words, int r, int C) {
    const int64_t b = static_cast<int64_t>(r) * C;
    const int sh = static_cast<int>(b & 63);
    uint64_t v = __ldcg(words + (b >> 6)) >> sh;
    if (sh + C > 64) v |= __ldcg(words + (b >> 6) + 1) << (64 - sh);
    return C == 64 ? v : (v & ((1ull << C) - 1));
}

template <bool WIDE>
__device__ __forceinline__ Unit decode_unit(const GemmArgs& a, int prob, int u) {
    Unit t;
    t.prob = prob;
    // split-K (dsd only): the split index is the outermost coordinate
    const int T = a.tail_rows;
    const int head_rows = a.n_row_tiles - T;
    const int head_units = head_rows * a.n_col_units;
    const int base_units = head_units + T * 2 * a.n_col_units;
    const int split = u / base_units;
    u -= split * base_units;
    t.split = split;
    t.tile = u;
    int i, cu;
    bool half = false;
    if (u < head_units) {
        // Grouped rasterization: tile rows (sorted heaviest first) are taken in
        // groups of kGroupRows; inside a group units go column-unit-major. The
        // CTAs in flight then share a few operand column/row slabs (L2 reuse),
        // heavy groups still go first, and for sdd the units carrying MMA work
        // (kept blocks are packed into the low column units) precede the
        // zero-fill-only units of their group.
        const int g = u / (kGroupRows * a.n_col_units);
        const int rem_u = u - g * kGroupRows * a.n_col_units;
        const int rows_in_group = min(kGroupRows, head_rows - g * kGroupRows);
        cu = rem_u / rows_in_group;
        i = g * kGroupRows + (rem_u - cu * rows_in_group);
    } else {
        // Tail: the lightest rows, handed out last, in half-width units so the
        // final wave is fine-grained (shorter idle tail across SMs).
        u -= head_units;
        cu = u / T;
        i = head_rows + (u - cu * T);
        half = true;
    }
    const int rt = a.row_order ? __ldcg(a.row_order + i) : i;
    t.row0 = rt * kBM;
    t.list_row = t.row0 / a.out_row_blk;
    t.nslots = 0;
    t.nzero = 0;
    t.first_entry = 0;
    const int width = half ? KCfg<WIDE>::kWidth / 2 : KCfg<WIDE>::kWidth;
    t.width = width;
    if (!(a.flags & kFlagSDD)) {
        t.n0 = cu * width;
        const int rem = a.cols_out - t.n0;
        t.n_eff = rem < width ? (rem > 0 ? rem : 0) : width;
        const int cnt = a.list_cnt ? __ldcg(a.list_cnt + t.list_row) : a.red / a.red_blk;
        // this split's contiguous share [lo, hi) of the row's kept blocks
        const int lo = static_cast<int>((static_cast<int64_t>(cnt) * split) / a.splits);
        const int hi = static_cast<int>((static_cast<int64_t>(cnt) * (split + 1)) / a.splits);
        t.first_entry = lo;
        t.nstages = (hi - lo) * (a.red_blk / kBK);
        if (hi == lo) t.n_eff = 0;
    } else {
        // Pack the row's KEPT output blocks (compacted list, ascending) into
        // full-width units, so every unit but the row's last runs full-N MMAs;
        // the same unit index also zero-fills the row's DROPPED blocks (kept at
        // the tail of the list by the mask kernel).
        const int per_unit = width / a.out_col_blk;
        const int cnt = __ldcg(a.list_cnt + t.list_row);
        const int ndrop = a.mask_cols - cnt;
        const int32_t* row = a.list_idx + static_cast<int64_t>(t.list_row) * a.list_stride;
        t.n0 = 0;
        if (a.flags & kFlagPairs) {
            // row-pair split (sd_gemm2.cu): the column blocks this row and its
            // pair partner both keep, taken in ascending pairs, are the 2-CTA
            // kernel's; this unit packs the REMAINING kept blocks (and zero-fills
            // the dropped ones from the list tail as usual)
            const uint64_t mine = pair_row_bits(a.words, t.list_row, a.mask_cols);
            const uint64_t common = mine & pair_row_bits(a.words, t.list_row ^ 1, a.mask_cols);
            uint64_t paired = common;
            for (int i = __popcll(common) & ~1; i < __popcll(common); ++i) paired &= ~(1ull << (63 - __clzll(paired)));
            uint64_t rem = mine & ~paired;
            for (int i = 0; i < cu * per_unit && rem; ++i) rem &= rem - 1;  // skip earlier units' blocks
            // slots and zero blocks fill in prefix order: constant indices after
            // unrolling keep the Unit in registers (no local-memory stack frame)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (j >= per_unit) break;
                const int li = cu * per_unit + j;
                if (rem) {
                    t.slot_blk[j] = __ffsll(static_cast<long long>(rem)) - 1;
                    t.nslots = j + 1;
                    rem &= rem - 1;
                }
                if (li < ndrop) {
                    t.zero_blk[j] = __ldcg(row + a.mask_cols - 1 - li);
                    t.nzero = j + 1;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (j >= per_unit) break;
                const int li = cu * per_unit + j;
                if (li < cnt) {
                    t.slot_blk[j] = __ldcg(row + li);
                    t.nslots = j + 1;
                }
                if (li < ndrop) {
                    t.zero_blk[j] = __ldcg(row + a.mask_cols - 1 - li);
                    t.nzero = j + 1;
                }
            }
        }
        t.n_eff = t.nslots * a.out_col_blk;
        t.nstages = a.red / kBK;
    }
    return t;
}

// ---- hash mode (small plans): decode without the mask workspace ----------
__device__ __forceinline__ uint64_t mix64_d(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Kept bits of list `idx` (a mask row for hash mode 1, a mask column for 2) over
// its hash_len <= 64 entries, from the counter hash (block_mask.cpp:70; the
// mask kernel's keep_bit). Whole scheduler warp; every lane gets the set.
__device__ __forceinline__ uint64_t hash_list_bits(const GemmArgs& a, int idx, uint32_t lane) {
    const int li = idx + a.hash_list_off;
    bool k0 = false, k1 = false;
    if (a.hash_mode == 1) {
        const uint64_t hr = mix64_d(a.hash_seed_mix ^ static_cast<uint64_t>(li + a.hash_row_off));
        if (static_cast<int>(lane) < a.hash_len) k0 = (mix64_d(hr ^ lane) >> 11) >= a.hash_threshold;
        if (static_cast<int>(lane) + 32 < a.hash_len) k1 = (mix64_d(hr ^ (lane + 32)) >> 11) >= a.hash_threshold;
    } else {
        const uint64_t c = static_cast<uint64_t>(li);
        if (static_cast<int>(lane) < a.hash_len)
            k0 = (mix64_d(mix64_d(a.hash_seed_mix ^ static_cast<uint64_t>(lane + a.hash_row_off)) ^ c) >> 11) >=
                 a.hash_threshold;
        if (static_cast<int>(lane) + 32 < a.hash_len)
            k1 = (mix64_d(mix64_d(a.hash_seed_mix ^ static_cast<uint64_t>(lane + 32 + a.hash_row_off)) ^ c) >> 11) >=
                 a.hash_threshold;
    }
    return static_cast<uint64_t>(__ballot_sync(0xffffffffu, k0)) |
           (static_cast<uint64_t>(__ballot_sync(0xffffffffu, k1)) << 32);
}

// Position of the (n+1)-th set bit of v (n < popcount(v)).
__device__ __forceinline__ int nth_set_bit64(uint64_t v, int n) {
    const uint32_t lo = static_cast<uint32_t>(v), hi = static_cast<uint32_t>(v >> 32);
    const int cl = __popc(lo);
    return n < cl ? static_cast<int>(__fns(lo, 0, n + 1)) : 32 + static_cast<int>(__fns(hi, 0, n - cl + 1));
}

// decode_unit's coordinates (no list reads; the tile-row order is not used)
template <bool WIDE>
__device__ __forceinline__ Unit decode_coords_h(const GemmArgs& a, int prob, int u, int& cu_out) {
    Unit t;
    t.prob = prob;
    const int T = a.tail_rows;
    const int head_rows = a.n_row_tiles - T;
    const int head_units = head_rows * a.n_col_units;
    const int base_units = head_units + T * 2 * a.n_col_units;
    const int split = u / base_units;
    u -= split * base_units;
    t.split = split;
    t.tile = u;
    int i, cu;
    bool half = false;
    if (u < head_units) {
        const int g = u / (kGroupRows * a.n_col_units);
        const int rem_u = u - g * kGroupRows * a.n_col_units;
        const int rows_in_group = min(kGroupRows, head_rows - g * kGroupRows);
        cu = rem_u / rows_in_group;
        i = g * kGroupRows + (rem_u - cu * rows_in_group);
    } else {
        u -= head_units;
        cu = u / T;
        i = head_rows + (u - cu * T);
        half = true;
    }
    t.row0 = i * kBM;
    t.list_row = t.row0 / a.out_row_blk;
    t.nslots = 0;
    t.nzero = 0;
    t.first_entry = 0;
    t.width = half ? KCfg<WIDE>::kWidth / 2 : KCfg<WIDE>::kWidth;
    cu_out = cu;
    return t;
}

// decode_unit's list-dependent fields, from the unit's kept bits
template <bool WIDE>
__device__ __forceinline__ void decode_finish_h(const GemmArgs& a, Unit& t, int cu, uint64_t hbits) {
    const int width = t.width;
    const int cnt = __popcll(hbits);
    if (!(a.flags & kFlagSDD)) {
        t.n0 = cu * width;
        const int rem = a.cols_out - t.n0;
        t.n_eff = rem < width ? (rem > 0 ? rem : 0) : width;
        const int lo = static_cast<int>((static_cast<int64_t>(cnt) * t.split) / a.splits);
        const int hi = static_cast<int>((static_cast<int64_t>(cnt) * (t.split + 1)) / a.splits);
        t.first_entry = lo;
        t.nstages = (hi - lo) * (a.red_blk / kBK);
        if (hi == lo) t.n_eff = 0;
    } else {
        // kept blocks ascending; dropped blocks ascending (each unit of the row
        // zero-fills its own share, every dropped block exactly once)
        const int per_unit = width / a.out_col_blk;
        const uint64_t all = a.mask_cols == 64 ? ~0ull : ((1ull << a.mask_cols) - 1);
        const int ndrop = a.mask_cols - cnt;
        t.n0 = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j >= per_unit) break;
            const int li = cu * per_unit + j;
            if (li < cnt) {
                t.slot_blk[j] = nth_set_bit64(hbits, li);
                t.nslots = j + 1;
            }
            if (li < ndrop) {
                t.zero_blk[j] = nth_set_bit64(~hbits & all, li);
                t.nzero = j + 1;
            }
        }
        t.n_eff = t.nslots * a.out_col_blk;
        t.nstages = a.red / kBK;
    }
}

// This CTA is done reading the mask workspaces of the launch (release counters).
__device__ __forceinline__ void release_workspaces(const LaunchArgs& L) {
    for (int r = 0; r < 2; ++r) {
        if (L.release[r]) {
            __threadfence();
            atomicAdd(L.release[r], 1u);
        }
    }
}

template <bool WIDE>
__device__ __forceinline__ Unit decode_global(const LaunchArgs& L, int u) {
    if (L.nprob > 1 && u >= L.p[1].unit_begin) return decode_unit<WIDE>(L.p[1], 1, u - L.p[1].unit_begin);
    return decode_unit<WIDE>(L.p[0], 0, u);
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

// Epilogue of one unit for one warp (32 output rows).
//   narrow: the unit's accumulator is TMEM region (acc_iter & 1), released at the end
//   WIDE:   columns [0,256) / [256,512) are regions 0 / 1, each released (tempty)
//           as soon as it is drained, so the next unit's MMAs start on region 0
//           while region 1 is still being stored
template <bool WIDE, bool OUT_F32>
__device__ __forceinline__ void epilogue_unit(const GemmArgs& a, const CUtensorMap* tmOut, const Unit& t,
                                              uint32_t q, uint32_t lane, uint32_t tmem_base,
                                              uint64_t* tfull_bar, uint64_t* tempty_bar, uint8_t* ebuf,
                                              uint32_t ebuf_addr, uint32_t& bi, uint32_t& acc_iter,
                                              unsigned int* turn_base, long long* tr) {
    (void)tr;
    constexpr int kChunkCols = OUT_F32 ? 32 : 64;  // 128 bytes of output per row
    const bool sdd = a.flags & kFlagSDD;
    const int row_first = t.row0 + 32 * q;
    // Split-K in a FIXED order (run-to-run deterministic, like the reference's
    // serial reduction): split 0 of an output tile stores its
    // partial, split j > 0 waits on the tile quarter's turnstile for j, reduce-
    // adds, waits for its writes to complete and passes the turnstile on (the
    // last split resets it to 0 for the next launch). Splits are claimed in
    // order (split-outermost unit numbering), so every wait is on a unit claimed
    // earlier by a resident CTA: no deadlock.
    const bool reduce = a.flags & kFlagReduce;
    unsigned int* turn = reduce ? turn_base + 4 * t.tile + q : nullptr;
    const auto turn_wait = [&] {
        if (lane == 0 && t.split > 0) {
            while (ptx::ld_acquire_gpu(turn) != static_cast<uint32_t>(t.split)) __nanosleep(32);
            ptx::fence_proxy_async_global();
        }
    };
    const auto turn_pass = [&] {
        if (lane == 0) {
            ptx::bulk_wait_group<0>();  // this unit's stores / reduce-adds have completed
            ptx::fence_proxy_async_global();
            ptx::st_release_gpu(turn, t.split + 1 == a.splits ? 0u : static_cast<uint32_t>(t.split + 1));
        }
    };
    if (sdd) {
#pragma unroll
        for (int z = 0; z < 4; ++z)
            if (z < t.nzero) zero_rows<OUT_F32>(a, row_first, t.zero_blk[z] * a.out_col_blk, a.out_col_blk, lane);
    }
    if (t.n_eff == 0) {
        const int rem = a.cols_out - t.n0;
        const int w = t.width;
        if (!sdd && (!reduce || t.split == 0)) {
            if (rem > 0) zero_rows<OUT_F32>(a, row_first, t.n0, rem < w ? rem : w, lane);
        }
        if (reduce) {
            __threadfence();
            __syncwarp();
            turn_wait();
            turn_pass();
            __syncwarp();
        }
        return;
    }
    uint32_t acc_col0, full_idx, full_phase;
    if constexpr (WIDE) {
        acc_col0 = 0;
        full_idx = 0;
        full_phase = acc_iter & 1;
    } else {
        acc_col0 = (acc_iter & 1) * kBN;
        full_idx = acc_iter & 1;
        full_phase = (acc_iter >> 1) & 1;
    }
    ++acc_iter;
    SD_TWAIT(5, ptx::mbar_wait(tfull_bar + full_idx, full_phase));
    ptx::tc_fence_after();
    const int nchunks = t.n_eff / kChunkCols;
    for (int c = 0; c < nchunks; ++c) {
        const uint32_t taddr = tmem_base + ((32 * q) << 16) + acc_col0 + c * kChunkCols;
        uint32_t v[kChunkCols];
        ptx::tmem_ld_32x32b_x32(taddr, v);
        if constexpr (!OUT_F32) ptx::tmem_ld_32x32b_x32(taddr + 32, v + 32);
        ptx::tmem_ld_wait();
        const bool last = c == nchunks - 1;
        if constexpr (WIDE) {
            // region 0 drained (columns [0,256) read out): the next unit may start on it;
            // region 1 is released at the end of every unit (used or not)
            const bool end_r0 = (c + 1) * kChunkCols == kBN;
            if (end_r0 || last) {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (end_r0 || t.n_eff <= kBN) ptx::mbar_arrive(tempty_bar + 0);
                    if (last) ptx::mbar_arrive(tempty_bar + 1);
                }
            }
        } else {
            if (last) {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(tempty_bar + full_idx);
            }
        }
        // staging buffer bi must no longer be read by the TMA store issued 2 chunks ago
        if (lane == 0) {
            if constexpr (KCfg<WIDE>::kEpiBufs == 2) ptx::bulk_wait_group_read<1>();
            else ptx::bulk_wait_group_read<0>();
        }
        __syncwarp();
        const uint32_t row_addr = ebuf_addr + bi * kEpiBufBytes + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t w0, w1, w2, w3;
            if constexpr (OUT_F32) {
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
        if (reduce && c == 0) turn_wait();
        if (lane == 0) {
            int col;
            if (sdd) {
                const int tcol = c * kChunkCols;
                const int sl = tcol / a.out_col_blk;
                const int blk = sl == 0 ? t.slot_blk[0] : sl == 1 ? t.slot_blk[1] : sl == 2 ? t.slot_blk[2] : t.slot_blk[3];
                col = blk * a.out_col_blk + (tcol - sl * a.out_col_blk);
            } else {
                col = t.n0 + c * kChunkCols;
            }
            if (reduce && t.split > 0)
                ptx::tma_reduce_add_2d(tmOut, ebuf + bi * kEpiBufBytes, col, row_first);
            else
                ptx::tma_store_2d(tmOut, ebuf + bi * kEpiBufBytes, col, row_first);
            ptx::bulk_commit_group();
        }
        if constexpr (KCfg<WIDE>::kEpiBufs == 2) bi ^= 1;
    }
    if (reduce) {
        turn_pass();
        __syncwarp();
    }
}

template <bool WIDE, bool HASH>
__global__ void __launch_bounds__(kThreads, 1)
    sd_gemm_kernel(const __grid_constant__ TensorMaps tms, const __grid_constant__ LaunchArgs L) {
    using C = KCfg<WIDE>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    const uint32_t sbase = ptx::smem_u32(smem);

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* full_bar = bars;                 // B slot (+ its stage's A tile) landed
    uint64_t* empty_bar = bars + C::kSB;       // B slot (narrow: the whole stage) consumed
    uint64_t* aempty_bar = bars + 2 * C::kSB;  // WIDE: A slot consumed (both halves of its stage)
    uint64_t* tfull_bar = aempty_bar + C::kSA;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint64_t* sfull_bar = tempty_bar + 2;
    uint64_t* sempty_bar = sfull_bar + kSchedDepth;
    uint64_t* claim_bar = sempty_bar + kSchedDepth;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffTmemSlot);
    Unit* sched_unit = reinterpret_cast<Unit*>(smem + C::kOffSched);
    int32_t* sched_list = reinterpret_cast<int32_t*>(smem + C::kOffList);  // [kSchedDepth][kListCap]

    const uint32_t warp = threadIdx.x / 32;
    const uint32_t lane = ptx::lane_id();
    const int num_units = L.total_units;
#ifdef SD_TRACE
    if (threadIdx.x == 0) atomicMin(&g_sd_timeline[(L.trace_id & 255) * 4 + 0], gtimer());
#endif

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < 3 * L.nprob; ++i) ptx::prefetch_tmap(&tms.m[i]);
        for (int i = 0; i < C::kSB; ++i) {
            ptx::mbar_init(full_bar + i, 1);
            ptx::mbar_init(empty_bar + i, 1);
        }
        for (int i = 0; i < C::kSA; ++i) ptx::mbar_init(aempty_bar + i, 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(tfull_bar + i, 1);
            ptx::mbar_init(tempty_bar + i, kEpiWarps);
        }
        for (int i = 0; i < kSchedDepth; ++i) {
            ptx::mbar_init(sfull_bar + i, 32);  // every scheduler lane publishes its own list stores
            ptx::mbar_init(sempty_bar + i, 2 + 32 * kEpiWarps);  // producer, MMA, every epilogue lane
        }
        ptx::mbar_init(claim_bar, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // Everything above overlapped the previous kernel's tail (PDL); from here on
    // we read its outputs (mask lists, operands), so wait for it to complete —
    // unless the launch is independent of it (no_wait: a plan's backward right
    // after its forward). Mask lists are read with ld.global.cg (L2), never
    // through a possibly stale L1 line of an earlier grid.
    if (!L.no_wait) ptx::pdl_wait();
    ptx::pdl_launch_dependents();
#ifdef SD_TRACE
    long long tr[16] = {0};
#else
    long long* tr = nullptr;  // per-role wait counters exist only in SD_TRACE builds
#endif
#ifdef SD_TRACE
    const long long t_start = clock64();
    const unsigned long long g_start = gtimer();
    if (threadIdx.x == 0) atomicMin(&g_sd_timeline[(L.trace_id & 255) * 4 + 1], gtimer());
#endif

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_normal();
            int stage = 0;      // B slot
            uint32_t phase = 0;
            int sa = 0;         // WIDE: A slot
            uint32_t pa = 0;
            int sslot = 0;
            uint32_t sphase = 0;
            // Units come from the scheduler warp through the ring; kClaimLead
            // stages before this unit's loads are all issued, the scheduler is
            // told to claim the next one (see warp 3).
            constexpr int kClaimLead = C::kClaimLead;
            while (true) {
                SD_TWAIT(1, ptx::mbar_wait(sfull_bar + sslot, sphase));
                const Unit cur = sched_unit[sslot];
                const int cur_slot = sslot;
                if (++sslot == kSchedDepth) {
                    sslot = 0;
                    sphase ^= 1;
                }
                if (cur.prob < 0) {
                    ptx::mbar_arrive(sempty_bar + cur_slot);
                    // lists were read here (units too long to stage): the mask
                    // workspace is released now that every load is issued
                    if (cur.nslots) release_workspaces(L);
                    break;
                }
                const int nst = cur.n_eff == 0 ? 0 : cur.nstages;
                const int claim_at = nst > kClaimLead ? nst - kClaimLead : 0;
                if (nst == 0) {
                    // no loads (zero fill only): the scheduler claimed the next
                    // unit without waiting for a claim signal
                    ptx::mbar_arrive(sempty_bar + cur_slot);
                    continue;
                }
                const GemmArgs& a = L.p[cur.prob];
                const CUtensorMap* tmA = &tms.m[3 * cur.prob];
                const CUtensorMap* tmB = &tms.m[3 * cur.prob + 1];
                const bool a_mn = a.flags & kFlagAMN;
                const bool b_mn = a.flags & kFlagBMN;
                const bool sdd = a.flags & kFlagSDD;
                const int nh = WIDE ? (cur.n_eff + kBN - 1) / kBN : 1;  // 256-column halves
                const int per_half = sdd ? kBN / a.out_col_blk : 0;    // sdd blocks per B slot
                const int spb = a.red_blk / kBK;
                const int li0 = sdd ? 0 : cur.first_entry;
                const int scol0 = cur.slot_blk[0] * a.out_col_blk, scol1 = cur.slot_blk[1] * a.out_col_blk;
                const int scol2 = cur.slot_blk[2] * a.out_col_blk, scol3 = cur.slot_blk[3] * a.out_col_blk;
                // kept-block indices: staged in smem by the scheduler (lists up to
                // kListCap, and every hash-mode list), else read from global one
                // block ahead
                const int32_t* slist = sched_list + cur_slot * kListCap;
                const int32_t* lst =
                    HASH ? (sdd ? nullptr : slist)
                         : ((!sdd && a.list_idx) ? a.list_idx + static_cast<int64_t>(cur.list_row) * a.list_stride + li0
                                                 : nullptr);
                const bool staged = HASH || cur.nstages / spb <= kListCap;
                int kb_next = lst ? (staged ? slist[0] : __ldcg(lst)) : 0;
                int kb = 0;
                for (int s = 0, li = 0, sub = 0; s < cur.nstages; ++s) {
                    if (s == claim_at) ptx::mbar_arrive(claim_bar);
                    int r0;
                    if (!sdd) {
                        if (sub == 0) {
                            kb = lst ? kb_next : li0 + li;
                            if (lst && li + 1 < cur.nstages / spb) kb_next = staged ? slist[li + 1] : __ldcg(lst + li + 1);
                        }
                        r0 = kb * a.red_blk + sub * kBK;
                        if (++sub == spb) {
                            sub = 0;
                            ++li;
                        }
                    } else {
                        r0 = s * kBK;
                    }
                    for (int h = 0; h < nh; ++h) {
                        const int ncols = WIDE ? min(kBN, cur.n_eff - kBN * h) : cur.n_eff;
                        uint32_t tx_bytes = static_cast<uint32_t>(ncols) * kBK * 2;
                        SD_TWAIT(0, ptx::mbar_wait(empty_bar + stage, phase ^ 1));
                        uint8_t* sA = smem + C::kOffA + (WIDE ? sa : stage) * kABytes;
                        if (h == 0) {
                            if constexpr (WIDE) SD_TWAIT(0, ptx::mbar_wait(aempty_bar + sa, pa ^ 1));
                            tx_bytes += kABytes;
                        }
                        uint64_t* fb = full_bar + stage;
#ifdef SD_DIAG_NO_TMA
                        ptx::mbar_arrive(fb);
                        (void)tx_bytes;
                        (void)per_half;
                        (void)sA;
#else
                        ptx::mbar_arrive_expect_tx(fb, tx_bytes);
                        if (h == 0) {
                            if (!a_mn) ptx::tma_load_2d(tmA, fb, sA, r0, cur.row0, pol);
                            else ptx::tma_load_3d(tmA, fb, sA, 0, r0, cur.row0 / 64, pol);
                        }
                        uint8_t* sB = smem + C::kOffB + stage * kBBytes;
                        if (!sdd) {
                            const int c0 = cur.n0 + kBN * h;
                            for (int j = 0; j < ncols / 128; ++j) {
                                if (!b_mn) ptx::tma_load_2d(tmB, fb, sB + j * 16384, r0, c0 + 128 * j, pol);
                                else ptx::tma_load_3d(tmB, fb, sB + j * 16384, 0, r0, (c0 + 128 * j) / 64, pol);
                            }
                        } else {
                            const int per = a.out_col_blk / 128;
                            // slot columns by select from per-unit scalars: a runtime index
                            // into cur puts the Unit in local memory, and unrolling with
                            // constant indices bloated this single-thread loop (sdd 4-7%
                            // slower: profiles/r02_local_memory_ab.txt)
                            const int sl_end = min(cur.nslots, (h + 1) * per_half);
                            for (int sl = h * per_half; sl < sl_end; ++sl) {
                                const int col0 = (sl == 0 ? scol0 : sl == 1 ? scol1 : sl == 2 ? scol2 : scol3);
                                const int off = (sl - h * per_half) * per;
                                for (int j = 0; j < per; ++j) {
                                    if (!b_mn)
                                        ptx::tma_load_2d(tmB, fb, sB + (off + j) * 16384, r0, col0 + 128 * j, pol);
                                    else
                                        ptx::tma_load_3d(tmB, fb, sB + (off + j) * 16384, 0, r0, (col0 + 128 * j) / 64,
                                                         pol);
                                }
                            }
                        }
#endif
                        if (++stage == C::kSB) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    if constexpr (WIDE) {
                        if (++sa == C::kSA) {
                            sa = 0;
                            pa ^= 1;
                        }
                    }
                }
                ptx::mbar_arrive(sempty_bar + cur_slot);  // done with the slot's staged list
            }
        }
    } else if (HASH && warp == 3) {
        // ===================== scheduler (hash mode) =====================
        // As below, but each unit's kept list comes from the counter hash
        // (one warp, no loads): the launch reads nothing of the mask workspace.
        int sslot = 0;
        uint32_t sphase = 0;
        uint32_t cphase = 0;
        int u = blockIdx.x;
        while (true) {
            Unit t;
            int cu = 0;
            int prob = -1;
            if (lane == 0) {
                if (u < num_units) {
                    prob = (L.nprob > 1 && u >= L.p[1].unit_begin) ? 1 : 0;
                    t = decode_coords_h<WIDE>(L.p[prob], prob, u - L.p[prob].unit_begin, cu);
                } else {
                    t.prob = -1;
                    t.nslots = 0;
                }
            }
            prob = __shfl_sync(0xffffffffu, prob, 0);
            uint64_t hbits = 0;
            if (prob >= 0) hbits = hash_list_bits(L.p[prob], __shfl_sync(0xffffffffu, t.list_row, 0), lane);
            int nblk = 0, li0 = 0;
            if (lane == 0 && prob >= 0) {
                decode_finish_h<WIDE>(L.p[prob], t, cu, hbits);
                const GemmArgs& a = L.p[prob];
                if (!(a.flags & kFlagSDD) && t.n_eff > 0) {
                    nblk = t.nstages / (a.red_blk / kBK);
                    li0 = t.first_entry;
                }
            }
            nblk = __shfl_sync(0xffffffffu, nblk, 0);
            li0 = __shfl_sync(0xffffffffu, li0, 0);
            SD_TWAIT(1, ptx::mbar_wait(sempty_bar + sslot, sphase ^ 1));
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = static_cast<int>(lane) + 32 * h;
                if ((hbits >> j) & 1ull) {
                    const int pos = __popcll(hbits & ((1ull << j) - 1ull)) - li0;
                    if (pos >= 0 && pos < nblk) sched_list[sslot * kListCap + pos] = j;
                }
            }
            if (lane == 0) sched_unit[sslot] = t;
            ptx::mbar_arrive(sfull_bar + sslot);
            if (++sslot == kSchedDepth) {
                sslot = 0;
                sphase ^= 1;
            }
            if (prob < 0) break;
            const bool loads = __shfl_sync(0xffffffffu, (t.n_eff > 0 && t.nstages > 0) ? 1 : 0, 0);
            if (lane == 0) {
                if (loads) ptx::mbar_wait(claim_bar, cphase);
                u = static_cast<int>(gridDim.x) + static_cast<int>(atomicAdd(L.sched, 1u));
            }
            if (loads) cphase ^= 1;
        }
    } else if (warp == 3) {
        // ===================== scheduler =====================
        // Dynamic persistent scheduling: first unit = blockIdx.x, then work
        // stealing through a global atomic counter (units are ordered heaviest
        // first, so this is greedy longest-processing-time). The next unit is
        // claimed only when the producer nears the end of its current one:
        // late enough that a CTA never sits on a claimed unit while others idle
        // at the tail (claiming two units ahead cost 15-40% tail imbalance),
        // early enough that the atomic and the decode's dependent loads (here,
        // off the TMA issue path) finish before the producer needs the unit.
        // The whole warp stages the unit's kept-block list (dsd) into the slot's
        // smem list, so the producer never waits on a list load between TMAs.
        int sslot = 0;
        uint32_t sphase = 0;
        uint32_t cphase = 0;
        int u = blockIdx.x;
        bool unstaged = false;  // a unit's list was too long to stage: the producer reads it
        while (true) {
            Unit t;
            if (lane == 0) {
                if (u < num_units) {
                    t = decode_global<WIDE>(L, u);
                } else {
                    t.prob = -1;
                    t.nslots = unstaged ? 1 : 0;  // end marker: who releases the mask workspace
                }
            }
            // list source of this unit (dsd with a list): entries [li0, li0 + nblk)
            const int32_t* src = nullptr;
            int nblk = 0;
            if (lane == 0 && t.prob >= 0 && t.n_eff > 0) {
                const GemmArgs& a = L.p[t.prob];
                if (!(a.flags & kFlagSDD) && a.list_idx) {
                    src = a.list_idx + static_cast<int64_t>(t.list_row) * a.list_stride + t.first_entry;
                    nblk = t.nstages / (a.red_blk / kBK);
                }
            }
            src = reinterpret_cast<const int32_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src), 0));
            nblk = __shfl_sync(0xffffffffu, nblk, 0);
            unstaged = unstaged || nblk > kListCap;
            // every lane acquires the slot itself (it overwrites list entries the
            // producer read under the previous phase) and releases its own
            // stores on sfull below: no reliance on __syncwarp for cross-lane
            // ordering (compute-sanitizer racecheck reported the list reads as
            // racing with these stores when only lane 0 waited and arrived)
            SD_TWAIT(1, ptx::mbar_wait(sempty_bar + sslot, sphase ^ 1));
            for (int i = lane; i < nblk && i < kListCap; i += 32) sched_list[sslot * kListCap + i] = __ldcg(src + i);
            const int prob = __shfl_sync(0xffffffffu, t.prob, 0);
            // the last unit of the launch decoded: nothing reads the mask
            // workspaces any more (every other unit was decoded before its
            // counter increment), whatever the CTAs still have to compute
            if (L.release_all && prob >= 0 && lane == 0 &&
                atomicAdd(L.sched + 2, 1u) == static_cast<unsigned int>(num_units) - 1u) {
#ifdef SD_TRACE
                g_sd_timeline[(L.trace_id & 255) * 4 + 3] = gtimer();  // mask workspaces released
#endif
                for (int r = 0; r < 2; ++r) {
                    if (L.release[r]) {
                        __threadfence();
                        atomicAdd(L.release[r], gridDim.x);
                    }
                }
            }
            if (lane == 0) sched_unit[sslot] = t;
            ptx::mbar_arrive(sfull_bar + sslot);  // release: this lane's list / unit stores are visible
            if (++sslot == kSchedDepth) {
                sslot = 0;
                sphase ^= 1;
            }
            if (prob < 0) {
                // Every unit this CTA will run is decoded and its list staged in
                // smem: the mask workspace (lists, counts, row order) is no longer
                // read, so the next generation into it may start (reader
                // tracking, sd_internal.h) while this CTA's last units still run.
                if (lane == 0 && !unstaged && !L.release_all) release_workspaces(L);
                break;
            }
            // A unit without MMA work (an sdd unit that only zero-fills dropped
            // blocks, a dsd unit of a fully dropped row) has no loads to wait
            // for: claim the next unit right away instead of after the
            // producer's signal (the epilogue zero-fills it in turn).
            const bool loads = __shfl_sync(0xffffffffu, (t.n_eff > 0 && t.nstages > 0) ? 1 : 0, 0);
            if (lane == 0) {
                if (loads) ptx::mbar_wait(claim_bar, cphase);
                u = static_cast<int>(gridDim.x) + static_cast<int>(atomicAdd(L.sched, 1u));
            }
            if (loads) cphase ^= 1;
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int sa = 0;
            uint32_t acc_iter = 0;
            int sslot = 0;
            uint32_t sphase = 0;
            while (true) {
                SD_TWAIT(4, ptx::mbar_wait(sfull_bar + sslot, sphase));
                const Unit t = sched_unit[sslot];
                ptx::mbar_arrive(sempty_bar + sslot);
                if (++sslot == kSchedDepth) {
                    sslot = 0;
                    sphase ^= 1;
                }
                if (t.prob < 0) break;
                if (t.n_eff == 0) continue;
                const GemmArgs& a = L.p[t.prob];
                const bool a_mn = a.flags & kFlagAMN;
                const bool b_mn = a.flags & kFlagBMN;
                const uint32_t a_step = a_mn ? 2048u : 32u, b_step = b_mn ? 2048u : 32u;
                const uint32_t a_lbo = a_mn ? 8192u : 0u, b_lbo = b_mn ? 8192u : 0u;
                if constexpr (!WIDE) {
                    const uint32_t acc = acc_iter & 1;
                    const uint32_t acc_phase = (acc_iter >> 1) & 1;
                    ++acc_iter;
                    SD_TWAIT(3, ptx::mbar_wait(tempty_bar + acc, acc_phase ^ 1));
                    ptx::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * kBN;
                    const uint32_t idesc = ptx::make_idesc_bf16(kBM, t.n_eff, a_mn, b_mn);
                    for (int s = 0; s < t.nstages; ++s) {
                        SD_TWAIT(2, ptx::mbar_wait(full_bar + stage, phase));
                        SD_TADD(8, 1);
                        ptx::tc_fence_after();
                        const uint32_t a_addr = sbase + C::kOffA + stage * kABytes;
                        const uint32_t b_addr = sbase + C::kOffB + stage * kBBytes;
#ifndef SD_DIAG_NO_MMA
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            const uint64_t ad = ptx::make_sw128_desc(a_addr + k * a_step, a_lbo, 1024);
                            const uint64_t bd = ptx::make_sw128_desc(b_addr + k * b_step, b_lbo, 1024);
                            ptx::mma_bf16_ss(d_tmem, ad, bd, idesc, (s > 0 || k > 0) ? 1u : 0u);
                        }
#else
                        (void)a_addr; (void)b_addr; (void)idesc; (void)a_step; (void)b_step; (void)a_lbo; (void)b_lbo;
#endif
                        ptx::mma_commit(empty_bar + stage);
                        if (++stage == C::kSB) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    ptx::mma_commit(tfull_bar + acc);
                } else {
                    // one 128 x 512 accumulator: half h = TMEM columns [256h, 256h + 256)
                    const int nh = (t.n_eff + kBN - 1) / kBN;
                    const uint32_t rphase = acc_iter & 1;
                    ++acc_iter;
                    SD_TWAIT(3, ptx::mbar_wait(tempty_bar + 0, rphase ^ 1));
                    ptx::tc_fence_after();
                    const uint32_t idesc0 = ptx::make_idesc_bf16(kBM, min(kBN, t.n_eff), a_mn, b_mn);
                    const uint32_t idesc1 = ptx::make_idesc_bf16(kBM, max(16, t.n_eff - kBN), a_mn, b_mn);
                    for (int s = 0; s < t.nstages; ++s) {
                        const uint32_t a_addr = sbase + C::kOffA + sa * kABytes;
                        for (int h = 0; h < nh; ++h) {
                            if (h == 1 && s == 0) {
                                // half 1: free once the previous unit's epilogue drained it
                                SD_TWAIT(3, ptx::mbar_wait(tempty_bar + 1, rphase ^ 1));
                                ptx::tc_fence_after();
                            }
                            SD_TWAIT(2, ptx::mbar_wait(full_bar + stage, phase));
                            SD_TADD(8, 1);
                            ptx::tc_fence_after();
                            const uint32_t b_addr = sbase + C::kOffB + stage * kBBytes;
#ifndef SD_DIAG_NO_MMA
#pragma unroll
                            for (int k = 0; k < kBK / 16; ++k) {
                                const uint64_t ad = ptx::make_sw128_desc(a_addr + k * a_step, a_lbo, 1024);
                                const uint64_t bd = ptx::make_sw128_desc(b_addr + k * b_step, b_lbo, 1024);
                                ptx::mma_bf16_ss(tmem_base + kBN * h, ad, bd, h ? idesc1 : idesc0,
                                                 (s > 0 || k > 0) ? 1u : 0u);
                            }
#else
                            (void)a_addr; (void)b_addr; (void)idesc0; (void)idesc1; (void)a_step; (void)b_step; (void)a_lbo;
                            (void)b_lbo;
#endif
                            ptx::mma_commit(empty_bar + stage);
                            if (++stage == C::kSB) {
                                stage = 0;
                                phase ^= 1;
                            }
                        }
                        ptx::mma_commit(aempty_bar + sa);
                        if (++sa == C::kSA) sa = 0;
                    }
                    ptx::mma_commit(tfull_bar + 0);
                }
                if (a.counters)
                    atomicAdd(a.counters + t.row0 / kBM,
                              static_cast<unsigned long long>(t.nstages / 2) * (t.n_eff / 128));
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue =====================
        const uint32_t q = warp & 3;  // TMEM lane quarter == output row quarter
        uint8_t* ebuf = smem + C::kOffEpi + q * C::kEpiBufs * kEpiBufBytes;
        const uint32_t ebuf_addr = sbase + C::kOffEpi + q * C::kEpiBufs * kEpiBufBytes;
        uint32_t bi = 0;
        uint32_t acc_iter = 0;
        int sslot = 0;
        uint32_t sphase = 0;
        while (true) {
            SD_TWAIT(6, ptx::mbar_wait(sfull_bar + sslot, sphase));
            const Unit t = sched_unit[sslot];
            ptx::mbar_arrive(sempty_bar + sslot);  // each lane releases its own read of the slot
            if (++sslot == kSchedDepth) {
                sslot = 0;
                sphase ^= 1;
            }
            if (t.prob < 0) break;
            const GemmArgs& a = L.p[t.prob];
            const CUtensorMap* tmOut = &tms.m[3 * t.prob + 2];
            unsigned int* turn_base = L.sched + kSchedWords + t.prob * kTurnPerProb;
            if (a.flags & kFlagF32)
                epilogue_unit<WIDE, true>(a, tmOut, t, q, lane, tmem_base, tfull_bar, tempty_bar, ebuf, ebuf_addr,
                                          bi, acc_iter, turn_base, tr);
            else
                epilogue_unit<WIDE, false>(a, tmOut, t, q, lane, tmem_base, tfull_bar, tempty_bar, ebuf, ebuf_addr,
                                           bi, acc_iter, turn_base, tr);
            SD_TADD(11, 1);
        }
        if (lane == 0) ptx::bulk_wait_group<0>();
        __syncwarp();
    }

#ifdef SD_TRACE
    {
        const long long t_role_end = clock64();
        // warp 0 lane 0 (producer) -> slots 0,1,9 ; warp 1 lane 0 (MMA) -> 2,3,4,7,8 ; warp 4 lane 0 -> 5,6,10,11
        unsigned long long* out = g_sd_trace + blockIdx.x * kTraceSlots;
        if (warp == 0 && lane == 0) {
            atomicAdd(out + 0, tr[0]); atomicAdd(out + 1, tr[1]); atomicAdd(out + 9, t_role_end - t_start);
        } else if (warp == 1 && lane == 0) {
            atomicAdd(out + 2, tr[2]); atomicAdd(out + 3, tr[3]); atomicAdd(out + 4, tr[4]);
            atomicAdd(out + 7, t_role_end - t_start); atomicAdd(out + 8, tr[8]);
            // globaltimer of this CTA's run (ns) and its start relative to the launch's first CTA
            atomicAdd(out + 12, gtimer() - g_start);
            atomicAdd(out + 13, g_start);
        } else if (warp == 4 && lane == 0) {
            atomicAdd(out + 5, tr[5]); atomicAdd(out + 6, tr[6]); atomicAdd(out + 10, t_role_end - t_start);
            atomicAdd(out + 11, tr[11]);
            atomicAdd(out + 14, gtimer() - g_start);  // epilogue role end (ns after start)
        }
    }
#else
    (void)tr;
#endif
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc<kTmemCols>(tmem_base);
#ifdef SD_TRACE
    if (threadIdx.x == 0) atomicMax(&g_sd_timeline[(L.trace_id & 255) * 4 + 2], gtimer());
#endif
    if (threadIdx.x == 0) {
        // last CTA out re-arms the scheduler slot for the next launch
        __threadfence();
        if (atomicAdd(L.sched + 1, 1u) == gridDim.x - 1) {
            L.sched[0] = 0u;
            L.sched[1] = 0u;
            L.sched[2] = 0u;
            __threadfence();
        }
    }
}

}  // namespace

// Scheduler tuning switches (A/B experiments), all features on by default;
// SD_TUNING (environment) overrides the default for whole-process A/B runs.
static int initial_tuning() {
    const char* e = std::getenv("SD_TUNING");
    return e ? std::atoi(e) : 0;
}
static int g_tuning = initial_tuning();
int tuning() { return g_tuning; }
void set_tuning(int t) { g_tuning = t; }

// Unit width of a launch. 128 x 512 units cut operand bytes per MAC by a sixth
// but hold the whole TMEM (no second accumulator to overlap the epilogue
// with). Measured in one process on the same buffers (tools/ab_libs.py, one
// B200): dsd forward 2-6% faster at 4096^3-8192^3 for p <= 0.5, dW within +-2%,
// sdd (dX) 4-8% slower, and near p = 0.9 the units get too short (+30-45%). So:
// wide for launches of dsd problems only, with 512+ columns, unless the mask
// keeps under 20%; no keep hint (generic C-ABI calls) counts as dense enough.
static bool wide_units(const GemmCall* const* calls, int n) {
    if (g_tuning & kTuneNarrow) return false;
    if (g_tuning & kTuneWide) return true;
    // fewer wide units than SMs: the launch is latency-bound and twice as many
    // narrow units finish sooner (1024^3 layer step -6.5%, 2048^3 -2%) —
    // unless a problem will be split along its long reduction instead (fp32
    // dsd: the MLP's dW), which fills the SMs either way
    int64_t wide_count = 0;
    bool splittable = false;
    for (int i = 0; i < n; ++i) {
        const GemmArgs& a = calls[i]->args;
        wide_count += static_cast<int64_t>(a.n_row_tiles) * ((a.cols_out + 2 * kBN - 1) / (2 * kBN));
        splittable = splittable || (!(g_tuning & kTuneNoSplitK) && !(a.flags & kFlagSDD) && (a.flags & kFlagF32) &&
                                    a.red / kBK >= 64);
    }
    if (!splittable && wide_count < num_sms()) return false;
    for (int i = 0; i < n; ++i) {
        const GemmArgs& a = calls[i]->args;
        if ((a.flags & kFlagSDD) || a.cols_out <= kBN) return false;
        // a ragged 256-column unit per row costs a whole single-buffered wide
        // accumulator: the ViT fc2 forward (N = 768) is 3-5% faster narrow
        // (profiles/r01_cfg3_width_ab.txt)
        if (a.cols_out % (2 * kBN) != 0 && a.cols_out < 8 * kBN) return false;
        if (a.keep_hint >= 0.f && a.keep_hint < 0.2f) return false;
    }
    return true;
}

void launch_gemms(const GemmCall* const* calls, int n, cudaStream_t s, bool no_wait) {
    if (n < 1 || n > kMaxProblems) fail(SD_EINVAL, "launch_gemms: 1 or 2 problems per launch");
    configure_once_per_device(0, [] {
        check_cuda(cudaFuncSetAttribute(sd_gemm_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        KCfg<false>::kSmem),
                   "cudaFuncSetAttribute(max dynamic smem)");
        check_cuda(cudaFuncSetAttribute(sd_gemm_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        KCfg<true>::kSmem),
                   "cudaFuncSetAttribute(max dynamic smem, wide)");
        check_cuda(cudaFuncSetAttribute(sd_gemm_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        KCfg<false>::kSmem),
                   "cudaFuncSetAttribute(max dynamic smem, hash)");
    });
    // dense problems go to the 2-CTA kernel (half the per-SM operand traffic
    // per MAC: tools/gemm2_check.py, +10-25% over this kernel at 4096-8192)
    {
        bool dense = true;
        for (int i = 0; i < n; ++i) dense = dense && gemm2_routed(calls[i]->args);
        if (dense) {
            // the problems of one call are independent: the second launch needs
            // nothing from the first (and the first's own wait, or its caller's
            // no_wait guarantee, covers everything before), so it never waits
            for (int i = 0; i < n; ++i)
                launch_gemm2(calls[i]->ta, calls[i]->tb, calls[i]->tout, calls[i]->args, nullptr, nullptr, 0, s,
                             i == 0 ? no_wait : true, calls[i]->release);
            return;
        }
        for (int i = 0; i < n; ++i)
            if (calls[i]->args.flags & kFlagOutMask) fail(SD_ERUNTIME, "masked dense GEMM not routable to the 2-CTA kernel");
    }
    TensorMaps tms;
    LaunchArgs L;
    std::memset(&L, 0, sizeof L);
    const int sms = num_sms();
    // split-K for dsd problems with too few output tiles to fill the GPU (e.g.
    // the MLP's dW, 72 tiles over a 65536-long reduction): fp32 outputs only;
    // split 0 stores, the others reduce-add in split order behind a per-tile
    // turnstile, so the result is bit-reproducible run to run.
    // unit width: 128 x 512 (wide) or 128 x 256, one choice per launch
    // hash mode (small plans): every problem decodes its lists from the mask's
    // counter hash; narrow units, no tile-row order, no mask-workspace reads
    bool hash = true;
    for (int i = 0; i < n; ++i) hash = hash && calls[i]->args.hash_mode != 0;
    const bool wide = !hash && wide_units(calls, n);
    const int width = wide ? 2 * kBN : kBN;
    GemmArgs pa[kMaxProblems];
    float cost[kMaxProblems];
    for (int i = 0; i < n; ++i) {
        pa[i] = calls[i]->args;
        pa[i].splits = 1;
        pa[i].tail_rows = 0;
        pa[i].n_col_units = (pa[i].cols_out + width - 1) / width;
        const int base = pa[i].n_row_tiles * pa[i].n_col_units;
        const bool sdd = pa[i].flags & kFlagSDD;
        const int red_stages = pa[i].red / kBK;
        // The split count is a function of the PROBLEM only (its 128 x 256
        // tile count, or that of the full problem a row slab belongs to), never
        // of the launch's unit width or of slabbing: the splits fix the fp32
        // summation order, so the wide and narrow kernels and the dW row slabs
        // of the data-parallel backward stay bit-identical to the full dW.
        const int split_rows = pa[i].split_rows > 0 ? pa[i].split_rows : pa[i].rows_out;
        const int base_narrow = (split_rows / kBM) * ((pa[i].cols_out + kBN - 1) / kBN);
        if (!(g_tuning & kTuneNoSplitK) && !sdd && (pa[i].flags & kFlagF32) && base_narrow < 2 * sms &&
            red_stages >= 64) {
            int sp = (2 * sms + base_narrow - 1) / base_narrow;
            sp = std::min(sp, red_stages / 32);
            if (sp > 1) {
                if (base * 4 > kTurnPerProb) fail(SD_ERUNTIME, "split-K turnstile capacity exceeded");
                pa[i].splits = sp;
                pa[i].flags |= kFlagReduce;
            }
        }
        cost[i] = static_cast<float>(red_stages) / pa[i].splits;  // stages per unit (upper bound)
    }
    // one shared queue, heaviest units first: the problem with the larger
    // per-unit cost is handed out first
    // (dsd cost is an upper bound — only kept blocks are reduced — while sdd
    // units always run the full reduction, so ties go to the sdd problem)
    int order[kMaxProblems] = {0, 1};
    const bool sdd0 = pa[0].flags & kFlagSDD, sdd1 = n == 2 && (pa[1].flags & kFlagSDD);
    if (n == 2 && (cost[1] > cost[0] || (cost[1] == cost[0] && sdd1 && !sdd0))) {
        order[0] = 1;
        order[1] = 0;
    }
    if (hash) {
        // small plans: dX's full-reduction units are the backward's critical
        // path and the step leaves SMs idle, so dX takes one kept block per unit
        // (1024^3 layer step -8% at p = 0.5, -18% at p = 0.9), and when the whole
        // step still fits on the SMs with every unit halved, the forward and dW
        // units are halved too (512^3 -12%, 768^3 -10%; at 1024^3 they would
        // not fit and the step is 15-28% slower; profiles/r02_small_hash_ab.txt)
        for (int i = 0; i < n; ++i) {
            const bool sdd = pa[i].flags & kFlagSDD;
            const bool fits = pa[i].hash_plan_units <= sms, all_fit = 2 * pa[i].hash_plan_units <= sms;
            if (pa[i].splits == 1 && ((sdd && fits && pa[i].out_col_blk == 128) || (!sdd && all_fit)))
                pa[i].tail_rows = pa[i].n_row_tiles;
        }
    }
    // tail halving on the problem handed out last, when the launch is only a
    // few waves deep: its lightest ~half wave of units become half-width
    {
        int total_units = 0;
        for (int i = 0; i < n; ++i) total_units += gemm_units(pa[i]);
        GemmArgs& last = pa[order[n - 1]];
        const bool sdd = last.flags & kFlagSDD;
        // not for launches of less than one wave: there the halved units only
        // add epilogues, and a plan's forward and early backward no longer fit
        // on the SMs side by side (1024^3 layer step at p = 0.1: 24.3 -> 18.1
        // us, p = 0.5: 18.5 -> 17.6 us; profiles/r02_small_ab.txt)
        if (!wide && !(g_tuning & kTuneNoTailHalving) && last.splits == 1 && total_units >= sms &&
            total_units < 12 * sms &&
            (!sdd || last.out_col_blk == 128)) {
            // about half a wave of half-width units: measured -2.5% on the 4096^3
            // fused backward at p = 0.5 and -5% on dX at p = 0.1; two waves' worth
            // cost more operand traffic than the shorter tail saves
            // (profiles/r01_tail_halving_ab.txt)
            const int T = (sms + 4 * last.n_col_units - 1) / (4 * last.n_col_units);
            last.tail_rows = std::min(T, last.n_row_tiles);
        }
    }
    int total = 0;
    for (int j = 0; j < n; ++j) {
        const int i = order[j];
        tms.m[3 * j] = calls[i]->ta;
        tms.m[3 * j + 1] = calls[i]->tb;
        tms.m[3 * j + 2] = calls[i]->tout;
        L.p[j] = pa[i];
        if ((g_tuning & kTuneNoRowOrder) || hash) L.p[j].row_order = nullptr;
        L.p[j].unit_begin = total;
        L.p[j].num_units = gemm_units(L.p[j]);
        total += L.p[j].num_units;
    }
    L.nprob = n;
    L.total_units = total;
    int cap = sms;
#ifdef SD_TRACE
    if (const char* e = std::getenv("SD_MAX_CTAS")) cap = std::max(1, std::min(cap, std::atoi(e)));
#endif
    const int grid = total < cap ? total : cap;
    if (grid <= 0) return;
    L.sched = sched_slot(s);
    L.trace_id = static_cast<int>(sd_launch_count());
    L.no_wait = no_wait && !(g_tuning & kTuneNoEarlyBackward);
    // bound mask workspaces read by this launch (lists, counts, row orders)
    int nrel = 0;
    bool may_unstage = false;  // a dsd list longer than the scheduler's smem staging
    for (int i = 0; i < n && !hash; ++i) {
        unsigned int* r = calls[i]->release;
        if (r && !(nrel > 0 && L.release[0] == r)) L.release[nrel++] = r;
        const GemmArgs& a = L.p[i];
        if (!(a.flags & kFlagSDD) && a.list_idx && a.red / a.red_blk > kListCap) may_unstage = true;
    }
    L.release_all = may_unstage ? 0 : 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = wide ? KCfg<true>::kSmem : KCfg<false>::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (hash) check_cuda(cudaLaunchKernelEx(&cfg, sd_gemm_kernel<false, true>, tms, L), "sd_gemm_kernel<hash> launch");
    else if (wide) check_cuda(cudaLaunchKernelEx(&cfg, sd_gemm_kernel<true, false>, tms, L), "sd_gemm_kernel<wide> launch");
    else check_cuda(cudaLaunchKernelEx(&cfg, sd_gemm_kernel<false, false>, tms, L), "sd_gemm_kernel launch");
    note_launch();
    for (int r = 0; r < nrel; ++r) mask_note_readers(L.release[r], grid, s);
}

}  // namespace sd

#ifdef SD_TRACE
// timeline: per launch id (mod 256) {first CTA start, first CTA past griddepcontrol.wait, last CTA end}
extern "C" SD_API int sd_timeline_read(unsigned long long* host) {
    if (cudaDeviceSynchronize() != cudaSuccess) return SD_ERUNTIME;
    if (cudaMemcpyFromSymbol(host, g_sd_timeline, sizeof(unsigned long long) * 256 * 4) != cudaSuccess)
        return SD_ERUNTIME;
    static unsigned long long init[256 * 4];
    for (int i = 0; i < 256; ++i) init[4 * i] = init[4 * i + 1] = ~0ull, init[4 * i + 2] = init[4 * i + 3] = 0;
    cudaMemcpyToSymbol(g_sd_timeline, init, sizeof init);
    return SD_OK;
}

extern "C" SD_API int sd_trace_read(unsigned long long* host, int n) {
    if (cudaDeviceSynchronize() != cudaSuccess) return SD_ERUNTIME;
    if (cudaMemcpyFromSymbol(host, g_sd_trace, sizeof(unsigned long long) * n) != cudaSuccess) return SD_ERUNTIME;
    static unsigned long long zeros[1024 * kTraceSlots] = {0};
    cudaMemcpyToSymbol(g_sd_trace, zeros, sizeof zeros);
    return SD_OK;
}
#endif
