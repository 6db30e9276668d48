// sd_internal.h — declarations shared by the CUDA translation units of
// libsparsedrop_b200.so (not part of the public C-ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>

#include "../../include/sparsedrop_b200.h"

namespace sd {

// Thrown inside the library, converted to a status code at the C boundary.
struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void set_last_error(const std::string& msg);  // sd_last_error() of the calling thread
void check_cuda(cudaError_t e, const char* what);
int num_sms();
// Runs `fn` once per (key, current device) under a lock: kernel attributes such
// as the dynamic shared-memory limit are per device context. Keys: 0 sd_gemm,
// 1 sd_gemm2, 2 mask kernels, 3 elementwise kernels.
void configure_once_per_device(int key, const std::function<void()>& fn);
void note_launch(uint64_t n = 1);

// ---------------------------------------------------------------- mask readers
// Lets a mask generation overlap the tail of the GEMM that still reads the
// previous mask of the same workspace (sd_capi.cu, "reader tracking"): every
// persistent GEMM CTA that reads a bound workspace's lists adds 1 to the
// workspace's release counter (ticket[1]) once its last list read is done; the
// next generation into that workspace waits for the count of reader CTAs
// launched since the previous one instead of for the whole preceding grid.
void mask_register_workspace(void* ws, size_t bytes, unsigned int* rel);  // sd_mask_bind
unsigned int* mask_release_counter(const sd_block_mask* m);  // m's counter if m is a live sd_mask_bind binding
void mask_note_readers(unsigned int* rel, int ctas, cudaStream_t s);  // after a successful launch
void mask_note_untracked(const void* p);  // a reader that does not release: next generation waits
// At a generation into the workspace of `rel`: true (and *target) when the
// generation may wait on the counter instead of griddepcontrol.wait. Resets the
// workspace's pending count either way (the kernel zeroes the counter).
bool mask_take_release(unsigned int* rel, cudaStream_t s, uint32_t* target);
void note_counter_wait();  // a generation launched in counter mode (sd_dev_mask_counter_waits)

// ---------------------------------------------------------------- mask plan
// off_path (small plans whose GEMMs hash their lists): every block lets the
// next launch start at once and waits for the preceding grid before writing;
// the generation's number is published in ticket word 2 by its last block and
// the next off-path generation into the workspace waits for it before writing
// (generations stay ordered by construction). Returns the number (0: none).
uint32_t launch_mask_plan(const sd_block_mask& m, bool from_words, uint64_t seed_mix,
                          uint64_t threshold, cudaStream_t s, bool off_path = false);
// the workspace's last off-path generation number, replaced by `gen`
uint32_t mask_swap_last_gen(unsigned int* rel, uint32_t gen);
void launch_mask_transpose(const sd_block_mask& in, sd_block_mask& out, cudaStream_t s);
// graph replays of a plan step: the generation kernel and its seed in a parameter block
const void* mask_plan_kernel_func();
size_t mask_plan_args_size();
void mask_plan_patch_seed(void* args, uint64_t seed_mix);
void launch_mask_retile(const sd_block_mask& in, int split_m, int split_k, sd_block_mask& out,
                        cudaStream_t s);

// ---------------------------------------------------------------- GEMM
// Output tile: 128 rows x up to 256 columns; 64-element reduction stages.
constexpr int kBM = 128;
constexpr int kBN = 256;
constexpr int kBK = 64;

// Operand / output layout flags of one GEMM problem.
enum GemmFlags : uint32_t {
    kFlagAMN = 1u,  // A is MN-major (contiguous along the output rows), else K-major
    kFlagBMN = 2u,  // B is MN-major (contiguous along the output columns), else K-major
    kFlagSDD = 4u,  // output-block skipping (sdd) instead of reduction-block skipping (dsd)
    kFlagF32 = 8u,  // fp32 output, else bf16
    kFlagReduce = 16u,  // split-K: split 0 stores, split j > 0 reduce-adds after split j - 1 (fixed order)
    kFlagOutMask = 32u,  // 2-CTA dense only: output blocks dropped in `words` (128x128, mask_cols
                         // per row) are written as +0.0 (dX at low p: masked dense, see sd_capi.cu)
    kFlagPairs = 64u,    // dX split by mask-row pairs: the 2-CTA kernel computes the column blocks both
                         // rows of a pair keep (taken in ascending pairs), the 1-CTA sdd kernel the
                         // remainder and the zero fill (sd_gemm2.cu; mask_cols <= 64)
};

struct GemmArgs {
    uint32_t flags;    // GemmFlags
    int rows_out;      // output rows (multiple of 128)
    int cols_out;      // output columns (multiple of 128)
    int red;           // reduction length (multiple of 64)
    int n_row_tiles;   // rows_out / 128
    int n_col_units;   // ceil(cols_out / 256)
    // dsd: per output-row-block list of kept reduction blocks (null = dense)
    // sdd: per output-row-block list of kept output blocks (+ dropped at the tail)
    const int32_t* list_cnt;
    const int32_t* list_idx;
    int list_stride;
    int red_blk;       // reduction block (mask block along the reduction), multiple of 64
    int out_row_blk;   // output rows per list/mask row (multiple of 128)
    const int32_t* row_order;  // optional tile-row permutation (when out_row_blk == 128)
    const uint64_t* words;     // mask bits (informational)
    int mask_cols;     // mask block columns (sdd: output column blocks)
    int out_col_blk;   // sdd output column block (128 or 256)
    float scale;
    void* out;
    unsigned long long* counters;
    int splits;        // dsd split-K factor (>= 1): each unit reduces a contiguous 1/splits of its list
    int tail_rows;     // the last tail_rows tile rows (lightest, end of the queue) use half-width units
    float keep_hint;   // nominal kept fraction of the mask (1 - p) when known, else < 0
    int split_rows;    // rows of the full problem that fix the split-K factor (0: rows_out; a dW row
                       // slab passes the full dW's rows so its reduction order equals the full call's)
    // Hash mode (small plans, sd_gemm_kernel<false, true>): the unit's kept list
    // comes from the mask's counter hash instead of the list arrays, so the
    // launch reads nothing of the mask workspace and need not follow the mask
    // generation: keep(r, c) = (mix64(mix64(seed_mix ^ (r + row_off)) ^ c) >> 11)
    // >= threshold over hash_len <= 64 entries. 0 = off; 1 = the list of mask
    // ROW list_row + list_off (forward, dX); 2 = of mask COLUMN list_row +
    // list_off (dW).
    int hash_mode;
    int hash_len;
    int hash_row_off;   // the mask's row_block_offset (row shards hash their global rows)
    int hash_list_off;
    uint64_t hash_seed_mix;
    uint64_t hash_threshold;
    int hash_plan_units;  // 128 x 256 units of the small plan's whole step (forward + dX + dW)
    int unit_begin;    // filled by launch_gemms: first global unit of this problem
    int num_units;     // filled by launch_gemms
};

inline int gemm_units(const GemmArgs& a) {
    const int T = a.tail_rows;
    return ((a.n_row_tiles - T) * a.n_col_units + T * 2 * a.n_col_units) * (a.splits > 0 ? a.splits : 1);
}

// Zeroed {next unit, CTAs done, units decoded, spare} counters for one
// persistent-kernel launch, followed by kTurnstiles split-K turnstiles (two
// problems x up to kTurnPerProb/4 output tiles x 4 epilogue row quarters). A
// ring of slots per stream (sched_slot), re-armed by the last CTA of the launch that used
// it (turnstiles are reset by each tile's last split). A launch captured into a
// CUDA graph gets a dedicated slot that is never handed out again (it is
// replayed later, possibly beside eager launches).
constexpr int kSchedWords = 64;
constexpr int kTurnPerProb = 1216;  // split-K only below 2 x 148 narrow tiles: <= 295 tiles x 4 quarters
constexpr int kTurnstiles = 2 * kTurnPerProb;
constexpr int kSlotWords = kSchedWords + kTurnstiles;
unsigned int* sched_slot(cudaStream_t s);

// A fully validated, ready-to-launch GEMM problem (tensor maps encoded).
struct GemmCall {
    CUtensorMap ta, tb, tout;
    GemmArgs args;
    unsigned int* release = nullptr;  // release counter of the mask whose lists args reads (host side)
};

// Scheduler tuning switches (bitmask; 0 = everything on), for A/B runs.
enum TuneFlags : int {
    kTuneNoTailHalving = 1,
    kTuneNoSplitK = 2,
    kTuneNoRowOrder = 4,
    kTuneNoFusedBackward = 8,   // the backward is always two launches
    kTuneNoGemm2 = 16,  // dense problems on the 1-CTA kernel instead of the 2-CTA one
    kTuneWide = 32,     // force 128 x 512 units on the 1-CTA kernel
    kTuneNarrow = 64,   // force 128 x 256 units on the 1-CTA kernel
    kTuneNoEarlyBackward = 128,  // a plan's backward waits for its forward grid (griddepcontrol.wait)
    kTuneNoMaskOverlap = 256,    // mask generation waits for the whole preceding grid
    kTuneNoGeluTable = 512,      // GELU' evaluated per element instead of from the shared-memory table
    kTuneNoMaskedDense = 1024,   // low-p dX stays on the sdd kernel instead of the masked 2-CTA dense GEMM
    kTuneSplitDwFirst = 32768,   // a two-launch backward launches dW before dX (default: dX first)
    kTuneForceFused = 65536,     // the backward is always one fused launch (default: two launches when the
                                 // fused launch would have >= 48 waves of units)
    kTunePairs = 16384,          // mid-p plans split dX by mask-row pairs (2-CTA + 1-CTA remainder); off
                                 // by default: bit-identical but not faster (profiles/r02_row_pairs_ab.txt)
    kTuneGemm2Narrow = 4096,     // 2-CTA kernel: always 256 x 256 pair tiles
    kTuneGemm2Wide = 8192,       // 2-CTA kernel: 256 x 512 pair tiles whenever the columns allow
    kTuneDxt = 1048576,          // a plan's dX on the transposed 2-CTA kernel (sd_dxt.cu) + dW on its own launch
    kTuneNoSmallHash = 2097152,  // small plans keep the mask generation ahead of list-reading GEMMs
    kTuneNoOwnBits = 2048,       // masked 2-CTA dX reads keep bits per chunk and releases at exit (the
                                 // > kMaxOwnUnits fallback, forced for tests)
};
int tuning();
void set_tuning(int t);

// Launch 1 or 2 independent GEMM problems as ONE persistent kernel sharing a
// single heaviest-first work queue (problem 0's units are handed out first).
// no_wait: the launch reads nothing the immediately preceding grid writes and
// writes nothing it reads (a plan's backward right after its forward), so its
// CTAs skip griddepcontrol.wait and start on the SMs the previous grid's tail
// frees. Every earlier grid is complete by then (the previous grid's CTAs
// passed their own wait before triggering this launch).
void launch_gemms(const GemmCall* const* calls, int n, cudaStream_t s, bool no_wait = false);
inline void launch_gemm(const GemmCall& c, cudaStream_t s, bool no_wait = false) {
    const GemmCall* p = &c;
    launch_gemms(&p, 1, s, no_wait);
}

// 2-CTA (cta_group::2) kernel for dense problems (no mask list): 256 x 256
// pair tiles, static schedule. Used by launch_gemms when every problem of the
// launch is dense and has at least one wave of pair tiles.
bool gemm2_supported(const GemmArgs& a);
bool gemm2_pairs_supported(const GemmArgs& a);
void launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tout, const GemmArgs& g,
                  const int32_t* pair_cnt, const int32_t* pair_idx, int pair_stride, cudaStream_t s,
                  bool no_wait = false, unsigned int* release = nullptr);
// launch_gemms sends a problem to the 2-CTA kernel when this holds
bool gemm2_routed(const GemmArgs& a);

// 2D row-major tensor map: `inner` contiguous elements, `outer` rows, 128B swizzle.
CUtensorMap make_tmap_2d(const void* base, bool f32, uint64_t inner, uint64_t outer,
                         uint32_t box_inner, uint32_t box_outer);
// bf16 [red][mn] operand (mn contiguous, row pitch ld) as 3D (64, red, mn / 64): box = 128 mn
// x 64 red in two atom-major 8 KB SW128 atoms; coordinates (0, red0, mn0 / 64).
CUtensorMap make_tmap_mn_atoms(const void* base, uint64_t mn, uint64_t red, uint64_t ld, uint32_t atoms = 2);
// 2D map without swizzle (the transposed dX epilogue's 32 x 32 store boxes)
CUtensorMap make_tmap_2d_noswizzle(const void* base, bool f32, uint64_t inner, uint64_t outer, uint32_t box_inner,
                                   uint32_t box_outer);

// dX on 2-CTA pairs in the transposed form dX^T = W dY^T (sd_dxt.cu): a
// layer's bf16 dX over 128 x 128 mask blocks, from its prepared sdd call.
bool dxt_supported(const GemmArgs& dx);
void launch_dxt(const GemmCall& dx, const void* dy, const void* w, cudaStream_t s, bool no_wait);

// ---------------------------------------------------------------- NCCL (sd_comm.cu)
// In-place sum all-reduce of `count` elements (SD_DTYPE_*) on stream s.
void comm_allreduce_sum(sd_comm* c, void* buf, size_t count, int dtype, cudaStream_t s);
int comm_nranks(const sd_comm* c);
int comm_device(const sd_comm* c);

}  // namespace sd
