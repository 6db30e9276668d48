// sd_internal.h — declarations shared by the CUDA translation units of
// libsparsedrop_b200.so (not part of the public C-ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/sparsedrop_b200.h"

namespace sd {

// Thrown inside the library, converted to a status code at the C boundary.
struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
int num_sms();
void note_launch(uint64_t n = 1);

// ---------------------------------------------------------------- mask plan
void launch_mask_plan(const sd_block_mask& m, bool from_words, uint64_t seed_mix,
                      uint64_t threshold, cudaStream_t s);
void launch_mask_transpose(const sd_block_mask& in, sd_block_mask& out, cudaStream_t s);
void launch_mask_retile(const sd_block_mask& in, int split_m, int split_k, sd_block_mask& out,
                        cudaStream_t s);

// ---------------------------------------------------------------- GEMM
// Output tile: 128 rows x up to 256 columns; 64-element reduction stages.
constexpr int kBM = 128;
constexpr int kBN = 256;
constexpr int kBK = 64;

struct GemmArgs {
    int rows_out;      // output rows (multiple of 128)
    int cols_out;      // output columns (multiple of 128)
    int red;           // reduction length (multiple of 64)
    int n_row_tiles;   // rows_out / 128
    int n_col_units;   // ceil(cols_out / 256)
    // dsd: per output-row-block list of kept reduction blocks (null = dense)
    const int32_t* list_cnt;
    const int32_t* list_idx;
    int list_stride;
    int red_blk;       // reduction block (mask block along the reduction), multiple of 64
    int out_row_blk;   // output rows per list/mask row (multiple of 128)
    const int32_t* row_order;  // optional tile-row permutation (when out_row_blk == 128)
    // sdd: output-block mask bits
    const uint64_t* words;
    int mask_cols;     // mask block columns (output column blocks)
    int out_col_blk;   // output column block (128 or 256)
    float scale;
    void* out;
    unsigned long long* counters;
    unsigned int* sched;  // {next-unit counter, CTAs-done counter}, zero between launches
};

// A zeroed {counter, done} pair for one persistent-kernel launch (ring of
// slots per device, re-armed by the last CTA of the launch that used it).
unsigned int* sched_slot();

// A_MN / B_MN: operand is MN-major (contiguous along the output dimension)
// rather than K-major (contiguous along the reduction).
enum class GemmKind { dsd, sdd };

void launch_gemm(bool a_mn, bool b_mn, GemmKind kind, bool out_f32, const CUtensorMap& ta,
                 const CUtensorMap& tb, const CUtensorMap& tout, const GemmArgs& args,
                 cudaStream_t s);

// 2D row-major tensor map: `inner` contiguous elements, `outer` rows, 128B swizzle.
CUtensorMap make_tmap_2d(const void* base, bool f32, uint64_t inner, uint64_t outer,
                         uint32_t box_inner, uint32_t box_outer);

}  // namespace sd
