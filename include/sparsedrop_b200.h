/*
 * sparsedrop_b200.h — the C-ABI drop-in boundary of the B200 SparseDrop path.
 *
 * Plain C: device pointers, sizes, a stream handle (cudaStream_t passed as
 * void*). No torch or C++ types cross this boundary. Every entry point replaces
 * one symbol of the reference's C++ operator API (namespace sparsedrop,
 * /root/reference/proj/include/sparsedrop/), cited per function below; the C++
 * wrapper include/sparsedrop_b200.hpp and the Python package
 * paper_2411_01238_b200 restore the reference's names, ownership and exception
 * types on top of it.
 *
 * Conventions
 *  - All matrices are dense row-major (matrix.hpp:11, element (i,j) at
 *    i*cols+j), bf16 (1) or fp32 (0) as tagged, 16-byte aligned.
 *  - Calls are stream-ordered and asynchronous; nothing allocates on the hot
 *    path. Buffers are caller-owned device memory.
 *  - Status codes: SD_OK, or SD_EINVAL (the reference throws
 *    std::invalid_argument), SD_ERANGE (std::out_of_range), SD_ERUNTIME
 *    (std::runtime_error: CUDA errors, missing device). sd_last_error() returns
 *    the message of the calling thread's last failure; messages keep the
 *    reference substrings ("m_blk", "k_blk", "does not divide",
 *    "gemm shape mismatch", "mask geometry").
 *  - There is no CPU fallback: without a B200 (sm_100) device every compute
 *    call returns SD_ERUNTIME.
 */
#ifndef SPARSEDROP_B200_H
#define SPARSEDROP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SD_API __attribute__((visibility("default")))
#else
#define SD_API
#endif

#define SD_OK 0
#define SD_EINVAL 1
#define SD_ERANGE 2
#define SD_ERUNTIME 3

#define SD_DTYPE_F32 0
#define SD_DTYPE_BF16 1

#define SD_ABI_VERSION 1

/* Device-resident block mask plus the compaction products the GEMMs consume.
 * Mirrors sparsedrop::BlockMask (block_mask.hpp:31-76): grid block_rows x
 * block_cols of m_blk x k_blk blocks, bit b = r*block_cols + c LSB-first in
 * words[b/64], set = KEEP, padding bits zero. row_block_offset is the GLOBAL
 * index of local block row 0 for a row shard (0 for an unsharded mask).
 * Bind the pointers with sd_mask_bind() over one device workspace of
 * sd_mask_workspace_bytes() bytes (zero-initialised once before first use). */
typedef struct sd_block_mask {
    int32_t block_rows, block_cols, m_blk, k_blk, row_block_offset, reserved;
    uint64_t* words;      /* ceil(R*C/64) mask words                              */
    int64_t* keep_count;  /* 1: popcount of the words                             */
    int32_t* row_cnt;     /* R: kept blocks per block row                          */
    int32_t* row_idx;     /* R*C: kept_blocks_in_row(mask, r), row stride C        */
    int32_t* col_cnt;     /* C: kept blocks per block column                      */
    int32_t* col_idx;     /* C*R: kept_blocks_in_row(transpose_mask(mask), c)     */
    int32_t* row_order;   /* R: block rows by kept count, descending (scheduling)  */
    int32_t* col_order;   /* C: block columns by kept count, descending           */
    uint32_t* ticket;     /* internal counters (keep zero; sd_mask_bind reserves 256 B:
                             [0] completion ticket, [1] reader release count,
                             [2] last off-path generation number) */
} sd_block_mask;

SD_API int sd_abi_version(void);
SD_API const char* sd_last_error(void);
/* Number of usable sm_100 devices (0 when none: compute calls then fail). */
SD_API int sd_device_count(void);

/* Minimal device-memory plumbing so FFI callers (and the C++ wrapper
 * include/sparsedrop_b200.hpp) need no CUDA headers. kind: 0 host->device,
 * 1 device->host, 2 device->device. stream may be NULL (legacy stream). */
SD_API int sd_device_alloc(void** ptr, size_t bytes);
SD_API int sd_device_free(void* ptr);
SD_API int sd_memcpy(void* dst, const void* src, size_t bytes, int32_t kind, void* stream);
SD_API int sd_memset(void* dst, int32_t value, size_t bytes, void* stream);
SD_API int sd_stream_synchronize(void* stream);

/* Workspace size for a block_rows x block_cols mask and its compaction lists. */
SD_API size_t sd_mask_workspace_bytes(int32_t block_rows, int32_t block_cols);
/* Carve `workspace` into the mask's arrays and record the geometry
 * (block_mask.hpp:31-41, BlockMask(block_rows, block_cols, m_blk, k_blk)). */
SD_API int sd_mask_bind(sd_block_mask* mask, void* workspace, int32_t block_rows, int32_t block_cols,
                 int32_t m_blk, int32_t k_blk, int32_t row_block_offset);

/* Replaces sparsedrop::sample_mask(const DropoutSpec&, int rows, int cols)
 * (block_mask.hpp:81, block_mask.cpp:52-80): validates p in [0,1) and that
 * m_blk | rows, k_blk | cols against `mask`'s block extents, then draws one
 * splitmix64 counter-hash bit per block, keep iff
 * unit_interval(counter_hash(seed, row_block_offset + r, c)) >= p — bit-exact
 * with the reference — and fills the compaction lists (kept_blocks_in_row on
 * the mask and on transpose_mask(mask), block_mask.cpp:117-135) in the same
 * launch. `rows` x `cols` are the LOCAL element extents of the mask. */
SD_API int sd_mask_sample(sd_block_mask* mask, uint64_t seed, double p, int32_t rows, int32_t cols,
                   void* stream);

/* Replaces mask_from_words + the compaction: `mask->words` already holds the
 * bits (e.g. uploaded from a host BlockMask); rebuild keep_count and lists.
 * (block_mask.cpp:82-98 — padding validation is the host wrapper's job.) */
SD_API int sd_mask_compact(sd_block_mask* mask, void* stream);

/* Replaces sparsedrop::transpose_mask (block_mask.cpp:117-123): `out` must be
 * bound with the swapped geometry (block_cols x block_rows, k_blk x m_blk). */
SD_API int sd_mask_transpose(const sd_block_mask* in, sd_block_mask* out, void* stream);

/* Replaces sparsedrop::retile (block_mask.cpp:100-115): `out` must be bound
 * with grid (R*split_m) x (C*split_k) and blocks (m_blk/split_m) x (k_blk/split_k). */
SD_API int sd_mask_retile(const sd_block_mask* in, int32_t split_m, int32_t split_k, sd_block_mask* out,
                   void* stream);

/* Replaces sparsedrop::dense_gemm (gemm.hpp:104-128): c = a * b,
 * a: m x k bf16, b: k x n bf16, c: m x n (c_dtype). tcgen05 GEMM.
 * Requires m % 128 == 0, n % 128 == 0, k % 64 == 0. */
SD_API int sd_dense_gemm(const void* a, const void* b, void* c, int32_t c_dtype, int32_t m, int32_t n,
                  int32_t k, void* stream);

/* Replaces sparsedrop::dsd_matmul (gemm.hpp:133-170):
 * c = scale * (a (.) expand(mask)) * b — dropped K-blocks of `a` are never
 * read. mask geometry must equal (m/m_blk) x (k/k_blk) blocks of m_blk x k_blk
 * (gemm.hpp:139-140). kblock_per_tile_row (optional, m/128 u64 device
 * counters, zeroed by the caller) accumulates executed 128x128x128 block
 * products per 128-row tile row (KernelCounters, gemm.hpp:31-37, n_blk = 128). */
SD_API int sd_dsd_matmul(const void* a, const sd_block_mask* mask, const void* b, float scale, void* c,
                  int32_t c_dtype, int32_t m, int32_t n, int32_t k,
                  unsigned long long* kblock_per_tile_row, void* stream);

/* Replaces sparsedrop::sdd_matmul (gemm.hpp:176-213):
 * c = scale * (a * b) restricted to kept OUTPUT blocks, a: m x k, b: k x n
 * row-major; dropped output blocks are written as exact +0.0 (never computed).
 * mask geometry must equal (m/m_blk) x (n/n_blk) with n_blk = mask->k_blk. */
SD_API int sd_sdd_matmul(const void* a, const void* b, const sd_block_mask* mask, float scale, void* c,
                  int32_t c_dtype, int32_t m, int32_t n, int32_t k,
                  unsigned long long* kblock_per_tile_row, void* stream);

/* Fused dropout+linear layer (layer.hpp:85-162), operands in place — no
 * materialised transposes (the reference copies W^T and x^T, layer.hpp:158-160).
 * x: m x k bf16, w: k x n bf16, dy: m x n bf16, mask over x (m/m_blk x k/k_blk).
 *  forward:      y  = scale * (x (.) m) w                          (layer.hpp:115)
 *  backward dX:  dx = scale * (dy w^T) (.) m   (sdd, W read K-major) (layer.hpp:158)
 *  backward dW:  dw = scale * (x (.) m)^T dy   (dsd over column lists) (layer.hpp:159-160)
 * scale = float(1.0/(1.0-p)) as dropout_scale<float> (layer.hpp:78-81). */
SD_API int sd_linear_forward(const void* x, const sd_block_mask* mask, const void* w, float scale, void* y,
                      int32_t y_dtype, int32_t m, int32_t n, int32_t k, void* stream);
SD_API int sd_linear_backward_dx(const void* dy, const void* w, const sd_block_mask* mask, float scale,
                          void* dx, int32_t dx_dtype, int32_t m, int32_t n, int32_t k,
                          void* stream);
SD_API int sd_linear_backward_dw(const void* x, const sd_block_mask* mask, const void* dy, float scale,
                          void* dw, int32_t dw_dtype, int32_t m, int32_t n, int32_t k,
                          void* stream);

/* Dense backward GEMMs for the dense fwd+bwd baseline (layer.hpp:140-145):
 * dx = dy w^T (w read in place), dw = x^T dy (x read in place). */
SD_API int sd_dense_gemm_nt(const void* a, const void* b_t, void* c, int32_t c_dtype, int32_t m,
                     int32_t n, int32_t k, void* stream); /* c[m,n] = a[m,k] * b_t[n,k]^T */
SD_API int sd_dense_gemm_tn(const void* a_t, const void* b, void* c, int32_t c_dtype, int32_t m,
                     int32_t n, int32_t k, void* stream); /* c[m,n] = a_t[k,m]^T * b[k,n] */

/* Layer plan: the fused dropout+linear layer of layer.hpp:85-162 with every
 * operand bound once (tensor maps encoded once, no per-step host work beyond
 * the launches) — the runtime object a trainer keeps per layer instance.
 * Buffers: x (m x k), w (k x n), dy (m x n) bf16 inputs; y (m x n), dx (m x k),
 * dw (k x n) outputs in the given dtypes; `mask` bound with geometry
 * (m/m_blk) x (k/k_blk) (row_block_offset selects a row shard's global rows).
 * p fixes the drop rate and the scale float(1/(1-p)) (layer.hpp:78-81).
 *   forward : sample_mask(seed) + y = s (x (.) m) w          (2 launches)
 *   backward: dw = s (x (.) m)^T dy, then dx = s (dy w^T) (.) m  (2 launches)
 * backward_dw / backward_dx split the two so a data-parallel caller can
 * all-reduce dw on another stream while dx runs. */
typedef struct sd_layer_plan sd_layer_plan;
SD_API int sd_layer_plan_create(sd_layer_plan** plan, const void* x, const void* w, const void* dy,
                                void* y, int32_t y_dtype, void* dx, int32_t dx_dtype, void* dw,
                                int32_t dw_dtype, int32_t m, int32_t n, int32_t k, double p,
                                const sd_block_mask* mask);
SD_API int sd_layer_plan_forward(sd_layer_plan* plan, uint64_t seed, void* stream);
SD_API int sd_layer_plan_backward(sd_layer_plan* plan, void* stream);
/* dW rows of mask-column blocks [C*part/nparts, C*(part+1)/nparts) only — the
 * same tiles and reduction order as sd_layer_plan_backward_dw, so the parts
 * together equal it bit for bit. Data-parallel callers all-reduce each part
 * while the next part and dX compute. SD_ERANGE for a bad part/nparts. */
SD_API int sd_layer_plan_backward_dw_part(sd_layer_plan* plan, int32_t part, int32_t nparts, void* stream);
SD_API int sd_layer_plan_backward_dw(sd_layer_plan* plan, void* stream);
SD_API int sd_layer_plan_backward_dx(sd_layer_plan* plan, void* stream);
/* Dense baseline with the same buffers (layer.hpp:98-99, 140-145): y = x w,
 * dw = x^T dy, dx = dy w^T on the same tcgen05 kernel, no mask. */
SD_API int sd_layer_plan_dense_forward(sd_layer_plan* plan, void* stream);
SD_API int sd_layer_plan_dense_backward(sd_layer_plan* plan, void* stream);
/* Plan options (bit set; default 0):
 * SD_PLAN_DY_READY  the caller guarantees dY — and everything else the backward
 *   reads — is written BEFORE sd_layer_plan_forward is enqueued, and nothing
 *   writes it between the forward and the backward (e.g. a fixed synthetic dY,
 *   or one uploaded before the step). The first backward launch right after the
 *   forward then skips griddepcontrol.wait and starts on the SMs the forward's
 *   last wave frees. Without it the backward always waits for the preceding
 *   grid, which is required when a caller kernel computes dY from Y in between:
 *   such a kernel may trigger its dependents early (PDL). */
#define SD_PLAN_DY_READY 1
SD_API int sd_layer_plan_set_options(sd_layer_plan* plan, int32_t options);
/* One CUDA-graph launch per step, for host-bound callers (small layers, many
 * layers per step): what = 1 replays sample_mask(seed) + forward, what = 3 the
 * whole step (+ backward). The plan's launches are captured once per `what` on
 * a private stream (same kernels, same PDL edges as the eager calls) and the
 * seed is patched into the graph's mask node per call; results equal the eager
 * calls'. Isolated 1024^3 steps: 35 -> 26 us (profiles/r02_isolated_probe.jsonl). */
SD_API int sd_layer_plan_graph_step(sd_layer_plan* plan, uint64_t seed, int32_t what, void* stream);
SD_API int sd_layer_plan_destroy(sd_layer_plan* plan);

/* ---- Data-parallel backward over row shards (the reference's
 * decomposition: tile rows are independent, gemm.hpp:84-100, and the keep
 * decision depends only on (seed, global row, column), block_mask.cpp:70).
 * Rank g owns rows [g*M/G, (g+1)*M/G) of X, dY, Y, dX (its plan is created with
 * row_block_offset = first global block row); W is replicated; each rank's dW
 * is the partial sum over its rows and ONE sum all-reduce (NCCL, NVLink)
 * gives every rank the full dW. The library owns the NCCL communicator; NCCL
 * is loaded at run time (the copy already in the process if any, else
 * libnccl.so.2; SD_NCCL_LIBRARY overrides). */
typedef struct sd_comm sd_comm;
#define SD_COMM_ID_BYTES 128
/* rank 0: a fresh 128-byte NCCL unique id, to be broadcast by the caller */
SD_API int sd_comm_unique_id(void* id_out);
/* every rank, on its own device (cudaSetDevice first): collective */
SD_API int sd_comm_init(sd_comm** comm, int32_t nranks, int32_t rank, const void* id);
SD_API int sd_comm_destroy(sd_comm* comm);
SD_API int sd_comm_nccl_version(int32_t* version);
/* in-place sum all-reduce of `count` elements (SD_DTYPE_F32 / SD_DTYPE_BF16) */
SD_API int sd_comm_allreduce_sum(sd_comm* comm, void* buf, size_t count, int32_t dtype, void* stream);
/* backward(layer, ctx, dy) of a row shard (layer.hpp:128-162) with the dW
 * all-reduce: dW in `nparts` row slabs (mask-column blocks, bit-identical to
 * the full dW's rows), slab i all-reduced on `comm_stream` while slab i+1 and
 * then dX compute on `stream`; `stream` waits for the last all-reduce before
 * anything enqueued after this call (comm_stream NULL: all on `stream`). */
SD_API int sd_layer_plan_backward_allreduce(sd_layer_plan* plan, sd_comm* comm, int32_t nparts, void* stream,
                                            void* comm_stream);

/* The MLP block's activation between two SparseDrop Linears (configs[2]):
 * exact GELU and its backward, one HBM pass each over n bf16 values
 * (n % 8 == 0, 16-byte aligned). act = h*Phi(h); dh = grad*(Phi(h) + h*phi(h)). */
SD_API int sd_gelu_forward(const void* h, void* act, int64_t n, void* stream);
SD_API int sd_gelu_backward(const void* h, const void* grad, void* dh, int64_t n, void* stream);

/* Generic dense tcgen05 GEMM c[m,n] = scale * A * B. a_mn = 0: a is m x k
 * row-major (K-major); 1: a is k x m row-major (read transposed in place).
 * b_mn = 1: b is k x n row-major; 0: b is n x k row-major (read transposed). */
SD_API int sd_gemm_ex(const void* a, int32_t a_mn, const void* b, int32_t b_mn, void* c, int32_t c_dtype,
                      int32_t m, int32_t n, int32_t k, float scale, void* stream);

/* The paper's comparison baselines (layer.hpp:69-76,105-111,
 * 148-156): out = in (.) m * scale, bf16 rows x cols (cols % 8 == 0), with m
 * the reference's per-element counter-hash mask sample_element_mask(seed, p)
 * (block_mask == NULL, bit-exact) or the expansion of a device BlockMask. */
SD_API int sd_dropout_apply(const void* in, void* out, int32_t rows, int32_t cols, uint64_t seed, double p,
                            float scale, const sd_block_mask* block_mask, void* stream);

/* Effective FLOPs (gemm.hpp:217-228): kind 0 = dsd (2*n*m_blk*k_blk*keep),
 * 1 = sdd (2*k*m_blk*n_blk*keep). */
SD_API uint64_t sd_flops_dense(int64_t m, int64_t n, int64_t k);
SD_API uint64_t sd_flops_effective(int64_t n, int64_t k, int32_t m_blk, int32_t n_blk, int32_t k_blk,
                            int64_t keep, int32_t kind);

/* Launch counter: number of kernels this library has enqueued (evidence that the
 * native path ran; see bench.py "gpu_launches"). */
SD_API uint64_t sd_launch_count(void);

/* Scheduler tuning switches for A/B measurements (default 0):
 * 1 no tail halving (half-width units for about the last half wave of narrow launches),
 * 2 no split-K, 4 no heaviest-first row order,
 * 8 backward always as two launches (default: one fused launch, or two — dX
 *    then dW, the second not waiting for the first — when the fused launch
 *    would have at least 48 waves of units, where dW's 128x512 units pay),
 * 16 dense (unmasked) GEMMs on the 1-CTA kernel instead of the 2-CTA
 *    (cta_group::2) kernel,
 * 32 force 128x512 tiles on the 1-CTA kernel, 64 force 128x256 tiles
 *    (default: 128x512 for dsd-only launches with a keep hint >= 0.2),
 * 128 a layer plan's backward waits for its forward grid even with
 *    SD_PLAN_DY_READY (default with that option: the first backward launch right
 *    after the plan's forward starts on the SMs the forward's last wave frees;
 *    it reads nothing the forward writes),
 * 256 mask generation waits for the whole preceding grid (default, for a
 *    workspace bound by sd_mask_bind: only for the GEMM CTAs still reading its
 *    previous lists, which release it when their last list read is done),
 * 512 GELU' evaluated per element instead of from the shared-memory table,
 * 1024 a low-p plan's dX stays on the sdd kernel (default: p <= 0.2, or <= 0.3
 *    on large problems, computes dX as the 2-CTA dense GEMM with dropped output
 *    blocks written as +0.0; bit-identical),
 * 2048 the masked 2-CTA dX reads its keep bits per output chunk and releases the
 *    mask workspace at exit (the path for CTAs with more than 512 units,
 *    forced here for tests),
 * 4096 the 2-CTA kernel always uses 256x256 pair tiles, 8192 always 256x512
 *    where the columns allow (default: 256x512 with at least two waves of them),
 * 16384 a plan with 0.3 < p <= 0.7 splits dX by mask-row pairs: the column
 *    blocks both rows of a pair keep run on the 2-CTA kernel, the rest on the
 *    1-CTA sdd kernel (bit-identical; off by default: not faster, measured),
 * 32768 a two-launch backward launches dW first, 65536 always one fused launch,
 * 1048576 a plan's dX on the transposed 2-CTA kernel (dX^T = W dY^T, two kept
 *    blocks of one mask row per pair MMA; bit-identical; off by default: slower,
 *    measured),
 * 2097152 small plans keep the list-reading path (default: a plan whose whole
 *    step fits on the SMs at once, with a mask grid of at most 64 x 64, runs its
 *    GEMMs from the mask's counter hash and generates the mask after the
 *    forward, off the critical path; bit-identical).
 * The environment variable SD_TUNING sets the initial value. */
SD_API int sd_set_tuning(int32_t flags);

#ifdef __cplusplus
}
#endif

#endif /* SPARSEDROP_B200_H */
