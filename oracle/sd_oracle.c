/*
 * sd_oracle.c — CPU restatement of the SparseDrop reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the B200 CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load the
 * library built from it (oracle/libsdoracle.so). The product path never links
 * or calls it, and there is no CPU fallback anywhere in paper_2411_01238_b200.
 *
 * Parity pinning: every function here is checked (tests/test_oracle.py) against
 *   (1) golden vectors produced by running the UNMODIFIED reference
 *       (oracle/_ref/libsdref.so built by oracle/Makefile from /root/reference),
 *       committed under tests/golden/ with the script that made them
 *       (tests/golden/make_golden.py), and
 *   (2) the live reference library whenever /root/reference is present.
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).
 *
 * Status codes follow include/sparsedrop_b200.h: 0 ok, 1 invalid_argument,
 * 2 out_of_range. The message of the last error is kept per thread.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

static _Thread_local char g_err[512];

const char* sdo_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ---- rng.hpp ----------------------------------------------------------- */

/* rng.hpp:11-16 — splitmix64 finalizer. */
uint64_t sdo_mix64(uint64_t z) {
    z += UINT64_C(0x9E3779B97F4A7C15);
    z = (z ^ (z >> 30)) * UINT64_C(0xBF58476D1CE4E5B9);
    z = (z ^ (z >> 27)) * UINT64_C(0x94D049BB133111EB);
    return z ^ (z >> 31);
}

/* rng.hpp:18-20 — counter_hash(seed, a, b). */
uint64_t sdo_counter_hash(uint64_t seed, uint64_t a, uint64_t b) {
    return sdo_mix64(sdo_mix64(sdo_mix64(seed) ^ a) ^ b);
}

/* rng.hpp:28-30 — top 53 bits mapped to [0, 1). */
double sdo_unit_interval(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }

/* layer.hpp:64-67 — effective_seed(spec, step_seed, layer_index). */
uint64_t sdo_effective_seed(uint64_t seed, uint64_t step_seed, int layer_index) {
    return sdo_counter_hash(seed, step_seed, (uint64_t)(int64_t)layer_index);
}

/* Integer form of the keep test used by the device kernel: with u = h >> 11
 * (< 2^53, exactly representable), unit_interval(h) >= p  <=>  u >= ceil(p*2^53).
 * p*2^53 is exact in double (power-of-two scaling), so the threshold is exact. */
uint64_t sdo_keep_threshold(double p) { return (uint64_t)ceil(p * 0x1.0p53); }

/* ---- block_mask.cpp ---------------------------------------------------- */

static int64_t word_count(int64_t bits) { return (bits + 63) / 64; }

static int popcount64(uint64_t w) { return __builtin_popcountll(w); }

static int get_bit(const uint64_t* words, int64_t b) { return (int)((words[b >> 6] >> (b & 63)) & 1u); }

/* block_mask.cpp:52-80 — sample_mask(spec, rows, cols).
 * Validation (:53-61) with the reference's messages; one draw per block
 * keep = unit_interval(counter_hash(seed, r, c)) >= p (:70); bits packed
 * LSB-first, b = r*C + c (:71-77, block_mask.hpp:28-30); popcount (:78).
 * row_block_offset (our extension for row shards, 0 = the reference) hashes the
 * GLOBAL block row r0 + r while packing the LOCAL index r: the reference's
 * decision depends only on (seed, r, c), so a shard's rows equal the global
 * mask's rows. */
int sdo_sample_mask(double p, int m_blk, int k_blk, uint64_t seed, int rows, int cols,
                    int row_block_offset, uint64_t* words, int64_t* keep_count) {
    char msg[256];
    if (p < 0.0 || p >= 1.0) {
        snprintf(msg, sizeof msg, "dropout rate must lie in [0, 1), got %f", p);
        return fail(1, msg);
    }
    if (m_blk <= 0 || rows % m_blk != 0) {
        snprintf(msg, sizeof msg, "mask block size m_blk=%d does not divide rows=%d", m_blk, rows);
        return fail(1, msg);
    }
    if (k_blk <= 0 || cols % k_blk != 0) {
        snprintf(msg, sizeof msg, "mask block size k_blk=%d does not divide cols=%d", k_blk, cols);
        return fail(1, msg);
    }
    const int R = rows / m_blk, C = cols / k_blk;
    if (R <= 0 || C <= 0) return fail(1, "BlockMask geometry must be positive");
    const int64_t total = (int64_t)R * C, nw = word_count(total);
    memset(words, 0, (size_t)nw * sizeof(uint64_t));
    int64_t keep = 0;
    for (int64_t b = 0; b < total; ++b) {
        const int r = (int)(b / C), c = (int)(b % C);
        const uint64_t h = sdo_counter_hash(seed, (uint64_t)(r + row_block_offset), (uint64_t)c);
        const int k = sdo_unit_interval(h) >= p;
        words[b >> 6] |= (uint64_t)k << (b & 63);
    }
    for (int64_t i = 0; i < nw; ++i) keep += popcount64(words[i]);
    *keep_count = keep;
    return 0;
}

/* block_mask.cpp:82-98 — mask_from_words: word count and zero padding bits. */
int sdo_mask_from_words(int R, int C, const uint64_t* words, int64_t nwords, int64_t* keep_count) {
    if (R <= 0 || C <= 0) return fail(1, "BlockMask geometry must be positive");
    const int64_t bits = (int64_t)R * C;
    if (nwords != word_count(bits)) return fail(1, "BlockMask word count does not match grid");
    if (bits & 63) {
        const uint64_t padding = ~(uint64_t)0 << (bits & 63);
        if (words[nwords - 1] & padding) return fail(1, "BlockMask has nonzero bits past the block grid");
    }
    int64_t keep = 0;
    for (int64_t i = 0; i < nwords; ++i) keep += popcount64(words[i]);
    *keep_count = keep;
    return 0;
}

/* block_mask.cpp:125-135 — kept_blocks_in_row: strictly increasing kept
 * block columns of one row; out_of_range for a bad row. */
int sdo_kept_blocks_in_row(const uint64_t* words, int R, int C, int row, int32_t* idx, int32_t* n) {
    if (row < 0 || row >= R) {
        char msg[128];
        snprintf(msg, sizeof msg, "block row %d outside grid with %d rows", row, R);
        return fail(2, msg);
    }
    int32_t k = 0;
    for (int c = 0; c < C; ++c)
        if (get_bit(words, (int64_t)row * C + c)) idx[k++] = c;
    *n = k;
    return 0;
}

/* block_mask.cpp:117-123 — transpose_mask: grid (C, R), bit (c, r) = bit (r, c). */
void sdo_transpose_mask(const uint64_t* words, int R, int C, uint64_t* out) {
    memset(out, 0, (size_t)word_count((int64_t)R * C) * sizeof(uint64_t));
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c)
            if (get_bit(words, (int64_t)r * C + c)) {
                const int64_t b = (int64_t)c * R + r;
                out[b >> 6] |= (uint64_t)1 << (b & 63);
            }
}

/* block_mask.cpp:100-115 — retile: each bit replicated split_m x split_k. */
int sdo_retile(const uint64_t* words, int R, int C, int m_blk, int k_blk, int split_m, int split_k,
               uint64_t* out) {
    if (split_m <= 0 || m_blk % split_m != 0) return fail(1, "split_m does not divide m_blk");
    if (split_k <= 0 || k_blk % split_k != 0) return fail(1, "split_k does not divide k_blk");
    const int R2 = R * split_m, C2 = C * split_k;
    memset(out, 0, (size_t)word_count((int64_t)R2 * C2) * sizeof(uint64_t));
    for (int r = 0; r < R2; ++r)
        for (int c = 0; c < C2; ++c)
            if (get_bit(words, (int64_t)(r / split_m) * C + c / split_k)) {
                const int64_t b = (int64_t)r * C2 + c;
                out[b >> 6] |= (uint64_t)1 << (b & 63);
            }
    return 0;
}

/* layer.hpp:69-76 — sample_element_mask: m(i,j) = unit_interval(counter_hash(seed, i, j)) >= p. */
void sdo_element_mask(uint64_t seed, double p, int rows, int cols, uint8_t* out) {
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j)
            out[(size_t)i * cols + j] = sdo_unit_interval(sdo_counter_hash(seed, (uint64_t)i, (uint64_t)j)) >= p;
}

/* block_mask.cpp:137-186 — write_mask: "BMSK", version 0x01, LE u32 block_rows,
 * block_cols, m_blk, k_blk, then the words as LE u64. Returns the byte count. */
int64_t sdo_write_mask(const uint64_t* words, int R, int C, int m_blk, int k_blk, uint8_t* out) {
    int64_t n = 0;
    out[n++] = 'B'; out[n++] = 'M'; out[n++] = 'S'; out[n++] = 'K'; out[n++] = 0x01;
    const uint32_t hdr[4] = {(uint32_t)R, (uint32_t)C, (uint32_t)m_blk, (uint32_t)k_blk};
    for (int h = 0; h < 4; ++h)
        for (int b = 0; b < 4; ++b) out[n++] = (uint8_t)(hdr[h] >> (8 * b));
    const int64_t nw = word_count((int64_t)R * C);
    for (int64_t w = 0; w < nw; ++w)
        for (int b = 0; b < 8; ++b) out[n++] = (uint8_t)(words[w] >> (8 * b));
    return n;
}

/* ---- tests/oracles.hpp ------------------------------------------------- */

/* tests/oracles.hpp:31-41 — random_matrix<float>: |v| in [0.25, 1.25),
 * sign from bit 0 of the same draw; computed in double, then narrowed. */
void sdo_random_matrix_f32(int rows, int cols, uint64_t seed, float* out) {
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) {
            const uint64_t bits = sdo_counter_hash(seed, (uint64_t)i, (uint64_t)j);
            const double mag = 0.25 + sdo_unit_interval(bits);
            out[(size_t)i * cols + j] = (float)((bits & 1) ? mag : -mag);
        }
}

/* float -> bf16 with round-to-nearest-even (the device inputs' rounding). */
void sdo_f32_to_bf16(const float* in, uint16_t* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        uint32_t u;
        memcpy(&u, &in[i], 4);
        if ((u & 0x7fffffffu) > 0x7f800000u) {
            out[i] = (uint16_t)((u >> 16) | 0x40u);
        } else {
            u += 0x7fffu + ((u >> 16) & 1u);
            out[i] = (uint16_t)(u >> 16);
        }
    }
}

void sdo_bf16_to_f64(const uint16_t* in, double* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        const uint32_t u = (uint32_t)in[i] << 16;
        float f;
        memcpy(&f, &u, 4);
        out[i] = f;
    }
}

/* ---- gemm.hpp ---------------------------------------------------------- */

/* Row-parallel helper (the reference's for_each_tile_row, gemm.hpp:86-100,
 * interleaves tile rows over std::threads; rows are disjoint, so any schedule
 * gives identical bits). */
typedef void (*row_fn)(void* ctx, int row);
struct par_ctx { row_fn fn; void* ctx; int lo, hi, stride, start; };

static void* par_worker(void* arg) {
    struct par_ctx* p = (struct par_ctx*)arg;
    for (int i = p->lo + p->start; i < p->hi; i += p->stride) p->fn(p->ctx, i);
    return NULL;
}

static void parallel_rows(int lo, int hi, int threads, row_fn fn, void* ctx) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (threads > hi - lo) threads = hi - lo > 0 ? hi - lo : 1;
    pthread_t tid[256];
    struct par_ctx pc[256];
    for (int t = 0; t < threads; ++t) {
        pc[t] = (struct par_ctx){fn, ctx, lo, hi, threads, t};
        if (t > 0) pthread_create(&tid[t], NULL, par_worker, &pc[t]);
    }
    par_worker(&pc[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* gemm.hpp:133-170 — dsd_matmul, restated per output row in double:
 * c[i][j] = scale * sum over kept K-blocks tk of row block i/m_blk (ascending,
 * :151-152) of sum_k a[i][k] * b[k][j]; dropped blocks are never read. Rows
 * [row_lo, row_hi) only (a row slab of the full product; 0, m for all).
 * kblock_per_tile_row (gemm.hpp:31-37) counts K-block iterations per tile row
 * with tile width n_blk, as the reference does (:156, :165). */
struct dsd_ctx {
    const double *a, *b;
    const uint64_t* words;
    int n, k, m_blk, k_blk, C, row_lo;
    double scale;
    double* c;
};

static void dsd_row(void* vp, int i) {
    const struct dsd_ctx* p = (const struct dsd_ctx*)vp;
    const int ti = i / p->m_blk, n = p->n, k = p->k;
    double* crow = p->c + (size_t)(i - p->row_lo) * n;
    for (int j = 0; j < n; ++j) crow[j] = 0.0;
    for (int tk = 0; tk < p->C; ++tk) {
        if (!get_bit(p->words, (int64_t)ti * p->C + tk)) continue;
        for (int kk = tk * p->k_blk; kk < (tk + 1) * p->k_blk; ++kk) {
            const double aik = p->a[(size_t)i * k + kk];
            const double* brow = p->b + (size_t)kk * n;
            for (int j = 0; j < n; ++j) crow[j] += aik * brow[j];
        }
    }
    for (int j = 0; j < n; ++j) crow[j] *= p->scale;
}

int sdo_dsd_matmul_f64(const double* a, const uint64_t* words, const double* b, int m, int n, int k,
                       int m_blk, int n_blk, int k_blk, double scale, int row_lo, int row_hi,
                       int threads, double* c, uint64_t* kblock_per_tile_row) {
    if (m_blk <= 0 || m % m_blk) return fail(1, "tile size m_blk does not divide dimension");
    if (n_blk <= 0 || n % n_blk) return fail(1, "tile size n_blk does not divide dimension");
    if (k_blk <= 0 || k % k_blk) return fail(1, "tile size k_blk does not divide dimension");
    struct dsd_ctx ctx = {a, b, words, n, k, m_blk, k_blk, k / k_blk, row_lo, scale, c};
    parallel_rows(row_lo, row_hi, threads, dsd_row, &ctx);
    if (kblock_per_tile_row) {
        for (int ti = row_lo / m_blk; ti < (row_hi + m_blk - 1) / m_blk; ++ti) {
            uint64_t kept = 0;
            for (int tk = 0; tk < ctx.C; ++tk) kept += (uint64_t)get_bit(words, (int64_t)ti * ctx.C + tk);
            kblock_per_tile_row[ti - row_lo / m_blk] = kept * (uint64_t)(n / n_blk);
        }
    }
    return 0;
}

/* gemm.hpp:176-213 — sdd_matmul: the mask sits on the OUTPUT, grid
 * (m/m_blk, n/n_blk); dropped output blocks are exactly +0.0 (never computed,
 * :184, :193); kept blocks get the full K reduction times scale. */
struct sdd_ctx {
    const double *a, *b;
    const uint64_t* words;
    int n, k, m_blk, n_blk, Cn, row_lo;
    double scale;
    double* c;
};

static void sdd_row(void* vp, int i) {
    const struct sdd_ctx* p = (const struct sdd_ctx*)vp;
    const int ti = i / p->m_blk, n = p->n, k = p->k;
    double* crow = p->c + (size_t)(i - p->row_lo) * n;
    for (int j = 0; j < n; ++j) crow[j] = 0.0;
    for (int kk = 0; kk < k; ++kk) {
        const double aik = p->a[(size_t)i * k + kk];
        const double* brow = p->b + (size_t)kk * n;
        for (int tj = 0; tj < p->Cn; ++tj) {
            if (!get_bit(p->words, (int64_t)ti * p->Cn + tj)) continue;
            for (int j = tj * p->n_blk; j < (tj + 1) * p->n_blk; ++j) crow[j] += aik * brow[j];
        }
    }
    for (int j = 0; j < n; ++j) crow[j] *= p->scale;
}

int sdo_sdd_matmul_f64(const double* a, const double* b, const uint64_t* words, int m, int n, int k,
                       int m_blk, int n_blk, double scale, int row_lo, int row_hi, int threads,
                       double* c) {
    if (m_blk <= 0 || m % m_blk) return fail(1, "tile size m_blk does not divide dimension");
    if (n_blk <= 0 || n % n_blk) return fail(1, "tile size n_blk does not divide dimension");
    struct sdd_ctx ctx = {a, b, words, n, k, m_blk, n_blk, n / n_blk, row_lo, scale, c};
    parallel_rows(row_lo, row_hi, threads, sdd_row, &ctx);
    return 0;
}

/* layer.hpp:158 — dX = sdd_matmul(dy, transpose(W), m, s, tiles_dx) without
 * materialising W^T: dx[i][kk] = s * sum_j dy[i][j] * w[kk][j] on kept mask
 * blocks (i/m_blk, kk/k_blk), exactly +0.0 elsewhere. Rows [row_lo, row_hi). */
struct dx_ctx {
    const double *dy, *w;
    const uint64_t* words;
    int n, k, m_blk, k_blk, C, row_lo;
    double scale;
    double* dx;
};

static void dx_row(void* vp, int i) {
    const struct dx_ctx* p = (const struct dx_ctx*)vp;
    const int ti = i / p->m_blk, n = p->n, k = p->k;
    double* out = p->dx + (size_t)(i - p->row_lo) * k;
    const double* dyr = p->dy + (size_t)i * n;
    for (int kk = 0; kk < k; ++kk) {
        if (!get_bit(p->words, (int64_t)ti * p->C + kk / p->k_blk)) {
            out[kk] = 0.0;
            continue;
        }
        const double* wr = p->w + (size_t)kk * n;
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += dyr[j] * wr[j];
        out[kk] = p->scale * s;
    }
}

int sdo_layer_dx_f64(const double* dy, const double* w, const uint64_t* words, int m, int n, int k,
                     int m_blk, int k_blk, double scale, int row_lo, int row_hi, int threads,
                     double* dx) {
    if (m_blk <= 0 || m % m_blk) return fail(1, "tile size m_blk does not divide dimension");
    if (k_blk <= 0 || k % k_blk) return fail(1, "tile size k_blk does not divide dimension");
    struct dx_ctx ctx = {dy, w, words, n, k, m_blk, k_blk, k / k_blk, row_lo, scale, dx};
    parallel_rows(row_lo, row_hi, threads, dx_row, &ctx);
    return 0;
}

/* layer.hpp:159-160 — dW = dsd_matmul(transpose(x), transpose_mask(m), dy, s,
 * tiles_dw) without materialising x^T: dw[kk][j] = s * sum over M-blocks ti kept
 * in mask column kk/k_blk (ascending, block_mask.cpp:117-123) of
 * sum_{i in ti} x[i][kk] * dy[i][j]. dW rows [krow_lo, krow_hi), all n columns. */
struct dw_ctx {
    const double *x, *dy;
    const uint64_t* words;
    int n, k, m_blk, k_blk, R, C, krow_lo;
    double scale;
    double* dw;
};

static void dw_row(void* vp, int kk) {
    const struct dw_ctx* p = (const struct dw_ctx*)vp;
    const int n = p->n, k = p->k;
    double* out = p->dw + (size_t)(kk - p->krow_lo) * n;
    for (int j = 0; j < n; ++j) out[j] = 0.0;
    const int tc = kk / p->k_blk;
    for (int ti = 0; ti < p->R; ++ti) {
        if (!get_bit(p->words, (int64_t)ti * p->C + tc)) continue;
        for (int i = ti * p->m_blk; i < (ti + 1) * p->m_blk; ++i) {
            const double xik = p->x[(size_t)i * k + kk];
            const double* dyr = p->dy + (size_t)i * n;
            for (int j = 0; j < n; ++j) out[j] += xik * dyr[j];
        }
    }
    for (int j = 0; j < n; ++j) out[j] *= p->scale;
}

int sdo_layer_dw_f64(const double* x, const double* dy, const uint64_t* words, int m, int n, int k,
                     int m_blk, int k_blk, double scale, int krow_lo, int krow_hi, int threads,
                     double* dw) {
    if (m_blk <= 0 || m % m_blk) return fail(1, "tile size m_blk does not divide dimension");
    if (k_blk <= 0 || k % k_blk) return fail(1, "tile size k_blk does not divide dimension");
    struct dw_ctx ctx = {x, dy, words, n, k, m_blk, k_blk, m / m_blk, k / k_blk, krow_lo, scale, dw};
    parallel_rows(krow_lo, krow_hi, threads, dw_row, &ctx);
    return 0;
}

/* gemm.hpp:104-128 — dense_gemm, rows [row_lo, row_hi). */
struct dense_ctx {
    const double *a, *b;
    int n, k, row_lo;
    double* c;
};

static void dense_row(void* vp, int i) {
    const struct dense_ctx* p = (const struct dense_ctx*)vp;
    const int n = p->n, k = p->k;
    double* crow = p->c + (size_t)(i - p->row_lo) * n;
    for (int j = 0; j < n; ++j) crow[j] = 0.0;
    for (int kk = 0; kk < k; ++kk) {
        const double aik = p->a[(size_t)i * k + kk];
        const double* brow = p->b + (size_t)kk * n;
        for (int j = 0; j < n; ++j) crow[j] += aik * brow[j];
    }
}

int sdo_dense_gemm_f64(const double* a, const double* b, int m, int n, int k, int row_lo, int row_hi,
                       int threads, double* c) {
    (void)m;
    struct dense_ctx ctx = {a, b, n, k, row_lo, c};
    parallel_rows(row_lo, row_hi, threads, dense_row, &ctx);
    return 0;
}

/* gemm.hpp:217-228 — flops_dense / flops_effective. kind 0 = dsd, 1 = sdd. */
uint64_t sdo_flops_dense(int64_t m, int64_t n, int64_t k) { return (uint64_t)2 * m * n * k; }
uint64_t sdo_flops_effective(int64_t n, int64_t k, int m_blk, int n_blk, int k_blk, int64_t keep,
                             int kind) {
    if (kind == 0) return 2ull * (uint64_t)n * m_blk * k_blk * (uint64_t)keep;
    return 2ull * (uint64_t)k * m_blk * n_blk * (uint64_t)keep;
}
