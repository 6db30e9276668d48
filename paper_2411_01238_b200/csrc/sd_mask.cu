// sd_mask.cu — block-mask generation and compaction (one launch).
//
// K1 (sample_mask, block_mask.cpp:52-80): the keep bit of block (r, c) is the
//     reference's splitmix64 counter hash, keep iff
//       unit_interval(counter_hash(seed, r, c)) >= p
//     evaluated exactly in integers: (h >> 11) >= ceil(p * 2^53). The decision
//     depends only on (seed, r, c), so a row shard hashes its GLOBAL rows
//     r0 + r and is bit-identical to the matching rows of the global mask.
// K2 (kept_blocks_in_row, block_mask.cpp:125-135, on the mask and on
//     transpose_mask, :117-123): warp-ballot compaction, one warp per block row
//     (row lists; the dropped columns fill the row's tail for the sdd zero
//     fill) and one block per block column (column lists); positions are the
//     popcount of the ballot below the lane, so lists come out strictly
//     increasing like the reference's.
// The three parts read nothing but (seed, r, c) — each recomputes the hash — so
// they run as independent blocks of a single grid; keep_count and the
// cost-ordered row / column permutations the persistent GEMM scheduler walks
// (heaviest first) come from one extra block that recomputes the counts itself
// (grids up to 32768 blocks; larger ones: the last block to finish, threadfence
// + ticket). All of this is latency-bound integer work (a 512x64 grid is 4 KB
// of words), so it is kept off the layer step's critical path: a generation
// into a workspace waits only for the reader CTAs of its previous contents to
// release it (wait_workspace_free), i.e. it runs during the tail of the
// backward that still finishes on the old mask.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "sd_internal.h"

namespace sd {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxOrderBins = 8192;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

#ifdef SD_TRACE
__device__ unsigned long long g_sd_timeline[256 * 4];  // this TU's copy (mask launches)
__device__ __forceinline__ unsigned long long gtimer_m() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

struct PlanArgs {
    int trace_id;
    sd_block_mask m;
    int from_words;
    uint64_t seed_mix;   // mix64(seed): counter_hash = mix64(mix64(seed_mix ^ r) ^ c)
    uint64_t threshold;  // ceil(p * 2^53)
    int nb_words, nb_rows, nb_cols;
    int inline_order;  // one extra block computes counts, keep_count and the orders itself
    // reader tracking (sd_internal.h): the bound workspace's release counter
    // (null: not a bound workspace); rel_wait: wait for rel >= rel_target
    // instead of griddepcontrol.wait
    unsigned int* rel;
    uint32_t rel_target;
    int rel_wait;
    // small plans (hash-mode GEMMs, sd_capi.cu): nothing on the GPU reads this
    // generation's lists, so every block lets its dependents launch at once
    // (trigger_early); gen_seq is published in ticket word 2 by the last block
    // out, and prev_gen (the previous generation into the workspace) is waited
    // for before the first write, so generations stay ordered by construction
    int trigger_early;
    uint32_t gen_seq;
    uint32_t prev_gen;
};

__device__ __forceinline__ void publish_generation(const PlanArgs& a) {
    if (a.gen_seq) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.m.ticket + 2), "r"(a.gen_seq) : "memory");
}

__device__ __forceinline__ unsigned long long gclock() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Wait until the previous contents of the workspace are no longer needed.
// Counter mode: the reader CTAs launched since the last generation have all
// released (their scheduler/producer list reads are done), so this grid runs
// during the tail of the GEMM still finishing on the old mask. Bounded: past
// 20 ms it falls back to griddepcontrol.wait (always sufficient; the bound only
// matters if the workspace was re-zeroed behind the library's back).
__device__ __forceinline__ void wait_previous_generation(const PlanArgs& a) {
    if (!a.prev_gen) return;
    if (threadIdx.x == 0) {
        const unsigned long long t0 = gclock();
        while (true) {
            unsigned int v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.m.ticket + 2) : "memory");
            if (v == a.prev_gen || gclock() - t0 > 20000000ull) break;
            __nanosleep(32);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void wait_workspace_free(const PlanArgs& a) {
    if (!a.rel_wait) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        wait_previous_generation(a);
        return;
    }
    __shared__ int fallback;
    if (threadIdx.x == 0) {
        const unsigned long long t0 = gclock();
        int fb = 0;
        while (true) {
            unsigned int v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.rel) : "memory");
            if (static_cast<int>(v - a.rel_target) >= 0) break;
            if (gclock() - t0 > 20000000ull) {
                fb = 1;
                break;
            }
            __nanosleep(32);
        }
        fallback = fb;
    }
    __syncthreads();
    if (fallback) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Exit count for a bound workspace in inline-order mode: the last block out
// zeroes the release counter for the next round of readers (they can only
// start releasing after this grid completes).
__device__ __forceinline__ void finish_block(const PlanArgs& a) {
    if (!a.rel) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.m.ticket, 1u) == gridDim.x - 1) {
            *a.rel = 0u;
            *a.m.ticket = 0u;
            __threadfence();
            // counter mode never waited for the preceding grid: the last block
            // out does, so this grid's completion implies its predecessor's
            // under the documented PDL semantics (not only by transitivity)
            if (a.rel_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
            publish_generation(a);
        }
    }
}

__device__ __forceinline__ bool keep_bit(const PlanArgs& a, int r, int c) {
    if (a.from_words) {
        const int64_t b = static_cast<int64_t>(r) * a.m.block_cols + c;
        return (a.m.words[b >> 6] >> (b & 63)) & 1ull;
    }
    const uint64_t h =
        mix64(mix64(a.seed_mix ^ static_cast<uint64_t>(r + a.m.row_block_offset)) ^ static_cast<uint64_t>(c));
    return (h >> 11) >= a.threshold;
}

// Exclusive scan of n ints in smem, DESCENDING index order:
// out[v] = sum_{w > v} in[v]. 256 threads.
__device__ void scan_desc(int* bins, int n, int* warp_tot) {
    const int tid = threadIdx.x;
    const int per = (n + kThreads - 1) / kThreads;
    // thread t owns reversed positions [t*per, t*per+per): index n-1-pos
    int local = 0;
    for (int i = 0; i < per; ++i) {
        const int pos = tid * per + i;
        if (pos < n) local += bins[n - 1 - pos];
    }
    // block exclusive scan of `local`
    const int lane = tid & 31, wid = tid >> 5;
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int w = lane < kThreads / 32 ? warp_tot[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += v;
        }
        if (lane < kThreads / 32) warp_tot[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    int run = incl - local + (wid > 0 ? warp_tot[wid - 1] : 0);
    for (int i = 0; i < per; ++i) {
        const int pos = tid * per + i;
        if (pos < n) {
            const int idx = n - 1 - pos;
            const int v = bins[idx];
            bins[idx] = run;
            run += v;
        }
    }
    __syncthreads();
}

// Counting sort of `count` (values in [0, max_val]) into a descending order.
// `count` is global memory written by other blocks of this grid (read through
// L2), or this block's shared memory.
template <bool SMEM>
__device__ __forceinline__ int read_count(const int32_t* count, int i) {
    if constexpr (SMEM) return count[i];
    else return __ldcg(count + i);
}
template <bool SMEM = false>
__device__ void order_by_count(const int32_t* count, int n, int max_val, int32_t* order, int* bins,
                               int* warp_tot) {
    if (max_val + 1 > kMaxOrderBins) {
        for (int i = threadIdx.x; i < n; i += kThreads) order[i] = i;
        return;
    }
    const int nb = max_val + 1;
    for (int i = threadIdx.x; i < nb; i += kThreads) bins[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kThreads) atomicAdd(&bins[read_count<SMEM>(count, i)], 1);
    __syncthreads();
    scan_desc(bins, nb, warp_tot);
    for (int i = threadIdx.x; i < n; i += kThreads) {
        const int pos = atomicAdd(&bins[read_count<SMEM>(count, i)], 1);
        order[pos] = i;
    }
    __syncthreads();
}

// Descending order of n <= 64 counts (smem) by one warp: rank = #greater +
// #equal at a lower index (stable). No block barrier: the row and column
// orders run in two warps at once (the counting sort above needs ~6 block
// barriers per order, ~1 us each on the critical path of a layer step).
__device__ __forceinline__ void warp_rank_order(const int* cnt, int n, int32_t* order) {
    const int lane = threadIdx.x & 31;
    const int i0 = lane, i1 = lane + 32;
    const int v0 = i0 < n ? cnt[i0] : 0, v1 = i1 < n ? cnt[i1] : 0;
    int r0 = 0, r1 = 0;
    for (int j = 0; j < n; ++j) {
        const int w = cnt[j];
        r0 += (w > v0) | ((w == v0) & (j < i0));
        r1 += (w > v1) | ((w == v1) & (j < i1));
    }
    if (i0 < n) order[r0] = i0;
    if (i1 < n) order[r1] = i1;
}

__global__ void __launch_bounds__(kThreads) mask_plan_kernel(const PlanArgs a) {
    extern __shared__ int dyn_smem[];
    __shared__ int warp_tot[kThreads / 32];
    __shared__ unsigned long long keep_part[kThreads / 32];
    __shared__ bool is_last;
    const int R = a.m.block_rows, C = a.m.block_cols;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    // the order block (the longest) is block 0 so it is dispatched first when
    // SMs free up at the end of the previous GEMM
    int blk = a.inline_order ? (blockIdx.x == 0 ? a.nb_words + a.nb_rows + a.nb_cols : blockIdx.x - 1)
                             : static_cast<int>(blockIdx.x);
#ifdef SD_TRACE
    if (threadIdx.x == 0) atomicMin(&g_sd_timeline[(a.trace_id & 255) * 4 + 0], gtimer_m());
#define SD_PAST_WAIT() \
    if (threadIdx.x == 0) atomicMax(&g_sd_timeline[(a.trace_id & 255) * 4 + 1], gtimer_m());  // last block past wait
#else
#define SD_PAST_WAIT()
#endif
    // Compact mode reads the given words, written by earlier work: wait first.
    // Seed mode reads nothing, so every block computes its part first and waits
    // (for the workspace's previous readers) only before its first global write.
    if (a.trigger_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const bool early = !a.from_words;
    if (!early) {
        wait_workspace_free(a);
        SD_PAST_WAIT()
    }

    if (a.inline_order && blk == a.nb_words + a.nb_rows + a.nb_cols) {
        // ---- counts, keep_count and cost orders, recomputed by this block alone
        // from (seed, r, c) (or the given words) while the other blocks write the
        // words and lists: no grid-wide ticket and serial last block on the
        // critical path (that phase cost 4-8 us per mask, ~3% of a 4096^3 step).
        int* rc = dyn_smem;
        int* cc = rc + R;
        int* ro = cc + C;   // fast path: orders staged here until the wait
        int* co = ro + R;
        int* bins = co + C;
        for (int i = threadIdx.x; i < R + C; i += kThreads) rc[i] = 0;
        __syncthreads();
        // warp w owns rows w, w + 8, ...: row counts accumulate in smem without
        // atomics, column counts in a register per lane (one smem atomic per
        // lane and chunk); four rows per pass keep four hash chains in flight
        constexpr int kW = kThreads / 32;
        for (int c0 = 0; c0 < C; c0 += 32) {
            const int c = c0 + lane;
            int colacc = 0;
            for (int r = wid; r < R; r += 4 * kW) {
                bool k[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int rr = r + u * kW;
                    k[u] = c < C && rr < R && keep_bit(a, rr, c);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int rr = r + u * kW;
                    const int n = __popc(__ballot_sync(0xffffffffu, k[u]));
                    if (lane == 0 && rr < R) rc[rr] += n;
                    colacc += k[u];
                }
            }
            if (c < C && colacc) atomicAdd(&cc[c], colacc);
        }
        __syncthreads();
        if (R <= 64 && C <= 64) {
            if (wid == 0) warp_rank_order(rc, R, ro);
            else if (wid == 1) warp_rank_order(cc, C, co);
            __syncthreads();
            if (early) {
                wait_workspace_free(a);
                SD_PAST_WAIT()
            }
            for (int i = threadIdx.x; i < R; i += kThreads) a.m.row_order[i] = ro[i];
            for (int i = threadIdx.x; i < C; i += kThreads) a.m.col_order[i] = co[i];
            if (wid == 2) {
                int kc = 0;
                for (int r = lane; r < R; r += 32) kc += rc[r];
                for (int o = 16; o > 0; o >>= 1) kc += __shfl_xor_sync(0xffffffffu, kc, o);
                if (lane == 0) *a.m.keep_count = static_cast<int64_t>(kc);
            }
        } else {
            if (early) {
                wait_workspace_free(a);
                SD_PAST_WAIT()
            }
            unsigned long long kc = 0;
            for (int r = threadIdx.x; r < R; r += kThreads) kc += static_cast<unsigned long long>(rc[r]);
            for (int o = 16; o > 0; o >>= 1) kc += __shfl_xor_sync(0xffffffffu, kc, o);
            if (lane == 0) keep_part[wid] = kc;
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long sum = 0;
                for (int i = 0; i < kThreads / 32; ++i) sum += keep_part[i];
                *a.m.keep_count = static_cast<int64_t>(sum);
            }
            order_by_count<true>(rc, R, C, a.m.row_order, bins, warp_tot);
            order_by_count<true>(cc, C, R, a.m.col_order, bins, warp_tot);
        }
        __syncthreads();
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef SD_TRACE
        if (threadIdx.x == 0) atomicMax(&g_sd_timeline[(a.trace_id & 255) * 4 + 3], gtimer_m());  // order block end
#endif
        finish_block(a);
        return;
    }
    if (blk < a.nb_words) {
        // ---- words: one warp per 64-bit word, two bits per lane, ballot-packed
        const int64_t total = static_cast<int64_t>(R) * C;
        const int64_t nwords = (total + 63) / 64;
        const int64_t w = static_cast<int64_t>(blk) * (kThreads / 32) + wid;
        uint64_t word = 0;
        if (w < nwords) {
            const int64_t b0 = w * 64 + lane, b1 = b0 + 32;
            const bool k0 = b0 < total && keep_bit(a, static_cast<int>(b0 / C), static_cast<int>(b0 % C));
            const bool k1 = b1 < total && keep_bit(a, static_cast<int>(b1 / C), static_cast<int>(b1 % C));
            const uint32_t lo = __ballot_sync(0xffffffffu, k0);
            const uint32_t hi = __ballot_sync(0xffffffffu, k1);
            word = (static_cast<uint64_t>(hi) << 32) | lo;
        }
        if (early) {
            wait_workspace_free(a);
            SD_PAST_WAIT()
        }
        if (w < nwords && lane == 0) a.m.words[w] = word;
    } else if ((blk -= a.nb_words) < a.nb_rows) {
        // ---- row lists: one warp per block row. Kept columns ascending from the
        // front (kept_blocks_in_row), dropped columns from the back (the sdd
        // kernel's zero-fill list). Keep bits of up to 32 column chunks are held
        // in a register across the wait.
        const int r = blk * (kThreads / 32) + wid;
        const int nch = (C + 31) / 32;
        const bool held = early && nch <= 32;
        uint32_t kbits = 0;
        if (held && r < R) {
            for (int j = 0; j < nch; ++j) {
                const int c = j * 32 + lane;
                kbits |= static_cast<uint32_t>(c < C && keep_bit(a, r, c)) << j;
            }
        }
        if (early) {
            wait_workspace_free(a);
            SD_PAST_WAIT()
        }
        if (r < R) {
            int base = 0, dbase = 0;
            int32_t* dst = a.m.row_idx + static_cast<int64_t>(r) * C;
            for (int j = 0, c0 = 0; c0 < C; ++j, c0 += 32) {
                const int c = c0 + lane;
                const bool valid = c < C;
                const bool k = valid && (held ? ((kbits >> j) & 1u) : keep_bit(a, r, c));
                const uint32_t bal = __ballot_sync(0xffffffffu, k);
                const uint32_t dbal = __ballot_sync(0xffffffffu, valid && !k);
                if (k) dst[base + __popc(bal & lt)] = c;
                if (valid && !k) dst[C - 1 - (dbase + __popc(dbal & lt))] = c;
                base += __popc(bal);
                dbase += __popc(dbal);
            }
            if (lane == 0) a.m.row_cnt[r] = base;
        }
    } else {
        // ---- column lists: one block per block column; warps take contiguous
        // 32-row chunks, ballots parked in smem, block scan, then scatter.
        const int c = blk - a.nb_rows;
        uint32_t* bal_s = reinterpret_cast<uint32_t*>(dyn_smem);
        const int nchunks = (R + 31) / 32;
        const int per_warp = (nchunks + kThreads / 32 - 1) / (kThreads / 32);
        const int ch0 = wid * per_warp;
        const int ch1 = min(nchunks, ch0 + per_warp);
        int cnt = 0;
        for (int ch = ch0; ch < ch1; ++ch) {
            const int r = ch * 32 + lane;
            const bool k = r < R && keep_bit(a, r, c);
            const uint32_t bal = __ballot_sync(0xffffffffu, k);
            if (lane == 0) bal_s[ch] = bal;
            cnt += __popc(bal);
        }
        if (lane == 0) warp_tot[wid] = cnt;
        __syncthreads();
        if (early) {
            wait_workspace_free(a);
            SD_PAST_WAIT()
        }
        int base = 0;
        for (int i = 0; i < wid; ++i) base += warp_tot[i];
        int32_t* dst = a.m.col_idx + static_cast<int64_t>(c) * R;
        for (int ch = ch0; ch < ch1; ++ch) {
            const uint32_t bal = bal_s[ch];
            if ((bal >> lane) & 1u) dst[base + __popc(bal & lt)] = ch * 32 + lane;
            base += __popc(bal);
        }
        if (threadIdx.x == kThreads - 1) {
            int tot = 0;
            for (int i = 0; i < kThreads / 32; ++i) tot += warp_tot[i];
            a.m.col_cnt[c] = tot;
        }
        __syncthreads();
    }

    // Only now let the consumer GEMM launch: its 1-CTA-per-SM blocks (227 KB of
    // shared memory) would otherwise take the SMs freed by the previous GEMM's
    // tail and wait there for this grid, starving our own blocks (measured: the
    // mask took ~15 us after the previous backward instead of ~6). Its
    // griddepcontrol.wait still orders all of its reads after this grid.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (a.inline_order) {
#ifdef SD_TRACE
        if (threadIdx.x == 0) atomicMax(&g_sd_timeline[(a.trace_id & 255) * 4 + 2], gtimer_m());
#endif
        finish_block(a);
        return;
    }

    // ---- last block: keep_count and cost orders
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(a.m.ticket, 1u);
        is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
#ifdef SD_TRACE
    if (threadIdx.x == 0) g_sd_timeline[(a.trace_id & 255) * 4 + 3] = gtimer_m();  // ordering phase starts
#endif

    unsigned long long kc = 0;
    for (int r = threadIdx.x; r < R; r += kThreads) kc += static_cast<unsigned long long>(__ldcg(a.m.row_cnt + r));
    for (int o = 16; o > 0; o >>= 1) kc += __shfl_xor_sync(0xffffffffu, kc, o);
    if (lane == 0) keep_part[wid] = kc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int i = 0; i < kThreads / 32; ++i) s += keep_part[i];
        *a.m.keep_count = static_cast<int64_t>(s);
    }
    order_by_count(a.m.row_cnt, R, C, a.m.row_order, dyn_smem, warp_tot);
    order_by_count(a.m.col_cnt, C, R, a.m.col_order, dyn_smem, warp_tot);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a.rel) *a.rel = 0u;  // every block has passed its wait: next round of readers
        *a.m.ticket = 0u;        // re-arm for the next launch on this workspace
        __threadfence();
        // counter mode: complete only after the preceding grid (see finish_block)
        if (a.rel_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
        publish_generation(a);
    }
#ifdef SD_TRACE
    if (threadIdx.x == 0) atomicMax(&g_sd_timeline[(a.trace_id & 255) * 4 + 2], gtimer_m());
#endif
}

__device__ __forceinline__ bool in_bit(const uint64_t* w, int64_t b) { return (w[b >> 6] >> (b & 63)) & 1ull; }

// transpose_mask (block_mask.cpp:117-123): out bit (c, r) = in bit (r, c).
__global__ void mask_transpose_kernel(const uint64_t* in, int R, int C, uint64_t* out) {
    const int64_t total = static_cast<int64_t>(R) * C;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w >= (total + 63) / 64) return;
    uint64_t word = 0;
    for (int i = 0; i < 64; ++i) {
        const int64_t b = w * 64 + i;  // bit of the (C x R) output grid
        if (b >= total) break;
        const int64_t c = b / R, r = b % R;
        word |= static_cast<uint64_t>(in_bit(in, r * C + c)) << i;
    }
    out[w] = word;
}

// retile (block_mask.cpp:100-115): out bit (r, c) = in bit (r / sm, c / sk).
__global__ void mask_retile_kernel(const uint64_t* in, int R, int C, int sm, int sk, uint64_t* out) {
    const int R2 = R * sm, C2 = C * sk;
    const int64_t total = static_cast<int64_t>(R2) * C2;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w >= (total + 63) / 64) return;
    uint64_t word = 0;
    for (int i = 0; i < 64; ++i) {
        const int64_t b = w * 64 + i;
        if (b >= total) break;
        const int64_t r = b / C2, c = b % C2;
        word |= static_cast<uint64_t>(in_bit(in, (r / sm) * C + c / sk)) << i;
    }
    out[w] = word;
}

}  // namespace

uint32_t launch_mask_plan(const sd_block_mask& m, bool from_words, uint64_t seed_mix, uint64_t threshold,
                          cudaStream_t s, bool off_path) {
    static std::atomic<uint32_t> g_gen_seq{0x5d000000u};  // process-wide: never repeats per workspace
    PlanArgs a;
    a.trigger_early = 0;
    a.gen_seq = 0;
    a.prev_gen = 0;
    a.trace_id = static_cast<int>(sd_launch_count());
    a.m = m;
    a.from_words = from_words ? 1 : 0;
    a.seed_mix = seed_mix;
    a.threshold = threshold;
    a.rel = mask_release_counter(&m);
    a.rel_target = 0;
    a.rel_wait = 0;
    if (a.rel) {
        uint32_t target = 0;
        const bool ok = mask_take_release(a.rel, s, &target);
        if (ok && !from_words && !off_path && !(tuning() & kTuneNoMaskOverlap)) {
            a.rel_wait = 1;
            a.rel_target = target;
            note_counter_wait();
        }
        if (off_path && !from_words) {
            // every block waits for the preceding grid (normal mode) but lets the
            // next launch start right away; generations into this workspace are
            // chained through ticket word 2
            a.trigger_early = 1;
            uint32_t v = g_gen_seq.fetch_add(1) + 1;
            if (v == 0) v = g_gen_seq.fetch_add(1) + 1;
            a.gen_seq = v;
            a.prev_gen = mask_swap_last_gen(a.rel, v);  // the workspace's previous off-path generation
        }
    }
    const int64_t nwords = (static_cast<int64_t>(m.block_rows) * m.block_cols + 63) / 64;
    a.nb_words = from_words ? 0 : static_cast<int>((nwords + kThreads / 32 - 1) / (kThreads / 32));
    a.nb_rows = (m.block_rows + kThreads / 32 - 1) / (kThreads / 32);
    a.nb_cols = m.block_cols;
    // counts + orders in one extra block when the grid is small enough for one
    // block to re-evaluate every bit cheaply (every BASELINE config up to
    // 512 x 64; cfg5's 4096 x 64 single-GPU shard uses the ticketed last block)
    const int64_t nbits = static_cast<int64_t>(m.block_rows) * m.block_cols;
    a.inline_order = (nbits <= 32768 && m.block_rows <= 4096 && m.block_cols <= 4096) ? 1 : 0;
    const int grid = a.nb_words + a.nb_rows + a.nb_cols + a.inline_order;
    const int bins = std::min(std::max(m.block_rows, m.block_cols) + 1, kMaxOrderBins);
    const int chunks = (m.block_rows + 31) / 32;
    const int inline_ints = a.inline_order ? 2 * (m.block_rows + m.block_cols) + bins : 0;
    const size_t smem = static_cast<size_t>(std::max({bins, chunks, inline_ints})) * sizeof(int);
    if (smem > 48 * 1024) {
        configure_once_per_device(2, [] {
            check_cuda(cudaFuncSetAttribute(mask_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
                       "mask_plan_kernel smem");
        });
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    check_cuda(cudaLaunchKernelEx(&cfg, mask_plan_kernel, a), "mask_plan_kernel launch");
    note_launch();
    return a.gen_seq;
}

// CUDA-graph replays of a plan step (sd_capi.cu): the generation kernel's
// function and its parameter block, whose seed is patched per replay.
const void* mask_plan_kernel_func() { return reinterpret_cast<const void*>(&mask_plan_kernel); }
size_t mask_plan_args_size() { return sizeof(PlanArgs); }
void mask_plan_patch_seed(void* args, uint64_t seed_mix) { static_cast<PlanArgs*>(args)->seed_mix = seed_mix; }

void launch_mask_transpose(const sd_block_mask& in, sd_block_mask& out, cudaStream_t s) {
    const int64_t nwords = (static_cast<int64_t>(in.block_rows) * in.block_cols + 63) / 64;
    const int grid = static_cast<int>((nwords + kThreads - 1) / kThreads);
    mask_transpose_kernel<<<grid, kThreads, 0, s>>>(in.words, in.block_rows, in.block_cols, out.words);
    check_cuda(cudaGetLastError(), "mask_transpose_kernel launch");
    note_launch();
    launch_mask_plan(out, true, 0, 0, s);
}

void launch_mask_retile(const sd_block_mask& in, int split_m, int split_k, sd_block_mask& out,
                        cudaStream_t s) {
    const int64_t nwords =
        (static_cast<int64_t>(out.block_rows) * out.block_cols + 63) / 64;
    const int grid = static_cast<int>((nwords + kThreads - 1) / kThreads);
    mask_retile_kernel<<<grid, kThreads, 0, s>>>(in.words, in.block_rows, in.block_cols, split_m,
                                                 split_k, out.words);
    check_cuda(cudaGetLastError(), "mask_retile_kernel launch");
    note_launch();
    launch_mask_plan(out, true, 0, 0, s);
}

}  // namespace sd

#ifdef SD_TRACE
extern "C" SD_API int sd_mask_timeline_read(unsigned long long* host) {
    if (cudaDeviceSynchronize() != cudaSuccess) return SD_ERUNTIME;
    if (cudaMemcpyFromSymbol(host, sd::g_sd_timeline, sizeof(unsigned long long) * 256 * 4) != cudaSuccess)
        return SD_ERUNTIME;
    static unsigned long long init[256 * 4];
    // {first block start (min), last block past griddepcontrol.wait (max), end (max), ordering start}
    for (int i = 0; i < 256; ++i) init[4 * i] = ~0ull, init[4 * i + 1] = init[4 * i + 2] = init[4 * i + 3] = 0;
    cudaMemcpyToSymbol(sd::g_sd_timeline, init, sizeof init);
    return SD_OK;
}
#endif
