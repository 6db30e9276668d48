// sd_capi.cu — the extern "C" boundary (include/sparsedrop_b200.h).
//
// Validation mirrors the reference's exceptions and messages:
//   sample_mask            block_mask.cpp:53-61
//   check_gemm_shapes      gemm.hpp:62-70 (check_divides :55-60)
//   check_mask_geometry    gemm.hpp:72-82
// plus the B200 kernels' own geometry limits (128-row output tiles, 64-element
// reduction stages, 128/256-wide mask blocks along the skipped dimension).
// Errors never cross the boundary as exceptions: sd::Error -> status code +
// thread-local message (sd_last_error).
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "sd_internal.h"

namespace sd {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return SD_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SD_ERUNTIME;
    }
}

std::string str(long long v) { return std::to_string(v); }

void require_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        fail(SD_ERUNTIME, "no CUDA device available (the B200 path has no CPU fallback)");
    }
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major != 10) fail(SD_ERUNTIME, "device is not sm_100 (B200); this library targets sm_100a only");
}

// gemm.hpp:55-60
void check_divides(int block, int extent, const char* which) {
    if (block <= 0 || extent % block != 0)
        fail(SD_EINVAL, std::string("tile size ") + which + "=" + str(block) +
                            " does not divide dimension " + str(extent));
}

// gemm.hpp:62-70 for c = a(m x k) * b(k x n), with the B200 tile limits.
void check_gemm(int m, int n, int k) {
    if (m <= 0 || n <= 0 || k <= 0)
        fail(SD_EINVAL, "gemm shape mismatch: dimensions must be positive, got m=" + str(m) +
                            " n=" + str(n) + " k=" + str(k));
    check_divides(128, m, "m_blk");
    check_divides(128, n, "n_blk");
    check_divides(64, k, "k_blk");
}

// gemm.hpp:72-82
void check_mask_geometry(const sd_block_mask* mask, int grid_rows, int grid_cols, int blk_rows,
                         int blk_cols, const char* where) {
    if (!mask) fail(SD_EINVAL, std::string(where) + ": null mask");
    if (mask->block_rows != grid_rows || mask->block_cols != grid_cols || mask->m_blk != blk_rows ||
        mask->k_blk != blk_cols)
        fail(SD_EINVAL, std::string(where) + ": mask geometry (" + str(mask->block_rows) + "x" +
                            str(mask->block_cols) + " blocks of " + str(mask->m_blk) + "x" +
                            str(mask->k_blk) + ") does not match problem (" + str(grid_rows) + "x" +
                            str(grid_cols) + " blocks of " + str(blk_rows) + "x" + str(blk_cols) +
                            ")");
}

void check_ptr(const void* p, const char* name) {
    if (!p) fail(SD_EINVAL, std::string("null pointer: ") + name);
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
        fail(SD_EINVAL, std::string(name) + " must be 16-byte aligned");
}

void check_dtype(int dt) {
    if (dt != SD_DTYPE_F32 && dt != SD_DTYPE_BF16) fail(SD_EINVAL, "unknown output dtype " + str(dt));
}

// Mask-block limits of the tcgen05 kernels: the mask block along the OUTPUT
// rows must cover whole 128-row tiles; along the reduction it must cover whole
// 64-element stages; along sdd output columns it must be 128 or 256.
void check_row_blk(int blk, const char* which) {
    if (blk <= 0 || blk % 128 != 0)
        fail(SD_EINVAL, std::string("mask block size ") + which + "=" + str(blk) +
                            " unsupported on B200: must be a multiple of 128");
}
void check_red_blk(int blk, const char* which) {
    if (blk <= 0 || blk % 64 != 0)
        fail(SD_EINVAL, std::string("mask block size ") + which + "=" + str(blk) +
                            " unsupported on B200: must be a multiple of 64");
}
void check_col_blk(int blk, const char* which) {
    if (blk != 128 && blk != 256)
        fail(SD_EINVAL, std::string("mask block size ") + which + "=" + str(blk) +
                            " unsupported on B200: must be 128 or 256");
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
uint64_t threshold_of(double p);
uint64_t mix64_host(uint64_t z);

GemmArgs base_args(int rows_out, int cols_out, int red, float scale, void* out) {
    GemmArgs a;
    std::memset(&a, 0, sizeof a);
    a.rows_out = rows_out;
    a.cols_out = cols_out;
    a.red = red;
    a.n_row_tiles = rows_out / kBM;
    a.n_col_units = (cols_out + kBN - 1) / kBN;
    a.red_blk = kBK;
    a.out_row_blk = kBM;
    a.out_col_blk = 128;
    a.scale = scale;
    a.out = out;
    a.keep_hint = -1.0f;
    return a;
}

// Output tensor map: store box = 32 rows x 128 bytes.
CUtensorMap out_map(void* c, int dt, int rows, int cols) {
    const bool f32 = dt == SD_DTYPE_F32;
    return make_tmap_2d(c, f32, cols, rows, f32 ? 32 : 64, 32);
}

// bf16 operand maps, 16 KB boxes. K-major (reduction contiguous): box 64 x
// 128 rows. MN-major (output dimension contiguous): a 3D box of two 64-wide
// atoms x 64 reduction rows. Per-SM TMA throughput is bound by boxes, not
// bytes (tools/l2_bench.cu: five boxes per 48 KB stage cap an SM at ~117 GB/s,
// two reach ~240 GB/s), so an operand tile is loaded in as few boxes as the
// 128B swizzle allows.
CUtensorMap kmajor_map(const void* p, int red, int rows) { return make_tmap_2d(p, false, red, rows, 64, 128); }
CUtensorMap mnmajor_map(const void* p, int mn, int red) { return make_tmap_mn_atoms(p, mn, red, mn); }

}  // namespace

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }
void set_last_error(const std::string& msg) { g_last_error = msg; }

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(SD_ERUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}

int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
    int n = 0;
    check_cuda(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "SM count");
    if (dev >= 0 && dev < 64) cached[dev] = n;
    return n;
}

void configure_once_per_device(int key, const std::function<void()>& fn) {
    static std::mutex mu;
    static bool done[8][64] = {};
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (key < 0 || key >= 8 || dev < 0 || dev >= 64) fail(SD_ERUNTIME, "configure_once_per_device: bad key/device");
    std::lock_guard<std::mutex> lock(mu);
    if (done[key][dev]) return;
    fn();
    done[key][dev] = true;
}

void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Scheduler-counter slots (sd_internal.h). Eager launches take slots
// round-robin from a ring owned by their STREAM: launches of one stream overlap
// at most a few deep (PDL), so a 64-slot ring is never reused while a launch
// that used a slot still runs, and launches of another stream — however many,
// however long this one runs — never share its slots. A launch captured into a
// graph gets a dedicated slot that is never handed out again (it is replayed
// later, possibly beside eager launches).
unsigned int* sched_slot(cudaStream_t s) {
    constexpr int kRing = 64;        // eager launches per stream, round-robin
    constexpr int kCaptured = 4096;  // launches captured into graphs, never reused (~10 KB each)
    constexpr size_t kSlotBytes = static_cast<size_t>(kSlotWords) * sizeof(unsigned int);
    struct Ring {
        unsigned int* base = nullptr;
        uint32_t next = 0;
    };
    struct DevSlots {
        unsigned int* captured = nullptr;
        uint32_t next_captured = 0;
        std::unordered_map<cudaStream_t, Ring> rings;
    };
    static std::mutex mu;
    static DevSlots devs[64];
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= 64) fail(SD_ERUNTIME, "device index out of range");
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (s != nullptr && cudaStreamIsCapturing(s, &cap) != cudaSuccess) {
        cudaGetLastError();
        cap = cudaStreamCaptureStatusNone;
    }
    std::lock_guard<std::mutex> lock(mu);
    DevSlots& d = devs[dev];
    if (!d.captured) {
        // first use on this device (sd_layer_plan_create calls this outside any
        // capture): the captured-launch slots, zeroed once
        unsigned int* p = nullptr;
        check_cuda(cudaMalloc(&p, kCaptured * kSlotBytes), "cudaMalloc(scheduler slots)");
        check_cuda(cudaMemset(p, 0, kCaptured * kSlotBytes), "cudaMemset(scheduler slots)");
        check_cuda(cudaDeviceSynchronize(), "scheduler slots init");
        d.captured = p;
    }
    if (cap == cudaStreamCaptureStatusActive) {
        const uint32_t i = d.next_captured++;
        if (i >= static_cast<uint32_t>(kCaptured))
            fail(SD_ERUNTIME, "too many captured GEMM launches (" + std::to_string(kCaptured) + " per device)");
        return d.captured + static_cast<size_t>(i) * kSlotWords;
    }
    // past kMaxRings distinct streams (640 KB each) the remaining streams share
    // one overflow ring (the pre-round-2 behaviour: safe unless a launch on one
    // of them outlives 64 launches on the others)
    constexpr size_t kMaxRings = 256;
    const cudaStream_t key =
        (d.rings.count(s) || d.rings.size() < kMaxRings) ? s : reinterpret_cast<cudaStream_t>(~uintptr_t{0});
    Ring& r = d.rings[key];
    if (!r.base) {
        // a stream's first eager launch: its ring, zeroed in stream order (the
        // launch that follows on the same stream sees the zeros; the overflow
        // ring is zeroed synchronously, it serves several streams)
        unsigned int* p = nullptr;
        check_cuda(cudaMalloc(&p, kRing * kSlotBytes), "cudaMalloc(stream scheduler slots)");
        if (key == s) {
            check_cuda(cudaMemsetAsync(p, 0, kRing * kSlotBytes, s), "cudaMemsetAsync(stream scheduler slots)");
        } else {
            check_cuda(cudaMemset(p, 0, kRing * kSlotBytes), "cudaMemset(overflow scheduler slots)");
            check_cuda(cudaDeviceSynchronize(), "overflow scheduler slots init");
        }
        r.base = p;
    }
    return r.base + static_cast<size_t>(r.next++ % kRing) * kSlotWords;
}

// ---------------------------------------------------------------- reader tracking
// One entry per workspace bound by sd_mask_bind: its byte range, its release
// counter (the second word of the 256-byte ticket slot) and the reader CTAs
// launched since the last generation into it. The counter protocol is only
// used when every such reader ran on the generation's own stream (so each of
// them is either complete or resident when the generation starts: no reader
// can wait for SMs held by the generation's spinning blocks) and outside
// stream capture; any doubt -> the generation falls back to
// griddepcontrol.wait, which covers every earlier grid of the stream.
namespace {
struct ReaderEntry {
    uintptr_t base, end;
    unsigned int* rel;
    uint32_t pending;
    cudaStream_t stream;
    bool mixed;
    uint32_t last_gen;  // the last off-path generation number published into the workspace (0: none)
};
std::mutex g_reader_mu;
std::vector<ReaderEntry> g_readers;

ReaderEntry* find_reader_entry(uintptr_t p) {
    for (auto& e : g_readers)
        if (p >= e.base && p < e.end) return &e;
    return nullptr;
}
}  // namespace

void mask_register_workspace(void* ws, size_t bytes, unsigned int* rel) {
    std::lock_guard<std::mutex> lock(g_reader_mu);
    const uintptr_t b = reinterpret_cast<uintptr_t>(ws), e = b + bytes;
    for (size_t i = 0; i < g_readers.size();) {
        if (g_readers[i].base < e && b < g_readers[i].end) {
            g_readers[i] = g_readers.back();
            g_readers.pop_back();
        } else {
            ++i;
        }
    }
    if (g_readers.size() >= 4096) g_readers.erase(g_readers.begin());  // untracked from now on: safe
    g_readers.push_back({b, e, rel, 0u, nullptr, false, 0u});
}

// Exact match on the counter address: only a struct filled by sd_mask_bind
// (whose ticket slot is 256 bytes) gets a counter; the library never writes
// the counter of a range it merely overlaps.
unsigned int* mask_release_counter(const sd_block_mask* m) {
    if (!m || !m->ticket) return nullptr;
    unsigned int* rel = m->ticket + 1;
    std::lock_guard<std::mutex> lock(g_reader_mu);
    for (const auto& e : g_readers)
        if (e.rel == rel) return rel;
    return nullptr;
}

void mask_note_readers(unsigned int* rel, int ctas, cudaStream_t s) {
    std::lock_guard<std::mutex> lock(g_reader_mu);
    for (auto& e : g_readers) {
        if (e.rel != rel) continue;
        if (e.pending > 0 && e.stream != s) e.mixed = true;
        e.stream = s;
        e.pending += static_cast<uint32_t>(ctas);
        return;
    }
}

void mask_note_untracked(const void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lock(g_reader_mu);
    if (ReaderEntry* e = find_reader_entry(reinterpret_cast<uintptr_t>(p))) e->mixed = true;
}

uint32_t mask_swap_last_gen(unsigned int* rel, uint32_t gen) {
    std::lock_guard<std::mutex> lock(g_reader_mu);
    for (auto& e : g_readers) {
        if (e.rel != rel) continue;
        const uint32_t prev = e.last_gen;
        e.last_gen = gen;
        return prev;
    }
    return 0;
}

std::atomic<uint64_t> g_counter_waits{0};
void note_counter_wait() { g_counter_waits.fetch_add(1, std::memory_order_relaxed); }

bool mask_take_release(unsigned int* rel, cudaStream_t s, uint32_t* target) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) {
        cudaGetLastError();
        cap = cudaStreamCaptureStatusActive;
    }
    std::lock_guard<std::mutex> lock(g_reader_mu);
    for (auto& e : g_readers) {
        if (e.rel != rel) continue;
        const bool ok = !e.mixed && e.pending > 0 && e.stream == s && cap == cudaStreamCaptureStatusNone;
        *target = e.pending;
        e.pending = 0;
        e.mixed = false;
        e.stream = s;
        return ok;
    }
    return false;
}

static CUtensorMap encode_tmap(const void* base, bool f32, cuuint32_t rank, const cuuint64_t* dims,
                               const cuuint64_t* strides, const cuuint32_t* box,
                               CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    std::call_once(g_encode_once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<EncodeTiledFn>(fn);
        else
            cudaGetLastError();
    });
    if (!g_encode) {
        require_device();  // no device: report the missing B200 (there is no CPU fallback)
        fail(SD_ERUNTIME, "cuTensorMapEncodeTiled unavailable (driver too old?)");
    }
    CUtensorMap map;
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = g_encode(&map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
                                const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::string shape;
        for (cuuint32_t i = 0; i < rank; ++i) shape += (i ? "x" : "") + std::to_string(dims[rank - 1 - i]);
        fail(SD_ERUNTIME, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ") for a " +
                              shape + " tensor");
    }
    return map;
}

CUtensorMap make_tmap_2d(const void* base, bool f32, uint64_t inner, uint64_t outer, uint32_t box_inner,
                         uint32_t box_outer) {
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner * (f32 ? 4 : 2)};
    const cuuint32_t box[2] = {box_inner, box_outer};
    return encode_tmap(base, f32, 2, dims, strides, box);
}

CUtensorMap make_tmap_2d_noswizzle(const void* base, bool f32, uint64_t inner, uint64_t outer, uint32_t box_inner,
                                   uint32_t box_outer) {
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner * (f32 ? 4 : 2)};
    const cuuint32_t box[2] = {box_inner, box_outer};
    return encode_tmap(base, f32, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

CUtensorMap make_tmap_mn_atoms(const void* base, uint64_t mn, uint64_t red, uint64_t ld, uint32_t atoms) {
    // view [red][mn] (mn contiguous, row pitch ld >= mn elements) as
    // (64 mn_in, red, mn / 64 atoms): one box = `atoms` (2, or 1 for a half
    // tile) 64-wide SW128 atoms of 64 reduction rows, atom-major in smem
    const cuuint64_t dims[3] = {64, red, mn / 64};
    const cuuint64_t strides[2] = {(ld ? ld : mn) * 2, 128};
    const cuuint32_t box[3] = {64, 64, atoms};
    return encode_tmap(base, false, 3, dims, strides, box);
}

}  // namespace sd

using namespace sd;

extern "C" {

int sd_abi_version(void) { return SD_ABI_VERSION; }

const char* sd_last_error(void) { return g_last_error.c_str(); }

uint64_t sd_launch_count(void) { return g_launches.load(); }

int sd_set_tuning(int32_t flags) {
    set_tuning(flags);
    return SD_OK;
}

int sd_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int ok = 0;
    for (int d = 0; d < n; ++d) {
        int major = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) == cudaSuccess && major == 10)
            ++ok;
    }
    return ok;
}

int sd_device_alloc(void** ptr, size_t bytes) {
    return guarded([&] {
        if (!ptr) fail(SD_EINVAL, "sd_device_alloc: null out pointer");
        require_device();
        check_cuda(cudaMalloc(ptr, bytes), "cudaMalloc");
    });
}

int sd_device_free(void* ptr) {
    return guarded([&] {
        if (ptr) check_cuda(cudaFree(ptr), "cudaFree");
    });
}

int sd_memcpy(void* dst, const void* src, size_t bytes, int32_t kind, void* stream) {
    return guarded([&] {
        const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                 : kind == 1 ? cudaMemcpyDeviceToHost
                                 : kind == 2 ? cudaMemcpyDeviceToDevice
                                             : cudaMemcpyDefault;
        if (kind < 0 || kind > 2) fail(SD_EINVAL, "sd_memcpy: kind must be 0, 1 or 2");
        check_cuda(cudaMemcpyAsync(dst, src, bytes, k, as_stream(stream)), "cudaMemcpyAsync");
        if (kind == 1 && !stream) check_cuda(cudaStreamSynchronize(nullptr), "cudaStreamSynchronize");
    });
}

int sd_memset(void* dst, int32_t value, size_t bytes, void* stream) {
    return guarded([&] { check_cuda(cudaMemsetAsync(dst, value, bytes, as_stream(stream)), "cudaMemsetAsync"); });
}

int sd_stream_synchronize(void* stream) {
    return guarded([&] { check_cuda(cudaStreamSynchronize(as_stream(stream)), "cudaStreamSynchronize"); });
}

// Layout of the mask workspace (each array 256-byte aligned):
// words | keep_count | ticket | row_cnt | row_idx | col_cnt | col_idx | row_order | col_order
static size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

size_t sd_mask_workspace_bytes(int32_t R, int32_t C) {
    if (R <= 0 || C <= 0) return 0;
    const size_t rc = static_cast<size_t>(R) * C;
    const size_t nwords = (rc + 63) / 64;
    return align256(nwords * 8) + align256(8) + align256(4) + align256(4 * R) + align256(4 * rc) +
           align256(4 * C) + align256(4 * rc) + align256(4 * R) + align256(4 * C);
}

int sd_mask_bind(sd_block_mask* m, void* ws, int32_t R, int32_t C, int32_t m_blk, int32_t k_blk,
                 int32_t row_block_offset) {
    return guarded([&] {
        if (!m || !ws) fail(SD_EINVAL, "sd_mask_bind: null mask or workspace");
        if (R <= 0 || C <= 0 || m_blk <= 0 || k_blk <= 0)
            fail(SD_EINVAL, "BlockMask geometry must be positive: grid " + str(R) + "x" + str(C) +
                                ", blocks " + str(m_blk) + "x" + str(k_blk));
        if (row_block_offset < 0) fail(SD_EINVAL, "row_block_offset must be non-negative");
        if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) fail(SD_EINVAL, "mask workspace must be 256-byte aligned");
        const size_t rc = static_cast<size_t>(R) * C;
        char* p = static_cast<char*>(ws);
        m->block_rows = R;
        m->block_cols = C;
        m->m_blk = m_blk;
        m->k_blk = k_blk;
        m->row_block_offset = row_block_offset;
        m->reserved = 0;
        m->words = reinterpret_cast<uint64_t*>(p);
        p += align256((rc + 63) / 64 * 8);
        m->keep_count = reinterpret_cast<int64_t*>(p);
        p += align256(8);
        m->ticket = reinterpret_cast<uint32_t*>(p);
        p += align256(4);
        m->row_cnt = reinterpret_cast<int32_t*>(p);
        p += align256(4 * static_cast<size_t>(R));
        m->row_idx = reinterpret_cast<int32_t*>(p);
        p += align256(4 * rc);
        m->col_cnt = reinterpret_cast<int32_t*>(p);
        p += align256(4 * static_cast<size_t>(C));
        m->col_idx = reinterpret_cast<int32_t*>(p);
        p += align256(4 * rc);
        m->row_order = reinterpret_cast<int32_t*>(p);
        p += align256(4 * static_cast<size_t>(R));
        m->col_order = reinterpret_cast<int32_t*>(p);
        // the ticket slot is 256 bytes: word 1 is the reader release counter
        mask_register_workspace(ws, sd_mask_workspace_bytes(R, C), m->ticket + 1);
    });
}

// block_mask.cpp:52-80
int sd_mask_sample(sd_block_mask* m, uint64_t seed, double p, int32_t rows, int32_t cols, void* stream) {
    return guarded([&] {
        if (!m) fail(SD_EINVAL, "sd_mask_sample: null mask");
        if (!(p >= 0.0 && p < 1.0)) {
            char buf[64];
            std::snprintf(buf, sizeof buf, "%f", p);
            fail(SD_EINVAL, std::string("dropout rate must lie in [0, 1), got ") + buf);
        }
        if (m->m_blk <= 0 || rows % m->m_blk != 0)
            fail(SD_EINVAL, "mask block size m_blk=" + str(m->m_blk) + " does not divide rows=" + str(rows));
        if (m->k_blk <= 0 || cols % m->k_blk != 0)
            fail(SD_EINVAL, "mask block size k_blk=" + str(m->k_blk) + " does not divide cols=" + str(cols));
        if (rows / m->m_blk != m->block_rows || cols / m->k_blk != m->block_cols)
            fail(SD_EINVAL, "sd_mask_sample: mask geometry (" + str(m->block_rows) + "x" + str(m->block_cols) +
                                " blocks) does not match rows=" + str(rows) + " cols=" + str(cols));
        require_device();
        // keep iff (h >> 11) * 2^-53 >= p  <=>  (h >> 11) >= ceil(p * 2^53)  (exact: p*2^53 is exact)
        launch_mask_plan(*m, false, mix64_host(seed), threshold_of(p), as_stream(stream));
    });
}

int sd_mask_compact(sd_block_mask* m, void* stream) {
    return guarded([&] {
        if (!m || !m->words) fail(SD_EINVAL, "sd_mask_compact: unbound mask");
        require_device();
        launch_mask_plan(*m, true, 0, 0, as_stream(stream));
    });
}

int sd_mask_transpose(const sd_block_mask* in, sd_block_mask* out, void* stream) {
    return guarded([&] {
        if (!in || !out) fail(SD_EINVAL, "sd_mask_transpose: null mask");
        if (out->block_rows != in->block_cols || out->block_cols != in->block_rows ||
            out->m_blk != in->k_blk || out->k_blk != in->m_blk)
            fail(SD_EINVAL, "sd_mask_transpose: output mask must have the swapped geometry");
        require_device();
        launch_mask_transpose(*in, *out, as_stream(stream));
    });
}

int sd_mask_retile(const sd_block_mask* in, int32_t split_m, int32_t split_k, sd_block_mask* out,
                   void* stream) {
    return guarded([&] {
        if (!in || !out) fail(SD_EINVAL, "sd_mask_retile: null mask");
        if (split_m <= 0 || in->m_blk % split_m != 0)
            fail(SD_EINVAL, "split_m=" + str(split_m) + " does not divide m_blk=" + str(in->m_blk));
        if (split_k <= 0 || in->k_blk % split_k != 0)
            fail(SD_EINVAL, "split_k=" + str(split_k) + " does not divide k_blk=" + str(in->k_blk));
        if (out->block_rows != in->block_rows * split_m || out->block_cols != in->block_cols * split_k ||
            out->m_blk != in->m_blk / split_m || out->k_blk != in->k_blk / split_k)
            fail(SD_EINVAL, "sd_mask_retile: output mask geometry does not match the split");
        require_device();
        launch_mask_retile(*in, split_m, split_k, *out, as_stream(stream));
    });
}

// ---------------------------------------------------------------- GEMMs
}  // extern "C"

namespace sd {
namespace {

uint32_t flags_of(bool a_mn, bool b_mn, bool sdd, int out_dtype) {
    return (a_mn ? kFlagAMN : 0u) | (b_mn ? kFlagBMN : 0u) | (sdd ? kFlagSDD : 0u) |
           (out_dtype == SD_DTYPE_F32 ? kFlagF32 : 0u);
}

// dense c[m,n] = A * B with A (K-major | MN-major) and B (K-major | MN-major)
GemmCall prep_dense(const void* a, bool a_mn, const void* b, bool b_mn, void* c, int c_dtype, int m, int n,
                    int k) {
    check_gemm(m, n, k);
    check_ptr(a, "a"), check_ptr(b, "b"), check_ptr(c, "c"), check_dtype(c_dtype);
    GemmCall g;
    g.ta = a_mn ? mnmajor_map(a, m, k) : kmajor_map(a, k, m);
    g.tb = b_mn ? mnmajor_map(b, n, k) : kmajor_map(b, k, n);
    g.tout = out_map(c, c_dtype, m, n);
    g.args = base_args(m, n, k, 1.0f, c);
    g.args.flags = flags_of(a_mn, b_mn, false, c_dtype);
    return g;
}

// gemm.hpp:133-170 / layer.hpp:115: c = s (a (.) m) b, skipping dropped K-blocks.
GemmCall prep_dsd_forward(const void* a, const sd_block_mask* mask, const void* b, float scale, void* c,
                          int c_dtype, int m, int n, int k, unsigned long long* counters, const char* where) {
    check_gemm(m, n, k);
    check_ptr(a, "a"), check_ptr(b, "b"), check_ptr(c, "c"), check_dtype(c_dtype);
    if (!mask) fail(SD_EINVAL, std::string(where) + ": null mask");
    check_divides(mask->m_blk, m, "m_blk");
    check_divides(mask->k_blk, k, "k_blk");
    check_mask_geometry(mask, m / mask->m_blk, k / mask->k_blk, mask->m_blk, mask->k_blk, where);
    check_row_blk(mask->m_blk, "m_blk");
    check_red_blk(mask->k_blk, "k_blk");
    GemmCall g;
    g.ta = kmajor_map(a, k, m);
    g.tb = mnmajor_map(b, n, k);
    g.tout = out_map(c, c_dtype, m, n);
    g.args = base_args(m, n, k, scale, c);
    g.args.flags = flags_of(false, true, false, c_dtype);
    g.args.list_cnt = mask->row_cnt;
    g.args.list_idx = mask->row_idx;
    g.release = mask_release_counter(mask);
    g.args.list_stride = mask->block_cols;
    g.args.red_blk = mask->k_blk;
    g.args.out_row_blk = mask->m_blk;
    g.args.row_order = mask->m_blk == kBM ? mask->row_order : nullptr;
    g.args.counters = counters;
    return g;
}

// gemm.hpp:176-213: c[m,n] = s (a[m,k] b[k,n]) on kept output blocks. b_kmajor: b is
// supplied as b^T (n x k row-major), e.g. the layer's W for dX (layer.hpp:158).
GemmCall prep_sdd(const void* a, const void* b, bool b_kmajor, const sd_block_mask* mask, float scale,
                  void* c, int c_dtype, int m, int n, int k, unsigned long long* counters, const char* where) {
    check_gemm(m, n, k);
    check_ptr(a, "a"), check_ptr(b, "b"), check_ptr(c, "c"), check_dtype(c_dtype);
    if (!mask) fail(SD_EINVAL, std::string(where) + ": null mask");
    check_divides(mask->m_blk, m, "m_blk");
    check_divides(mask->k_blk, n, "n_blk");
    check_mask_geometry(mask, m / mask->m_blk, n / mask->k_blk, mask->m_blk, mask->k_blk, where);
    check_row_blk(mask->m_blk, "m_blk");
    check_col_blk(mask->k_blk, "n_blk");
    GemmCall g;
    g.ta = kmajor_map(a, k, m);
    g.tb = b_kmajor ? kmajor_map(b, k, n) : mnmajor_map(b, n, k);
    g.tout = out_map(c, c_dtype, m, n);
    g.args = base_args(m, n, k, scale, c);
    g.args.flags = flags_of(false, !b_kmajor, true, c_dtype);
    g.args.words = mask->words;
    g.args.list_cnt = mask->row_cnt;
    g.args.list_idx = mask->row_idx;
    g.release = mask_release_counter(mask);
    g.args.list_stride = mask->block_cols;
    g.args.mask_cols = mask->block_cols;
    g.args.out_col_blk = mask->k_blk;
    g.args.out_row_blk = mask->m_blk;
    g.args.row_order = mask->m_blk == kBM ? mask->row_order : nullptr;
    g.args.counters = counters;
    return g;
}

// layer.hpp:158: dx (m x k) = s (dy (m x n) W^T) (.) m — the sdd problem (M, K_out=k, N_red=n).
GemmCall prep_layer_dx(const void* dy, const void* w, const sd_block_mask* mask, float scale, void* dx,
                       int dx_dtype, int m, int n, int k) {
    return prep_sdd(dy, w, true, mask, scale, dx, dx_dtype, m, k, n, nullptr, "layer backward dx");
}

// Rows [kb0, kb1) (mask-column blocks) of the layer's dW problem: the same
// tiles, lists and reduction order as the full call, so each part is
// bit-identical to those rows of the full dW (no cost order across parts).
GemmCall prep_layer_dw_part(const GemmCall& full, const void* x, const sd_block_mask* mask, int m, int k, int n,
                            int kb0, int kb1) {
    const int kblk = mask->k_blk;
    const int r0 = kb0 * kblk, rows = (kb1 - kb0) * kblk;
    GemmCall g = full;
    g.ta = make_tmap_mn_atoms(static_cast<const uint16_t*>(x) + r0, rows, m, k);
    const bool f32 = full.args.flags & kFlagF32;
    void* out = static_cast<char*>(full.args.out) + static_cast<size_t>(r0) * n * (f32 ? 4 : 2);
    g.tout = out_map(out, f32 ? SD_DTYPE_F32 : SD_DTYPE_BF16, rows, n);
    g.args.out = out;
    g.args.rows_out = rows;
    g.args.n_row_tiles = rows / kBM;
    g.args.list_cnt = full.args.list_cnt + kb0;
    g.args.list_idx = full.args.list_idx + static_cast<int64_t>(kb0) * full.args.list_stride;
    g.args.row_order = nullptr;
    g.args.split_rows = full.args.rows_out;  // the full dW's split-K factor (same summation order)
    g.args.hash_list_off = kb0;              // hash mode: the slab's first mask column
    return g;
}

// layer.hpp:159-160: dw (k x n) = s (x (.) m)^T dy over the mask's column lists —
// the dsd problem (K_out = k rows, N, M_red = m) with x read MN-major in place.
GemmCall prep_layer_dw(const void* x, const sd_block_mask* mask, const void* dy, float scale, void* dw,
                       int dw_dtype, int m, int n, int k) {
    check_gemm(k, n, m);
    check_ptr(x, "x"), check_ptr(dy, "dy"), check_ptr(dw, "dw"), check_dtype(dw_dtype);
    if (!mask) fail(SD_EINVAL, "layer backward dw: null mask");
    check_divides(mask->m_blk, m, "m_blk");
    check_divides(mask->k_blk, k, "k_blk");
    check_mask_geometry(mask, m / mask->m_blk, k / mask->k_blk, mask->m_blk, mask->k_blk, "layer backward dw");
    check_row_blk(mask->k_blk, "k_blk");
    check_red_blk(mask->m_blk, "m_blk");
    GemmCall g;
    g.ta = mnmajor_map(x, k, m);
    g.tb = mnmajor_map(dy, n, m);
    g.tout = out_map(dw, dw_dtype, k, n);
    g.args = base_args(k, n, m, scale, dw);
    g.args.flags = flags_of(true, true, false, dw_dtype);
    g.args.list_cnt = mask->col_cnt;
    g.args.list_idx = mask->col_idx;
    g.release = mask_release_counter(mask);
    g.args.list_stride = mask->block_rows;
    g.args.red_blk = mask->m_blk;
    g.args.out_row_blk = mask->k_blk;
    g.args.row_order = mask->k_blk == kBM ? mask->col_order : nullptr;
    return g;
}

uint64_t threshold_of(double p) { return static_cast<uint64_t>(std::ceil(std::ldexp(p, 53))); }

uint64_t mix64_host(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

float dropout_scale_f32(double p) { return static_cast<float>(1.0 / (1.0 - p)); }

}  // namespace
}  // namespace sd

struct sd_layer_plan {
    sd_block_mask mask;
    double p;
    uint64_t threshold;
    int device;
    sd::GemmCall fwd, dw, dx, dense_fwd, dense_dw, dense_dx;
    // dW split by mask-column blocks (data-parallel overlap of the all-reduce)
    std::vector<sd::GemmCall> dw_part;
    int dw_parts = 0;
    const void* x = nullptr;
    const void* dy = nullptr;
    const void* w = nullptr;
    // small plans (the whole step fits on the SMs at once, mask grid <= 64 x 64):
    // the GEMMs evaluate their kept lists from the counter hash (hash mode,
    // sd_gemm_kernel<false, true>), so the forward runs first and the mask
    // generation after it, off the critical path (launch_mask_plan off_path)
    bool small = false;
    bool hash_active = false;  // the last forward ran in hash mode (its backward must too)
    int m = 0, n = 0, k = 0;
    // launch count right after this plan's last forward and its stream: the
    // next backward launch may skip the wait for the forward grid if nothing
    // of ours was launched in between (sd::launch_gemms no_wait)
    uint64_t fwd_mark = ~0ull;
    cudaStream_t fwd_stream = nullptr;
    bool early_backward = true;  // false when buffers alias (sd_layer_plan_create)
    // SD_PLAN_DY_READY (sd_layer_plan_set_options): the caller guarantees that
    // nothing the backward reads (dY in particular) is written between this
    // plan's forward and its backward. Off by default: a caller kernel that
    // writes dY there may trigger its dependents early (PDL), and a backward
    // that skipped griddepcontrol.wait would then read dY before it is written.
    bool dy_ready = false;
    // low p: dX as the 2-CTA dense GEMM with dropped output blocks written as
    // +0.0 (every kept block is reduced over the same 64-deep stages in the same
    // order as in the sdd kernel: bit-identical)
    sd::GemmCall dx_masked;
    bool dx_masked_ok = false;
    // mid p: dX split by mask-row pairs (sd_gemm2.cu kFlagPairs): the column
    // blocks both rows of a pair keep on the 2-CTA kernel, the remainder and
    // the zero fill on the 1-CTA sdd kernel (bit-identical to the plain sdd)
    sd::GemmCall dx_pairs, dx_rem;
    bool pairs_ok = false;
    // data-parallel backward (sd_layer_plan_backward_allreduce): one event per
    // dW slab (compute -> comm stream) and one for the last all-reduce
    std::vector<cudaEvent_t> slab_done;
    cudaEvent_t reduced = nullptr;
    // CUDA-graph replays of the step (sd_layer_plan_graph_step): [0] forward,
    // [1] forward + backward; captured once on a private stream, the mask
    // kernel node's seed patched per replay
    struct GraphStep {
        cudaGraph_t graph = nullptr;  // kept: its mask node is the handle the exec update needs
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t mask_node = nullptr;
        cudaKernelNodeParams mask_params{};
        std::vector<unsigned char> mask_args;
        uint64_t kernels = 0;
    } graph[2];
    cudaStream_t capture_stream = nullptr;
    ~sd_layer_plan() {
        for (cudaEvent_t e : slab_done) cudaEventDestroy(e);
        if (reduced) cudaEventDestroy(reduced);
        for (auto& g : graph) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            if (g.graph) cudaGraphDestroy(g.graph);
        }
        if (capture_stream) cudaStreamDestroy(capture_stream);
    }
};

namespace {
constexpr double kMaskedDenseMaxP = 0.3;
constexpr double kPairsMaxP = 0.7;  // above: too few common kept blocks per row pair to pay a launch

// Measured (tools/ab_steps.py, profiles/r01_masked_dx_ab.txt): at 4096^3 the
// split backward gains 1-2% at p <= 0.2 and loses 3% at p = 0.3 (the fused
// dW+dX queue's shared tail is worth more there); at 8192^3, -12% at p = 0.1
// and -5% at p = 0.3. So p <= 0.2, or p <= 0.3 with at least four waves of
// 256x256 pair tiles.
bool use_masked_dx(const sd_layer_plan* plan) {
    if (plan->hash_active) return false;  // the masked dense dX reads the mask words
    if (!plan->dx_masked_ok || (sd::tuning() & sd::kTuneNoMaskedDense) || !sd::gemm2_routed(plan->dx_masked.args))
        return false;
    const int64_t tiles = static_cast<int64_t>(plan->dx_masked.args.rows_out / 256) * (plan->dx_masked.args.cols_out / 256);
    return plan->p <= 0.2 || tiles >= 4 * static_cast<int64_t>(sd::num_sms());
}

bool use_pairs(const sd_layer_plan* plan) {
    return !plan->hash_active && plan->pairs_ok && (sd::tuning() & sd::kTunePairs) && plan->p > 0.0 && plan->p <= kPairsMaxP &&
           !use_masked_dx(plan);
}

// dX of a mid-p plan: the row-pair 2-CTA part, then (never waiting for it: the
// output blocks are disjoint) the 1-CTA remainder (+ dW when fused).
void launch_dx_pairs(const sd_layer_plan* plan, cudaStream_t s, bool no_wait) {
    const sd::GemmCall& g = plan->dx_pairs;
    sd::launch_gemm2(g.ta, g.tb, g.tout, g.args, nullptr, nullptr, 0, s, no_wait, g.release);
}

// The backward reads X, W, dY and the mask lists and writes dX, dW; the forward
// reads X, W and the lists and writes Y. So when the caller has declared dY
// ready before the forward (SD_PLAN_DY_READY), the first backward launch right
// after the plan's forward (no launch of ours in between, same stream) needs
// nothing from the forward grid: its CTAs start on the SMs the forward's last
// wave leaves idle. Without the declaration every backward waits for the
// preceding grid (a caller kernel writing dY may trigger early under PDL).
// Consumed by the first backward launch.
// dW split into `nparts` row slabs by mask-column blocks (cached per nparts).
void prepare_dw_parts(sd_layer_plan* plan, int nparts) {
    if (plan->dw_parts == nparts) return;
    const int cblocks = plan->mask.block_cols;
    plan->dw_part.clear();
    for (int i = 0; i < nparts; ++i) {
        const int kb0 = static_cast<int>(static_cast<int64_t>(cblocks) * i / nparts);
        const int kb1 = static_cast<int>(static_cast<int64_t>(cblocks) * (i + 1) / nparts);
        plan->dw_part.push_back(prep_layer_dw_part(plan->dw, plan->x, &plan->mask, plan->m, plan->k, plan->n, kb0, kb1));
    }
    plan->dw_parts = nparts;
}

bool take_no_wait(sd_layer_plan* plan, cudaStream_t s) {
    const bool ok = plan->dy_ready && plan->early_backward && plan->fwd_mark == sd_launch_count() &&
                    plan->fwd_stream == s;
    plan->fwd_mark = ~0ull;
    return ok;
}

// The backward's two GEMMs are independent: run them as ONE persistent launch
// with a shared heaviest-first queue — dX's coarse full-reduction units first,
// dW's finer units fill the tail.
// Fused or two launches? One launch shares its tail between dX and dW but runs
// both on 128x256 units; two launches let dW run alone on 128x512 units (20
// instead of 24 KB of operands per 1M MACs) at the cost of one more tail.
// Measured (tools/ab_steps.py, profiles/r02_split_backward_ab.txt): two
// launches lose 6% at 4096^3 and 1-2% at 8192^3 (27 waves of fused units),
// win 3-4% at M = 32768-65536 with K = N = 8192 (69-124 waves), tie at p = 0.3.
bool split_backward(const sd::GemmCall& dx, const sd::GemmCall& dw) {
    const int t = sd::tuning();
    if (t & sd::kTuneNoFusedBackward) return true;
    if (t & sd::kTuneForceFused) return false;
    const auto units = [](const sd::GemmArgs& a) {
        return static_cast<int64_t>(a.n_row_tiles) * ((a.cols_out + sd::kBN - 1) / sd::kBN);
    };
    return units(dx.args) + units(dw.args) >= 48LL * sd::num_sms();
}

void fused_backward(const sd::GemmCall& dx, const sd::GemmCall& dw, cudaStream_t s, bool no_wait) {
    if (split_backward(dx, dw)) {
        // two launches; the second reads nothing the first writes, so it never
        // waits for it (its CTAs take the SMs the first one's tail frees).
        // dX's coarse full-reduction units first, dW's finer ones fill the tail
        if (sd::tuning() & sd::kTuneSplitDwFirst) {
            sd::launch_gemm(dw, s, no_wait);
            sd::launch_gemm(dx, s, true);
        } else {
            sd::launch_gemm(dx, s, no_wait);
            sd::launch_gemm(dw, s, true);
        }
        return;
    }
    const sd::GemmCall* calls[2] = {&dx, &dw};
    sd::launch_gemms(calls, 2, s, no_wait);
}
}  // namespace

extern "C" {

int sd_dense_gemm(const void* a, const void* b, void* c, int32_t c_dtype, int32_t m, int32_t n, int32_t k,
                  void* stream) {
    return guarded([&] {
        auto g = prep_dense(a, false, b, true, c, c_dtype, m, n, k);
        require_device();
        launch_gemm(g, as_stream(stream));
    });
}

int sd_gemm_ex(const void* a, int32_t a_mn, const void* b, int32_t b_mn, void* c, int32_t c_dtype, int32_t m,
               int32_t n, int32_t k, float scale, void* stream) {
    return guarded([&] {
        auto g = prep_dense(a, a_mn != 0, b, b_mn != 0, c, c_dtype, m, n, k);
        g.args.scale = scale;
        require_device();
        launch_gemm(g, as_stream(stream));
    });
}

int sd_dense_gemm_nt(const void* a, const void* b_t, void* c, int32_t c_dtype, int32_t m, int32_t n,
                     int32_t k, void* stream) {
    return guarded([&] {
        auto g = prep_dense(a, false, b_t, false, c, c_dtype, m, n, k);
        require_device();
        launch_gemm(g, as_stream(stream));
    });
}

int sd_dense_gemm_tn(const void* a_t, const void* b, void* c, int32_t c_dtype, int32_t m, int32_t n,
                     int32_t k, void* stream) {
    return guarded([&] {
        auto g = prep_dense(a_t, true, b, true, c, c_dtype, m, n, k);
        require_device();
        launch_gemm(g, as_stream(stream));
    });
}

int sd_dsd_matmul(const void* a, const sd_block_mask* mask, const void* b, float scale, void* c,
                  int32_t c_dtype, int32_t m, int32_t n, int32_t k, unsigned long long* counters,
                  void* stream) {
    return guarded([&] {
        auto g = prep_dsd_forward(a, mask, b, scale, c, c_dtype, m, n, k, counters, "dsd_matmul");
        require_device();
        launch_gemm(g, as_stream(stream));
    });
}

// Development entry (not in the public header): a dsd GEMM on the 2-CTA kernel
// in union mode, from caller-built pair lists ((block << 2) | owner bits per
// 256-row pair). a_mn selects the dW operand layout (A = X read MN-major).
SD_API int sd_dev_dsd_pairs(const void* a, const void* b, void* c, int32_t c_dtype, int32_t m, int32_t n, int32_t k,
                            int32_t a_mn, int32_t red_blk, const int32_t* pair_cnt, const int32_t* pair_idx,
                            int32_t pair_stride, float scale, void* stream) {
    return guarded([&] {
        check_gemm(m, n, k);
        GemmCall g;
        g.ta = a_mn ? mnmajor_map(a, m, k) : kmajor_map(a, k, m);
        g.tb = mnmajor_map(b, n, k);
        g.tout = out_map(c, c_dtype, m, n);
        g.args = base_args(m, n, k, scale, c);
        g.args.flags = flags_of(a_mn != 0, true, false, c_dtype);
        g.args.red_blk = red_blk;
        if (!gemm2_supported(g.args)) fail(SD_EINVAL, "sd_dev_dsd_pairs: unsupported shape");
        require_device();
        launch_gemm2(g.ta, g.tb, g.tout, g.args, pair_cnt, pair_idx, pair_stride, as_stream(stream));
    });
}

// Development entry (not in the public header): how many mask generations
// waited on their workspace's reader release counter instead of the whole
// preceding grid (evidence for the overlap tests).
SD_API uint64_t sd_dev_mask_counter_waits(void) { return g_counter_waits.load(); }

int sd_linear_forward(const void* x, const sd_block_mask* mask, const void* w, float scale, void* y,
                      int32_t y_dtype, int32_t m, int32_t n, int32_t k, void* stream) {
    return guarded([&] {
        auto g = prep_dsd_forward(x, mask, w, scale, y, y_dtype, m, n, k, nullptr, "layer forward");
        require_device();
        launch_gemm(g, as_stream(stream));
    });
}

int sd_sdd_matmul(const void* a, const void* b, const sd_block_mask* mask, float scale, void* c,
                  int32_t c_dtype, int32_t m, int32_t n, int32_t k, unsigned long long* counters,
                  void* stream) {
    return guarded([&] {
        auto g = prep_sdd(a, b, false, mask, scale, c, c_dtype, m, n, k, counters, "sdd_matmul");
        require_device();
        launch_gemm(g, as_stream(stream));
    });
}

int sd_linear_backward_dx(const void* dy, const void* w, const sd_block_mask* mask, float scale, void* dx,
                          int32_t dx_dtype, int32_t m, int32_t n, int32_t k, void* stream) {
    return guarded([&] {
        auto g = prep_layer_dx(dy, w, mask, scale, dx, dx_dtype, m, n, k);
        require_device();
        launch_gemm(g, as_stream(stream));
    });
}

int sd_linear_backward_dw(const void* x, const sd_block_mask* mask, const void* dy, float scale, void* dw,
                          int32_t dw_dtype, int32_t m, int32_t n, int32_t k, void* stream) {
    return guarded([&] {
        auto g = prep_layer_dw(x, mask, dy, scale, dw, dw_dtype, m, n, k);
        require_device();
        launch_gemm(g, as_stream(stream));
    });
}

// ---------------------------------------------------------------- layer plan

int sd_layer_plan_create(sd_layer_plan** out, const void* x, const void* w, const void* dy, void* y,
                         int32_t y_dtype, void* dx, int32_t dx_dtype, void* dw, int32_t dw_dtype, int32_t m,
                         int32_t n, int32_t k, double p, const sd_block_mask* mask) {
    return guarded([&] {
        if (!out) fail(SD_EINVAL, "sd_layer_plan_create: null plan pointer");
        *out = nullptr;
        if (!(p >= 0.0 && p < 1.0)) {
            char buf[64];
            std::snprintf(buf, sizeof buf, "%f", p);
            fail(SD_EINVAL, std::string("dropout rate must lie in [0, 1), got ") + buf);
        }
        if (!mask) fail(SD_EINVAL, "sd_layer_plan_create: null mask");
        const float s = dropout_scale_f32(p);
        sd_layer_plan tmp;
        tmp.mask = *mask;
        tmp.p = p;
        tmp.threshold = threshold_of(p);
        tmp.fwd = prep_dsd_forward(x, mask, w, s, y, y_dtype, m, n, k, nullptr, "layer forward");
        tmp.dw = prep_layer_dw(x, mask, dy, s, dw, dw_dtype, m, n, k);
        tmp.dx = prep_layer_dx(dy, w, mask, s, dx, dx_dtype, m, n, k);
        // nominal keep fraction: lets the GEMM launcher pick the unit kind (tile shape)
        tmp.fwd.args.keep_hint = tmp.dw.args.keep_hint = tmp.dx.args.keep_hint = static_cast<float>(1.0 - p);
        require_device();
        cudaGetDevice(&tmp.device);
        (void)sched_slot(nullptr);  // allocate the scheduler slots now (keeps launches capturable)
        tmp.dense_fwd = prep_dense(x, false, w, true, y, y_dtype, m, n, k);
        tmp.dense_dw = prep_dense(x, true, dy, true, dw, dw_dtype, k, n, m);
        tmp.dense_dx = prep_dense(dy, false, w, false, dx, dx_dtype, m, k, n);
        tmp.x = x;
        tmp.dy = dy;
        tmp.w = w;
        tmp.m = m, tmp.n = n, tmp.k = k;
        {
            // small: every 128 x 256 unit of the forward, dX and dW runs at once
            // (< one wave together) and every kept list fits the 64-entry hash
            // decode; then the mask generation is better off the critical path
            const auto units = [](const GemmArgs& a) {
                return static_cast<int64_t>(a.n_row_tiles) * ((a.cols_out + kBN - 1) / kBN);
            };
#ifndef SD_SMALL_ANY
#define SD_SMALL_ANY 0
#endif
            tmp.small = p > 0.0 && mask->block_rows <= 64 && mask->block_cols <= 64 &&
                        (SD_SMALL_ANY || units(tmp.fwd.args) + units(tmp.dx.args) + units(tmp.dw.args) <= num_sms());
        }
        // Masked dense dX: sdd over the kept fraction (1 - p) of the blocks on
        // 1-CTA tiles costs ~1.2-1.4x the 2-CTA kernel's time per MAC
        // (profiles/r01_masked_dx_ab.txt), so below p = kMaskedDenseMaxP the
        // full dense product with zeroed dropped blocks is faster.
        tmp.dx_masked = tmp.dense_dx;
        tmp.dx_masked.args.scale = s;
        tmp.dx_masked.args.flags |= kFlagOutMask;
        tmp.dx_masked.args.words = mask->words;
        tmp.dx_masked.args.mask_cols = mask->block_cols;
        tmp.dx_masked.release = mask_release_counter(mask);
        tmp.dx_masked_ok = p <= kMaskedDenseMaxP && mask->m_blk == 128 && mask->k_blk == 128 &&
                           gemm2_supported(tmp.dx_masked.args);
        // row-pair split of dX: A = dY (K-major), B = W (K-major, read in place)
        tmp.dx_pairs.ta = tmp.dx.ta;
        tmp.dx_pairs.tb = tmp.dx.tb;
        tmp.dx_pairs.tout = tmp.dx.tout;
        tmp.dx_pairs.args = base_args(m, k, n, s, dx);
        tmp.dx_pairs.args.flags = kFlagPairs | (dx_dtype == SD_DTYPE_F32 ? kFlagF32 : 0u);
        tmp.dx_pairs.args.words = mask->words;
        tmp.dx_pairs.args.mask_cols = mask->block_cols;
        tmp.dx_pairs.args.out_row_blk = mask->m_blk;
        tmp.dx_pairs.args.out_col_blk = mask->k_blk;
        tmp.dx_pairs.release = mask_release_counter(mask);
        tmp.dx_rem = tmp.dx;
        tmp.dx_rem.args.flags |= kFlagPairs;
        tmp.pairs_ok = mask->m_blk == 128 && mask->k_blk == 128 && mask->block_rows % 2 == 0 &&
                       gemm2_pairs_supported(tmp.dx_pairs.args);
        // the early backward relies on the forward writing nothing the backward
        // touches: with Y overlapping X, W, dY, dX or dW, or the mask workspace
        // overlapping any buffer, every backward waits for the forward grid
        {
            const auto el = [](int dt) -> size_t { return dt == SD_DTYPE_F32 ? 4 : 2; };
            struct Range {
                uintptr_t b, e;
            };
            const auto rg = [](const void* p, size_t bytes) {
                return Range{reinterpret_cast<uintptr_t>(p), reinterpret_cast<uintptr_t>(p) + bytes};
            };
            const Range ry = rg(y, static_cast<size_t>(m) * n * el(y_dtype));
            const Range others[5] = {rg(x, static_cast<size_t>(m) * k * 2), rg(w, static_cast<size_t>(k) * n * 2),
                                     rg(dy, static_cast<size_t>(m) * n * 2),
                                     rg(dx, static_cast<size_t>(m) * k * el(dx_dtype)),
                                     rg(dw, static_cast<size_t>(k) * n * el(dw_dtype))};
            const size_t mws = sd_mask_workspace_bytes(mask->block_rows, mask->block_cols);
            const Range rm = rg(mask->words, mws);
            const auto overlap = [](Range a, Range b) { return a.b < b.e && b.b < a.e; };
            bool alias = false;
            for (const Range& o : others) alias = alias || overlap(ry, o) || overlap(rm, o);
            alias = alias || overlap(rm, ry);
            tmp.early_backward = !alias;
        }
        *out = new sd_layer_plan(tmp);
    });
}

// p = 0 keeps every block: the step is the dense layer, and the dense kernels
// (2-CTA when the shape allows) give bit-identical outputs — every element is
// reduced over the same 16-deep MMA steps in the same order
// (tests/test_gpu_kernel_modes.py::test_p0_plan_equals_sparse_kernels). The
// (all-kept) mask is still generated: the caller's BlockMask stays valid.
static bool plan_dense(const sd_layer_plan* plan) { return plan->p == 0.0 && !(tuning() & kTuneNarrow); }

// Hash mode of a small plan's GEMMs (GemmArgs::hash_mode): set on the forward,
// dX and dW calls (and the dW slabs) for this forward's seed, or cleared.
static void set_hash(sd::GemmArgs& a, int mode, int len, uint64_t seed_mix, const sd_layer_plan* plan) {
    a.hash_mode = mode;
    a.hash_len = len;
    a.hash_row_off = plan->mask.row_block_offset;
    a.hash_seed_mix = seed_mix;
    a.hash_threshold = plan->threshold;
}

static void plan_set_hash(sd_layer_plan* plan, uint64_t seed_mix, bool on) {
    const int R = plan->mask.block_rows, C = plan->mask.block_cols;
    set_hash(plan->fwd.args, on ? 1 : 0, C, seed_mix, plan);
    set_hash(plan->dx.args, on ? 1 : 0, C, seed_mix, plan);
    set_hash(plan->dw.args, on ? 2 : 0, R, seed_mix, plan);
    for (auto& g : plan->dw_part) set_hash(g.args, on ? 2 : 0, R, seed_mix, plan);
    const auto units = [](const sd::GemmArgs& a) { return a.n_row_tiles * ((a.cols_out + sd::kBN - 1) / sd::kBN); };
    const int total = units(plan->fwd.args) + units(plan->dx.args) + units(plan->dw.args);
    plan->fwd.args.hash_plan_units = plan->dx.args.hash_plan_units = plan->dw.args.hash_plan_units = total;
    for (auto& g : plan->dw_part) g.args.hash_plan_units = total;
}

static bool stream_capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return st != cudaStreamCaptureStatusNone;
}

static void plan_forward_impl(sd_layer_plan* plan, uint64_t seed, cudaStream_t s, bool allow_small = true) {
    const uint64_t sm = mix64_host(seed);
    const bool dense = plan_dense(plan);
    const bool small = plan->small && allow_small && !dense && !(sd::tuning() & sd::kTuneNoSmallHash) &&
                       !stream_capturing(s);
    plan_set_hash(plan, sm, small);
    plan->hash_active = small;
    if (small) {
        // the forward needs nothing from the mask generation: it goes first, the
        // generation (for the plan's mask outputs and list readers) after it
        launch_gemm(plan->fwd, s);
        launch_mask_plan(plan->mask, false, sm, plan->threshold, s, true);
    } else {
        launch_mask_plan(plan->mask, false, sm, plan->threshold, s);
        launch_gemm(dense ? plan->dense_fwd : plan->fwd, s);
    }
    plan->fwd_mark = sd_launch_count();
    plan->fwd_stream = s;
}

int sd_layer_plan_forward(sd_layer_plan* plan, uint64_t seed, void* stream) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        plan_forward_impl(plan, seed, as_stream(stream));
    });
}

int sd_layer_plan_backward_dw(sd_layer_plan* plan, void* stream) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        launch_gemm(plan->dw, as_stream(stream), take_no_wait(plan, as_stream(stream)));
    });
}

int sd_layer_plan_backward_dw_part(sd_layer_plan* plan, int32_t part, int32_t nparts, void* stream) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        const int cblocks = plan->mask.block_cols;
        if (nparts < 1 || part < 0 || part >= nparts || nparts > cblocks)
            fail(SD_ERANGE, "backward_dw_part: part " + str(part) + " of " + str(nparts) + " out of range for " +
                                str(cblocks) + " mask columns");
        prepare_dw_parts(plan, nparts);
        launch_gemm(plan->dw_part[part], as_stream(stream), take_no_wait(plan, as_stream(stream)));
    });
}

int sd_layer_plan_backward_allreduce(sd_layer_plan* plan, sd_comm* comm, int32_t nparts, void* stream,
                                     void* comm_stream) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        if (!comm) fail(SD_EINVAL, "sd_layer_plan_backward_allreduce: null communicator");
        if (comm_device(comm) != plan->device)
            fail(SD_EINVAL, "sd_layer_plan_backward_allreduce: communicator on device " + str(comm_device(comm)) +
                                ", plan on device " + str(plan->device));
        const int cblocks = plan->mask.block_cols;
        if (nparts < 1 || nparts > cblocks)
            fail(SD_ERANGE, "backward_allreduce: nparts " + str(nparts) + " out of range for " + str(cblocks) +
                                " mask columns");
        prepare_dw_parts(plan, nparts);
        const cudaStream_t s = as_stream(stream);
        const cudaStream_t cs = comm_stream ? as_stream(comm_stream) : s;
        while (static_cast<int>(plan->slab_done.size()) < nparts) {
            cudaEvent_t e;
            check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            plan->slab_done.push_back(e);
        }
        if (!plan->reduced) check_cuda(cudaEventCreateWithFlags(&plan->reduced, cudaEventDisableTiming), "cudaEventCreate");
        const bool f32 = plan->dw.args.flags & kFlagF32;
        const bool nw = take_no_wait(plan, s);
        // dW slab by slab (mask-column blocks, the same tiles and reduction
        // order as the full dW): slab i's all-reduce runs on the comm stream
        // while slab i+1 and then dX compute on `stream`
        for (int i = 0; i < nparts; ++i) {
            const GemmCall& g = plan->dw_part[i];
            launch_gemm(g, s, i == 0 && nw);
            if (cs != s) {
                check_cuda(cudaEventRecord(plan->slab_done[i], s), "cudaEventRecord(dW slab)");
                check_cuda(cudaStreamWaitEvent(cs, plan->slab_done[i], 0), "cudaStreamWaitEvent(dW slab)");
            }
            comm_allreduce_sum(comm, g.args.out, static_cast<size_t>(g.args.rows_out) * g.args.cols_out,
                               f32 ? SD_DTYPE_F32 : SD_DTYPE_BF16, cs);
        }
        // dX reads nothing the dW slabs write: it does not wait for them, and
        // its CTAs start on the SMs the last slab's tail frees
        if (use_pairs(plan)) {
            launch_dx_pairs(plan, s, true);
            launch_gemm(plan->dx_rem, s, true);
        } else {
            launch_gemm(use_masked_dx(plan) ? plan->dx_masked : plan->dx, s, true);
        }
        if (cs != s) {
            check_cuda(cudaEventRecord(plan->reduced, cs), "cudaEventRecord(all-reduce)");
            check_cuda(cudaStreamWaitEvent(s, plan->reduced, 0), "cudaStreamWaitEvent(all-reduce)");
        }
    });
}

int sd_layer_plan_backward_dx(sd_layer_plan* plan, void* stream) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        const bool nw = take_no_wait(plan, as_stream(stream));
        if ((sd::tuning() & sd::kTuneDxt) && sd::dxt_supported(plan->dx.args)) {
            sd::launch_dxt(plan->dx, plan->dy, plan->w, as_stream(stream), nw);
        } else if (use_pairs(plan)) {
            launch_dx_pairs(plan, as_stream(stream), nw);
            launch_gemm(plan->dx_rem, as_stream(stream), true);
        } else {
            launch_gemm(use_masked_dx(plan) ? plan->dx_masked : plan->dx, as_stream(stream), nw);
        }
    });
}

static void plan_backward_impl(sd_layer_plan* plan, cudaStream_t s) {
    const bool nw = take_no_wait(plan, s);
    if (plan_dense(plan)) {
        fused_backward(plan->dense_dx, plan->dense_dw, s, nw);
    } else if (use_masked_dx(plan)) {
        // dW on the 1-CTA kernel, dX on the 2-CTA kernel: independent
        // launches, the second never waits for the first
        launch_gemm(plan->dw, s, nw);
        launch_gemm(plan->dx_masked, s, true);
    } else if ((sd::tuning() & sd::kTuneDxt) && sd::dxt_supported(plan->dx.args)) {
        // dX on the transposed 2-CTA kernel, then dW as its own 1-CTA launch
        // (never waiting for dX: independent outputs)
        sd::launch_dxt(plan->dx, plan->dy, plan->w, s, nw);
        launch_gemm(plan->dw, s, true);
    } else if (use_pairs(plan)) {
        // dX's row-pair part on the 2-CTA kernel, then dX's remainder and dW
        // as one 1-CTA launch that fills the SMs the first one leaves
        launch_dx_pairs(plan, s, nw);
        fused_backward(plan->dx_rem, plan->dw, s, true);
    } else {
        fused_backward(plan->dx, plan->dw, s, nw);
    }
}

int sd_layer_plan_backward(sd_layer_plan* plan, void* stream) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        plan_backward_impl(plan, as_stream(stream));
    });
}

// One CUDA-graph launch per step for host-bound callers (small layers, many
// layers per step): the step's kernels (mask generation, forward and, with
// what = 3, the backward — the same launches and PDL edges as the eager
// calls) are captured once per plan on a private stream; each call patches the
// seed into the graph's mask node and launches the graph on `stream`. Results
// equal the eager calls'. Inside the graph the mask generation waits for its
// predecessor grid (the release-counter overlap needs host tracking), and the
// next eager generation into the workspace does too.
int sd_layer_plan_graph_step(sd_layer_plan* plan, uint64_t seed, int32_t what, void* stream) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        if (what != 1 && what != 3) fail(SD_EINVAL, "sd_layer_plan_graph_step: what must be 1 (forward) or 3 (step)");
        auto& g = plan->graph[what == 3 ? 1 : 0];
        if (!g.exec) {
            if (!plan->capture_stream)
                check_cuda(cudaStreamCreateWithFlags(&plan->capture_stream, cudaStreamNonBlocking),
                           "cudaStreamCreate(capture)");
            const cudaStream_t cs = plan->capture_stream;
            const uint64_t l0 = sd_launch_count();
            check_cuda(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
            cudaGraph_t graph = nullptr;
            try {
                plan_forward_impl(plan, seed, cs, false);
                if (what == 3) plan_backward_impl(plan, cs);
            } catch (...) {
                cudaStreamEndCapture(cs, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            check_cuda(cudaStreamEndCapture(cs, &graph), "cudaStreamEndCapture");
            g.kernels = sd_launch_count() - l0;
            size_t n = 0;
            check_cuda(cudaGraphGetNodes(graph, nullptr, &n), "cudaGraphGetNodes");
            std::vector<cudaGraphNode_t> nodes(n);
            check_cuda(cudaGraphGetNodes(graph, nodes.data(), &n), "cudaGraphGetNodes");
            for (cudaGraphNode_t node : nodes) {
                cudaGraphNodeType type;
                check_cuda(cudaGraphNodeGetType(node, &type), "cudaGraphNodeGetType");
                if (type != cudaGraphNodeTypeKernel) continue;
                cudaKernelNodeParams kp{};
                check_cuda(cudaGraphKernelNodeGetParams(node, &kp), "cudaGraphKernelNodeGetParams");
                if (kp.func != mask_plan_kernel_func()) continue;
                g.mask_node = node;
                g.mask_params = kp;
                g.mask_args.assign(static_cast<unsigned char*>(kp.kernelParams[0]),
                                   static_cast<unsigned char*>(kp.kernelParams[0]) + mask_plan_args_size());
                break;
            }
            if (!g.mask_node) {
                cudaGraphDestroy(graph);
                fail(SD_ERUNTIME, "sd_layer_plan_graph_step: no mask node in the captured step");
            }
            const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
            if (e != cudaSuccess) {
                cudaGraphDestroy(graph);
                g.mask_node = nullptr;
                check_cuda(e, "cudaGraphInstantiate");
            }
            g.graph = graph;
        }
        mask_plan_patch_seed(g.mask_args.data(), mix64_host(seed));
        void* args[1] = {g.mask_args.data()};
        cudaKernelNodeParams kp = g.mask_params;
        kp.kernelParams = args;
        kp.extra = nullptr;
        check_cuda(cudaGraphExecKernelNodeSetParams(g.exec, g.mask_node, &kp), "cudaGraphExecKernelNodeSetParams");
        check_cuda(cudaGraphLaunch(g.exec, as_stream(stream)), "cudaGraphLaunch");
        note_launch(g.kernels);
        // the replay's readers release the workspace counter without host
        // tracking: the next eager generation waits for the whole grid instead
        mask_note_untracked(plan->mask.words);
        plan->fwd_mark = ~0ull;
    });
}

int sd_layer_plan_dense_forward(sd_layer_plan* plan, void* stream) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        launch_gemm(plan->dense_fwd, as_stream(stream));
        plan->fwd_mark = sd_launch_count();
        plan->fwd_stream = as_stream(stream);
    });
}

int sd_layer_plan_dense_backward(sd_layer_plan* plan, void* stream) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        fused_backward(plan->dense_dx, plan->dense_dw, as_stream(stream), take_no_wait(plan, as_stream(stream)));
    });
}

int sd_layer_plan_set_options(sd_layer_plan* plan, int32_t options) {
    return guarded([&] {
        if (!plan) fail(SD_EINVAL, "null plan");
        if (options & ~SD_PLAN_DY_READY) fail(SD_EINVAL, "sd_layer_plan_set_options: unknown option bits");
        plan->dy_ready = (options & SD_PLAN_DY_READY) != 0;
    });
}

int sd_layer_plan_destroy(sd_layer_plan* plan) {
    delete plan;
    return SD_OK;
}

uint64_t sd_flops_dense(int64_t m, int64_t n, int64_t k) { return 2ull * m * n * k; }

uint64_t sd_flops_effective(int64_t n, int64_t k, int32_t m_blk, int32_t n_blk, int32_t k_blk, int64_t keep,
                            int32_t kind) {
    const uint64_t kp = static_cast<uint64_t>(keep);
    if (kind == 0) return 2ull * static_cast<uint64_t>(n) * m_blk * k_blk * kp;
    return 2ull * static_cast<uint64_t>(k) * m_blk * n_blk * kp;
}

}  // extern "C"
