// sparsedrop_b200.hpp — C++ host API over the C-ABI (sparsedrop_b200.h),
// mirroring the reference's operator API (namespace sparsedrop,
// /root/reference/proj/include/sparsedrop/{block_mask,gemm,layer}.hpp) on B200
// device memory. Header-only; needs no CUDA headers (device memory goes through
// sd_device_alloc / sd_memcpy). Link against libsparsedrop_b200.so.
//
// Differences from the reference, all forced by the device:
//  * matrices live in device memory (DeviceMatrix<T>, T = bf16 inputs,
//    bf16 or float outputs); host Matrix-like data is uploaded with
//    DeviceMatrix<bf16>::from_host (round-to-nearest-even) and read back with
//    to_host();
//  * the `threads` argument is replaced by a stream handle (void*, NULL =
//    legacy default stream);
//  * TileConfig describes the mask blocks only: the B200 kernels use fixed
//    128 x 256 x 64 tiles, and require m_blk % 128 == 0 and k_blk % 64 == 0
//    (sdd: n_blk in {128, 256}).
// Errors: the same exception classes and message substrings as the reference
// (std::invalid_argument, std::out_of_range, std::runtime_error).
#pragma once

#include <cmath>
#include <array>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sparsedrop_b200.h"

namespace sparsedrop::b200 {

inline void check(int status) {
    if (status == SD_OK) return;
    const std::string msg = sd_last_error();
    if (status == SD_EINVAL) throw std::invalid_argument(msg);
    if (status == SD_ERANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

// bf16 storage (bit pattern), round-to-nearest-even from float.
struct bf16 {
    std::uint16_t bits = 0;
    static bf16 from_float(float f) {
        std::uint32_t u;
        std::memcpy(&u, &f, 4);
        bf16 b;
        if ((u & 0x7fffffffu) > 0x7f800000u)
            b.bits = static_cast<std::uint16_t>((u >> 16) | 0x40u);
        else
            b.bits = static_cast<std::uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
        return b;
    }
    float to_float() const {
        const std::uint32_t u = static_cast<std::uint32_t>(bits) << 16;
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    }
};

template <typename T>
constexpr int dtype_code() {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, bf16>, "bf16 or float");
    return std::is_same_v<T, float> ? SD_DTYPE_F32 : SD_DTYPE_BF16;
}

// Owning device allocation.
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t bytes) : bytes_(bytes) {
        void* p = nullptr;
        check(sd_device_alloc(&p, bytes));
        ptr_.reset(p);
    }
    void* get() const { return ptr_.get(); }
    std::size_t bytes() const { return bytes_; }

private:
    struct Free {
        void operator()(void* p) const { sd_device_free(p); }
    };
    std::unique_ptr<void, Free> ptr_;
    std::size_t bytes_ = 0;
};

// Dense row-major device matrix (matrix.hpp:11 layout).
template <typename T>
class DeviceMatrix {
public:
    DeviceMatrix() = default;
    DeviceMatrix(int rows, int cols) : rows_(rows), cols_(cols) {
        if (rows <= 0 || cols <= 0)
            throw std::invalid_argument("Matrix dimensions must be positive, got " + std::to_string(rows) + "x" +
                                        std::to_string(cols));
        buf_ = std::make_shared<DeviceBuffer>(static_cast<std::size_t>(rows) * cols * sizeof(T));
    }
    static DeviceMatrix from_host(int rows, int cols, const std::vector<float>& data, void* stream = nullptr) {
        if (data.size() != static_cast<std::size_t>(rows) * cols)
            throw std::invalid_argument("Matrix data length does not match shape");
        DeviceMatrix m(rows, cols);
        std::vector<T> host(data.size());
        for (std::size_t i = 0; i < data.size(); ++i) {
            if constexpr (std::is_same_v<T, bf16>)
                host[i] = bf16::from_float(data[i]);
            else
                host[i] = data[i];
        }
        check(sd_memcpy(m.data(), host.data(), host.size() * sizeof(T), 0, stream));
        check(sd_stream_synchronize(stream));
        return m;
    }
    std::vector<float> to_host(void* stream = nullptr) const {
        std::vector<T> host(size());
        check(sd_memcpy(host.data(), data(), host.size() * sizeof(T), 1, stream));
        check(sd_stream_synchronize(stream));
        std::vector<float> out(host.size());
        for (std::size_t i = 0; i < host.size(); ++i) {
            if constexpr (std::is_same_v<T, bf16>)
                out[i] = host[i].to_float();
            else
                out[i] = host[i];
        }
        return out;
    }
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    std::size_t size() const { return static_cast<std::size_t>(rows_) * cols_; }
    T* data() const { return static_cast<T*>(buf_ ? buf_->get() : nullptr); }
    std::string shape_string() const { return std::to_string(rows_) + "x" + std::to_string(cols_); }

private:
    int rows_ = 0, cols_ = 0;
    std::shared_ptr<DeviceBuffer> buf_;
};

// block_mask.hpp:14-26
struct TileConfig {
    int m_blk = 128;
    int n_blk = 128;
    int k_blk = 128;
};

struct DropoutSpec {
    double p = 0.0;
    int m_blk = 128;
    int k_blk = 128;
    std::uint64_t seed = 0;
};

// Device-resident BlockMask (block_mask.hpp:31-76) with its compaction lists.
class BlockMask {
public:
    BlockMask() = default;
    BlockMask(int block_rows, int block_cols, int m_blk, int k_blk, int row_block_offset = 0) {
        if (block_rows <= 0 || block_cols <= 0 || m_blk <= 0 || k_blk <= 0)
            throw std::invalid_argument("BlockMask geometry must be positive: grid " + std::to_string(block_rows) +
                                        "x" + std::to_string(block_cols) + ", blocks " + std::to_string(m_blk) +
                                        "x" + std::to_string(k_blk));
        const std::size_t bytes = sd_mask_workspace_bytes(block_rows, block_cols);
        ws_ = std::make_shared<DeviceBuffer>(bytes);  // cudaMalloc: 256-byte aligned
        check(sd_memset(ws_->get(), 0, bytes, nullptr));
        check(sd_stream_synchronize(nullptr));
        c_ = std::make_shared<sd_block_mask>();
        check(sd_mask_bind(c_.get(), ws_->get(), block_rows, block_cols, m_blk, k_blk, row_block_offset));
    }
    int block_rows() const { return c_->block_rows; }
    int block_cols() const { return c_->block_cols; }
    int m_blk() const { return c_->m_blk; }
    int k_blk() const { return c_->k_blk; }
    int rows() const { return block_rows() * m_blk(); }
    int cols() const { return block_cols() * k_blk(); }
    std::int64_t total_blocks() const { return static_cast<std::int64_t>(block_rows()) * block_cols(); }
    std::int64_t keep_count(void* stream = nullptr) const {
        std::int64_t k = 0;
        check(sd_memcpy(&k, c_->keep_count, sizeof k, 1, stream));
        check(sd_stream_synchronize(stream));
        return k;
    }
    double realized_sparsity(void* stream = nullptr) const {
        return total_blocks() == 0 ? 0.0 : 1.0 - static_cast<double>(keep_count(stream)) / total_blocks();
    }
    std::vector<std::uint64_t> words(void* stream = nullptr) const {
        std::vector<std::uint64_t> w(static_cast<std::size_t>((total_blocks() + 63) / 64));
        check(sd_memcpy(w.data(), c_->words, w.size() * 8, 1, stream));
        check(sd_stream_synchronize(stream));
        return w;
    }
    bool kept(int block_row, int block_col) const {
        const auto w = words();
        const std::uint64_t b = static_cast<std::uint64_t>(block_row) * block_cols() + block_col;
        return (w[b >> 6] >> (b & 63)) & 1u;
    }
    const sd_block_mask* c() const { return c_.get(); }
    sd_block_mask* c() { return c_.get(); }

private:
    std::shared_ptr<DeviceBuffer> ws_;
    std::shared_ptr<sd_block_mask> c_;
};

// block_mask.cpp:52-80 (on device, bit-exact)
inline BlockMask sample_mask(const DropoutSpec& spec, int rows, int cols, void* stream = nullptr,
                             int row_block_offset = 0) {
    if (spec.p < 0.0 || spec.p >= 1.0)
        throw std::invalid_argument("dropout rate must lie in [0, 1), got " + std::to_string(spec.p));
    if (spec.m_blk <= 0 || rows % spec.m_blk != 0)
        throw std::invalid_argument("mask block size m_blk=" + std::to_string(spec.m_blk) +
                                    " does not divide rows=" + std::to_string(rows));
    if (spec.k_blk <= 0 || cols % spec.k_blk != 0)
        throw std::invalid_argument("mask block size k_blk=" + std::to_string(spec.k_blk) +
                                    " does not divide cols=" + std::to_string(cols));
    BlockMask m(rows / spec.m_blk, cols / spec.k_blk, spec.m_blk, spec.k_blk, row_block_offset);
    check(sd_mask_sample(m.c(), spec.seed, spec.p, rows, cols, stream));
    return m;
}

// block_mask.cpp:82-98
inline BlockMask mask_from_words(int block_rows, int block_cols, int m_blk, int k_blk,
                                 const std::vector<std::uint64_t>& words, void* stream = nullptr) {
    const std::int64_t bits = static_cast<std::int64_t>(block_rows) * block_cols;
    if (static_cast<std::int64_t>(words.size()) != (bits + 63) / 64)
        throw std::invalid_argument("BlockMask word count " + std::to_string(words.size()) +
                                    " does not match grid of " + std::to_string(bits) + " bits");
    if ((bits & 63) && (words.back() & (~std::uint64_t(0) << (bits & 63))))
        throw std::invalid_argument("BlockMask has nonzero bits past the block grid");
    BlockMask m(block_rows, block_cols, m_blk, k_blk);
    check(sd_memcpy(m.c()->words, words.data(), words.size() * 8, 0, stream));
    check(sd_mask_compact(m.c(), stream));
    return m;
}

// block_mask.cpp:117-123
inline BlockMask transpose_mask(const BlockMask& mask, void* stream = nullptr) {
    BlockMask out(mask.block_cols(), mask.block_rows(), mask.k_blk(), mask.m_blk());
    check(sd_mask_transpose(mask.c(), out.c(), stream));
    return out;
}

// block_mask.cpp:100-115
inline BlockMask retile(const BlockMask& mask, int split_m, int split_k, void* stream = nullptr) {
    if (split_m <= 0 || mask.m_blk() % split_m != 0)
        throw std::invalid_argument("split_m=" + std::to_string(split_m) + " does not divide m_blk=" +
                                    std::to_string(mask.m_blk()));
    if (split_k <= 0 || mask.k_blk() % split_k != 0)
        throw std::invalid_argument("split_k=" + std::to_string(split_k) + " does not divide k_blk=" +
                                    std::to_string(mask.k_blk()));
    BlockMask out(mask.block_rows() * split_m, mask.block_cols() * split_k, mask.m_blk() / split_m,
                  mask.k_blk() / split_k);
    check(sd_mask_retile(mask.c(), split_m, split_k, out.c(), stream));
    return out;
}

// block_mask.cpp:125-135 (from the device row lists)
inline std::vector<int> kept_blocks_in_row(const BlockMask& mask, int block_row, void* stream = nullptr) {
    if (block_row < 0 || block_row >= mask.block_rows())
        throw std::out_of_range("block row " + std::to_string(block_row) + " outside grid with " +
                                std::to_string(mask.block_rows()) + " rows");
    std::int32_t cnt = 0;
    check(sd_memcpy(&cnt, mask.c()->row_cnt + block_row, 4, 1, stream));
    check(sd_stream_synchronize(stream));
    std::vector<std::int32_t> idx(static_cast<std::size_t>(cnt));
    if (cnt) {
        check(sd_memcpy(idx.data(), mask.c()->row_idx + static_cast<std::int64_t>(block_row) * mask.block_cols(),
                        idx.size() * 4, 1, stream));
        check(sd_stream_synchronize(stream));
    }
    return std::vector<int>(idx.begin(), idx.end());
}

// ---------------------------------------------------------------- BMSK (block_mask.cpp:137-219)
// Byte-compatible with the reference's container; read_mask re-compacts the
// mask on the device so it can drive the GEMMs directly.
inline void write_mask(const BlockMask& mask, std::ostream& out) {
    auto put = [&](std::uint64_t v, int n) {
        for (int i = 0; i < n; ++i) out.put(static_cast<char>((v >> (8 * i)) & 0xff));
    };
    out.write("BMSK", 4);
    out.put(static_cast<char>(0x01));
    put(static_cast<std::uint32_t>(mask.block_rows()), 4);
    put(static_cast<std::uint32_t>(mask.block_cols()), 4);
    put(static_cast<std::uint32_t>(mask.m_blk()), 4);
    put(static_cast<std::uint32_t>(mask.k_blk()), 4);
    for (std::uint64_t w : mask.words()) put(w, 8);
}

inline BlockMask read_mask(std::istream& in, const std::string& name, void* stream = nullptr) {
    char magic[4];
    if (!in.read(magic, 4) || std::memcmp(magic, "BMSK", 4) != 0)
        throw std::runtime_error(name + ": not a BMSK file (bad magic)");
    const int version = in.get();
    if (version != 0x01) throw std::runtime_error(name + ": unsupported BMSK version " + std::to_string(version));
    auto get = [&](int n, const char* what) {
        unsigned char b[8];
        if (!in.read(reinterpret_cast<char*>(b), n)) throw std::runtime_error(name + ": truncated BMSK " + what);
        std::uint64_t v = 0;
        for (int i = 0; i < n; ++i) v |= std::uint64_t(b[i]) << (8 * i);
        return v;
    };
    const auto br = static_cast<int>(get(4, "header")), bc = static_cast<int>(get(4, "header"));
    const auto mb = static_cast<int>(get(4, "header")), kb = static_cast<int>(get(4, "header"));
    if (br <= 0 || bc <= 0 || mb <= 0 || kb <= 0) throw std::runtime_error(name + ": BMSK header has non-positive geometry");
    std::vector<std::uint64_t> words(static_cast<std::size_t>((static_cast<std::int64_t>(br) * bc + 63) / 64));
    for (auto& w : words) w = get(8, "payload");
    try {
        return mask_from_words(br, bc, mb, kb, words, stream);
    } catch (const std::invalid_argument& e) {
        throw std::runtime_error(name + ": " + e.what());
    }
}

inline void save_mask(const BlockMask& mask, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open " + path + " for writing");
    write_mask(mask, out);
    if (!out) throw std::runtime_error("write failed: " + path);
}

inline BlockMask load_mask(const std::string& path, void* stream = nullptr) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    return read_mask(in, path, stream);
}

// gemm.hpp:31-37 (128-row tile rows; n_blk = 128 on B200)
struct KernelCounters {
    std::uint64_t kblock_iterations = 0;
    std::vector<std::uint64_t> kblock_per_tile_row;
};

namespace detail {
inline void check_shapes(int a_rows, int a_cols, int b_rows, int b_cols) {
    if (a_cols != b_rows)
        throw std::invalid_argument("gemm shape mismatch: " + std::to_string(a_rows) + "x" + std::to_string(a_cols) +
                                    " * " + std::to_string(b_rows) + "x" + std::to_string(b_cols));
}
struct CounterBuf {
    DeviceBuffer buf;
    int n = 0;
    CounterBuf(KernelCounters* c, int rows) {
        if (!c) return;
        n = rows / 128;
        buf = DeviceBuffer(static_cast<std::size_t>(n) * 8);
        check(sd_memset(buf.get(), 0, buf.bytes(), nullptr));
    }
    unsigned long long* ptr() const { return static_cast<unsigned long long*>(buf.get()); }
    void fill(KernelCounters* c, void* stream) const {
        if (!c) return;
        c->kblock_per_tile_row.assign(n, 0);
        check(sd_memcpy(c->kblock_per_tile_row.data(), buf.get(), buf.bytes(), 1, stream));
        check(sd_stream_synchronize(stream));
        c->kblock_iterations = 0;
        for (auto v : c->kblock_per_tile_row) c->kblock_iterations += v;
    }
};
}  // namespace detail

// gemm.hpp:104-128
template <typename OutT = bf16>
DeviceMatrix<OutT> dense_gemm(const DeviceMatrix<bf16>& a, const DeviceMatrix<bf16>& b, void* stream = nullptr) {
    detail::check_shapes(a.rows(), a.cols(), b.rows(), b.cols());
    DeviceMatrix<OutT> c(a.rows(), b.cols());
    check(sd_dense_gemm(a.data(), b.data(), c.data(), dtype_code<OutT>(), a.rows(), b.cols(), a.cols(), stream));
    return c;
}

// gemm.hpp:133-170
template <typename OutT = bf16>
DeviceMatrix<OutT> dsd_matmul(const DeviceMatrix<bf16>& a, const BlockMask& mask, const DeviceMatrix<bf16>& b,
                              float scale_factor, KernelCounters* counters = nullptr, void* stream = nullptr) {
    detail::check_shapes(a.rows(), a.cols(), b.rows(), b.cols());
    DeviceMatrix<OutT> c(a.rows(), b.cols());
    detail::CounterBuf cb(counters, a.rows());
    check(sd_dsd_matmul(a.data(), mask.c(), b.data(), scale_factor, c.data(), dtype_code<OutT>(), a.rows(),
                        b.cols(), a.cols(), cb.ptr(), stream));
    cb.fill(counters, stream);
    return c;
}

// gemm.hpp:176-213
template <typename OutT = bf16>
DeviceMatrix<OutT> sdd_matmul(const DeviceMatrix<bf16>& a, const DeviceMatrix<bf16>& b, const BlockMask& mask,
                              float scale_factor, KernelCounters* counters = nullptr, void* stream = nullptr) {
    detail::check_shapes(a.rows(), a.cols(), b.rows(), b.cols());
    DeviceMatrix<OutT> c(a.rows(), b.cols());
    detail::CounterBuf cb(counters, a.rows());
    check(sd_sdd_matmul(a.data(), b.data(), mask.c(), scale_factor, c.data(), dtype_code<OutT>(), a.rows(),
                        b.cols(), a.cols(), cb.ptr(), stream));
    cb.fill(counters, stream);
    return c;
}

inline std::uint64_t flops_dense(std::int64_t m, std::int64_t n, std::int64_t k) { return sd_flops_dense(m, n, k); }

// ---------------------------------------------------------------- layer.hpp

enum class LinearVariant { dense, dropout_dense, sparsedrop };

inline std::uint64_t mix64(std::uint64_t z) {
    z += UINT64_C(0x9E3779B97F4A7C15);
    z = (z ^ (z >> 30)) * UINT64_C(0xBF58476D1CE4E5B9);
    z = (z ^ (z >> 27)) * UINT64_C(0x94D049BB133111EB);
    return z ^ (z >> 31);
}
inline std::uint64_t counter_hash(std::uint64_t seed, std::uint64_t a, std::uint64_t b) {
    return mix64(mix64(mix64(seed) ^ a) ^ b);
}

// layer.hpp:29-47
struct LinearLayer {
    LinearVariant kind = LinearVariant::dense;
    DeviceMatrix<bf16> weight;  // K x N
    DropoutSpec spec;
    TileConfig tiles;
    int layer_index = 0;

    LinearLayer() = default;
    LinearLayer(LinearVariant kind_, DeviceMatrix<bf16> weight_, DropoutSpec spec_, TileConfig tiles_,
                int layer_index_ = 0)
        : kind(kind_), weight(std::move(weight_)), spec(spec_), tiles(tiles_), layer_index(layer_index_) {
        if (kind == LinearVariant::dropout_dense)
            throw std::invalid_argument("dropout_dense is not implemented on the B200 path");
        if (kind == LinearVariant::sparsedrop && (spec.m_blk != tiles.m_blk || spec.k_blk != tiles.k_blk))
            throw std::invalid_argument("sparsedrop mask block sizes must equal the GEMM tile sizes");
    }
};

// layer.hpp:51-58 (the input is referenced, not copied)
struct LayerContext {
    DeviceMatrix<bf16> input;
    std::optional<BlockMask> block_mask;
    bool training = false;
    std::uint64_t step_seed = 0;
};

struct LayerGrads {
    DeviceMatrix<bf16> dx;
    DeviceMatrix<float> dw;
};

namespace detail {
// layer.hpp:64-67, 78-81
inline std::uint64_t effective_seed(const DropoutSpec& spec, std::uint64_t step_seed, int layer_index) {
    return counter_hash(spec.seed, step_seed, static_cast<std::uint64_t>(layer_index));
}
inline float dropout_scale(double p) { return static_cast<float>(1.0 / (1.0 - p)); }
}  // namespace detail

// layer.hpp:85-117
inline std::pair<DeviceMatrix<bf16>, LayerContext> forward(const LinearLayer& layer, const DeviceMatrix<bf16>& x,
                                                           bool train, std::uint64_t step_seed,
                                                           void* stream = nullptr) {
    if (x.cols() != layer.weight.rows())
        throw std::invalid_argument("layer forward: input " + x.shape_string() + " does not match weight " +
                                    layer.weight.shape_string());
    LayerContext ctx;
    ctx.input = x;
    ctx.training = train;
    ctx.step_seed = step_seed;
    if (!train || layer.kind == LinearVariant::dense) return {dense_gemm<bf16>(x, layer.weight, stream), ctx};
    DropoutSpec spec = layer.spec;
    spec.seed = detail::effective_seed(layer.spec, step_seed, layer.layer_index);
    ctx.block_mask = sample_mask(spec, x.rows(), x.cols(), stream);
    DeviceMatrix<bf16> y(x.rows(), layer.weight.cols());
    check(sd_linear_forward(x.data(), ctx.block_mask->c(), layer.weight.data(), detail::dropout_scale(layer.spec.p),
                            y.data(), SD_DTYPE_BF16, x.rows(), layer.weight.cols(), x.cols(), stream));
    return {std::move(y), std::move(ctx)};
}

// layer.hpp:128-162 (no materialised transposes)
inline LayerGrads backward(const LinearLayer& layer, const LayerContext& ctx, const DeviceMatrix<bf16>& dy,
                           void* stream = nullptr) {
    const DeviceMatrix<bf16>& x = ctx.input;
    if (dy.rows() != x.rows() || dy.cols() != layer.weight.cols())
        throw std::invalid_argument("layer backward: dy " + dy.shape_string() + " does not match forward shapes " +
                                    x.shape_string() + " * " + layer.weight.shape_string());
    const int m = x.rows(), k = x.cols(), n = dy.cols();
    LayerGrads g{DeviceMatrix<bf16>(m, k), DeviceMatrix<float>(k, n)};
    if (!ctx.training || layer.kind == LinearVariant::dense || !ctx.block_mask) {
        check(sd_dense_gemm_tn(x.data(), dy.data(), g.dw.data(), SD_DTYPE_F32, k, n, m, stream));
        check(sd_dense_gemm_nt(dy.data(), layer.weight.data(), g.dx.data(), SD_DTYPE_BF16, m, k, n, stream));
        return g;
    }
    const float s = detail::dropout_scale(layer.spec.p);
    check(sd_linear_backward_dw(x.data(), ctx.block_mask->c(), dy.data(), s, g.dw.data(), SD_DTYPE_F32, m, n, k,
                                stream));
    check(sd_linear_backward_dx(dy.data(), layer.weight.data(), ctx.block_mask->c(), s, g.dx.data(), SD_DTYPE_BF16,
                                m, n, k, stream));
    return g;
}

// ---------------------------------------------------------------- runtime objects

// NCCL communicator owned by the library (sd_comm_*): rank 0 makes the id,
// the caller broadcasts its 128 bytes (MPI, a file, a TCP store), every rank
// constructs on its own device.
class Communicator {
public:
    using Id = std::array<unsigned char, SD_COMM_ID_BYTES>;
    static Id unique_id() {
        Id id{};
        check(sd_comm_unique_id(id.data()));
        return id;
    }
    Communicator(int nranks, int rank, const Id& id) {
        sd_comm* c = nullptr;
        check(sd_comm_init(&c, nranks, rank, id.data()));
        c_.reset(c);
    }
    void allreduce_sum(DeviceMatrix<float>& m, void* stream = nullptr) {
        check(sd_comm_allreduce_sum(c_.get(), m.data(), m.size(), SD_DTYPE_F32, stream));
    }
    sd_comm* c() const { return c_.get(); }

private:
    struct Destroy {
        void operator()(sd_comm* c) const { sd_comm_destroy(c); }
    };
    std::unique_ptr<sd_comm, Destroy> c_;
};

// A bound SparseDrop layer (sd_layer_plan): the forward/backward of
// layer.hpp:85-162 on fixed device buffers, tensor maps encoded once — the
// object a training loop keeps per layer. A row shard passes the global block
// row of its first row (row_block_offset) so its mask rows equal the global
// mask's; backward_allreduce then sums the shards' dW.
class LayerPlan {
public:
    LayerPlan(const DeviceMatrix<bf16>& x, const DeviceMatrix<bf16>& w, const DeviceMatrix<bf16>& dy, double p,
              int m_blk = 128, int k_blk = 128, int row_block_offset = 0, bool dy_ready = false)
        : x_(x), w_(w), dy_(dy), y_(x.rows(), w.cols()), dx_(x.rows(), x.cols()), dw_(x.cols(), w.cols()),
          mask_(x.rows() / m_blk, x.cols() / k_blk, m_blk, k_blk, row_block_offset) {
        if (w.rows() != x.cols() || dy.rows() != x.rows() || dy.cols() != w.cols())
            throw std::invalid_argument("layer shapes: x " + x.shape_string() + " w " + w.shape_string() + " dy " +
                                        dy.shape_string());
        sd_layer_plan* pl = nullptr;
        check(sd_layer_plan_create(&pl, x.data(), w.data(), dy.data(), y_.data(), SD_DTYPE_BF16, dx_.data(),
                                   SD_DTYPE_BF16, dw_.data(), SD_DTYPE_F32, x.rows(), w.cols(), x.cols(), p,
                                   mask_.c()));
        plan_.reset(pl);
        if (dy_ready) check(sd_layer_plan_set_options(pl, SD_PLAN_DY_READY));
    }
    void forward(std::uint64_t seed, void* stream = nullptr) { check(sd_layer_plan_forward(plan_.get(), seed, stream)); }
    void backward(void* stream = nullptr) { check(sd_layer_plan_backward(plan_.get(), stream)); }
    void backward_allreduce(Communicator& comm, int nparts = 2, void* stream = nullptr, void* comm_stream = nullptr) {
        check(sd_layer_plan_backward_allreduce(plan_.get(), comm.c(), nparts, stream, comm_stream));
    }
    const DeviceMatrix<bf16>& y() const { return y_; }
    const DeviceMatrix<bf16>& dx() const { return dx_; }
    DeviceMatrix<float>& dw() { return dw_; }
    const BlockMask& mask() const { return mask_; }

private:
    struct Destroy {
        void operator()(sd_layer_plan* p) const { sd_layer_plan_destroy(p); }
    };
    DeviceMatrix<bf16> x_, w_, dy_, y_, dx_;
    DeviceMatrix<float> dw_;
    BlockMask mask_;
    std::unique_ptr<sd_layer_plan, Destroy> plan_;
};

}  // namespace sparsedrop::b200
