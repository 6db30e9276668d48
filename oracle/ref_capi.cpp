// oracle/_ref C shim — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Thin extern "C" entry points over the UNMODIFIED reference implementation,
// compiled from the sources where they lie under /root/reference/proj by
// oracle/Makefile into oracle/_ref/libsdref.so. Only tests/, bench.py's
// cpu_baseline / --impl reference leg and __graft_entry__.smoke() load it.
//
// Each wrapper calls the reference symbol named in its comment; the reference's
// exceptions are mapped to the same status codes the B200 C-ABI uses
// (include/sparsedrop_b200.h) so parity tests can compare error behaviour too.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracles.hpp"              // /root/reference/proj/tests/oracles.hpp
#include "sparsedrop/block_mask.hpp"
#include "sparsedrop/gemm.hpp"
#include "sparsedrop/layer.hpp"
#include "sparsedrop/rng.hpp"

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

sparsedrop::DropoutSpec make_spec(double p, int m_blk, int k_blk, uint64_t seed) {
    sparsedrop::DropoutSpec s;
    s.p = p;
    s.m_blk = m_blk;
    s.k_blk = k_blk;
    s.seed = seed;
    return s;
}

std::size_t word_count(int r, int c) { return (static_cast<std::size_t>(r) * c + 63) / 64; }

sparsedrop::BlockMask mask_of(const uint64_t* words, int br, int bc, int m_blk, int k_blk) {
    return sparsedrop::mask_from_words(br, bc, m_blk, k_blk,
                                       std::vector<uint64_t>(words, words + word_count(br, bc)));
}

template <typename T>
sparsedrop::Matrix<T> mat(const T* p, int r, int c) {
    return sparsedrop::Matrix<T>(r, c, std::vector<T>(p, p + static_cast<std::size_t>(r) * c));
}

template <typename T>
void out(const sparsedrop::Matrix<T>& m, T* dst) {
    std::memcpy(dst, m.data(), m.size() * sizeof(T));
}

}  // namespace

extern "C" {

const char* sdref_last_error(void) { return g_err.c_str(); }

// rng.hpp:11-16 / :18-20
uint64_t sdref_mix64(uint64_t z) { return sparsedrop::mix64(z); }
uint64_t sdref_counter_hash(uint64_t seed, uint64_t a, uint64_t b) {
    return sparsedrop::counter_hash(seed, a, b);
}
// layer.hpp:64-67
uint64_t sdref_effective_seed(uint64_t seed, uint64_t step_seed, int layer_index) {
    sparsedrop::DropoutSpec s;
    s.seed = seed;
    return sparsedrop::detail::effective_seed(s, step_seed, layer_index);
}
// layer.hpp:78-81
float sdref_dropout_scale_f32(double p) { return sparsedrop::detail::dropout_scale<float>(p); }

// block_mask.cpp:52-80  sample_mask(spec, rows, cols)
int sdref_sample_mask(double p, int m_blk, int k_blk, uint64_t seed, int rows, int cols,
                      uint64_t* words, int64_t nwords_cap, int64_t* keep_count) {
    return guarded([&] {
        auto m = sparsedrop::sample_mask(make_spec(p, m_blk, k_blk, seed), rows, cols);
        if (static_cast<int64_t>(m.words().size()) > nwords_cap)
            throw std::runtime_error("sdref_sample_mask: words buffer too small");
        std::memcpy(words, m.words().data(), m.words().size() * sizeof(uint64_t));
        *keep_count = m.keep_count();
    });
}

// block_mask.cpp:82-98  mask_from_words (validation only)
int sdref_mask_from_words(int br, int bc, int m_blk, int k_blk, const uint64_t* words,
                          int64_t nwords, int64_t* keep_count) {
    return guarded([&] {
        auto m = sparsedrop::mask_from_words(br, bc, m_blk, k_blk,
                                             std::vector<uint64_t>(words, words + nwords));
        *keep_count = m.keep_count();
    });
}

// block_mask.cpp:125-135  kept_blocks_in_row
int sdref_kept_blocks_in_row(const uint64_t* words, int br, int bc, int m_blk, int k_blk, int row,
                             int32_t* idx_out, int32_t* n_out) {
    return guarded([&] {
        auto v = sparsedrop::kept_blocks_in_row(mask_of(words, br, bc, m_blk, k_blk), row);
        for (std::size_t i = 0; i < v.size(); ++i) idx_out[i] = v[i];
        *n_out = static_cast<int32_t>(v.size());
    });
}

// block_mask.cpp:117-123  transpose_mask
int sdref_transpose_mask(const uint64_t* words, int br, int bc, int m_blk, int k_blk,
                         uint64_t* out_words) {
    return guarded([&] {
        auto t = sparsedrop::transpose_mask(mask_of(words, br, bc, m_blk, k_blk));
        std::memcpy(out_words, t.words().data(), t.words().size() * sizeof(uint64_t));
    });
}

// block_mask.cpp:100-115  retile
int sdref_retile(const uint64_t* words, int br, int bc, int m_blk, int k_blk, int split_m,
                 int split_k, uint64_t* out_words) {
    return guarded([&] {
        auto t = sparsedrop::retile(mask_of(words, br, bc, m_blk, k_blk), split_m, split_k);
        std::memcpy(out_words, t.words().data(), t.words().size() * sizeof(uint64_t));
    });
}

// tests/oracles.hpp:31-41  random_matrix<float>
void sdref_random_matrix_f32(int rows, int cols, uint64_t seed, float* dst) {
    out(sparsedrop::testing::random_matrix<float>(rows, cols, seed), dst);
}

// gemm.hpp:104-128  dense_gemm
#define SDREF_DENSE(T, suffix)                                                                   \
    int sdref_dense_gemm_##suffix(const T* a, const T* b, int m, int n, int k, int m_blk,       \
                                  int n_blk, int k_blk, int threads, T* c) {                    \
        return guarded([&] {                                                                     \
            out(sparsedrop::dense_gemm(mat(a, m, k), mat(b, k, n),                               \
                                       sparsedrop::TileConfig{m_blk, n_blk, k_blk}, threads),   \
                c);                                                                              \
        });                                                                                      \
    }
SDREF_DENSE(float, f32)
SDREF_DENSE(double, f64)

// gemm.hpp:133-170  dsd_matmul (mask on a: grid (m/m_blk, k/k_blk))
#define SDREF_DSD(T, suffix)                                                                     \
    int sdref_dsd_matmul_##suffix(const T* a, const uint64_t* words, const T* b, int m, int n,  \
                                  int k, int m_blk, int n_blk, int k_blk, T scale, int threads, \
                                  T* c, uint64_t* kblock_per_tile_row) {                         \
        return guarded([&] {                                                                     \
            sparsedrop::KernelCounters kc;                                                       \
            auto r = sparsedrop::dsd_matmul(                                                     \
                mat(a, m, k), mask_of(words, m / m_blk, k / k_blk, m_blk, k_blk), mat(b, k, n), \
                scale, sparsedrop::TileConfig{m_blk, n_blk, k_blk}, &kc, threads);               \
            out(r, c);                                                                           \
            if (kblock_per_tile_row)                                                             \
                for (std::size_t i = 0; i < kc.kblock_per_tile_row.size(); ++i)                  \
                    kblock_per_tile_row[i] = kc.kblock_per_tile_row[i];                          \
        });                                                                                      \
    }
SDREF_DSD(float, f32)
SDREF_DSD(double, f64)

// gemm.hpp:176-213  sdd_matmul (mask on the output: grid (m/m_blk, n/n_blk))
#define SDREF_SDD(T, suffix)                                                                     \
    int sdref_sdd_matmul_##suffix(const T* a, const T* b, const uint64_t* words, int m, int n,  \
                                  int k, int m_blk, int n_blk, int k_blk, T scale, int threads, \
                                  T* c, uint64_t* kblock_per_tile_row) {                         \
        return guarded([&] {                                                                     \
            sparsedrop::KernelCounters kc;                                                       \
            auto r = sparsedrop::sdd_matmul(                                                     \
                mat(a, m, k), mat(b, k, n), mask_of(words, m / m_blk, n / n_blk, m_blk, n_blk), \
                scale, sparsedrop::TileConfig{m_blk, n_blk, k_blk}, &kc, threads);               \
            out(r, c);                                                                           \
            if (kblock_per_tile_row)                                                             \
                for (std::size_t i = 0; i < kc.kblock_per_tile_row.size(); ++i)                  \
                    kblock_per_tile_row[i] = kc.kblock_per_tile_row[i];                          \
        });                                                                                      \
    }
SDREF_SDD(float, f32)
SDREF_SDD(double, f64)

// layer.hpp:85-117 forward(train=true) + layer.hpp:128-162 backward, sparsedrop variant.
// x: m x k, w: k x n, dy: m x n. Outputs y (m x n), dx (m x k), dw (k x n) and the mask words
// (grid m/m_blk x k/k_blk) that forward sampled.
#define SDREF_LAYER(T, suffix)                                                                   \
    int sdref_layer_fwd_bwd_##suffix(const T* x, const T* w, const T* dy, int m, int n, int k,   \
                                     double p, int m_blk, int k_blk, int n_blk, uint64_t seed,   \
                                     uint64_t step_seed, int layer_index, int threads, T* y,     \
                                     T* dx, T* dw, uint64_t* mask_words) {                       \
        return guarded([&] {                                                                     \
            sparsedrop::LinearLayer<T> layer(sparsedrop::LinearVariant::sparsedrop, mat(w, k, n), \
                                             make_spec(p, m_blk, k_blk, seed),                   \
                                             sparsedrop::TileConfig{m_blk, n_blk, k_blk},        \
                                             layer_index);                                       \
            auto fw = sparsedrop::forward(layer, mat(x, m, k), true, step_seed, threads);        \
            if (y) out(fw.first, y);                                                             \
            if (mask_words)                                                                      \
                std::memcpy(mask_words, fw.second.block_mask->words().data(),                    \
                            fw.second.block_mask->words().size() * sizeof(uint64_t));            \
            if (dx || dw) {                                                                      \
                auto g = sparsedrop::backward(layer, fw.second, mat(dy, m, n), threads);         \
                if (dx) out(g.dx, dx);                                                           \
                if (dw) out(g.dw, dw);                                                           \
            }                                                                                    \
        });                                                                                      \
    }
SDREF_LAYER(float, f32)
SDREF_LAYER(double, f64)

// layer.hpp:69-76, 105-111, 148-156: the dropout_dense variant (element mask), double.
int sdref_dropout_dense_fwd_bwd_f64(const double* x, const double* w, const double* dy, int m, int n, int k,
                                    double p, uint64_t seed, uint64_t step_seed, int layer_index, int threads,
                                    double* y, double* dx, double* dw) {
    return guarded([&] {
        sparsedrop::LinearLayer<double> layer(sparsedrop::LinearVariant::dropout_dense, mat(w, k, n),
                                              make_spec(p, 1, 1, seed), sparsedrop::TileConfig{32, 32, 32},
                                              layer_index);
        auto fw = sparsedrop::forward(layer, mat(x, m, k), true, step_seed, threads);
        if (y) out(fw.first, y);
        auto g = sparsedrop::backward(layer, fw.second, mat(dy, m, n), threads);
        if (dx) out(g.dx, dx);
        if (dw) out(g.dw, dw);
    });
}

// block_mask.cpp:137-219  write_mask / read_mask (BMSK container)
int sdref_write_mask(const uint64_t* words, int br, int bc, int m_blk, int k_blk, unsigned char* out,
                     int64_t cap, int64_t* n_out) {
    return guarded([&] {
        std::ostringstream os;
        sparsedrop::write_mask(mask_of(words, br, bc, m_blk, k_blk), os);
        const std::string b = os.str();
        if (static_cast<int64_t>(b.size()) > cap) throw std::runtime_error("sdref_write_mask: buffer too small");
        std::memcpy(out, b.data(), b.size());
        *n_out = static_cast<int64_t>(b.size());
    });
}

int sdref_read_mask(const unsigned char* bytes, int64_t n, int* geom4, uint64_t* words, int64_t cap) {
    return guarded([&] {
        std::istringstream is(std::string(reinterpret_cast<const char*>(bytes), static_cast<std::size_t>(n)));
        auto m = sparsedrop::read_mask(is, "buffer");
        geom4[0] = m.block_rows();
        geom4[1] = m.block_cols();
        geom4[2] = m.m_blk();
        geom4[3] = m.k_blk();
        if (static_cast<int64_t>(m.words().size()) > cap) throw std::runtime_error("sdref_read_mask: buffer too small");
        std::memcpy(words, m.words().data(), m.words().size() * 8);
    });
}

// gemm.hpp:217-228
uint64_t sdref_flops_dense(int64_t m, int64_t n, int64_t k) { return sparsedrop::flops_dense(m, n, k); }

}  // extern "C"
