// C++ drop-in test: the reference's own test cases (proj/tests/test_block_mask.cpp,
// test_gemm.cpp), restated against the B200 C++ API (include/sparsedrop_b200.hpp)
// and run on the GPU through the C-ABI. Built by __graft_entry__.build() into
// tests/cpp/build/, run by tests/test_cpp_api.py (-m gpu). Uses the same
// doctest subset as the reference (oracle/doctest_shim).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "sparsedrop_b200.hpp"

using namespace sparsedrop::b200;

namespace {

DropoutSpec spec_of(double p, int m_blk, int k_blk, std::uint64_t seed) {
    DropoutSpec s;
    s.p = p;
    s.m_blk = m_blk;
    s.k_blk = k_blk;
    s.seed = seed;
    return s;
}

double unit_interval(std::uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

// tests/oracles.hpp:31-41
std::vector<float> random_matrix(int rows, int cols, std::uint64_t seed) {
    std::vector<float> m(static_cast<std::size_t>(rows) * cols);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) {
            const std::uint64_t bits = counter_hash(seed, i, j);
            const double mag = 0.25 + unit_interval(bits);
            m[static_cast<std::size_t>(i) * cols + j] = static_cast<float>((bits & 1) ? mag : -mag);
        }
    return m;
}

std::vector<double> bf16_round(const std::vector<float>& v) {
    std::vector<double> out(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = bf16::from_float(v[i]).to_float();
    return out;
}

bool kept_host(const std::vector<std::uint64_t>& w, int C, int r, int c) {
    const std::uint64_t b = static_cast<std::uint64_t>(r) * C + c;
    return (w[b >> 6] >> (b & 63)) & 1u;
}

// scale * (a (.) m) b in double, a: m x k
std::vector<double> masked_matmul(const std::vector<double>& a, const std::vector<std::uint64_t>& w, int C,
                                  int m_blk, int k_blk, const std::vector<double>& b, int m, int n, int k,
                                  double scale) {
    std::vector<double> c(static_cast<std::size_t>(m) * n, 0.0);
    for (int i = 0; i < m; ++i)
        for (int kk = 0; kk < k; ++kk) {
            if (!kept_host(w, C, i / m_blk, kk / k_blk)) continue;
            const double aik = a[static_cast<std::size_t>(i) * k + kk];
            for (int j = 0; j < n; ++j) c[static_cast<std::size_t>(i) * n + j] += aik * b[static_cast<std::size_t>(kk) * n + j];
        }
    for (auto& v : c) v *= scale;
    return c;
}

double rel_frob(const std::vector<float>& got, const std::vector<double>& want) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < got.size(); ++i) {
        num += (got[i] - want[i]) * (got[i] - want[i]);
        den += want[i] * want[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1));
}

}  // namespace

// test_block_mask.cpp:27-33
TEST_CASE("sample_mask p=0 keeps everything") {
    auto m = sample_mask(spec_of(0.0, 128, 128, 123), 512, 1024);
    CHECK(m.block_rows() == 4);
    CHECK(m.block_cols() == 8);
    CHECK(m.keep_count() == 32);
    CHECK(m.realized_sparsity() == 0.0);
}

// test_block_mask.cpp:35-41
TEST_CASE("sample_mask is deterministic") {
    auto spec = spec_of(0.4, 128, 128, 99);
    auto a = sample_mask(spec, 8192, 8192);
    auto b = sample_mask(spec, 8192, 8192);
    CHECK(a.words() == b.words());
    CHECK(a.keep_count() == b.keep_count());
}

// test_block_mask.cpp:43-50
TEST_CASE("sample_mask validates arguments") {
    CHECK_THROWS_WITH_AS(sample_mask(spec_of(0.5, 3, 4, 0), 16, 16), doctest::Contains("m_blk"),
                         std::invalid_argument);
    CHECK_THROWS_WITH_AS(sample_mask(spec_of(0.5, 4, 5, 0), 16, 16), doctest::Contains("k_blk"),
                         std::invalid_argument);
    CHECK_THROWS_AS(sample_mask(spec_of(1.0, 4, 4, 0), 16, 16), std::invalid_argument);
    CHECK_THROWS_AS(sample_mask(spec_of(-0.1, 4, 4, 0), 16, 16), std::invalid_argument);
}

// test_block_mask.cpp:52-66 (1000 seeds, 32 x 32 grid, 3 sigma)
TEST_CASE("sample_mask keep fraction is unbiased over many seeds") {
    const double p = 0.5;
    std::int64_t kept = 0, total = 0;
    for (int s = 0; s < 1000; ++s) {
        auto m = sample_mask(spec_of(p, 1, 1, s), 32, 32);
        kept += m.keep_count();
        total += m.total_blocks();
    }
    const double mean_keep = double(kept) / double(total);
    const double sigma = std::sqrt(p * (1 - p) / double(total));
    CHECK(std::abs(mean_keep - (1 - p)) < 3 * sigma);
}

// the device draw equals the reference formula bit for bit
TEST_CASE("sample_mask bits equal the splitmix64 counter hash") {
    auto m = sample_mask(spec_of(0.3, 128, 128, 77), 128 * 13, 128 * 70);
    const auto w = m.words();
    for (int r = 0; r < 13; ++r)
        for (int c = 0; c < 70; ++c)
            CHECK(kept_host(w, 70, r, c) == (unit_interval(counter_hash(77, r, c)) >= 0.3));
    auto one = sample_mask(spec_of(0.5, 128, 128, 0), 1024, 1024);
    CHECK(one.words() == std::vector<std::uint64_t>{UINT64_C(0xe43d829a90c95084)});
}

// test_block_mask.cpp:127-152
TEST_CASE("transpose_mask is an involution") {
    auto m = sample_mask(spec_of(0.45, 128, 256, 13), 128 * 12, 256 * 9);
    auto t = transpose_mask(m);
    CHECK(t.block_rows() == 9);
    CHECK(t.block_cols() == 12);
    CHECK(t.m_blk() == 256);
    CHECK(t.k_blk() == 128);
    CHECK(transpose_mask(t).words() == m.words());
    const auto w = m.words(), wt = t.words();
    for (int r = 0; r < 12; ++r)
        for (int c = 0; c < 9; ++c) CHECK(kept_host(w, 9, r, c) == kept_host(wt, 12, c, r));
}

// test_block_mask.cpp:89-125
TEST_CASE("retile replicates each bit") {
    auto m = sample_mask(spec_of(0.5, 256, 256, 6), 2048, 2048);
    auto r = retile(m, 2, 1);
    CHECK(r.m_blk() == 128);
    CHECK(r.k_blk() == 256);
    CHECK(r.block_rows() == 2 * m.block_rows());
    CHECK(r.keep_count() == 2 * m.keep_count());
    const auto w = m.words(), rw = r.words();
    for (int br = 0; br < r.block_rows(); ++br)
        for (int bc = 0; bc < r.block_cols(); ++bc) CHECK(kept_host(rw, 8, br, bc) == kept_host(w, 8, br / 2, bc));
    CHECK_THROWS_AS(retile(m, 3, 1), std::invalid_argument);
    CHECK_THROWS_AS(retile(m, 1, 5), std::invalid_argument);
}

// test_block_mask.cpp:154-172
TEST_CASE("kept_blocks_in_row") {
    auto all = sample_mask(spec_of(0.0, 128, 128, 0), 1024, 768);
    CHECK(kept_blocks_in_row(all, 2) == std::vector<int>{0, 1, 2, 3, 4, 5});
    std::vector<std::uint64_t> w(1, 0);
    w[0] = std::uint64_t(1) << (1 * 4 + 3);  // grid 2 x 4, only (1, 3) kept
    auto empty_row = mask_from_words(2, 4, 128, 128, w);
    CHECK(kept_blocks_in_row(empty_row, 0).empty());
    CHECK(kept_blocks_in_row(empty_row, 1) == std::vector<int>{3});
    CHECK_THROWS_AS(kept_blocks_in_row(all, 8), std::out_of_range);
    auto m = sample_mask(spec_of(0.5, 128, 128, 31), 128 * 20, 128 * 20);
    const auto mw = m.words();
    for (int r = 0; r < 20; ++r) {
        std::vector<int> expected;
        for (int c = 0; c < 20; ++c)
            if (kept_host(mw, 20, r, c)) expected.push_back(c);
        CHECK(kept_blocks_in_row(m, r) == expected);
    }
}

// test_block_mask.cpp:247-253
TEST_CASE("mask_from_words rejects nonzero padding bits") {
    std::vector<std::uint64_t> words{~std::uint64_t(0)};
    CHECK_THROWS_AS(mask_from_words(3, 3, 128, 128, words), std::invalid_argument);
    std::vector<std::uint64_t> ok{(std::uint64_t(1) << 9) - 1};
    CHECK(mask_from_words(3, 3, 128, 128, ok).keep_count() == 9);
}

// test_gemm.cpp:57-68
TEST_CASE("dense_gemm validates shapes and divisibility") {
    auto a = DeviceMatrix<bf16>::from_host(256, 256, random_matrix(256, 256, 8));
    auto b = DeviceMatrix<bf16>::from_host(384, 256, random_matrix(384, 256, 9));
    CHECK_THROWS_WITH_AS(dense_gemm(a, b), doctest::Contains("gemm shape mismatch"), std::invalid_argument);
    auto c = DeviceMatrix<bf16>::from_host(100, 256, random_matrix(100, 256, 9));
    CHECK_THROWS_WITH_AS(dense_gemm(c, a), doctest::Contains("m_blk"), std::invalid_argument);
}

// test_gemm.cpp:70-80
TEST_CASE("dsd_matmul all-set equals dense, all-clear is zero") {
    const int M = 512, N = 384, K = 512;
    auto a = DeviceMatrix<bf16>::from_host(M, K, random_matrix(M, K, 1));
    auto b = DeviceMatrix<bf16>::from_host(K, N, random_matrix(K, N, 2));
    auto all = sample_mask(spec_of(0.0, 128, 128, 0), M, K);
    CHECK(dsd_matmul<float>(a, all, b, 1.0f).to_host() == dense_gemm<float>(a, b).to_host());
    auto none = mask_from_words(4, 4, 128, 128, std::vector<std::uint64_t>{0});
    KernelCounters kc;
    auto z = dsd_matmul<float>(a, none, b, 2.0f, &kc).to_host();
    for (float v : z) CHECK(v == 0.0f);
    CHECK(kc.kblock_iterations == 0);
}

// test_gemm.cpp:82-104 (tolerance instead of bitwise: bf16 inputs, fp32 accumulate)
TEST_CASE("dsd_matmul matches the masked dense oracle; work counter") {
    const int M = 512, N = 256, K = 1024;
    const auto ah = random_matrix(M, K, 1), bh = random_matrix(K, N, 2);
    auto a = DeviceMatrix<bf16>::from_host(M, K, ah);
    auto b = DeviceMatrix<bf16>::from_host(K, N, bh);
    auto mask = sample_mask(spec_of(0.5, 128, 128, 3), M, K);
    KernelCounters kc;
    auto got = dsd_matmul<float>(a, mask, b, 2.0f, &kc).to_host();
    const auto want = masked_matmul(bf16_round(ah), mask.words(), K / 128, 128, 128, bf16_round(bh), M, N, K, 2.0);
    CHECK(rel_frob(got, want) < 1e-5);
    CHECK(kc.kblock_iterations == static_cast<std::uint64_t>(N / 128) * mask.keep_count());
}

// test_gemm.cpp:116-152
TEST_CASE("sdd_matmul: masked output, exact zeros, counters") {
    const int M = 512, N = 512, K = 384;
    const auto ah = random_matrix(M, K, 4), bh = random_matrix(K, N, 5);
    auto a = DeviceMatrix<bf16>::from_host(M, K, ah);
    auto b = DeviceMatrix<bf16>::from_host(K, N, bh);
    auto mask = sample_mask(spec_of(0.5, 128, 128, 6), M, N);
    KernelCounters kc;
    auto got = sdd_matmul<float>(a, b, mask, 1.5f, &kc).to_host();
    std::vector<double> full(static_cast<std::size_t>(M) * N, 0.0);
    const auto ad = bf16_round(ah), bd = bf16_round(bh);
    for (int i = 0; i < M; ++i)
        for (int kk = 0; kk < K; ++kk)
            for (int j = 0; j < N; ++j) full[static_cast<std::size_t>(i) * N + j] += ad[static_cast<std::size_t>(i) * K + kk] * bd[static_cast<std::size_t>(kk) * N + j];
    const auto w = mask.words();
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            auto& v = full[static_cast<std::size_t>(i) * N + j];
            v = kept_host(w, N / 128, i / 128, j / 128) ? 1.5 * v : 0.0;
        }
    CHECK(rel_frob(got, full) < 1e-5);
    bool zeros_exact = true;
    for (std::size_t i = 0; i < got.size(); ++i)
        if ((full[i] == 0.0) != (got[i] == 0.0f) || std::signbit(got[i]) != std::signbit(full[i])) zeros_exact = false;
    CHECK(zeros_exact);
    CHECK(kc.kblock_iterations == static_cast<std::uint64_t>(K / 128) * mask.keep_count());
}

// test_gemm.cpp:199-213
TEST_CASE("a fully dropped mask row yields a zero output row") {
    const int M = 384, N = 256, K = 256;
    std::vector<std::uint64_t> w{0};
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 2; ++c)
            if (r != 1) w[0] |= std::uint64_t(1) << (r * 2 + c);
    auto mask = mask_from_words(3, 2, 128, 128, w);
    auto a = DeviceMatrix<bf16>::from_host(M, K, random_matrix(M, K, 1));
    auto b = DeviceMatrix<bf16>::from_host(K, N, random_matrix(K, N, 2));
    auto c = dsd_matmul<float>(a, mask, b, 2.0f).to_host();
    bool row_zero = true, others_nonzero = true;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            const float v = c[static_cast<std::size_t>(i) * N + j];
            if (i / 128 == 1 && (v != 0.0f || std::signbit(v))) row_zero = false;
            if (i / 128 != 1 && v == 0.0f) others_nonzero = false;
        }
    CHECK(row_zero);
    CHECK(others_nonzero);
}

// layer.hpp:85-162 forward + backward vs the double oracle
TEST_CASE("layer forward/backward (sparsedrop) match the oracle") {
    const int M = 384, N = 256, K = 512;
    const double p = 0.4;
    const auto xh = random_matrix(M, K, 1), wh = random_matrix(K, N, 2), dyh = random_matrix(M, N, 3);
    LinearLayer layer(LinearVariant::sparsedrop, DeviceMatrix<bf16>::from_host(K, N, wh), spec_of(p, 128, 128, 4),
                      TileConfig{128, 128, 128}, 1);
    auto x = DeviceMatrix<bf16>::from_host(M, K, xh);
    auto dy = DeviceMatrix<bf16>::from_host(M, N, dyh);
    auto [y, ctx] = forward(layer, x, true, 9);
    auto g = backward(layer, ctx, dy);
    REQUIRE(ctx.block_mask.has_value());
    const auto w = ctx.block_mask->words();
    const double s = static_cast<float>(1.0 / (1.0 - p));
    const auto xd = bf16_round(xh), wd = bf16_round(wh), dyd = bf16_round(dyh);
    CHECK(rel_frob(y.to_host(), masked_matmul(xd, w, K / 128, 128, 128, wd, M, N, K, s)) < 4e-3);
    std::vector<double> dx(static_cast<std::size_t>(M) * K, 0.0), dw(static_cast<std::size_t>(K) * N, 0.0);
    for (int i = 0; i < M; ++i)
        for (int kk = 0; kk < K; ++kk) {
            if (!kept_host(w, K / 128, i / 128, kk / 128)) continue;
            double acc = 0;
            for (int j = 0; j < N; ++j) acc += dyd[static_cast<std::size_t>(i) * N + j] * wd[static_cast<std::size_t>(kk) * N + j];
            dx[static_cast<std::size_t>(i) * K + kk] = s * acc;
            for (int j = 0; j < N; ++j)
                dw[static_cast<std::size_t>(kk) * N + j] += s * xd[static_cast<std::size_t>(i) * K + kk] * dyd[static_cast<std::size_t>(i) * N + j];
        }
    CHECK(rel_frob(g.dx.to_host(), dx) < 4e-3);
    CHECK(rel_frob(g.dw.to_host(), dw) < 1e-5);
    CHECK_THROWS_AS(backward(layer, ctx, x), std::invalid_argument);
}

// SURVEY §8e through the C++ API: two row shards of one layer, each with its own
// plan (row_block_offset = its first global block row) — their masks are the
// global mask's rows, and the sum of their dW (what the NCCL all-reduce forms on
// G GPUs) equals the unsharded dW within fp32 reassociation. backward_allreduce
// runs on a 1-rank communicator (one GPU here): the identity, so it must equal
// the plain backward bit for bit.
TEST_CASE("row-sharded layer plans and the dW all-reduce") {
    const int M = 512, N = 256, K = 384;
    const double p = 0.4;
    const auto xh = random_matrix(M, K, 11), wh = random_matrix(K, N, 12), dyh = random_matrix(M, N, 13);
    auto x = DeviceMatrix<bf16>::from_host(M, K, xh), w = DeviceMatrix<bf16>::from_host(K, N, wh);
    auto dy = DeviceMatrix<bf16>::from_host(M, N, dyh);
    LayerPlan full(x, w, dy, p);
    full.forward(77);
    full.backward();
    const auto dw_full = full.dw().to_host();
    const auto words_full = full.mask().words();
    std::vector<double> dw_sum(static_cast<std::size_t>(K) * N, 0.0);
    Communicator comm(1, 0, Communicator::unique_id());
    for (int shard = 0; shard < 2; ++shard) {
        const int r0 = shard * M / 2;
        std::vector<float> xs(xh.begin() + static_cast<std::ptrdiff_t>(r0) * K,
                              xh.begin() + static_cast<std::ptrdiff_t>(r0 + M / 2) * K);
        std::vector<float> dys(dyh.begin() + static_cast<std::ptrdiff_t>(r0) * N,
                               dyh.begin() + static_cast<std::ptrdiff_t>(r0 + M / 2) * N);
        auto xg = DeviceMatrix<bf16>::from_host(M / 2, K, xs), dyg = DeviceMatrix<bf16>::from_host(M / 2, N, dys);
        LayerPlan part(xg, w, dyg, p, 128, 128, r0 / 128);
        part.forward(77);
        part.backward();
        const auto dw_plain = part.dw().to_host();
        const auto ws = part.mask().words();
        for (int r = 0; r < M / 256; ++r)
            for (int c = 0; c < K / 128; ++c)
                CHECK(kept_host(ws, K / 128, r, c) == kept_host(words_full, K / 128, r0 / 128 + r, c));
        part.forward(77);
        part.backward_allreduce(comm, 3);
        CHECK(part.dw().to_host() == dw_plain);  // 1-rank all-reduce: identity, slabs bit-identical
        for (std::size_t i = 0; i < dw_sum.size(); ++i) dw_sum[i] += dw_plain[i];
    }
    CHECK(rel_frob(dw_full, dw_sum) < 1e-6);
}
