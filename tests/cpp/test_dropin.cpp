// C++ parity test of the drop-in krplev::KrpSampler (include/krplev/*.hpp over
// libkrpg.so) against the CPU oracle restatement (oracle/krp_oracle.h), in the
// style of the reference's test_krp_sampler.cpp. Built and run by
// tests/test_cpp_dropin.py (gpu marker); compile-only on CPU boxes.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <optional>
#include <string>
#include <vector>

#include "krp_oracle.h"
#include "krplev/krp_sampler.hpp"
#include "krplev/segment_tree_sampler.hpp"

using namespace krplev;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                               \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(cond)) {                                                            \
            ++g_fail;                                                             \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                         \
    } while (0)
#define CHECK_THROWS_AS(expr, type)       \
    do {                                  \
        bool thrown = false;              \
        try {                             \
            (void)(expr);                 \
        } catch (const type&) {           \
            thrown = true;                \
        } catch (...) {                   \
        }                                 \
        CHECK(thrown);                    \
    } while (0)

static Matrix random_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed) {
    Matrix m(rows, cols);
    CounterRng rng(seed, 0);
    for (double& v : m.data) v = rng.normal();
    return m;
}

// bit-exact indices except draws within 1e-10 of a threshold (either side's margin)
static void compare_with_oracle(const std::vector<Matrix>& fs, std::optional<std::size_t> excluded, std::size_t J,
                                std::uint64_t seed) {
    const KrpSampler s(fs);
    const SampleBatch b = s.sample(excluded, J, seed, KrpSampler::Mode::TwoStage, 0, true);
    std::vector<const double*> ptrs;
    std::vector<std::uint64_t> I;
    for (const Matrix& f : fs) {
        ptrs.push_back(f.data.data());
        I.push_back(f.rows);
    }
    ko_krp* o = nullptr;
    CHECK(ko_krp_create(ptrs.data(), I.data(), uint32_t(fs.size()), uint32_t(fs[0].cols), &o) == 0);
    const std::size_t N = fs.size(), R = fs[0].cols;
    std::vector<uint32_t> idx(J * N);
    std::vector<double> prob(J), rows(J * R), margin(J);
    CHECK(ko_krp_sample(o, excluded ? int64_t(*excluded) : -1, J, seed, 0, idx.data(), prob.data(), rows.data(),
                        margin.data()) == 0);
    std::size_t mism = 0, unexplained = 0;
    double perr = 0.0;
    for (std::size_t d = 0; d < J; ++d) {
        bool same = true;
        for (std::size_t k = 0; k < N; ++k) same &= b.index(d, k) == idx[d * N + k];
        if (!same) {
            ++mism;
            if (std::min(b.margin[d], margin[d]) > 1e-10) ++unexplained;
            continue;
        }
        perr = std::max(perr, std::abs(b.probabilities[d] - prob[d]) / std::abs(prob[d]));
    }
    CHECK(unexplained == 0);
    CHECK(perr <= 1e-10);
    std::printf("  compare N=%zu J=%zu excluded=%d: %zu mismatches (boundary), prob rel err %.2e\n", N, J,
                excluded ? int(*excluded) : -1, mism, perr);
    ko_krp_destroy(o);
}

int main() {
    // construct caches factor Grams (test_krp_sampler.cpp:63-80)
    {
        const KrpSampler s({Matrix::ones(2, 1), Matrix::ones(2, 1)});
        CHECK(std::abs(s.factor_gram(0)(0, 0) - 2.0) < 1e-12);
        CHECK_THROWS_AS(KrpSampler({Matrix::ones(2, 1), Matrix::ones(2, 2)}), std::invalid_argument);
        CHECK_THROWS_AS(KrpSampler({Matrix(2, 2), Matrix(2, 2)}), std::invalid_argument);
        CHECK_THROWS_AS(KrpSampler(std::vector<Matrix>{}), std::invalid_argument);
    }
    // bit-exact parity with the oracle, every exclusion setting
    {
        std::vector<Matrix> fs;
        for (int j = 0; j < 3; ++j) fs.push_back(random_matrix(2000 + 97 * j, 16, 900 + j));
        for (std::optional<std::size_t> e : {std::optional<std::size_t>(), std::optional<std::size_t>(0),
                                             std::optional<std::size_t>(1), std::optional<std::size_t>(2)})
            compare_with_oracle(fs, e, 4096, 17);
        std::vector<Matrix> gs;
        for (int j = 0; j < 3; ++j) gs.push_back(random_matrix(3001 + 13 * j, 64, 910 + j));
        compare_with_oracle(gs, std::nullopt, 4096, 18);
    }
    // exclusion consistency (test_krp_sampler.cpp:233-247)
    {
        std::vector<Matrix> fs;
        for (int j = 0; j < 3; ++j) fs.push_back(random_matrix(9, 3, 740 + j));
        const KrpSampler full(fs);
        const KrpSampler reduced({fs[0], fs[2]});
        const SampleBatch a = full.sample(1, 500, 741);
        const SampleBatch b = reduced.sample(std::nullopt, 500, 741);
        bool same = true;
        for (std::size_t d = 0; d < 500; ++d) same &= a.index(d, 0) == b.index(d, 0) && a.index(d, 2) == b.index(d, 1);
        CHECK(same);
        CHECK(a.index(0, 1) == SampleBatch::kExcluded);
    }
    // update_factor / update_factor_entry (test_krp_sampler.cpp:249-306)
    {
        std::vector<Matrix> fs;
        for (int j = 0; j < 3; ++j) fs.push_back(random_matrix(8, 4, 750 + j));
        KrpSampler s(fs);
        const Matrix unew = random_matrix(8, 4, 753);
        s.update_factor(2, unew);
        fs[2] = unew;
        const KrpSampler fresh(fs);
        CHECK(s.sample(std::nullopt, 300, 754).indices == fresh.sample(std::nullopt, 300, 754).indices);
        s.update_factor_entry(0, 4, 1, -2.5);
        CHECK(s.factor(0)(4, 1) == -2.5);
        s.validate();
        CHECK_THROWS_AS(s.update_factor_entry(0, 8, 0, 1.0), std::invalid_argument);
        CHECK_THROWS_AS(s.sample(std::nullopt, 0, 1), std::invalid_argument);
        CHECK_THROWS_AS(s.sample(3, 10, 1), std::invalid_argument);
    }
    // flat index + rows are Hadamard products (test_krp_sampler.cpp:308-333)
    {
        std::vector<Matrix> fs{random_matrix(2, 2, 770), random_matrix(3, 2, 771), random_matrix(4, 2, 772)};
        const KrpSampler s(fs);
        const SampleBatch b = s.sample(std::nullopt, 50, 773);
        bool ok = true;
        for (std::size_t d = 0; d < b.count; ++d) {
            const std::uint64_t i0 = b.index(d, 0), i1 = b.index(d, 1), i2 = b.index(d, 2);
            ok &= b.flat_index(d, RowOrder::Ascending) == (i0 * 3 + i1) * 4 + i2;
            ok &= b.flat_index(d, RowOrder::Reversed) == (i2 * 3 + i1) * 2 + i0;
            for (std::size_t c = 0; c < 2; ++c) {
                const double want = fs[0](i0, c) * fs[1](i1, c) * fs[2](i2, c);
                ok &= std::abs(b.rows(d, c) - want) <= 1e-12 * std::max(1.0, std::abs(want));
            }
        }
        CHECK(ok);
    }
    // SegmentTreeSampler drop-in (test_segment_tree.cpp's checks on the device tree)
    {
        // identity rows, y = ones, h = ones: every row has mass 1 -> uniform (known answer)
        Matrix eye(4, 4);
        for (std::size_t i = 0; i < 4; ++i) eye(i, i) = 1.0;
        const SegmentTreeSampler t(eye, 1, std::vector<double>(4, 1.0));
        const std::vector<double> h(4, 1.0);
        const std::vector<double> q = t.analytic_probabilities(h);
        bool uni = true;
        for (double v : q) uni &= std::abs(v - 0.25) < 1e-15;
        CHECK(uni);
        CounterRng rng(5, 0);
        const std::size_t r = t.row_sample(h, rng);
        CHECK(r < 4);
        CHECK(rng.draws() == 1);  // exactly one uniform consumed
        CHECK(std::abs(t.normalizer(h) - 4.0) < 1e-12);
        CHECK_THROWS_AS(SegmentTreeSampler(eye, 0, std::vector<double>(4, 1.0)), std::invalid_argument);
        CHECK_THROWS_AS(t.row_sample(std::vector<double>(3, 1.0), rng), std::invalid_argument);
        CHECK_THROWS_AS(t.row_sample(std::vector<double>(4, 0.0), rng), std::runtime_error);
    }
    {
        const Matrix U = random_matrix(777, 8, 780);
        Matrix Y(8, 8);
        const Matrix A = random_matrix(11, 8, 781);
        for (std::size_t a = 0; a < 8; ++a)
            for (std::size_t b = 0; b < 8; ++b) {
                double s = 0.0;
                for (std::size_t k = 0; k < 11; ++k) s += A(k, a) * A(k, b);
                Y(a, b) = s / 8.0;
            }
        const SegmentTreeSampler t(U, 5, Y, SegmentTreeSampler::Layout::Full);
        // children-sum invariant (segment_tree_sampler.cpp:180-186)
        bool sums = true;
        for (std::size_t v = 0; v < t.node_count(); ++v) {
            if (t.is_leaf(v)) continue;
            const Matrix p = t.node_gram(v), l = t.node_gram(t.left_child(v)), rr = t.node_gram(t.right_child(v));
            for (std::size_t e = 0; e < p.data.size(); ++e)
                sums &= std::abs(p.data[e] - l.data[e] - rr.data[e]) <= 1e-10 * (1.0 + std::abs(p.data[e]));
        }
        CHECK(sums);
        // draws vs the oracle restatement of the reference tree, same streams
        ko_tree* o = nullptr;
        CHECK(ko_tree_create(U.data.data(), U.rows, 8, 5, Y.data.data(), &o) == 0);
        std::vector<double> h(8);
        int same = 0;
        for (int d = 0; d < 300; ++d) {
            CounterRng hr(900 + d, 1);
            for (double& v : h) v = hr.normal();
            CounterRng rng(31, d);
            const std::size_t got = t.row_sample(h, rng);
            std::uint64_t ref = 0;
            CHECK(ko_tree_row_sample(o, h.data(), 31, uint64_t(d), 1, &ref) == 0);
            same += got == ref;
        }
        CHECK(same == 300);
        double tot = 0.0;
        for (double v : t.analytic_probabilities(h)) tot += v;
        CHECK(std::abs(tot - 1.0) < 1e-12);
        const auto seg = t.leaf_segment(3);
        CHECK(t.leaf_probabilities(h, 3).size() == seg.second - seg.first);
        ko_tree_destroy(o);
    }
    std::printf("%d/%d checks passed\n", g_checks - g_fail, g_checks);
    return g_fail ? 1 : 0;
}
