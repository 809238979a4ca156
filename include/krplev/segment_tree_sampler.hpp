// Drop-in for /root/reference/proj/include/krplev/segment_tree_sampler.hpp (:26-139),
// header-only, backed by the B200 C ABI (krpg_segtree_* in include/krpg.h).
//
// Same class, names, argument meaning and exception classes as the reference
// SegmentTreeSampler: the tree of partial Grams over U with leaf capacity F and a
// fixed PSD Y (general or rank-1) lives in HBM; row_sample consumes exactly one
// uniform of the caller's CounterRng (evaluated on the device from the
// generator's key and counter). Introspection (node_gram, node_segment,
// normalizer, left_subtree_mass, analytic_probabilities) is served from device
// data.
//
// Differences (documented in DESIGN.md):
//  * storage is always the compact layout (root + left children); with
//    Layout::Full, node_gram of a right child is formed as parent - left sibling;
//  * from_sparse keeps the reference's validation, Y = ones and greedy R^2-nonzero
//    leaf partition, but the device holds the densified rows (variable leaf segments
//    via krpg_segtree_create_segments); draws equal the reference's sparse tree's;
//  * extra: row_sample_batch (J draws, one history and one stream each).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "krpg.h"
#include "krplev/matrix.hpp"
#include "krplev/rng.hpp"

namespace krplev {

namespace detail {
inline void segtree_check(int rc) {
    if (rc == KRPG_OK) return;
    const std::string msg = krpg_last_error();
    if (rc == KRPG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
}  // namespace detail

class SegmentTreeSampler {
public:
    enum class Layout { Compact, Full };

    // General PSD Y. F is the leaf capacity.
    SegmentTreeSampler(const Matrix& U, std::size_t F, const Matrix& Y, Layout layout = Layout::Compact)
        : layout_(layout), u_(U), y_(Y) {
        if (U.empty()) throw std::invalid_argument("build_sampler: empty matrix");
        if (Y.rows != U.cols || Y.cols != U.cols) throw std::invalid_argument("build_sampler: Y must be R x R");
        create(F, Y.data.data(), nullptr);
    }
    // Rank-1 Y = y y^T.
    SegmentTreeSampler(const Matrix& U, std::size_t F, std::vector<double> y_rank1, Layout layout = Layout::Compact)
        : layout_(layout), u_(U), y_vec_(std::move(y_rank1)) {
        if (y_vec_.size() != U.cols) throw std::invalid_argument("SegmentTreeSampler: y must have R entries");
        create(F, nullptr, y_vec_.data());
    }

    // value semantics like the reference: a copy owns its own device tree
    SegmentTreeSampler(const SegmentTreeSampler& o)
        : layout_(o.layout_), u_(o.u_), y_(o.y_), y_vec_(o.y_vec_), F_(o.F_), sparse_(o.sparse_),
          row_ptr_(o.row_ptr_), col_idx_(o.col_idx_) {
        krpg_segtree_t t = nullptr;
        detail::segtree_check(krpg_segtree_clone(o.h_.get(), &t));
        h_.reset(t);
    }
    SegmentTreeSampler& operator=(const SegmentTreeSampler& o) {
        if (this != &o) {
            SegmentTreeSampler tmp(o);
            *this = std::move(tmp);
        }
        return *this;
    }
    SegmentTreeSampler(SegmentTreeSampler&&) noexcept = default;
    SegmentTreeSampler& operator=(SegmentTreeSampler&&) noexcept = default;

    // Sparse construction (segment_tree_sampler.cpp:67-109) with Y fixed to all-ones:
    // leaves by the greedy rule "at most R^2 stored nonzeros per leaf".
    static SegmentTreeSampler from_sparse(const SparseMatrixCoo& U, Layout layout = Layout::Compact) {
        if (U.rows < 1 || U.cols < 1) throw std::invalid_argument("build_sampler_sparse: empty matrix");
        if (U.entries.empty()) throw std::invalid_argument("build_sampler_sparse: matrix has no nonzeros");
        if (!U.sorted_row_major()) throw std::invalid_argument("build_sampler_sparse: entries must be sorted row-major");
        SegmentTreeSampler s(layout);
        s.sparse_ = true;
        s.u_ = Matrix(U.rows, U.cols);
        s.y_vec_.assign(U.cols, 1.0);
        s.row_ptr_.assign(U.rows + 1, 0);
        s.col_idx_.reserve(U.nnz());
        for (const auto& e : U.entries) {
            if (e.row >= U.rows || e.col >= U.cols) throw std::invalid_argument("build_sampler_sparse: entry out of range");
            if (!std::isfinite(e.value)) throw std::invalid_argument("build_sampler_sparse: non-finite entry");
            s.row_ptr_[e.row + 1]++;
            s.col_idx_.push_back(e.col);
            s.u_(e.row, e.col) = e.value;
        }
        for (std::size_t i = 0; i < U.rows; ++i) s.row_ptr_[i + 1] += s.row_ptr_[i];
        const std::size_t cap = U.cols * U.cols;
        std::vector<std::uint64_t> offs{0};
        std::size_t cur = 0;
        for (std::size_t i = 0; i < U.rows; ++i) {
            const std::size_t rn = s.row_ptr_[i + 1] - s.row_ptr_[i];
            if (cur + rn > cap && cur > 0) {
                offs.push_back(i);
                cur = 0;
            }
            cur += rn;
        }
        offs.push_back(U.rows);
        s.F_ = U.cols;  // nominal, as the reference
        krpg_segtree_t t = nullptr;
        detail::segtree_check(krpg_segtree_create_segments(s.u_.data.data(), s.u_.rows,
                                                           static_cast<std::uint32_t>(s.u_.cols), offs.data(),
                                                           offs.size() - 1, nullptr, s.y_vec_.data(), 0, &t));
        s.h_.reset(t);
        return s;
    }

    std::size_t rows() const { return u_.rows; }
    std::size_t cols() const { return u_.cols; }
    bool sparse() const { return sparse_; }

    // Draws one row index in [0, I); consumes exactly one uniform variate.
    std::size_t row_sample(std::span<const double> h, CounterRng& rng) const {
        check_h(h);
        const std::uint64_t key = rng.key(), counter = rng.draws() + 1;
        std::uint64_t out = 0;
        detail::segtree_check(krpg_segtree_sample_keyed(h_.get(), h.data(), 1, &key, &counter, &out, nullptr));
        (void)rng.uniform();  // the uniform the device consumed
        return static_cast<std::size_t>(out);
    }
    // Extra: J draws at once, draw d with history H[d] and its own generator.
    std::vector<std::size_t> row_sample_batch(const Matrix& H, std::vector<CounterRng>& rngs) const {
        if (H.cols != cols() || H.rows != rngs.size())
            throw std::invalid_argument("row_sample_batch: one history row and one generator per draw");
        std::vector<std::uint64_t> keys(H.rows), ctr(H.rows), out(H.rows);
        for (std::size_t d = 0; d < H.rows; ++d) {
            keys[d] = rngs[d].key();
            ctr[d] = rngs[d].draws() + 1;
        }
        detail::segtree_check(
            krpg_segtree_sample_keyed(h_.get(), H.data.data(), H.rows, keys.data(), ctr.data(), out.data(), nullptr));
        for (CounterRng& r : rngs) (void)r.uniform();
        return std::vector<std::size_t>(out.begin(), out.end());
    }

    // q_{h,U,Y} restricted to the rows of the given in-order leaf.
    std::vector<double> leaf_probabilities(std::span<const double> h, std::size_t leaf) const {
        const auto seg = leaf_segment(leaf);
        const std::vector<double> q = analytic_probabilities(h);
        return std::vector<double>(q.begin() + seg.first, q.begin() + seg.second);
    }

    void update_entry(std::size_t r, std::size_t c, double value) {
        if (sparse_ && r < rows() && c < cols() &&
            !std::binary_search(col_idx_.begin() + row_ptr_[r], col_idx_.begin() + row_ptr_[r + 1],
                                static_cast<std::uint32_t>(c)))
            throw std::invalid_argument("update_entry: entry outside the stored sparsity pattern");
        detail::segtree_check(krpg_segtree_update_entry(h_.get(), r, static_cast<std::uint32_t>(c), value));
        u_(r, c) = value;
    }

    // --- introspection and test support -------------------------------------
    std::size_t leaf_count() const { return shape().first; }
    std::size_t node_count() const { return shape().second; }
    std::pair<std::size_t, std::size_t> leaf_segment(std::size_t leaf) const {
        const std::size_t L = leaf_count();
        if (leaf >= L) throw std::invalid_argument("leaf_segment: leaf out of range");
        std::vector<std::uint64_t> offs(L + 1);
        detail::segtree_check(krpg_segtree_leaf_offsets(h_.get(), offs.data()));
        return {static_cast<std::size_t>(offs[leaf]), static_cast<std::size_t>(offs[leaf + 1])};
    }
    std::pair<std::size_t, std::size_t> node_segment(std::size_t node) const {
        std::uint64_t f = 0, l = 0;
        detail::segtree_check(krpg_segtree_node_rows(h_.get(), node, &f, &l));
        return {static_cast<std::size_t>(f), static_cast<std::size_t>(l)};
    }
    bool gram_stored(std::size_t node) const { return layout_ == Layout::Full || node == 0 || (node & 1); }
    Matrix node_gram(std::size_t node) const {
        if (node >= node_count()) throw std::invalid_argument("node_gram: node out of range");
        Matrix g(cols(), cols());
        if (node == 0 || (node & 1)) {
            detail::segtree_check(krpg_segtree_node_gram(h_.get(), node, g.data.data()));
            return g;
        }
        if (layout_ != Layout::Full) throw std::invalid_argument("node_gram: Gram of this node is not stored");
        const Matrix p = node_gram((node - 1) / 2), l = node_gram(node - 1);  // right = parent - left
        for (std::size_t e = 0; e < g.data.size(); ++e) g.data[e] = p.data[e] - l.data[e];
        return g;
    }
    std::size_t left_child(std::size_t node) const { return 2 * node + 1; }
    std::size_t right_child(std::size_t node) const { return 2 * node + 2; }
    bool is_leaf(std::size_t node) const { return 2 * node + 1 >= node_count(); }

    // Normalizer C = <h h^T, U^T U, Y>.
    double normalizer(std::span<const double> h) const { return gram_mass(node_gram(0), h); }
    // Normalised mass of the left subtree of an internal node: the branch threshold of
    // the sampling walk without the running offset (segment_tree_sampler.cpp:325-331).
    double left_subtree_mass(std::size_t node, std::span<const double> h) const {
        if (is_leaf(node)) throw std::invalid_argument("left_subtree_mass: node is a leaf");
        const double C = normalizer(h);
        if (C <= 0.0) throw std::runtime_error("left_subtree_mass: degenerate distribution");
        return gram_mass(node_gram(left_child(node)), h) / C;
    }
    std::vector<double> analytic_probabilities(std::span<const double> h) const {
        check_h(h);
        std::vector<double> q(rows());
        detail::segtree_check(krpg_segtree_probabilities(h_.get(), h.data(), q.data()));
        return q;
    }
    const Matrix& dense_matrix() const {
        if (sparse_) throw std::logic_error("dense_matrix: sampler was built from sparse input");
        return u_;
    }

private:
    struct Del {
        void operator()(krpg_segtree* t) const { krpg_segtree_destroy(t); }
    };

    explicit SegmentTreeSampler(Layout layout) : layout_(layout) {}

    void create(std::size_t F, const double* Y, const double* y) {
        if (u_.empty()) throw std::invalid_argument("SegmentTreeSampler: empty matrix");
        F_ = F;
        krpg_segtree_t t = nullptr;
        detail::segtree_check(
            krpg_segtree_create(u_.data.data(), u_.rows, static_cast<std::uint32_t>(u_.cols), F, Y, y, 0, &t));
        h_.reset(t);
    }
    std::pair<std::size_t, std::size_t> shape() const {
        std::uint64_t L = 0, n = 0;
        detail::segtree_check(krpg_segtree_shape(h_.get(), &L, &n));
        return {static_cast<std::size_t>(L), static_cast<std::size_t>(n)};
    }
    void check_h(std::span<const double> h) const {
        if (h.size() != cols()) throw std::invalid_argument("SegmentTreeSampler: history length must equal R");
    }
    // <h h^T o Y, G> for a dense node Gram (fold_weights + packed_inner semantics)
    double gram_mass(const Matrix& G, std::span<const double> h) const {
        check_h(h);
        const std::size_t R = cols();
        double acc = 0.0;
        for (std::size_t a = 0; a < R; ++a)
            for (std::size_t b = a; b < R; ++b) {
                const double y = y_vec_.empty() ? y_(a, b) : y_vec_[a] * y_vec_[b];
                acc += (a == b ? 1.0 : 2.0) * h[a] * h[b] * y * G(a, b);
            }
        return acc;
    }

    Layout layout_;
    Matrix u_, y_;
    std::vector<double> y_vec_;
    std::size_t F_ = 0;
    bool sparse_ = false;
    std::vector<std::size_t> row_ptr_;  // sparse-built: stored pattern (CSR)
    std::vector<std::uint32_t> col_idx_;
    std::unique_ptr<krpg_segtree, Del> h_;
};

}  // namespace krplev
