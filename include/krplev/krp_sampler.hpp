// Drop-in for /root/reference/proj/include/krplev/krp_sampler.hpp (:17-101),
// header-only, backed by the B200 C ABI (include/krpg.h, libkrpg.so).
//
// Same names, argument meaning, value semantics and exception classes as the
// reference KrpSampler: construct / factor / factor_gram / sample /
// conditional / update_factor / update_factor_entry / validate. Factors and
// segment trees live in HBM; the class keeps a host mirror of the factors so
// factor(j) can return a reference like the reference does.
//
// Differences (documented in DESIGN.md):
//  * tree(j) is not provided (the device tree is introspected through
//    node_gram(j, node) / tree_shape(j));
//  * validate(tol) compares with a Gram-relative tolerance (see krpg.h);
//  * extras: update_factor_entries (one batched device patch for a whole
//    sequence of single-entry updates), sample with draw_offset (sharding),
//    margins for boundary-draw accounting, the one-stage mode.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "krpg.h"
#include "krplev/matrix.hpp"
#include "krplev/rng.hpp"

namespace krplev {

enum class RowOrder { Ascending, Reversed };

struct SampleBatch {
    static constexpr std::uint32_t kExcluded = static_cast<std::uint32_t>(-1);

    std::optional<std::size_t> excluded;
    std::size_t count = 0;
    std::size_t factor_count = 0;
    std::vector<std::uint64_t> dims;
    std::vector<std::uint32_t> indices;  // J x N
    std::vector<double> probabilities;
    Matrix rows;                         // J x R
    std::vector<double> margin;          // B200 extra: boundary-draw margins (optional)

    std::uint32_t index(std::size_t draw, std::size_t factor) const { return indices[draw * factor_count + factor]; }
    std::uint64_t flat_index(std::size_t draw, RowOrder order) const {
        std::uint64_t flat = 0;
        auto step = [&](std::size_t k) {
            if (excluded && *excluded == k) return;
            flat = flat * dims[k] + index(draw, k);
        };
        if (order == RowOrder::Ascending)
            for (std::size_t k = 0; k < factor_count; ++k) step(k);
        else
            for (std::size_t k = factor_count; k-- > 0;) step(k);
        return flat;
    }
    std::vector<std::uint64_t> flat_indices(RowOrder order) const {
        std::vector<std::uint64_t> out(count);
        for (std::size_t d = 0; d < count; ++d) out[d] = flat_index(d, order);
        return out;
    }
};

struct ConditionalDistribution {
    std::vector<double> probabilities;
    std::vector<double> mixture_weights;
};

namespace detail {
inline void krpg_check(int rc) {
    if (rc == KRPG_OK) return;
    const std::string msg = krpg_last_error();
    if (rc == KRPG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
}  // namespace detail

class KrpSampler {
public:
    enum class Mode : std::uint32_t { TwoStage = KRPG_MODE_TWO_STAGE, OneStage = KRPG_MODE_ONE_STAGE };

    explicit KrpSampler(std::vector<Matrix> factors, int device = 0, bool fp32_storage = false)
        : fp32_(fp32_storage), factors_(std::move(factors)) {
        if (factors_.empty()) throw std::invalid_argument("KrpSampler: factor list is empty");
        rank_ = factors_[0].cols;
        std::vector<const double*> ptrs;
        std::vector<std::uint64_t> I;
        for (const Matrix& U : factors_) {
            if (U.empty()) throw std::invalid_argument("KrpSampler: empty factor");
            if (U.cols != rank_) throw std::invalid_argument("KrpSampler: inconsistent column counts");
            ptrs.push_back(U.data.data());
            I.push_back(U.rows);
        }
        krpg_t h = nullptr;
        detail::krpg_check(krpg_create(ptrs.data(), I.data(), static_cast<std::uint32_t>(factors_.size()),
                                       static_cast<std::uint32_t>(rank_),
                                       fp32_storage ? KRPG_STORE_F32 : KRPG_STORE_F64, device, &h));
        h_.reset(h);
        if (fp32_storage)  // the host mirror holds exactly what the device stores
            for (std::size_t j = 0; j < factors_.size(); ++j) refresh_factor(j);
        refresh_grams();
    }

    std::size_t factor_count() const { return factors_.size(); }
    std::size_t rank() const { return rank_; }
    const Matrix& factor(std::size_t j) const { return factors_.at(j); }
    const Matrix& factor_gram(std::size_t j) const {
        if (gram_dirty_.at(j)) refresh_gram(j);  // single-entry updates since the last read
        return grams_.at(j);
    }

    SampleBatch sample(std::optional<std::size_t> excluded, std::size_t J, std::uint64_t seed) const {
        return sample(excluded, J, seed, Mode::TwoStage, 0, false);
    }
    SampleBatch sample(std::optional<std::size_t> excluded, std::size_t J, std::uint64_t seed, Mode mode,
                       std::uint64_t draw_offset, bool with_margin) const {
        if (J < 1) throw std::invalid_argument("KrpSample: sample count must be positive");
        SampleBatch b;
        b.excluded = excluded;
        b.count = J;
        b.factor_count = factors_.size();
        b.dims.assign(factors_.size(), 0);
        for (std::size_t k = 0; k < factors_.size(); ++k)
            if (!excluded || *excluded != k) b.dims[k] = factors_[k].rows;
        b.indices.resize(J * factors_.size());
        b.probabilities.resize(J);
        b.rows = Matrix(J, rank_);
        if (with_margin) b.margin.resize(J);
        const std::int64_t e = excluded ? static_cast<std::int64_t>(*excluded) : -1;
        detail::krpg_check(krpg_sample(h_.get(), e, J, seed, draw_offset, static_cast<std::uint32_t>(mode),
                                       b.indices.data(), b.probabilities.data(), b.rows.data.data(),
                                       with_margin ? b.margin.data() : nullptr));
        return b;
    }

    ConditionalDistribution conditional(std::optional<std::size_t> excluded, std::size_t k,
                                        std::span<const double> h) const {
        if (k >= factors_.size()) throw std::invalid_argument("conditional: factor k is not included");
        if (h.size() != rank_) throw std::invalid_argument("conditional: history vector has wrong length");
        ConditionalDistribution out;
        out.probabilities.resize(factors_[k].rows);
        out.mixture_weights.resize(rank_);
        const std::int64_t e = excluded ? static_cast<std::int64_t>(*excluded) : -1;
        detail::krpg_check(krpg_conditional(h_.get(), e, static_cast<std::uint32_t>(k), h.data(),
                                            out.probabilities.data(), out.mixture_weights.data()));
        return out;
    }

    void update_factor(std::size_t j, const Matrix& U) {
        if (j >= factors_.size()) throw std::invalid_argument("update_factor: index out of range");
        if (U.cols != rank_) throw std::invalid_argument("update_factor: column count mismatch");
        detail::krpg_check(krpg_update_factor(h_.get(), static_cast<std::uint32_t>(j), U.data.data(), U.rows));
        factors_[j] = U;
        refresh_gram(j);
    }

    void update_factor_entry(std::size_t j, std::size_t r, std::size_t c, double value) {
        const std::uint64_t rr = r;
        const std::uint32_t cc = static_cast<std::uint32_t>(c);
        update_factor_entries(j, std::span<const std::uint64_t>(&rr, 1), std::span<const std::uint32_t>(&cc, 1),
                              std::span<const double>(&value, 1));
    }

    // B200 extra: a whole sequence of update_factor_entry calls as one device patch
    void update_factor_entries(std::size_t j, std::span<const std::uint64_t> r, std::span<const std::uint32_t> c,
                               std::span<const double> v) {
        if (j >= factors_.size()) throw std::invalid_argument("update_factor_entry: index out of range");
        if (r.size() != c.size() || r.size() != v.size())
            throw std::invalid_argument("update_factor_entry: length mismatch");
        detail::krpg_check(krpg_update_entries(h_.get(), static_cast<std::uint32_t>(j), r.data(), c.data(),
                                               v.data(), v.size()));
        for (std::size_t i = 0; i < v.size(); ++i)  // mirror exactly what the device stores
            factors_[j](r[i], c[i]) = fp32_ ? static_cast<double>(static_cast<float>(v[i])) : v[i];
        gram_dirty_[j] = 1;  // the device queues the entries; G is re-read on the next factor_gram(j)
    }

    void validate(double tol = 1e-10) const { detail::krpg_check(krpg_validate(h_.get(), tol)); }

    // tree introspection (segment_tree_sampler.hpp:64-95 analogues)
    std::pair<std::uint64_t, std::uint64_t> tree_shape(std::size_t j) const {
        std::uint64_t L = 0, n = 0;
        detail::krpg_check(krpg_tree_shape(h_.get(), static_cast<std::uint32_t>(j), &L, &n));
        return {L, n};
    }
    Matrix node_gram(std::size_t j, std::size_t node) const {
        Matrix G(rank_, rank_);
        detail::krpg_check(krpg_node_gram(h_.get(), static_cast<std::uint32_t>(j), node, G.data.data()));
        return G;
    }

    krpg_t handle() const { return h_.get(); }

private:
    struct Closer {
        void operator()(krpg_t h) const { krpg_destroy(h); }
    };

    void refresh_grams() {
        grams_.assign(factors_.size(), Matrix(rank_, rank_));
        gram_dirty_.assign(factors_.size(), 0);
        for (std::size_t j = 0; j < factors_.size(); ++j) refresh_gram(j);
    }
    void refresh_gram(std::size_t j) const {
        if (grams_.size() != factors_.size()) grams_.assign(factors_.size(), Matrix(rank_, rank_));
        if (gram_dirty_.size() != factors_.size()) gram_dirty_.assign(factors_.size(), 0);
        detail::krpg_check(krpg_factor_gram(h_.get(), static_cast<std::uint32_t>(j), grams_[j].data.data()));
        gram_dirty_[j] = 0;
    }
    void refresh_factor(std::size_t j) {
        detail::krpg_check(krpg_factor(h_.get(), static_cast<std::uint32_t>(j), factors_[j].data.data()));
    }
    std::size_t rank_ = 0;
    bool fp32_ = false;
    std::vector<Matrix> factors_;
    mutable std::vector<Matrix> grams_;       // host mirror of the device Grams, refreshed lazily
    mutable std::vector<char> gram_dirty_;
    std::unique_ptr<krpg_sampler, Closer> h_;
};

}  // namespace krplev
