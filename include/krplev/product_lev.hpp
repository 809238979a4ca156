// Device CP-ARLS-LEV product-of-leverage sampler: the reference's
// product_lev_sample (/root/reference/proj/include/krplev/sketch.hpp:55-57,
// sketch.cpp:86-149), backed by krpg_product_lev_sample[_factors] (include/krpg.h).
//
// Same arguments, SampleBatch layout, per-draw CounterRng(seed, d) consumption
// (one uniform per included factor, in order) and exceptions. Indices equal the
// reference's up to counted boundary draws (cumulative tables are summed in a
// different order); probabilities and rows agree to 1e-10 relative.
//
// product_lev_sample_device(factors, ...) is the free function (factors copied to
// the device, gram(U) formed there); product_lev_sample_device(sampler, ...) uses a
// KrpSampler's resident factors and cached Grams. A build that replaces the
// reference's sketch.cpp definition forwards krplev::product_lev_sample to the
// former (tests/refsuite/product_lev_dropin.cpp).
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <vector>

#include "krpg.h"
#include "krplev/krp_sampler.hpp"
#include "krplev/matrix.hpp"

namespace krplev {

namespace detail {
inline SampleBatch lev_batch(std::optional<std::size_t> excluded, std::size_t J, std::size_t N, std::size_t R,
                             const std::vector<std::uint64_t>& rows_per_factor) {
    SampleBatch b;
    b.excluded = excluded;
    b.count = J;
    b.factor_count = N;
    b.dims.assign(N, 0);
    for (std::size_t k = 0; k < N; ++k)
        if (!excluded || *excluded != k) b.dims[k] = rows_per_factor[k];
    b.indices.resize(J * N);
    b.probabilities.resize(J);
    b.rows = Matrix(J, R);
    return b;
}
}  // namespace detail

inline SampleBatch product_lev_sample_device(const std::vector<Matrix>& factors, std::optional<std::size_t> excluded,
                                             std::size_t J, std::uint64_t seed, int device = 0) {
    if (factors.empty()) throw std::invalid_argument("product_lev_sample: factor list is empty");
    if (J < 1) throw std::invalid_argument("product_lev_sample: J must be positive");
    const std::size_t N = factors.size(), R = factors[0].cols;
    if (excluded && *excluded >= N) throw std::invalid_argument("product_lev_sample: excluded index out of range");
    std::vector<const double*> ptrs(N);
    std::vector<std::uint64_t> I(N);
    for (std::size_t k = 0; k < N; ++k) {
        if ((!excluded || *excluded != k) && factors[k].cols != R)
            throw std::invalid_argument("product_lev_sample: inconsistent column counts");
        ptrs[k] = factors[k].data.data();
        I[k] = factors[k].rows;
    }
    SampleBatch b = detail::lev_batch(excluded, J, N, R, I);
    const std::int64_t e = excluded ? static_cast<std::int64_t>(*excluded) : -1;
    detail::krpg_check(krpg_product_lev_sample_factors(ptrs.data(), I.data(), static_cast<std::uint32_t>(N),
                                                       static_cast<std::uint32_t>(R), e, J, seed, device,
                                                       b.indices.data(), b.probabilities.data(), b.rows.data.data(),
                                                       nullptr));
    return b;
}

inline SampleBatch product_lev_sample_device(const KrpSampler& s, std::optional<std::size_t> excluded, std::size_t J,
                                             std::uint64_t seed, std::uint64_t draw_offset = 0) {
    if (J < 1) throw std::invalid_argument("product_lev_sample: J must be positive");
    const std::size_t N = s.factor_count();
    std::vector<std::uint64_t> I(N);
    for (std::size_t k = 0; k < N; ++k) I[k] = s.factor(k).rows;
    SampleBatch b = detail::lev_batch(excluded, J, N, s.rank(), I);
    const std::int64_t e = excluded ? static_cast<std::int64_t>(*excluded) : -1;
    detail::krpg_check(krpg_product_lev_sample(s.handle(), e, J, seed, draw_offset, b.indices.data(),
                                               b.probabilities.data(), b.rows.data.data(), nullptr));
    return b;
}

}  // namespace krplev
