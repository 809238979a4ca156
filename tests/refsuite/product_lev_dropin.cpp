// Links the reference's own test_sketch.cpp product-sampler cases against the
// device implementation: oracle/Makefile compiles the reference sketch.cpp with its
// product_lev_sample renamed away and this definition takes its place.
#include "krplev/product_lev.hpp"
#include "krplev/sketch.hpp"

namespace krplev {

SampleBatch product_lev_sample(const std::vector<Matrix>& factors, std::optional<std::size_t> excluded,
                               std::size_t J, std::uint64_t seed) {
    return product_lev_sample_device(factors, excluded, J, seed);
}

}  // namespace krplev
