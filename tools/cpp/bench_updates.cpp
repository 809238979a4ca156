// Single-entry update throughput through the reference-facing C++ API
// (krplev::KrpSampler::update_factor_entry, krp_sampler.cpp:207-228), one call per
// entry exactly as a reference user writes it, on the SURVEY's measurement problem
// (factors 2^22 x 32, N(0,1); the reference did 1e5 calls in 0.20 s = 4.9e5/s).
// The timed region ends with factor_gram(j) and one sample() so the queued entries
// are applied on the device (and their Gram read back) inside it.
//
//   bench_updates [I] [R] [n]   -> one JSON line
#include <krplev/krp_sampler.hpp>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>

int main(int argc, char** argv) {
    const std::size_t I = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : (std::size_t(1) << 22);
    const std::size_t R = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 32;
    const std::size_t n = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 100000;
    std::mt19937_64 g(2301);
    std::normal_distribution<double> nd;
    std::vector<krplev::Matrix> fs;
    for (int k = 0; k < 3; ++k) {
        krplev::Matrix U(I, R);
        for (double& x : U.data) x = nd(g);
        fs.push_back(std::move(U));
    }
    krplev::KrpSampler s(std::move(fs));
    std::uniform_int_distribution<std::size_t> ri(0, I - 1), ci(0, R - 1);
    std::vector<std::size_t> r(n), c(n);
    std::vector<double> v(n);
    for (std::size_t i = 0; i < n; ++i) {
        r[i] = ri(g);
        c[i] = ci(g);
        v[i] = nd(g);
    }
    s.update_factor_entry(0, 0, 0, 1.0);  // warm: scratch buffers
    (void)s.factor_gram(0);
    const auto t0 = std::chrono::steady_clock::now();
    for (std::size_t i = 0; i < n; ++i) s.update_factor_entry(0, r[i], c[i], v[i]);
    const auto t1 = std::chrono::steady_clock::now();
    const krplev::Matrix& G = s.factor_gram(0);  // applies the queued entries on the device
    const auto t2 = std::chrono::steady_clock::now();
    const auto b = s.sample(std::nullopt, 65536, 7);
    const auto t3 = std::chrono::steady_clock::now();
    auto sec = [](auto a, auto z) { return std::chrono::duration<double>(z - a).count(); };
    std::printf("{\"api\": \"krplev::KrpSampler::update_factor_entry (one call per entry)\", \"I\": %zu, \"R\": %zu, "
                "\"calls\": %zu, \"queue_s\": %.6f, \"apply_s\": %.6f, \"seconds\": %.6f, \"updates_per_s\": %.1f, "
                "\"sample_after_s\": %.6f, \"G00\": %.17g, \"prob0\": %.17g}\n",
                I, R, n, sec(t0, t1), sec(t1, t2), sec(t0, t2), double(n) / sec(t0, t2), sec(t2, t3), G(0, 0),
                b.probabilities[0]);
    return 0;
}
