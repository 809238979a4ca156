// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Neutral C-ABI wrapper around the *unmodified* reference sources under
// /root/reference/proj (compiled by oracle/Makefile with -Dkrplev=krplev_ref so
// the reference namespace can never collide with the drop-in's krplev::).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg load the resulting oracle/_ref/libkrplev_ref.so.
//
// Every entry point forwards to a public reference API:
//   KrpSampler ctor/sample/conditional/update_*  krp_sampler.hpp:61-101
//   SegmentTreeSampler (Full layout introspection) segment_tree_sampler.hpp:26-95
//   eigh_psd / pinv_from_eigen / hadamard_chain    dense_kernels.hpp:29-47
//   materialize_krp / leverage_scores              reference/reference.hpp:28-32
//   CounterRng                                     rng.hpp:13-48
//   make_sampling_weights                          sketch.hpp:37-39
//   SparseTensorCoo::from_entries, sampled_rhs_rows,
//   gram / gram_cross / pinv_psd / matmul          tensor.hpp:23, cp_als.hpp:52, dense_kernels.hpp
//   (one STS-CP factor update, the StsCp branch of cp_als.cpp:279-313)
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "krplev/cp_als.hpp"
#include "krplev/dense_kernels.hpp"
#include "krplev/krp_sampler.hpp"
#include "krplev/rng.hpp"
#include "krplev/segment_tree_sampler.hpp"
#include "krplev/sketch.hpp"
#include "krplev/tensor.hpp"
#include "reference.hpp"

using namespace krplev;  // == krplev_ref via -D

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 runtime_error / other
template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Matrix to_matrix(const double* p, uint64_t rows, uint32_t cols) {
    Matrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data.data(), p, sizeof(double) * rows * cols);
    return m;
}

std::optional<std::size_t> excl(int64_t e) {
    if (e < 0) return std::nullopt;
    return static_cast<std::size_t>(e);
}

}  // namespace

extern "C" {

const char* kref_last_error() { return g_err.c_str(); }

// ---------------- CounterRng (rng.hpp:13-48) ----------------
void kref_uniforms(uint64_t seed, uint64_t stream, uint64_t n, double* out) {
    CounterRng r(seed, stream);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.uniform();
}
void kref_normals(uint64_t seed, uint64_t stream, uint64_t n, double* out) {
    CounterRng r(seed, stream);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.normal();
}
uint64_t kref_derive_seed(uint64_t seed, uint64_t a, uint64_t b) { return derive_seed(seed, a, b); }

// ---------------- dense kernels (dense_kernels.cpp) ----------------
int kref_gram(const double* U, uint64_t I, uint32_t R, double* out) {
    return guard([&] {
        Matrix g = gram(to_matrix(U, I, R));
        std::memcpy(out, g.data.data(), sizeof(double) * R * R);
    });
}
// values descending, vectors as columns (row-major n x n)
int kref_eigh(const double* G, uint32_t n, double* vectors, double* values) {
    return guard([&] {
        EigenPair e = eigh_psd(to_matrix(G, n, n));
        std::memcpy(vectors, e.vectors.data.data(), sizeof(double) * n * n);
        std::memcpy(values, e.values.data(), sizeof(double) * n);
    });
}
int kref_pinv(const double* G, uint32_t n, double* out, uint64_t* rank) {
    return guard([&] {
        EigenPair e = eigh_psd(to_matrix(G, n, n));
        *rank = numerical_rank(e);
        Matrix p = pinv_from_eigen(e);
        std::memcpy(out, p.data.data(), sizeof(double) * n * n);
    });
}

// ---------------- KrpSampler (krp_sampler.hpp:61-101) ----------------
int kref_create(const double* const* U, const uint64_t* I, uint32_t N, uint32_t R, void** out) {
    return guard([&] {
        std::vector<Matrix> fs;
        fs.reserve(N);
        for (uint32_t k = 0; k < N; ++k) fs.push_back(to_matrix(U[k], I[k], R));
        *out = new KrpSampler(std::move(fs));
    });
}
void kref_destroy(void* h) { delete static_cast<KrpSampler*>(h); }

int kref_factor_gram(void* h, uint32_t j, double* out) {
    return guard([&] {
        const Matrix& g = static_cast<KrpSampler*>(h)->factor_gram(j);
        std::memcpy(out, g.data.data(), sizeof(double) * g.data.size());
    });
}

// Stored (compact) node Gram of factor j's Z-tree, unpacked R x R.
int kref_node_gram(void* h, uint32_t j, uint64_t node, double* out) {
    return guard([&] {
        Matrix g = static_cast<KrpSampler*>(h)->tree(j).node_gram(node);
        std::memcpy(out, g.data.data(), sizeof(double) * g.data.size());
    });
}

int kref_sample(void* h, int64_t excluded, uint64_t J, uint64_t seed, uint32_t* idx,
                double* prob, double* rows) {
    return guard([&] {
        const KrpSampler& s = *static_cast<KrpSampler*>(h);
        SampleBatch b = s.sample(excl(excluded), J, seed);
        if (idx) std::memcpy(idx, b.indices.data(), sizeof(uint32_t) * b.indices.size());
        if (prob) std::memcpy(prob, b.probabilities.data(), sizeof(double) * J);
        if (rows) std::memcpy(rows, b.rows.data.data(), sizeof(double) * b.rows.data.size());
    });
}

int kref_conditional(void* h, int64_t excluded, uint32_t k, const double* hv, double* probs,
                     double* mixture) {
    return guard([&] {
        const KrpSampler& s = *static_cast<KrpSampler*>(h);
        ConditionalDistribution cd =
            s.conditional(excl(excluded), k, std::span<const double>(hv, s.rank()));
        std::memcpy(probs, cd.probabilities.data(), sizeof(double) * cd.probabilities.size());
        std::memcpy(mixture, cd.mixture_weights.data(),
                    sizeof(double) * cd.mixture_weights.size());
    });
}

int kref_update_factor(void* h, uint32_t j, const double* U, uint64_t I) {
    return guard([&] {
        KrpSampler& s = *static_cast<KrpSampler*>(h);
        s.update_factor(j, to_matrix(U, I, s.rank()));
    });
}

int kref_update_entries(void* h, uint32_t j, const uint64_t* r, const uint32_t* c,
                        const double* v, uint64_t n) {
    return guard([&] {
        KrpSampler& s = *static_cast<KrpSampler*>(h);
        for (uint64_t i = 0; i < n; ++i) s.update_factor_entry(j, r[i], c[i], v[i]);
    });
}

int kref_validate(void* h, double tol) {
    return guard([&] { static_cast<KrpSampler*>(h)->validate(tol); });
}

// One-stage (north_star "M = G+ o hh^T o G_{>k}") chain oracle, SURVEY §8(c):
// per included factor in ascending order build SegmentTreeSampler(U_k, R, G_{>k})
// (general-Y ctor, segment_tree_sampler.cpp:26-45) with G_{>k} computed with
// downstream_gram semantics (krp_sampler.cpp:74-80), and draw with the persistent
// CounterRng(seed, d) (one uniform per factor).
int kref_sample_one_stage(void* h, int64_t excluded, uint64_t J, uint64_t seed, uint32_t* idx,
                          double* prob, double* rows) {
    return guard([&] {
        const KrpSampler& s = *static_cast<KrpSampler*>(h);
        const std::size_t N = s.factor_count(), R = s.rank();
        std::vector<std::size_t> inc;
        for (std::size_t k = 0; k < N; ++k)
            if (excluded < 0 || static_cast<std::size_t>(excluded) != k) inc.push_back(k);
        if (inc.empty()) throw std::invalid_argument("one_stage: no factors left");
        std::vector<const Matrix*> gs;
        for (std::size_t k : inc) gs.push_back(&s.factor_gram(k));
        const Matrix G = hadamard_chain(gs, R, R);
        const EigenPair ge = eigh_psd(G);
        const std::size_t rank = numerical_rank(ge);
        if (rank == 0) throw std::runtime_error("one_stage: zero KRP");
        const Matrix gp = pinv_from_eigen(ge);
        std::vector<CounterRng> rngs;
        rngs.reserve(J);
        for (uint64_t d = 0; d < J; ++d) rngs.emplace_back(seed, d);
        Matrix H = Matrix::ones(J, R);
        for (uint64_t i = 0; i < J * N; ++i) idx[i] = SampleBatch::kExcluded;
        for (std::size_t pos = 0; pos < inc.size(); ++pos) {
            const std::size_t k = inc[pos];
            std::vector<const Matrix*> ds{&gp};
            for (std::size_t p = pos + 1; p < inc.size(); ++p) ds.push_back(&s.factor_gram(inc[p]));
            const Matrix Y = hadamard_chain(ds, R, R);
            const SegmentTreeSampler t(s.factor(k), R, Y);
            const Matrix& U = s.factor(k);
#pragma omp parallel for schedule(static)
            for (uint64_t d = 0; d < J; ++d) {
                double* hv = H.row(d);
                const std::size_t r = t.row_sample(std::span<const double>(hv, R), rngs[d]);
                idx[d * N + k] = static_cast<uint32_t>(r);
                const double* row = U.row(r);
                for (std::size_t c = 0; c < R; ++c) hv[c] *= row[c];
            }
        }
        for (uint64_t d = 0; d < J; ++d) {
            const std::span<const double> hv(H.row(d), R);
            if (prob) prob[d] = quadratic_form(hv, gp, hv) / static_cast<double>(rank);
        }
        if (rows) std::memcpy(rows, H.data.data(), sizeof(double) * J * R);
    });
}

// ---------------- SegmentTreeSampler (segment_tree_sampler.hpp:26-95) ----------------
// Y == nullptr -> rank-1 all-ones Y (the KrpSampler Z-tree configuration).
int kref_tree_create(const double* U, uint64_t I, uint32_t R, uint64_t F, const double* Y,
                     int full, void** out) {
    return guard([&] {
        const auto lay = full ? SegmentTreeSampler::Layout::Full : SegmentTreeSampler::Layout::Compact;
        if (Y)
            *out = new SegmentTreeSampler(to_matrix(U, I, R), F, to_matrix(Y, R, R), lay);
        else
            *out = new SegmentTreeSampler(to_matrix(U, I, R), F, std::vector<double>(R, 1.0), lay);
    });
}
// SegmentTreeSampler::from_sparse (segment_tree_sampler.cpp:67-109) over COO entries
int kref_tree_create_sparse(uint64_t rows, uint64_t cols, const uint32_t* er, const uint32_t* ec, const double* ev,
                            uint64_t nnz, int full, void** out) {
    return guard([&] {
        SparseMatrixCoo c;
        c.rows = rows;
        c.cols = cols;
        for (uint64_t k = 0; k < nnz; ++k) c.entries.push_back({er[k], ec[k], ev[k]});
        const auto lay = full ? SegmentTreeSampler::Layout::Full : SegmentTreeSampler::Layout::Compact;
        *out = new SegmentTreeSampler(SegmentTreeSampler::from_sparse(c, lay));
    });
}
void kref_tree_destroy(void* t) { delete static_cast<SegmentTreeSampler*>(t); }
uint64_t kref_tree_node_count(void* t) { return static_cast<SegmentTreeSampler*>(t)->node_count(); }
uint64_t kref_tree_leaf_count(void* t) { return static_cast<SegmentTreeSampler*>(t)->leaf_count(); }
int kref_tree_node_gram(void* t, uint64_t node, double* out) {
    return guard([&] {
        Matrix g = static_cast<SegmentTreeSampler*>(t)->node_gram(node);
        std::memcpy(out, g.data.data(), sizeof(double) * g.data.size());
    });
}
int kref_tree_node_segment(void* t, uint64_t node, uint64_t* first, uint64_t* last) {
    return guard([&] {
        auto [a, b] = static_cast<SegmentTreeSampler*>(t)->node_segment(node);
        *first = a;
        *last = b;
    });
}
// n draws from one CounterRng(seed, stream); out = row indices.
int kref_tree_row_sample(void* t, const double* h, uint64_t seed, uint64_t stream, uint64_t n,
                         uint64_t* out) {
    return guard([&] {
        const SegmentTreeSampler& s = *static_cast<SegmentTreeSampler*>(t);
        CounterRng rng(seed, stream);
        for (uint64_t i = 0; i < n; ++i) out[i] = s.row_sample(std::span<const double>(h, s.cols()), rng);
    });
}
int kref_tree_update_entry(void* t, uint64_t r, uint64_t c, double v) {
    return guard([&] { static_cast<SegmentTreeSampler*>(t)->update_entry(r, c, v); });
}
int kref_tree_analytic(void* t, const double* h, double* out) {
    return guard([&] {
        const SegmentTreeSampler& s = *static_cast<SegmentTreeSampler*>(t);
        auto p = s.analytic_probabilities(std::span<const double>(h, s.cols()));
        std::memcpy(out, p.data(), sizeof(double) * p.size());
    });
}
int kref_tree_left_mass(void* t, uint64_t node, const double* h, double* out) {
    return guard([&] {
        const SegmentTreeSampler& s = *static_cast<SegmentTreeSampler*>(t);
        *out = s.left_subtree_mass(node, std::span<const double>(h, s.cols()));
    });
}

// ---------------- exact leverage (reference/reference.cpp:30-48) ----------------
// normalized leverage of the KRP of the given factors, ascending row order.
int kref_leverage(const double* const* U, const uint64_t* I, uint32_t N, uint32_t R, double* out) {
    return guard([&] {
        std::vector<Matrix> fs;
        for (uint32_t k = 0; k < N; ++k) fs.push_back(to_matrix(U[k], I[k], R));
        const Matrix A = ref::materialize_krp(fs, RowOrder::Ascending);
        std::vector<double> l = ref::leverage_scores(A);
        double tot = 0.0;
        for (double v : l) tot += v;
        for (std::size_t i = 0; i < l.size(); ++i) out[i] = l[i] / tot;
    });
}

// ---------------- CP-ARLS-LEV product sampler (sketch.cpp:86-149) ----------------
int kref_product_lev_sample(const double* const* U, const uint64_t* I, uint32_t N, uint32_t R, int64_t excluded,
                            uint64_t J, uint64_t seed, uint32_t* idx, double* prob, double* rows, double* margin) {
    return guard([&] {
        std::vector<Matrix> fs;
        for (uint32_t k = 0; k < N; ++k) fs.push_back(to_matrix(U[k], I[k], R));
        std::optional<std::size_t> ex;
        if (excluded >= 0) ex = static_cast<std::size_t>(excluded);
        const SampleBatch b = product_lev_sample(fs, ex, J, seed);
        std::memcpy(idx, b.indices.data(), sizeof(uint32_t) * b.indices.size());
        std::memcpy(prob, b.probabilities.data(), sizeof(double) * J);
        std::memcpy(rows, b.rows.data.data(), sizeof(double) * J * R);
        if (margin)
            for (uint64_t d = 0; d < J; ++d) margin[d] = HUGE_VAL;
    });
}

// ---------------- STS-CP gather weights (sketch.cpp:36-52) ----------------
int kref_sampling_weights(const double* prob, uint64_t n, uint64_t J, double* w) {
    return guard([&] {
        std::vector<uint64_t> ids(n, 0);
        RowSampleWeights rw = make_sampling_weights(ids, std::span<const double>(prob, n), J);
        std::memcpy(w, rw.weights.data(), sizeof(double) * n);
    });
}

// Deduplicated, sorted entries of SparseTensorCoo::from_entries (tensor.cpp:34-75).
// Call with coords_out == nullptr to get the count.
int kref_tensor_entries(const uint64_t* dims, uint32_t N, const uint32_t* coords, const double* values, uint64_t nnz,
                        uint32_t* coords_out, double* values_out, uint64_t* nnz_out) {
    return guard([&] {
        SparseTensorCoo T = SparseTensorCoo::from_entries(std::vector<uint64_t>(dims, dims + N),
                                                          std::vector<uint32_t>(coords, coords + nnz * N),
                                                          std::vector<double>(values, values + nnz));
        *nnz_out = T.nnz();
        if (coords_out)
            for (std::size_t e = 0; e < T.nnz(); ++e)
                for (uint32_t k = 0; k < N; ++k) coords_out[e * N + k] = T.coords(e)[k];
        if (values_out) std::memcpy(values_out, T.values().data(), sizeof(double) * T.nnz());
    });
}

// One STS-CP factor update of mode j (cp_als.cpp:279-313, solver StsCp) through the
// reference's public functions; the column renormalisation of cp_als.cpp:39-52 is
// internal to that file and is restated here (norms into sigma, zero column ->
// unit basis vector c % I).
int kref_sts_step(const double* const* factors, const uint64_t* I, uint32_t N, uint32_t R, const uint32_t* coords,
                  const double* values, uint64_t nnz, uint32_t j, uint64_t J, uint64_t seed, double* unew,
                  double* sigma) {
    return guard([&] {
        std::vector<Matrix> fs;
        std::vector<uint64_t> dims(I, I + N);
        for (uint32_t k = 0; k < N; ++k) fs.push_back(to_matrix(factors[k], I[k], R));
        KrpSampler sampler(fs);
        SparseTensorCoo T = SparseTensorCoo::from_entries(dims, std::vector<uint32_t>(coords, coords + nnz * N),
                                                          std::vector<double>(values, values + nnz));
        SampleBatch batch = sampler.sample(j, J, seed);
        const RowSampleWeights w =
            make_sampling_weights(batch.flat_indices(RowOrder::Reversed), batch.probabilities, batch.count);
        Matrix sa = std::move(batch.rows);
        for (std::size_t d = 0; d < sa.rows; ++d)
            for (std::size_t c = 0; c < R; ++c) sa(d, c) *= w.weights[d];
        Matrix sb = sampled_rhs_rows(T, j, batch);
        for (std::size_t d = 0; d < sb.rows; ++d)
            for (std::size_t c = 0; c < sb.cols; ++c) sb(d, c) *= w.weights[d];
        const Matrix gs = gram(sa);
        Matrix u = transpose(matmul(pinv_psd(gs), gram_cross(sa, sb)));
        for (std::size_t c = 0; c < u.cols; ++c) {
            double nrm = 0.0;
            for (std::size_t i = 0; i < u.rows; ++i) nrm += u(i, c) * u(i, c);
            nrm = std::sqrt(nrm);
            sigma[c] = nrm;
            if (nrm > 0.0) {
                for (std::size_t i = 0; i < u.rows; ++i) u(i, c) /= nrm;
            } else {
                u(c % u.rows, c) = 1.0;
            }
        }
        std::memcpy(unew, u.data.data(), sizeof(double) * u.rows * u.cols);
    });
}

}  // extern "C"
