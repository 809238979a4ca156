// Small dense R x R host math for the sampler's per-call setup: Hadamard
// chains, symmetric PSD eigendecomposition, rank cutoff and pseudo-inverse.
// Semantics follow /root/reference/proj/src/dense_kernels.cpp:82-205; the
// eigensolver is a different (faster, O(R^3) with a small constant) algorithm:
// Householder tridiagonalisation followed by implicit-shift QL.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace krpg {

struct Eig {
    std::vector<double> vectors;  // n x n row-major, column k = eigenvector k
    std::vector<double> values;   // descending, clamped to >= 0
};

// Throws std::invalid_argument like eigh_psd (dense_kernels.cpp:93-176):
// non-finite input, asymmetry > 1e-10 * max(1, max|G|), or an eigenvalue below
// -1e-8 * lambda_max.
Eig eigh_psd(const double* G, std::size_t n);

double rank_cutoff(const Eig& e);                 // n * eps * lambda_max (:178-182)
std::size_t numerical_rank(const Eig& e);         // #{lambda > cutoff}  (:184-190)
std::vector<double> pinv_from_eigen(const Eig& e);  // sum_{lambda>cutoff} v v^T / lambda (:192-205)
// eigendecomposition of pinv_from_eigen(e) read off e (values 1/lambda descending, then
// the null space): equals eigh_psd(G+) up to rounding, without a second eigensolve
Eig eig_of_pinv(const Eig& e);

// out = ones o m_0 o m_1 ... (dense_kernels.cpp:82-91)
void hadamard_into(std::vector<double>& out, const double* m);

// packed upper triangle (row-major) of a symmetric n x n matrix
std::vector<double> pack_upper(const double* M, std::size_t n);
void unpack_upper(const double* packed, std::size_t n, double* M);

// x^T M y for dense n x n M (dense_kernels.cpp:232-243)
double quadratic_form(const double* x, const double* M, std::size_t n, const double* y);

}  // namespace krpg
