// Host R x R linear algebra for the sampler setup (see host_linalg.hpp).
#include "host_linalg.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <thread>

namespace krpg {

namespace {

// Householder tridiagonalisation of the full symmetric matrix a (n x n,
// row-major, both triangles kept): all updates are row-contiguous (symv +
// rank-2), so they vectorise. Reflector k (acting on coordinates k+1..n-1) is
// I - beta_k v_k v_k^T; v_k is stored in row k of `refl` at columns k+1..n-1.
// On return d/e hold the tridiagonal (e[i] couples i-1 and i, e[0] = 0).
void tridiagonalize_rowmajor(std::vector<double>& a, std::size_t n, std::vector<double>& d,
                             std::vector<double>& e, std::vector<double>& refl, std::vector<double>& beta) {
    std::vector<double> p(n), w(n);
    refl.assign(n * n, 0.0);
    beta.assign(n, 0.0);
    e.assign(n, 0.0);
    for (std::size_t k = 0; k + 2 < n; ++k) {
        double* ak = a.data() + k * n;
        const std::size_t m0 = k + 1;
        double sig = 0.0;
        for (std::size_t j = m0 + 1; j < n; ++j) sig += ak[j] * ak[j];
        const double x0 = ak[m0];
        d[k] = ak[k];
        if (sig == 0.0) {  // already tridiagonal in this column
            e[k + 1] = x0;
            continue;
        }
        const double nrm = std::sqrt(x0 * x0 + sig);
        const double alpha = x0 >= 0.0 ? -nrm : nrm;
        double* v = refl.data() + k * n;
        v[m0] = x0 - alpha;
        for (std::size_t j = m0 + 1; j < n; ++j) v[j] = ak[j];
        const double vtv = v[m0] * v[m0] + sig;
        const double b = 2.0 / vtv;
        beta[k] = b;
        e[k + 1] = alpha;
        // p = b * A22 v
        double pv = 0.0;
        for (std::size_t i = m0; i < n; ++i) {
            const double* ai = a.data() + i * n;
            double s = 0.0;
#pragma omp simd reduction(+ : s)
            for (std::size_t j = m0; j < n; ++j) s += ai[j] * v[j];
            p[i] = b * s;
            pv += p[i] * v[i];
        }
        const double K = 0.5 * b * pv;
        for (std::size_t i = m0; i < n; ++i) w[i] = p[i] - K * v[i];
        for (std::size_t i = m0; i < n; ++i) {
            double* ai = a.data() + i * n;
            const double vi = v[i], wi = w[i];
            for (std::size_t j = m0; j < n; ++j) ai[j] -= vi * w[j] + wi * v[j];
        }
    }
    if (n >= 2) {
        d[n - 2] = a[(n - 2) * n + (n - 2)];
        d[n - 1] = a[(n - 1) * n + (n - 1)];
        e[n - 1] = a[(n - 2) * n + (n - 1)];
    } else {
        d[0] = a[0];
    }
}

struct Rot {
    std::uint32_t i;  // rotates rows i, i+1 of Z^T
    double c, s;
};

// Implicit-shift QL on the tridiagonal (d, e), eigenvalues only; the Givens
// rotations that would update the eigenvector matrix are recorded in order
// (O(n^2) of them) and applied afterwards, in parallel over column slices.
void tridiagonal_ql(std::vector<double>& d, std::vector<double>& e, std::size_t n, std::vector<Rot>& rots) {
    for (std::size_t i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    const double eps = std::numeric_limits<double>::epsilon();
    for (std::size_t l = 0; l < n; ++l) {
        int iter = 0;
        std::size_t m;
        do {
            for (m = l; m + 1 < n; ++m) {
                const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
                if (std::abs(e[m]) <= eps * dd) break;
            }
            if (m != l) {
                if (++iter > 60) throw std::runtime_error("eigh_psd: QL iteration did not converge");
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = std::sqrt(g * g + 1.0);
                g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? std::abs(r) : -std::abs(r)));
                double s = 1.0, c = 1.0, p = 0.0;
                bool deflated = false;
                for (std::size_t i = m; i-- > l;) {
                    double f = s * e[i];
                    const double b = c * e[i];
                    r = std::sqrt(f * f + g * g);
                    e[i + 1] = r;
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[m] = 0.0;
                        deflated = true;
                        break;
                    }
                    const double ir = 1.0 / r;
                    s = f * ir;
                    c = g * ir;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    p = s * r;
                    d[i + 1] = g + p;
                    g = c * r - b;
                    rots.push_back(Rot{std::uint32_t(i), c, s});
                }
                if (deflated) continue;
                d[l] -= p;
                e[l] = g;
                e[m] = 0.0;
            }
        } while (m != l);
    }
}

// Apply the recorded rotations to columns [k0, k1) of zt (n x n, row-major).
void apply_rotations(const std::vector<Rot>& rots, double* zt, std::size_t n, std::size_t k0, std::size_t k1) {
    for (const Rot& q : rots) {
        double* __restrict__ zi = zt + q.i * n;
        double* __restrict__ zi1 = zi + n;
        const double c = q.c, s = q.s;
        for (std::size_t k = k0; k < k1; ++k) {
            const double a0 = zi[k], a1 = zi1[k];
            zi1[k] = s * a0 + c * a1;
            zi[k] = c * a0 - s * a1;
        }
    }
}

// Back-transform eigenvectors r in [r0, r1) (rows of zt): z <- H_0 ... H_{n-3} z.
void back_transform(const std::vector<double>& refl, const std::vector<double>& beta, double* zt, std::size_t n,
                    std::size_t r0, std::size_t r1) {
    for (std::size_t k = n - 2; k-- > 0;) {
        if (beta[k] == 0.0) continue;
        const double* __restrict__ v = refl.data() + k * n;
        for (std::size_t r = r0; r < r1; ++r) {
            double* __restrict__ z = zt + r * n;
            double sdot = 0.0;
#pragma omp simd reduction(+ : sdot)
            for (std::size_t j = k + 1; j < n; ++j) sdot += v[j] * z[j];
            sdot *= beta[k];
            for (std::size_t j = k + 1; j < n; ++j) z[j] -= sdot * v[j];
        }
    }
}

// fn(t) for t in [0, T): T-1 helper threads + the caller
template <typename F>
void run_parallel(unsigned T, F&& fn) {
    if (T <= 1) {
        fn(0u);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(T - 1);
    for (unsigned t = 1; t < T; ++t) th.emplace_back(fn, t);
    fn(0u);
    for (auto& x : th) x.join();
}

}  // namespace

Eig eigh_psd(const double* G, std::size_t n) {
    if (n == 0) throw std::invalid_argument("eigh_psd: matrix must be square");
    double maxabs = 0.0;
    for (std::size_t k = 0; k < n * n; ++k) {
        if (!std::isfinite(G[k])) throw std::invalid_argument("eigh_psd: non-finite entries");
        maxabs = std::max(maxabs, std::abs(G[k]));
    }
    double asym = 0.0;
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = i + 1; j < n; ++j) asym = std::max(asym, std::abs(G[i * n + j] - G[j * n + i]));
    if (asym > 1e-10 * std::max(1.0, maxabs))
        throw std::invalid_argument("eigh_psd: input not symmetric within tolerance");

    std::vector<double> a(n * n), d(n), e(n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) a[i * n + j] = 0.5 * (G[i * n + j] + G[j * n + i]);
    std::vector<double> zt(n * n, 0.0);  // rows = eigenvectors
    if (n == 1) {
        d[0] = a[0];
        zt[0] = 1.0;
    } else {
        std::vector<double> refl, beta;
        tridiagonalize_rowmajor(a, n, d, e, refl, beta);
        for (std::size_t i = 0; i < n; ++i) zt[i * n + i] = 1.0;
        std::vector<Rot> rots;
        rots.reserve(2 * n * n);
        tridiagonal_ql(d, e, n, rots);  // eigenvalues; rotations recorded
        // eigenvectors of the tridiagonal, then of A; both passes split the
        // work into independent slices (columns, then vectors) over threads
        const unsigned T = n >= 128 ? std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency() / 2)) : 1u;
        const std::size_t cw = (n + T - 1) / T;
        run_parallel(T, [&](unsigned t) {
            const std::size_t k0 = std::min(n, t * cw), k1 = std::min(n, k0 + cw);
            apply_rotations(rots, zt.data(), n, k0, k1);
        });
        run_parallel(T, [&](unsigned t) {
            const std::size_t r0 = std::min(n, t * cw), r1 = std::min(n, r0 + cw);
            back_transform(refl, beta, zt.data(), n, r0, r1);
        });
    }

    std::vector<std::size_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) { return d[x] > d[y]; });
    const double lmax = *std::max_element(d.begin(), d.end());
    Eig out;
    out.values.resize(n);
    out.vectors.assign(n * n, 0.0);
    for (std::size_t k = 0; k < n; ++k) {
        double lam = d[order[k]];
        if (lam < 0.0) {
            if (lam < -1e-8 * std::max(lmax, 0.0))
                throw std::invalid_argument("eigh_psd: significantly negative eigenvalue; input not PSD");
            lam = 0.0;
        }
        out.values[k] = lam;
        const double* z = zt.data() + order[k] * n;
        for (std::size_t i = 0; i < n; ++i) out.vectors[i * n + k] = z[i];
    }
    return out;
}

double rank_cutoff(const Eig& e) {
    const double lmax = e.values.empty() ? 0.0 : e.values.front();
    return static_cast<double>(e.values.size()) * std::numeric_limits<double>::epsilon() * lmax;
}

std::size_t numerical_rank(const Eig& e) {
    const double tau = rank_cutoff(e);
    std::size_t r = 0;
    for (double v : e.values)
        if (v > tau) ++r;
    return r;
}

std::vector<double> pinv_from_eigen(const Eig& e) {
    const std::size_t n = e.values.size();
    const double tau = rank_cutoff(e);
    // P = W V^T over the kept eigenpairs, W = V diag(1/lambda): row-by-row dot
    // products of contiguous rows (u runs along a row of `vectors`), upper triangle
    // then mirrored
    std::vector<double> inv(n, 0.0);
    for (std::size_t u = 0; u < n; ++u)
        if (e.values[u] > tau) inv[u] = 1.0 / e.values[u];
    std::vector<double> W(n * n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t u = 0; u < n; ++u) W[i * n + u] = e.vectors[i * n + u] * inv[u];
    std::vector<double> P(n * n, 0.0);
    for (std::size_t i = 0; i < n; ++i) {
        const double* wi = W.data() + i * n;
        for (std::size_t j = i; j < n; ++j) {
            const double* vj = e.vectors.data() + j * n;
            double acc = 0.0;
#pragma omp simd reduction(+ : acc)
            for (std::size_t u = 0; u < n; ++u) acc += wi[u] * vj[u];
            P[i * n + j] = acc;
            P[j * n + i] = acc;
        }
    }
    return P;
}

Eig eig_of_pinv(const Eig& e) {
    const std::size_t n = e.values.size();
    const double tau = rank_cutoff(e);
    Eig out;
    out.values.assign(n, 0.0);
    out.vectors.assign(n * n, 0.0);
    std::size_t k = 0;
    // 1/lambda descending = lambda ascending over the kept eigenpairs, then the null space
    for (std::size_t u = n; u-- > 0;) {
        if (e.values[u] <= tau) continue;
        out.values[k] = 1.0 / e.values[u];
        for (std::size_t i = 0; i < n; ++i) out.vectors[i * n + k] = e.vectors[i * n + u];
        ++k;
    }
    for (std::size_t u = 0; u < n; ++u) {
        if (e.values[u] > tau) continue;
        for (std::size_t i = 0; i < n; ++i) out.vectors[i * n + k] = e.vectors[i * n + u];
        ++k;
    }
    return out;
}

void hadamard_into(std::vector<double>& out, const double* m) {
    for (std::size_t k = 0; k < out.size(); ++k) out[k] *= m[k];
}

std::vector<double> pack_upper(const double* M, std::size_t n) {
    std::vector<double> p(n * (n + 1) / 2);
    std::size_t idx = 0;
    for (std::size_t a = 0; a < n; ++a)
        for (std::size_t b = a; b < n; ++b) p[idx++] = M[a * n + b];
    return p;
}

void unpack_upper(const double* packed, std::size_t n, double* M) {
    std::size_t idx = 0;
    for (std::size_t a = 0; a < n; ++a)
        for (std::size_t b = a; b < n; ++b, ++idx) {
            M[a * n + b] = packed[idx];
            M[b * n + a] = packed[idx];
        }
}

double quadratic_form(const double* x, const double* M, std::size_t n, const double* y) {
    double acc = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        double inner = 0.0;
        for (std::size_t j = 0; j < n; ++j) inner += M[i * n + j] * y[j];
        acc += x[i] * inner;
    }
    return acc;
}

}  // namespace krpg
