// Host R x R linear algebra for the sampler setup (see host_linalg.hpp).
#include "host_linalg.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>

namespace krpg {

namespace {

// Householder reduction of the symmetric matrix a (n x n, row-major, lower
// triangle used) to tridiagonal form. On return a holds the orthogonal Q with
// A = Q T Q^T, d the diagonal and e the sub-diagonal (e[0] = 0).
void tridiagonalize(std::vector<double>& a, std::size_t n, std::vector<double>& d,
                    std::vector<double>& e) {
    auto A = [&](std::size_t i, std::size_t j) -> double& { return a[i * n + j]; };
    for (std::size_t i = n - 1; i > 0; --i) {
        const std::size_t l = i - 1;
        double h = 0.0;
        if (l > 0) {
            double scale = 0.0;
            for (std::size_t k = 0; k <= l; ++k) scale += std::abs(A(i, k));
            if (scale == 0.0) {
                e[i] = A(i, l);
            } else {
                for (std::size_t k = 0; k <= l; ++k) {
                    A(i, k) /= scale;
                    h += A(i, k) * A(i, k);
                }
                double f = A(i, l);
                double g = f >= 0.0 ? -std::sqrt(h) : std::sqrt(h);
                e[i] = scale * g;
                h -= f * g;
                A(i, l) = f - g;
                f = 0.0;
                for (std::size_t j = 0; j <= l; ++j) {
                    A(j, i) = A(i, j) / h;
                    g = 0.0;
                    for (std::size_t k = 0; k <= j; ++k) g += A(j, k) * A(i, k);
                    for (std::size_t k = j + 1; k <= l; ++k) g += A(k, j) * A(i, k);
                    e[j] = g / h;
                    f += e[j] * A(i, j);
                }
                const double hh = f / (h + h);
                for (std::size_t j = 0; j <= l; ++j) {
                    f = A(i, j);
                    e[j] = g = e[j] - hh * f;
                    for (std::size_t k = 0; k <= j; ++k) A(j, k) -= (f * e[k] + g * A(i, k));
                }
            }
        } else {
            e[i] = A(i, l);
        }
        d[i] = h;
    }
    d[0] = 0.0;
    e[0] = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        if (d[i] != 0.0) {
            for (std::size_t j = 0; j < i; ++j) {
                double g = 0.0;
                for (std::size_t k = 0; k < i; ++k) g += A(i, k) * A(k, j);
                for (std::size_t k = 0; k < i; ++k) A(k, j) -= g * A(k, i);
            }
        }
        d[i] = A(i, i);
        A(i, i) = 1.0;
        for (std::size_t j = 0; j < i; ++j) A(j, i) = A(i, j) = 0.0;
    }
}

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

// Givens rotation of two contiguous rows (vectorised: the rows never alias)
inline void rotate_rows(double* __restrict__ zi, double* __restrict__ zi1, std::size_t n, double c, double s) {
    for (std::size_t k = 0; k < n; ++k) {
        const double a0 = zi[k], a1 = zi1[k];
        zi1[k] = s * a0 + c * a1;
        zi[k] = c * a0 - s * a1;
    }
}

// Implicit-shift QL on the tridiagonal (d, e); zt holds Q^T (rows = vectors)
// and is rotated alongside so its rows become the eigenvectors.
void tridiagonal_ql(std::vector<double>& d, std::vector<double>& e, std::vector<double>& zt,
                    std::size_t n) {
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
                    s = f / r;
                    c = g / r;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    p = s * r;
                    d[i + 1] = g + p;
                    g = c * r - b;
                    rotate_rows(zt.data() + i * n, zt.data() + (i + 1) * n, n, c, s);
                }
                if (deflated) continue;
                d[l] -= p;
                e[l] = g;
                e[m] = 0.0;
            }
        } while (m != l);
    }
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
        tridiagonal_ql(d, e, zt, n);  // zt rows: eigenvectors of the tridiagonal
        // back-transform all vectors at once, z <- H_0 H_1 ... H_{n-3} z, on the
        // coordinate-major copy zc[j][r] so every update is a contiguous axpy
        std::vector<double> zc(n * n), s(n);
        for (std::size_t r = 0; r < n; ++r)
            for (std::size_t j = 0; j < n; ++j) zc[j * n + r] = zt[r * n + j];
        for (std::size_t k = n - 2; k-- > 0;) {
            if (beta[k] == 0.0) continue;
            const double* v = refl.data() + k * n;
            std::fill(s.begin(), s.end(), 0.0);
            for (std::size_t j = k + 1; j < n; ++j) {
                const double vj = v[j];
                const double* __restrict__ zj = zc.data() + j * n;
                double* __restrict__ sp = s.data();
                for (std::size_t r = 0; r < n; ++r) sp[r] += vj * zj[r];
            }
            for (std::size_t r = 0; r < n; ++r) s[r] *= beta[k];
            for (std::size_t j = k + 1; j < n; ++j) {
                const double vj = v[j];
                double* __restrict__ zj = zc.data() + j * n;
                const double* __restrict__ sp = s.data();
                for (std::size_t r = 0; r < n; ++r) zj[r] -= vj * sp[r];
            }
        }
        for (std::size_t r = 0; r < n; ++r)
            for (std::size_t j = 0; j < n; ++j) zt[r * n + j] = zc[j * n + r];
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
    std::vector<double> P(n * n, 0.0);
    for (std::size_t u = 0; u < n; ++u) {
        if (e.values[u] <= tau) continue;
        const double inv = 1.0 / e.values[u];
        for (std::size_t i = 0; i < n; ++i) {
            const double vi = e.vectors[i * n + u] * inv;
            double* row = P.data() + i * n;
            for (std::size_t j = 0; j < n; ++j) row[j] += vi * e.vectors[j * n + u];
        }
    }
    return P;
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
