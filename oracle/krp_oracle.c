/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference krplev sampler (see krp_oracle.h).
 * The arithmetic is written in the same operation order as the reference so
 * that, compiled with -ffp-contract=off, results are bit-identical to the
 * reference built the same way (pinned by tests/test_oracle.py and the
 * committed fixtures in tests/golden/).
 *
 * Parity: pinned (oracle/_ref + tests/golden/*.npz).
 */
#include "krp_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}
const char* ko_last_error(void) { return g_err; }

#define KO_EXCLUDED 0xFFFFFFFFu

/* ------------------------------------------------------------------------ */
/* CounterRng — rng.hpp:13-48                                               */
/* ------------------------------------------------------------------------ */
uint64_t ko_mix(uint64_t z) { /* rng.hpp:36-43 */
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ull;
    z ^= z >> 33;
    return z;
}
typedef struct {
    uint64_t key, counter;
} rng_t;
static void rng_init(rng_t* r, uint64_t seed, uint64_t stream) { /* rng.hpp:16-18 */
    r->key = ko_mix(ko_mix(seed + 0x9e3779b97f4a7c15ull) ^ ko_mix(stream + 0xbf58476d1ce4e5b9ull));
    r->counter = 0;
}
static double rng_uniform(rng_t* r) { /* rng.hpp:21-24 */
    const uint64_t bits = ko_mix(r->key + (++r->counter) * 0x9e3779b97f4a7c15ull);
    return (double)(bits >> 11) * 0x1.0p-53;
}
static double rng_normal(rng_t* r) { /* rng.hpp:27-31 */
    const double u1 = 1.0 - rng_uniform(r);
    const double u2 = rng_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2);
}
void ko_uniforms(uint64_t seed, uint64_t stream, uint64_t n, double* out) {
    rng_t r;
    rng_init(&r, seed, stream);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng_uniform(&r);
}
void ko_normals(uint64_t seed, uint64_t stream, uint64_t n, double* out) {
    rng_t r;
    rng_init(&r, seed, stream);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng_normal(&r);
}
uint64_t ko_derive_seed(uint64_t seed, uint64_t a, uint64_t b) { /* rng.hpp:52-54 */
    return ko_mix(ko_mix(seed ^ (a * 0xd6e8feb86659fd93ull)) + b);
}

/* ------------------------------------------------------------------------ */
/* dense kernels — dense_kernels.cpp                                         */
/* ------------------------------------------------------------------------ */
void ko_gram(const double* U, uint64_t I, uint32_t R, double* G) { /* :19-42 */
    for (uint32_t a = 0; a < R; ++a)
        for (uint32_t b = a; b < R; ++b) {
            double acc = 0.0;
            for (uint64_t i = 0; i < I; ++i) acc += U[i * R + a] * U[i * R + b];
            G[a * R + b] = acc;
            G[b * R + a] = acc;
        }
}

static void hadamard_into(double* out, const double* m, size_t n) { /* :82-91 */
    for (size_t k = 0; k < n; ++k) out[k] *= m[k];
}

/* cyclic Jacobi eigh_psd, dense_kernels.cpp:93-176. V columns = eigenvectors. */
int ko_eigh(const double* G, uint32_t n, double* Vout, double* lam) {
    if (n == 0) return fail(1, "eigh_psd: matrix must be square");
    double maxabs = 0.0;
    for (size_t k = 0; k < (size_t)n * n; ++k) {
        if (!isfinite(G[k])) return fail(1, "eigh_psd: non-finite entries");
        maxabs = fmax(maxabs, fabs(G[k]));
    }
    double asym = 0.0;
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = i + 1; j < n; ++j) asym = fmax(asym, fabs(G[i * n + j] - G[j * n + i]));
    if (asym > 1e-10 * fmax(1.0, maxabs)) return fail(1, "eigh_psd: input not symmetric within tolerance");

    double* A = malloc(sizeof(double) * n * n);
    double* V = calloc((size_t)n * n, sizeof(double));
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < n; ++j) A[i * n + j] = 0.5 * (G[i * n + j] + G[j * n + i]);
    for (uint32_t i = 0; i < n; ++i) V[i * n + i] = 1.0;

    double frob = 0.0;
    for (size_t k = 0; k < (size_t)n * n; ++k) frob += A[k] * A[k];
    frob = sqrt(frob);
    const double off_target = 1e-12 * frob;

    for (int sweep = 0; sweep < 64; ++sweep) {
        double s = 0.0;
        for (uint32_t i = 0; i < n; ++i)
            for (uint32_t j = i + 1; j < n; ++j) s += 2.0 * A[i * n + j] * A[i * n + j];
        if (!(sqrt(s) > off_target)) break;
        for (uint32_t p = 0; p < n; ++p) {
            for (uint32_t q = p + 1; q < n; ++q) {
                const double apq = A[p * n + q];
                if (apq == 0.0) continue;
                const double app = A[p * n + p], aqq = A[q * n + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double sn = t * c;
                for (uint32_t k = 0; k < n; ++k) {
                    const double akp = A[k * n + p], akq = A[k * n + q];
                    A[k * n + p] = c * akp - sn * akq;
                    A[k * n + q] = sn * akp + c * akq;
                }
                for (uint32_t k = 0; k < n; ++k) {
                    const double apk = A[p * n + k], aqk = A[q * n + k];
                    A[p * n + k] = c * apk - sn * aqk;
                    A[q * n + k] = sn * apk + c * aqk;
                }
                for (uint32_t k = 0; k < n; ++k) {
                    const double vkp = V[k * n + p], vkq = V[k * n + q];
                    V[k * n + p] = c * vkp - sn * vkq;
                    V[k * n + q] = sn * vkp + c * vkq;
                }
            }
        }
    }
    double* vals = malloc(sizeof(double) * n);
    uint32_t* order = malloc(sizeof(uint32_t) * n);
    for (uint32_t i = 0; i < n; ++i) {
        vals[i] = A[i * n + i];
        order[i] = i;
    }
    /* stable sort descending (std::stable_sort with values[a] > values[b]) */
    for (uint32_t i = 1; i < n; ++i) {
        const uint32_t x = order[i];
        uint32_t j = i;
        while (j > 0 && vals[x] > vals[order[j - 1]]) {
            order[j] = order[j - 1];
            --j;
        }
        order[j] = x;
    }
    double lmax = vals[0];
    for (uint32_t i = 1; i < n; ++i) lmax = fmax(lmax, vals[i]);
    int rc = 0;
    for (uint32_t k = 0; k < n; ++k) {
        double l = vals[order[k]];
        if (l < 0.0) {
            if (l < -1e-8 * fmax(lmax, 0.0)) {
                rc = fail(1, "eigh_psd: significantly negative eigenvalue; input not PSD");
                break;
            }
            l = 0.0;
        }
        lam[k] = l;
        for (uint32_t i = 0; i < n; ++i) Vout[i * n + k] = V[i * n + order[k]];
    }
    free(A);
    free(V);
    free(vals);
    free(order);
    return rc;
}

static double rank_cutoff(const double* lam, uint32_t n) { /* :178-182 */
    return (double)n * DBL_EPSILON * lam[0];
}
static uint64_t numerical_rank(const double* lam, uint32_t n) { /* :184-190 */
    const double tau = rank_cutoff(lam, n);
    uint64_t r = 0;
    for (uint32_t i = 0; i < n; ++i)
        if (lam[i] > tau) ++r;
    return r;
}
static void pinv_from_eigen(const double* V, const double* lam, uint32_t n, double* P) { /* :192-205 */
    const double tau = rank_cutoff(lam, n);
    memset(P, 0, sizeof(double) * n * n);
    for (uint32_t u = 0; u < n; ++u) {
        if (lam[u] <= tau) continue;
        const double inv = 1.0 / lam[u];
        for (uint32_t i = 0; i < n; ++i) {
            const double vi = V[i * n + u] * inv;
            for (uint32_t j = 0; j < n; ++j) P[i * n + j] += vi * V[j * n + u];
        }
    }
}
int ko_pinv(const double* G, uint32_t n, double* out, uint64_t* rank) {
    double* V = malloc(sizeof(double) * n * n);
    double* l = malloc(sizeof(double) * n);
    int rc = ko_eigh(G, n, V, l);
    if (!rc) {
        *rank = numerical_rank(l, n);
        pinv_from_eigen(V, l, n, out);
    }
    free(V);
    free(l);
    return rc;
}

static double quadratic_form(const double* x, const double* M, uint32_t n, const double* y) { /* :232-243 */
    double acc = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        double inner = 0.0;
        for (uint32_t j = 0; j < n; ++j) inner += M[i * n + j] * y[j];
        acc += x[i] * inner;
    }
    return acc;
}

/* ------------------------------------------------------------------------ */
/* SegmentTreeSampler — segment_tree_sampler.cpp                             */
/* ------------------------------------------------------------------------ */
struct ko_tree {
    uint64_t I, R, F, L, n, P;
    uint64_t *seg0, *seg1, *leaf_node;
    double* grams; /* full store n * P */
    double* U;     /* I x R, owned or borrowed */
    int own_u;
    double* Y;  /* general Y (R x R) or NULL */
    double* y1; /* rank-1 factor or NULL */
    const uint64_t* offs; /* explicit leaf offsets (L + 1) during tree_topology, or NULL */
};

static uint64_t ceil_log2(uint64_t n) { /* :18-22 */
    uint64_t d = 0;
    while (((uint64_t)1 << d) < n) ++d;
    return d;
}
static int is_leaf(const ko_tree* t, uint64_t v) { return 2 * v + 1 >= t->n; } /* .hpp:82 */

static void tree_topology(ko_tree* t) { /* init_tree :111-149 */
    const uint64_t L = t->L, n = 2 * L - 1;
    t->n = n;
    t->seg0 = calloc(n, sizeof(uint64_t));
    t->seg1 = calloc(n, sizeof(uint64_t));
    t->leaf_node = calloc(L, sizeof(uint64_t));
    const uint64_t d = ceil_log2(L);
    const uint64_t bottom = 2 * L - ((uint64_t)1 << d);
    for (uint64_t l = 0; l < L; ++l) {
        const uint64_t node = (l < bottom) ? (((uint64_t)1 << d) - 1 + l) : (L - 1 + (l - bottom));
        t->leaf_node[l] = node;
        if (t->offs) { /* explicit leaf_segments (from_sparse's partition, :88-101) */
            t->seg0[node] = t->offs[l];
            t->seg1[node] = t->offs[l + 1];
        } else {
            t->seg0[node] = l * t->F;
            t->seg1[node] = (l * t->F + t->F < t->I) ? l * t->F + t->F : t->I;
        }
    }
    for (uint64_t v = n; v-- > 0;)
        if (!is_leaf(t, v)) {
            t->seg0[v] = t->seg0[2 * v + 1];
            t->seg1[v] = t->seg1[2 * v + 2];
        }
}

static void tree_build(ko_tree* t) { /* build_grams :151-191 (dense path) */
    const uint64_t P = t->P, R = t->R;
    memset(t->grams, 0, sizeof(double) * t->n * P);
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < (int64_t)t->L; ++l) {
        const uint64_t v = t->leaf_node[l];
        double* g = t->grams + v * P;
        for (uint64_t i = t->seg0[v]; i < t->seg1[v]; ++i) {
            const double* r = t->U + i * R;
            uint64_t idx = 0;
            for (uint64_t a = 0; a < R; ++a)
                for (uint64_t b = a; b < R; ++b, ++idx) g[idx] += r[a] * r[b];
        }
    }
    for (uint64_t v = t->n; v-- > 0;) {
        if (is_leaf(t, v)) continue;
        double* g = t->grams + v * P;
        const double* gl = t->grams + (2 * v + 1) * P;
        const double* gr = t->grams + (2 * v + 2) * P;
        for (uint64_t k = 0; k < P; ++k) g[k] = gl[k] + gr[k];
    }
}

static int tree_init(ko_tree* t, double* U, int own, uint64_t I, uint32_t R, uint64_t F,
                     const double* Y) {
    memset(t, 0, sizeof *t);
    if (I == 0 || R == 0) return fail(1, "build_sampler: empty matrix");
    if (F < 1) return fail(1, "build_sampler: leaf capacity must be positive");
    for (uint64_t k = 0; k < I * R; ++k)
        if (!isfinite(U[k])) return fail(1, "build_sampler: non-finite entries");
    t->I = I;
    t->R = R;
    t->F = F;
    t->P = (uint64_t)R * (R + 1) / 2;
    t->U = U;
    t->own_u = own;
    if (Y) {
        t->Y = malloc(sizeof(double) * R * R);
        memcpy(t->Y, Y, sizeof(double) * R * R);
    } else {
        t->y1 = malloc(sizeof(double) * R);
        for (uint32_t c = 0; c < R; ++c) t->y1[c] = 1.0;
    }
    t->L = (I + F - 1) / F;
    tree_topology(t);
    t->grams = malloc(sizeof(double) * t->n * t->P);
    tree_build(t);
    return 0;
}
static void tree_free(ko_tree* t) {
    free(t->seg0);
    free(t->seg1);
    free(t->leaf_node);
    free(t->grams);
    free(t->Y);
    free(t->y1);
    if (t->own_u) free(t->U);
}

int ko_tree_create(const double* U, uint64_t I, uint32_t R, uint64_t F, const double* Y,
                   ko_tree** out) {
    ko_tree* t = malloc(sizeof *t);
    double* u = malloc(sizeof(double) * (I * R ? I * R : 1));
    memcpy(u, U, sizeof(double) * I * R);
    int rc = tree_init(t, u, 1, I, R, F, Y);
    if (rc) {
        free(u);
        free(t);
        return rc;
    }
    *out = t;
    return 0;
}
/* init_tree over explicit leaf segments [offs[l], offs[l+1]) (:111-149); F becomes
 * the longest leaf (scan work size). Y == NULL -> rank-1 all-ones (from_sparse). */
int ko_tree_create_segments(const double* U, uint64_t I, uint32_t R, const uint64_t* offs, uint64_t L,
                            const double* Y, ko_tree** out) {
    if (L < 1 || offs[0] != 0 || offs[L] != I) return fail(1, "build_sampler: leaf segments must cover [0, I)");
    uint64_t fmax = 0;
    for (uint64_t l = 0; l < L; ++l) {
        if (offs[l + 1] <= offs[l]) return fail(1, "build_sampler: leaf segments must be non-empty and ascending");
        if (offs[l + 1] - offs[l] > fmax) fmax = offs[l + 1] - offs[l];
    }
    ko_tree* t = malloc(sizeof *t);
    double* u = malloc(sizeof(double) * (I * R ? I * R : 1));
    memcpy(u, U, sizeof(double) * I * R);
    memset(t, 0, sizeof *t);
    for (uint64_t k = 0; k < I * R; ++k)
        if (!isfinite(u[k])) {
            free(u);
            free(t);
            return fail(1, "build_sampler: non-finite entries");
        }
    t->I = I;
    t->R = R;
    t->F = fmax;
    t->P = (uint64_t)R * (R + 1) / 2;
    t->U = u;
    t->own_u = 1;
    if (Y) {
        t->Y = malloc(sizeof(double) * R * R);
        memcpy(t->Y, Y, sizeof(double) * R * R);
    } else {
        t->y1 = malloc(sizeof(double) * R);
        for (uint32_t c = 0; c < R; ++c) t->y1[c] = 1.0;
    }
    t->L = L;
    t->offs = offs;
    tree_topology(t);
    t->offs = NULL;
    t->grams = malloc(sizeof(double) * t->n * t->P);
    tree_build(t);
    *out = t;
    return 0;
}
void ko_tree_destroy(ko_tree* t) {
    if (!t) return;
    tree_free(t);
    free(t);
}
uint64_t ko_tree_node_count(const ko_tree* t) { return t->n; }
uint64_t ko_tree_leaf_count(const ko_tree* t) { return t->L; }
const double* ko_tree_node_packed(const ko_tree* t, uint64_t node) { return t->grams + node * t->P; }
void ko_tree_node_segment(const ko_tree* t, uint64_t node, uint64_t* first, uint64_t* last) {
    *first = t->seg0[node];
    *last = t->seg1[node];
}

static void fold_weights(const ko_tree* t, const double* h, double* folded) { /* :193-211 */
    const uint64_t R = t->R;
    uint64_t idx = 0;
    if (t->y1) {
        for (uint64_t a = 0; a < R; ++a) {
            const double za = h[a] * t->y1[a];
            for (uint64_t b = a; b < R; ++b, ++idx) {
                const double zb = h[b] * t->y1[b];
                folded[idx] = (a == b ? 1.0 : 2.0) * za * zb;
            }
        }
    } else {
        for (uint64_t a = 0; a < R; ++a)
            for (uint64_t b = a; b < R; ++b, ++idx)
                folded[idx] = (a == b ? 1.0 : 2.0) * h[a] * h[b] * t->Y[a * R + b];
    }
}
static double packed_inner(const ko_tree* t, uint64_t node, const double* folded) { /* :213-218 */
    const double* g = t->grams + node * t->P;
    double acc = 0.0;
    for (uint64_t k = 0; k < t->P; ++k) acc += g[k] * folded[k];
    return acc;
}
static void segment_masses(const ko_tree* t, uint64_t first, uint64_t last, const double* h,
                           const double* folded, double* out) { /* :220-252 */
    const uint64_t R = t->R;
    if (t->y1) {
        for (uint64_t i = first; i < last; ++i) {
            double dot = 0.0;
            const double* r = t->U + i * R;
            for (uint64_t c = 0; c < R; ++c) dot += r[c] * (h[c] * t->y1[c]);
            out[i - first] = dot * dot;
        }
    } else {
        for (uint64_t i = first; i < last; ++i) {
            const double* r = t->U + i * R;
            double acc = 0.0;
            uint64_t idx = 0;
            for (uint64_t a = 0; a < R; ++a) {
                const double ra = r[a];
                for (uint64_t b = a; b < R; ++b, ++idx) acc += folded[idx] * ra * r[b];
            }
            out[i - first] = acc;
        }
    }
}

/* row_sample :258-293. Returns 0 and *row on success. work: P + F doubles.
 * *margin (if non-NULL) is min-updated with |cutoff - d| of every comparison. */
static int row_sample(const ko_tree* t, const double* h, rng_t* rng, double* work, uint64_t* row,
                      double* margin) {
    double* folded = work;
    double* masses = work + t->P;
    fold_weights(t, h, folded);
    const double C = packed_inner(t, 0, folded);
    if (!isfinite(C)) return fail(2, "row_sample: non-finite normalizer");
    if (C <= 0.0) return fail(2, "row_sample: degenerate distribution (C <= 0)");
    const double inv_c = 1.0 / C;
    const double d = rng_uniform(rng);
    uint64_t node = 0;
    double low = 0.0;
    double mg = margin ? *margin : 0.0;
    while (!is_leaf(t, node)) {
        const double cutoff = low + inv_c * packed_inner(t, 2 * node + 1, folded);
        mg = fmin(mg, fabs(cutoff - d));
        if (cutoff >= d) {
            node = 2 * node + 1;
        } else {
            low = cutoff;
            node = 2 * node + 2;
        }
    }
    const uint64_t first = t->seg0[node], last = t->seg1[node];
    segment_masses(t, first, last, h, folded, masses);
    double cum = low;
    uint64_t last_nonzero = UINT64_MAX;
    for (uint64_t i = first; i < last; ++i) {
        const double m = inv_c * masses[i - first];
        if (m > 0.0) last_nonzero = i;
        cum += m;
        mg = fmin(mg, fabs(cum - d));
        if (cum >= d) {
            *row = i;
            if (margin) *margin = mg;
            return 0;
        }
    }
    *row = last_nonzero != UINT64_MAX ? last_nonzero : last - 1;
    if (margin) *margin = mg;
    return 0;
}

int ko_tree_row_sample(const ko_tree* t, const double* h, uint64_t seed, uint64_t stream,
                       uint64_t n, uint64_t* out) {
    rng_t rng;
    rng_init(&rng, seed, stream);
    double* work = malloc(sizeof(double) * (t->P + t->F));
    int rc = 0;
    for (uint64_t i = 0; i < n && !rc; ++i) rc = row_sample(t, h, &rng, work, out + i, NULL);
    free(work);
    return rc;
}

/* update_entry :358-409 (dense path; patches every node on the path — the
 * compact reference patches the stored subset with the same values). */
static void tree_patch(ko_tree* t, uint64_t r, uint64_t c, double old, double delta) {
    const uint64_t R = t->R;
    uint64_t node = 0;
    for (;;) {
        double* g = t->grams + node * t->P;
        const double* row = t->U + r * R;
        for (uint64_t b = 0; b < R; ++b) {
            if (b == c) continue;
            const uint64_t a0 = b < c ? b : c, b0 = b < c ? c : b;
            g[a0 * R - a0 * (a0 - 1) / 2 + (b0 - a0)] += delta * row[b];
        }
        g[c * R - c * (c - 1) / 2] += 2.0 * delta * old + delta * delta;
        if (is_leaf(t, node)) break;
        node = (r < t->seg1[2 * node + 1]) ? 2 * node + 1 : 2 * node + 2;
    }
}
int ko_tree_update_entry(ko_tree* t, uint64_t r, uint64_t c, double v) {
    if (!(r < t->I && c < t->R)) return fail(1, "update_entry: index out of range");
    if (!isfinite(v)) return fail(1, "update_entry: non-finite value");
    const double old = t->U[r * t->R + c];
    tree_patch(t, r, c, old, v - old);
    t->U[r * t->R + c] = v;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* KrpSampler — krp_sampler.cpp                                              */
/* ------------------------------------------------------------------------ */
struct ko_krp {
    uint32_t N, R;
    uint64_t* I;
    double** U; /* owned, shared with trees */
    double** G; /* cached gram(U) */
    ko_tree* trees;
};

int ko_krp_create(const double* const* U, const uint64_t* I, uint32_t N, uint32_t R,
                  ko_krp** out) { /* :41-62 */
    if (N == 0) return fail(1, "KrpSampler: factor list is empty");
    for (uint32_t k = 0; k < N; ++k) {
        if (I[k] == 0 || R == 0) return fail(1, "KrpSampler: empty factor");
        for (uint64_t e = 0; e < I[k] * R; ++e)
            if (!isfinite(U[k][e])) return fail(1, "KrpSampler: non-finite factor entries");
    }
    ko_krp* s = calloc(1, sizeof *s);
    s->N = N;
    s->R = R;
    s->I = malloc(sizeof(uint64_t) * N);
    s->U = malloc(sizeof(double*) * N);
    s->G = malloc(sizeof(double*) * N);
    s->trees = calloc(N, sizeof(ko_tree));
    for (uint32_t k = 0; k < N; ++k) {
        s->I[k] = I[k];
        s->U[k] = malloc(sizeof(double) * I[k] * R);
        memcpy(s->U[k], U[k], sizeof(double) * I[k] * R);
        s->G[k] = malloc(sizeof(double) * R * R);
        ko_gram(s->U[k], I[k], R, s->G[k]);
        tree_init(&s->trees[k], s->U[k], 0, I[k], R, R, NULL);
    }
    double* G = malloc(sizeof(double) * R * R);
    for (uint32_t e = 0; e < R * R; ++e) G[e] = 1.0;
    for (uint32_t k = 0; k < N; ++k) hadamard_into(G, s->G[k], (size_t)R * R);
    double tr = 0.0;
    for (uint32_t r = 0; r < R; ++r) tr += G[r * R + r];
    free(G);
    if (!(tr > 0.0)) {
        ko_krp_destroy(s);
        return fail(1, "KrpSampler: Khatri-Rao product is identically zero");
    }
    *out = s;
    return 0;
}
void ko_krp_destroy(ko_krp* s) {
    if (!s) return;
    for (uint32_t k = 0; k < s->N; ++k) {
        tree_free(&s->trees[k]);
        free(s->U[k]);
        free(s->G[k]);
    }
    free(s->trees);
    free(s->U);
    free(s->G);
    free(s->I);
    free(s);
}
int ko_krp_factor_gram(const ko_krp* s, uint32_t j, double* out) {
    if (j >= s->N) return fail(1, "factor_gram: index out of range");
    memcpy(out, s->G[j], sizeof(double) * s->R * s->R);
    return 0;
}
const double* ko_krp_node_packed(const ko_krp* s, uint32_t j, uint64_t node) {
    return ko_tree_node_packed(&s->trees[j], node);
}
uint64_t ko_krp_leaf_count(const ko_krp* s, uint32_t j) { return s->trees[j].L; }

static int included(const ko_krp* s, int64_t excluded, uint32_t* inc, uint32_t* ninc) { /* :64-72 */
    if (excluded >= 0 && (uint64_t)excluded >= s->N)
        return fail(1, "KrpSampler: excluded index out of range");
    *ninc = 0;
    for (uint32_t k = 0; k < s->N; ++k)
        if (excluded < 0 || (uint32_t)excluded != k) inc[(*ninc)++] = k;
    if (*ninc == 0) return fail(1, "KrpSampler: no factors left after exclusion");
    return 0;
}

/* G = hadamard of included Grams; eig; rank; pinv (krp_sampler.cpp:89-96) */
static int gram_pinv(const ko_krp* s, const uint32_t* inc, uint32_t ninc, double* gp,
                     uint64_t* rank) {
    const uint32_t R = s->R;
    double* G = malloc(sizeof(double) * R * R);
    double* V = malloc(sizeof(double) * R * R);
    double* l = malloc(sizeof(double) * R);
    for (uint32_t e = 0; e < R * R; ++e) G[e] = 1.0;
    for (uint32_t p = 0; p < ninc; ++p) hadamard_into(G, s->G[inc[p]], (size_t)R * R);
    int rc = ko_eigh(G, R, V, l);
    if (!rc) {
        *rank = numerical_rank(l, R);
        pinv_from_eigen(V, l, R, gp);
    }
    free(G);
    free(V);
    free(l);
    return rc;
}
static void downstream_gram(const ko_krp* s, const uint32_t* inc, uint32_t ninc, uint32_t pos,
                            const double* gp, double* out) { /* :74-80 */
    const uint32_t R = s->R;
    for (uint32_t e = 0; e < R * R; ++e) out[e] = 1.0;
    hadamard_into(out, gp, (size_t)R * R);
    for (uint32_t p = pos + 1; p < ninc; ++p) hadamard_into(out, s->G[inc[p]], (size_t)R * R);
}

int ko_krp_sample(const ko_krp* s, int64_t excluded, uint64_t J, uint64_t seed,
                  uint64_t draw_offset, uint32_t* idx, double* prob, double* rows,
                  double* margin) { /* :82-151; stream = draw_offset + d (0 = reference) */
    if (J < 1) return fail(1, "KrpSample: sample count must be positive");
    const uint32_t N = s->N, R = s->R;
    uint32_t inc[64], ninc;
    int rc = included(s, excluded, inc, &ninc);
    if (rc) return rc;
    double* gp = malloc(sizeof(double) * R * R);
    uint64_t rank = 0;
    rc = gram_pinv(s, inc, ninc, gp, &rank);
    if (!rc && rank == 0) rc = fail(2, "KRPSample: Khatri-Rao product of included factors is zero");
    if (rc) {
        free(gp);
        return rc;
    }
    for (uint64_t e = 0; e < J * N; ++e) idx[e] = KO_EXCLUDED;
    for (uint64_t e = 0; e < J * R; ++e) rows[e] = 1.0;
    if (margin)
        for (uint64_t d = 0; d < J; ++d) margin[d] = INFINITY;
    rng_t* rngs = malloc(sizeof(rng_t) * J);
    for (uint64_t d = 0; d < J; ++d) rng_init(&rngs[d], seed, draw_offset + d);

    double* gk = malloc(sizeof(double) * R * R);
    double* V = malloc(sizeof(double) * R * R);
    double* l = malloc(sizeof(double) * R);
    double* scaled = malloc(sizeof(double) * R * R);
    volatile int err = 0;
    for (uint32_t pos = 0; pos < ninc && !err; ++pos) {
        const uint32_t k = inc[pos];
        downstream_gram(s, inc, ninc, pos, gp, gk);
        rc = ko_eigh(gk, R, V, l);
        if (rc) break;
        for (uint32_t u = 0; u < R; ++u) {
            const double sq = sqrt(l[u]);
            for (uint32_t c = 0; c < R; ++c) scaled[u * R + c] = sq * V[c * R + u];
        }
        ko_tree est; /* SegmentTreeSampler(scaled, 1, grams_[k]) :123 */
        tree_init(&est, scaled, 0, R, R, 1, s->G[k]);
        const ko_tree* zk = &s->trees[k];
        const double* uk = s->U[k];
#pragma omp parallel
        {
            double* work = malloc(sizeof(double) * (zk->P + zk->F + est.P + 1));
            double* ht = malloc(sizeof(double) * R);
#pragma omp for schedule(static)
            for (int64_t d = 0; d < (int64_t)J; ++d) {
                double* h = rows + (uint64_t)d * R;
                uint64_t u, t;
                double* mg = margin ? margin + d : NULL;
                if (row_sample(&est, h, &rngs[d], work, &u, mg)) {
                    err = 1;
                    continue;
                }
                for (uint32_t c = 0; c < R; ++c) ht[c] = h[c] * V[c * R + u];
                if (row_sample(zk, ht, &rngs[d], work, &t, mg)) {
                    err = 1;
                    continue;
                }
                idx[(uint64_t)d * N + k] = (uint32_t)t;
                const double* row = uk + t * R;
                for (uint32_t c = 0; c < R; ++c) h[c] *= row[c];
            }
            free(work);
            free(ht);
        }
        tree_free(&est);
    }
    if (!rc && err) rc = 2;
    if (!rc && prob)
        for (uint64_t d = 0; d < J; ++d)
            prob[d] = quadratic_form(rows + d * R, gp, R, rows + d * R) / (double)rank;
    free(rngs);
    free(gk);
    free(V);
    free(l);
    free(scaled);
    free(gp);
    return rc;
}

int ko_krp_sample_one_stage(const ko_krp* s, int64_t excluded, uint64_t J, uint64_t seed,
                            uint64_t draw_offset, uint32_t* idx, double* prob, double* rows,
                            double* margin) {
    if (J < 1) return fail(1, "KrpSample: sample count must be positive");
    const uint32_t N = s->N, R = s->R;
    uint32_t inc[64], ninc;
    int rc = included(s, excluded, inc, &ninc);
    if (rc) return rc;
    double* gp = malloc(sizeof(double) * R * R);
    uint64_t rank = 0;
    rc = gram_pinv(s, inc, ninc, gp, &rank);
    if (!rc && rank == 0) rc = fail(2, "one_stage: zero KRP");
    if (rc) {
        free(gp);
        return rc;
    }
    for (uint64_t e = 0; e < J * N; ++e) idx[e] = KO_EXCLUDED;
    for (uint64_t e = 0; e < J * R; ++e) rows[e] = 1.0;
    if (margin)
        for (uint64_t d = 0; d < J; ++d) margin[d] = INFINITY;
    rng_t* rngs = malloc(sizeof(rng_t) * J);
    for (uint64_t d = 0; d < J; ++d) rng_init(&rngs[d], seed, draw_offset + d);
    double* Y = malloc(sizeof(double) * R * R);
    volatile int err = 0;
    for (uint32_t pos = 0; pos < ninc; ++pos) {
        const uint32_t k = inc[pos];
        downstream_gram(s, inc, ninc, pos, gp, Y);
        ko_tree t; /* SegmentTreeSampler(U_k, R, G_{>k}) shares the Z-tree Grams */
        t = s->trees[k];
        t.Y = Y;
        t.y1 = NULL;
        const double* uk = s->U[k];
#pragma omp parallel
        {
            double* work = malloc(sizeof(double) * (t.P + t.F));
#pragma omp for schedule(static)
            for (int64_t d = 0; d < (int64_t)J; ++d) {
                double* h = rows + (uint64_t)d * R;
                uint64_t r;
                if (row_sample(&t, h, &rngs[d], work, &r, margin ? margin + d : NULL)) {
                    err = 1;
                    continue;
                }
                idx[(uint64_t)d * N + k] = (uint32_t)r;
                const double* row = uk + r * R;
                for (uint32_t c = 0; c < R; ++c) h[c] *= row[c];
            }
            free(work);
        }
    }
    if (err) rc = 2;
    if (!rc && prob)
        for (uint64_t d = 0; d < J; ++d)
            prob[d] = quadratic_form(rows + d * R, gp, R, rows + d * R) / (double)rank;
    free(Y);
    free(rngs);
    free(gp);
    return rc;
}

int ko_krp_conditional(const ko_krp* s, int64_t excluded, uint32_t k, const double* h,
                       double* probs, double* mixture) { /* :153-196 */
    const uint32_t R = s->R;
    uint32_t inc[64], ninc, pos = UINT32_MAX;
    int rc = included(s, excluded, inc, &ninc);
    if (rc) return rc;
    for (uint32_t p = 0; p < ninc; ++p)
        if (inc[p] == k) pos = p;
    if (pos == UINT32_MAX) return fail(1, "conditional: factor k is not included");
    double* gp = malloc(sizeof(double) * R * R);
    double* gk = malloc(sizeof(double) * R * R);
    double* V = malloc(sizeof(double) * R * R);
    double* l = malloc(sizeof(double) * R);
    double* hc = malloc(sizeof(double) * R * R);
    double* ht = malloc(sizeof(double) * R);
    const uint64_t I = s->I[k];
    double* col = malloc(sizeof(double) * I);
    uint64_t rank;
    rc = gram_pinv(s, inc, ninc, gp, &rank);
    if (!rc) {
        downstream_gram(s, inc, ninc, pos, gp, gk);
        rc = ko_eigh(gk, R, V, l);
    }
    if (!rc) {
        for (uint32_t e = 0; e < R * R; ++e) hc[e] = 1.0;
        hadamard_into(hc, s->G[k], (size_t)R * R);
        hadamard_into(hc, gk, (size_t)R * R);
        const double C = quadratic_form(h, hc, R, h);
        if (!(C > 0.0)) rc = fail(2, "conditional: zero normalizer");
        else {
            const double* uk = s->U[k];
            for (uint64_t t = 0; t < I; ++t) probs[t] = 0.0;
            for (uint32_t u = 0; u < R; ++u) mixture[u] = 0.0;
            for (uint32_t u = 0; u < R; ++u) {
                if (l[u] == 0.0) continue;
                for (uint32_t c = 0; c < R; ++c) ht[c] = h[c] * V[c * R + u];
                double norm1 = 0.0;
                for (uint64_t t = 0; t < I; ++t) {
                    const double* row = uk + t * R;
                    double dot = 0.0;
                    for (uint32_t c = 0; c < R; ++c) dot += row[c] * ht[c];
                    col[t] = dot * dot;
                    norm1 += col[t];
                }
                if (norm1 == 0.0) continue;
                const double w = l[u] * norm1 / C;
                mixture[u] = w;
                for (uint64_t t = 0; t < I; ++t) probs[t] += w * col[t] / norm1;
            }
        }
    }
    free(gp);
    free(gk);
    free(V);
    free(l);
    free(hc);
    free(ht);
    free(col);
    return rc;
}

int ko_krp_update_factor(ko_krp* s, uint32_t j, const double* U, uint64_t I) { /* :198-205 */
    if (j >= s->N) return fail(1, "update_factor: index out of range");
    if (I == 0) return fail(1, "update_factor: invalid factor");
    for (uint64_t e = 0; e < I * s->R; ++e)
        if (!isfinite(U[e])) return fail(1, "update_factor: invalid factor");
    tree_free(&s->trees[j]);
    free(s->U[j]);
    s->I[j] = I;
    s->U[j] = malloc(sizeof(double) * I * s->R);
    memcpy(s->U[j], U, sizeof(double) * I * s->R);
    ko_gram(s->U[j], I, s->R, s->G[j]);
    return tree_init(&s->trees[j], s->U[j], 0, I, s->R, s->R, NULL);
}

int ko_krp_update_entries(ko_krp* s, uint32_t j, const uint64_t* r, const uint32_t* c,
                          const double* v, uint64_t n) { /* :207-228 */
    if (j >= s->N) return fail(1, "update_factor_entry: index out of range");
    const uint32_t R = s->R;
    for (uint64_t e = 0; e < n; ++e) {
        if (!(r[e] < s->I[j] && c[e] < R)) return fail(1, "update_factor_entry: entry out of range");
        if (!isfinite(v[e])) return fail(1, "update_factor_entry: non-finite value");
        double* U = s->U[j];
        const double old = U[r[e] * R + c[e]];
        const double delta = v[e] - old;
        tree_patch(&s->trees[j], r[e], c[e], old, delta);
        double* G = s->G[j];
        for (uint32_t b = 0; b < R; ++b) {
            if (b == c[e]) continue;
            G[c[e] * R + b] += delta * U[r[e] * R + b];
            G[b * R + c[e]] += delta * U[r[e] * R + b];
        }
        G[c[e] * R + c[e]] += 2.0 * delta * old + delta * delta;
        U[r[e] * R + c[e]] = v[e];
    }
    return 0;
}

/* reference.cpp:30-48 + normalization as in test_krp_sampler.cpp:53-59 */
int ko_leverage(const double* const* U, const uint64_t* I, uint32_t N, uint32_t R, double* out) {
    uint64_t rows = 1;
    for (uint32_t k = 0; k < N; ++k) rows *= I[k];
    double* A = malloc(sizeof(double) * rows * R);
    /* ascending KRP: first factor slowest (khatri_rao_columns :85-95) */
    for (uint64_t f = 0; f < rows; ++f) {
        uint64_t rem = f;
        uint64_t ik[64];
        for (uint32_t k = N; k-- > 0;) {
            ik[k] = rem % I[k];
            rem /= I[k];
        }
        for (uint32_t c = 0; c < R; ++c) {
            double v = U[0][ik[0] * R + c];
            for (uint32_t k = 1; k < N; ++k) v = v * U[k][ik[k] * R + c];
            A[f * R + c] = v;
        }
    }
    double* G = calloc((size_t)R * R, sizeof(double));
    for (uint64_t i = 0; i < rows; ++i)
        for (uint32_t a = 0; a < R; ++a)
            for (uint32_t b = 0; b < R; ++b) G[a * R + b] += A[i * R + a] * A[i * R + b];
    double* P = malloc(sizeof(double) * R * R);
    uint64_t rk;
    int rc = ko_pinv(G, R, P, &rk);
    if (!rc) {
        double tot = 0.0;
        for (uint64_t i = 0; i < rows; ++i) {
            out[i] = quadratic_form(A + i * R, P, R, A + i * R);
            tot += out[i];
        }
        for (uint64_t i = 0; i < rows; ++i) out[i] /= tot;
    }
    free(A);
    free(G);
    free(P);
    return rc;
}

int ko_sampling_weights(const double* prob, uint64_t n, uint64_t J, double* w) { /* sketch.cpp:36-52 */
    if (J < 1) return fail(1, "make_sampling_weights: J must be positive");
    for (uint64_t d = 0; d < n; ++d) {
        const double q = prob[d];
        if (!(q > 0.0) || !isfinite(q))
            return fail(1, "make_sampling_weights: sampled index has zero probability");
        w[d] = 1.0 / sqrt((double)J * q);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* CP-ARLS-LEV product sampler — sketch.cpp:86-149                           */
/* ------------------------------------------------------------------------ */
/* Per included factor: p_i = u_i^T pinv(gram(U)) u_i (quadratic_form order),
 * normalised by their sequential sum, cumulative table by a sequential running
 * sum (:104-122). Draw d: CounterRng(seed, d), per included factor in order one
 * uniform, t = min(lower_bound(cum, u * cum.back()), I - 1) (:19-26); prob = prod
 * p[t], rows = Hadamard of the drawn rows (:133-145). margin (nullable, J): per
 * draw the smallest |cum[x] - target| over the two bin edges of every pick. */
int ko_product_lev_sample(const double* const* U, const uint64_t* I, uint32_t N, uint32_t R, int64_t excluded,
                          uint64_t J, uint64_t seed, uint32_t* idx, double* prob, double* rows, double* margin) {
    if (N == 0) return fail(1, "product_lev_sample: factor list is empty");
    if (J < 1) return fail(1, "product_lev_sample: J must be positive");
    if (excluded >= 0 && (uint64_t)excluded >= N) return fail(1, "product_lev_sample: excluded index out of range");
    if (N == 1 && excluded == 0) return fail(1, "product_lev_sample: no factors left after exclusion");
    double** p = calloc(N, sizeof(double*));
    double** c = calloc(N, sizeof(double*));
    double* G = malloc(sizeof(double) * R * R);
    double* Gp = malloc(sizeof(double) * R * R);
    int rc = 0;
    for (uint32_t k = 0; k < N && !rc; ++k) {
        if ((int64_t)k == excluded) continue;
        ko_gram(U[k], I[k], R, G);
        uint64_t rk = 0;
        rc = ko_pinv(G, R, Gp, &rk);
        if (rc) break;
        p[k] = malloc(sizeof(double) * I[k]);
        c[k] = malloc(sizeof(double) * I[k]);
        double total = 0.0;
        for (uint64_t i = 0; i < I[k]; ++i) {
            p[k][i] = quadratic_form(U[k] + i * R, Gp, R, U[k] + i * R);
            total += p[k][i];
        }
        if (!(total > 0.0)) {
            rc = fail(2, "product_lev_sample: zero factor");
            break;
        }
        double run = 0.0;
        for (uint64_t i = 0; i < I[k]; ++i) {
            p[k][i] /= total;
            run += p[k][i];
            c[k][i] = run;
        }
    }
    if (!rc) {
#pragma omp parallel for schedule(static)
        for (int64_t d = 0; d < (int64_t)J; ++d) {
            rng_t rng;
            rng_init(&rng, seed, (uint64_t)d);
            double* h = rows + (uint64_t)d * R;
            for (uint32_t a = 0; a < R; ++a) h[a] = 1.0;
            double pr = 1.0, mg = INFINITY;
            for (uint32_t k = 0; k < N; ++k) {
                idx[(uint64_t)d * N + k] = 0xFFFFFFFFu;
                if ((int64_t)k == excluded) continue;
                const uint64_t n = I[k];
                const double target = rng_uniform(&rng) * c[k][n - 1];
                uint64_t lo = 0, hi = n; /* first x with c[x] >= target */
                while (lo < hi) {
                    const uint64_t mid = lo + (hi - lo) / 2;
                    if (c[k][mid] < target) lo = mid + 1;
                    else hi = mid;
                }
                const uint64_t t = lo < n - 1 ? lo : n - 1;
                mg = fmin(mg, fabs(c[k][t] - target));
                if (t > 0) mg = fmin(mg, fabs(c[k][t - 1] - target));
                idx[(uint64_t)d * N + k] = (uint32_t)t;
                pr *= p[k][t];
                const double* r = U[k] + t * R;
                for (uint32_t a = 0; a < R; ++a) h[a] *= r[a];
            }
            prob[d] = pr;
            if (margin) margin[d] = mg;
        }
    }
    for (uint32_t k = 0; k < N; ++k) {
        free(p[k]);
        free(c[k]);
    }
    free(p);
    free(c);
    free(G);
    free(Gp);
    return rc;
}
