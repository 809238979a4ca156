/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference's exact KRP leverage sampler
 * (/root/reference/proj, krplev). Every function cites the reference
 * file:line it restates. Pinned bit-for-bit against the reference itself
 * (oracle/_ref, built from the unmodified sources) by tests/test_oracle.py and
 * against committed fixtures in tests/golden/ (tests/golden/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 */
#ifndef KRP_ORACLE_H
#define KRP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 0 ok, 1 invalid_argument, 2 runtime_error (reference exception classes). */
const char* ko_last_error(void);

/* CounterRng, rng.hpp:13-48 */
uint64_t ko_mix(uint64_t z);
void ko_uniforms(uint64_t seed, uint64_t stream, uint64_t n, double* out);
void ko_normals(uint64_t seed, uint64_t stream, uint64_t n, double* out);
uint64_t ko_derive_seed(uint64_t seed, uint64_t a, uint64_t b);

/* dense_kernels.cpp */
void ko_gram(const double* U, uint64_t I, uint32_t R, double* G);
int ko_eigh(const double* G, uint32_t n, double* V, double* lam);
int ko_pinv(const double* G, uint32_t n, double* out, uint64_t* rank);

/* SegmentTreeSampler (full-store layout; Y == NULL -> rank-1 ones) */
typedef struct ko_tree ko_tree;
int ko_tree_create(const double* U, uint64_t I, uint32_t R, uint64_t F, const double* Y,
                   ko_tree** out);
int ko_tree_create_segments(const double* U, uint64_t I, uint32_t R, const uint64_t* offs, uint64_t L,
                            const double* Y, ko_tree** out);
void ko_tree_destroy(ko_tree* t);
uint64_t ko_tree_node_count(const ko_tree* t);
uint64_t ko_tree_leaf_count(const ko_tree* t);
/* packed upper triangle (P entries) of any node */
const double* ko_tree_node_packed(const ko_tree* t, uint64_t node);
void ko_tree_node_segment(const ko_tree* t, uint64_t node, uint64_t* first, uint64_t* last);
int ko_tree_row_sample(const ko_tree* t, const double* h, uint64_t seed, uint64_t stream,
                       uint64_t n, uint64_t* out);
int ko_tree_update_entry(ko_tree* t, uint64_t r, uint64_t c, double v);

/* CP-ARLS-LEV product_lev_sample (sketch.cpp:86-149); excluded < 0: none */
int ko_product_lev_sample(const double* const* U, const uint64_t* I, uint32_t N, uint32_t R, int64_t excluded,
                          uint64_t J, uint64_t seed, uint32_t* idx, double* prob, double* rows, double* margin);

/* KrpSampler */
typedef struct ko_krp ko_krp;
int ko_krp_create(const double* const* U, const uint64_t* I, uint32_t N, uint32_t R,
                  ko_krp** out);
void ko_krp_destroy(ko_krp* k);
int ko_krp_factor_gram(const ko_krp* k, uint32_t j, double* out);
/* compact-layout node (root or odd id) packed Gram */
const double* ko_krp_node_packed(const ko_krp* k, uint32_t j, uint64_t node);
uint64_t ko_krp_leaf_count(const ko_krp* k, uint32_t j);
/* two-stage sample, krp_sampler.cpp:82-151. margin (nullable, J): per draw the
 * smallest |cutoff - d| over every branch/scan comparison made. */
int ko_krp_sample(const ko_krp* k, int64_t excluded, uint64_t J, uint64_t seed,
                  uint64_t draw_offset, uint32_t* idx, double* prob, double* rows, double* margin);
/* one-stage chain */
int ko_krp_sample_one_stage(const ko_krp* k, int64_t excluded, uint64_t J, uint64_t seed,
                            uint64_t draw_offset, uint32_t* idx, double* prob, double* rows,
                            double* margin);
int ko_krp_conditional(const ko_krp* k, int64_t excluded, uint32_t kk, const double* h,
                       double* probs, double* mixture);
int ko_krp_update_factor(ko_krp* k, uint32_t j, const double* U, uint64_t I);
int ko_krp_update_entries(ko_krp* k, uint32_t j, const uint64_t* r, const uint32_t* c,
                          const double* v, uint64_t n);

/* reference/reference.cpp:30-48, normalized to sum 1 */
int ko_leverage(const double* const* U, const uint64_t* I, uint32_t N, uint32_t R, double* out);

/* sketch.cpp:36-52 */
int ko_sampling_weights(const double* prob, uint64_t n, uint64_t J, double* w);

#ifdef __cplusplus
}
#endif
#endif
