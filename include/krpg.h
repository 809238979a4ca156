/* krpg — B200-native exact Khatri-Rao-product leverage-score sampler (C ABI).
 *
 * This is the drop-in boundary beneath the reference's C++ KrpSampler API
 * (/root/reference/proj/include/krplev/krp_sampler.hpp). Every entry point is
 * plain C: handles, raw pointers and sizes, no torch / C++ types. All state
 * (factors, segment trees, scratch) lives in HBM on one device; host buffers
 * passed in or out are row-major fp64 like krplev::Matrix (matrix.hpp:13-48).
 *
 * Return codes mirror the reference's exception classes so a C++ wrapper can
 * rethrow the same types:
 *   KRPG_OK (0), KRPG_INVALID_ARGUMENT (1) -> std::invalid_argument,
 *   KRPG_RUNTIME_ERROR (2) -> std::runtime_error, KRPG_CUDA_ERROR (3).
 * krpg_last_error() returns the thread-local message of the last failure.
 *
 * Threading: create / update_* / destroy need exclusive access to a handle;
 * sample / conditional / *_gram may be called concurrently (each call is
 * serialised on the handle's stream internally).
 */
#ifndef KRPG_H
#define KRPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KRPG_OK 0
#define KRPG_INVALID_ARGUMENT 1
#define KRPG_RUNTIME_ERROR 2
#define KRPG_CUDA_ERROR 3

/* SampleBatch::kExcluded, krp_sampler.hpp:28 */
#define KRPG_EXCLUDED 0xFFFFFFFFu

/* factor storage precision on device (fp64 arithmetic either way) */
#define KRPG_STORE_F64 0u
#define KRPG_STORE_F32 1u

/* sampling modes */
#define KRPG_MODE_TWO_STAGE 0u /* bit-exact to KrpSampler::sample (krp_sampler.cpp:82-151) */
#define KRPG_MODE_ONE_STAGE 1u /* M = G+ o hh^T o G_{>k} per draw (SURVEY §8(c) chain) */

typedef struct krpg_sampler* krpg_t;

const char* krpg_last_error(void);
/* 1 if a CUDA device is usable (never falls back to the CPU otherwise). */
int krpg_device_count(void);

/* Replaces KrpSampler::KrpSampler(std::vector<Matrix>)  (krp_sampler.cpp:41-62).
 * factors[k] is an I[k] x R row-major fp64 host matrix. storage selects the
 * device copy precision (KRPG_STORE_F32 rounds each entry to fp32 once). */
int krpg_create(const double* const* factors, const uint64_t* I, uint32_t N, uint32_t R,
                uint32_t storage, int device, krpg_t* out);
/* Same, with factors already resident on `device` (row-major, storage dtype). */
int krpg_create_device(const void* const* dev_factors, const uint64_t* I, uint32_t N,
                       uint32_t R, uint32_t storage, int device, krpg_t* out);
int krpg_destroy(krpg_t h);

int krpg_info(krpg_t h, uint32_t* N, uint32_t* R, uint64_t* I /* N entries, nullable */);

/* Replaces KrpSampler::factor_gram(j) (krp_sampler.hpp:66): R x R, taken from
 * the segment-tree root (the device sum of all leaf Grams). */
int krpg_factor_gram(krpg_t h, uint32_t j, double* out);
/* Copy of factor j as stored on device, up-cast to fp64 (I x R). */
int krpg_factor(krpg_t h, uint32_t j, double* out);

/* Tree introspection (SegmentTreeSampler test support, segment_tree_sampler.hpp:64-95).
 * The device stores the reference's compact layout: slot 0 = root, slot s>=1 =
 * heap node 2s-1 (left children), each a packed upper triangle (hpp:111-115). */
int krpg_tree_shape(krpg_t h, uint32_t j, uint64_t* leaf_count, uint64_t* node_count);
/* unpacked R x R Gram of a stored node (root or odd heap id) */
int krpg_node_gram(krpg_t h, uint32_t j, uint64_t node, double* out);
/* all L stored packed Grams, slot order (L x R(R+1)/2) */
int krpg_tree_grams(krpg_t h, uint32_t j, double* out);

/* Replaces KrpSampler::sample(excluded, J, seed) (krp_sampler.cpp:82-151).
 * excluded < 0 means none. Host outputs (each nullable): idx J x N (excluded
 * column = KRPG_EXCLUDED), prob J, rows J x R. draw_offset shifts the CounterRng
 * stream ids (stream = draw_offset + d) so J can be sharded across devices with
 * results identical to one big call. margin (nullable, J): per draw the smallest
 * |cutoff - u| over all branch/scan comparisons (boundary-draw accounting). */
int krpg_sample(krpg_t h, int64_t excluded, uint64_t J, uint64_t seed, uint64_t draw_offset,
                uint32_t mode, uint32_t* idx, double* prob, double* rows, double* margin);
/* Same with device output pointers on the handle's device (any nullable);
 * stream 0 = the handle's own stream. Does not synchronise the host unless an
 * error check needs it (see krpg_sync). */
int krpg_sample_device(krpg_t h, int64_t excluded, uint64_t J, uint64_t seed,
                       uint64_t draw_offset, uint32_t mode, uint32_t* d_idx, double* d_prob,
                       double* d_rows, double* d_margin);
int krpg_sync(krpg_t h);
/* The handle's CUDA stream (cudaStream_t) for event timing by callers. */
void* krpg_stream(krpg_t h);

/* Replaces KrpSampler::conditional(excluded, k, h) (krp_sampler.cpp:153-196).
 * probs: I_k, mixture: R. */
int krpg_conditional(krpg_t h, int64_t excluded, uint32_t k, const double* hist, double* probs,
                     double* mixture);

/* Replaces KrpSampler::update_factor(j, U) (krp_sampler.cpp:198-205): full device rebuild. */
int krpg_update_factor(krpg_t h, uint32_t j, const double* U, uint64_t I);
/* Same with the new factor already on the handle's device (storage dtype), e.g.
 * produced by a device-side STS-CP solve (cp_als.cpp:293-313). */
int krpg_update_factor_device(krpg_t h, uint32_t j, const void* dU, uint64_t I);
/* Rebuild factor j's tree from its current device rows (timing / recovery). */
int krpg_rebuild(krpg_t h, uint32_t j);
/* Replaces a sequence of KrpSampler::update_factor_entry(j, r[i], c[i], v[i])
 * (krp_sampler.cpp:207-228) applied in order: all entries are validated first,
 * then each touched row's net change u'u'^T - uu^T is patched into every stored
 * node on its root-leaf path (segment_tree_sampler.cpp:358-409 semantics). */
int krpg_update_entries(krpg_t h, uint32_t j, const uint64_t* r, const uint32_t* c,
                        const double* v, uint64_t n);

/* Replaces KrpSampler::validate(tol) (krp_sampler.cpp:230-245), but with a
 * relative tolerance: root Gram vs a fresh device Gram, entrywise
 * |a-b| <= tol * sqrt(G_aa G_bb). */
int krpg_validate(krpg_t h, double tol);

/* STS-CP gather (cp_als.cpp:284-289, sketch.cpp:36-52) on device buffers:
 * w_d = 1/sqrt(J q_d); SA[d,:] = w_d * rows[d,:]. Fails (invalid argument) if
 * any q_d <= 0 or non-finite. */
int krpg_gather_sa_device(krpg_t h, uint64_t J, const double* d_prob, const double* d_rows,
                          double* d_weights, double* d_sa);

/* Timing of the last tree build (ms, device events) for the bench. */
int krpg_last_build_ms(krpg_t h, float* ms);

/* ---- instrumentation (bench / profiling support) ----
 * Every kernel launch is counted per category; when profiling is enabled each
 * category's launches are also bracketed by CUDA events on the handle's stream
 * and their device time accumulated. */
#define KRPG_PROF_TREE_LEAF 0   /* DMMA leaf/pair Gram kernel            */
#define KRPG_PROF_TREE_LEVELS 1 /* level-by-level packed reductions      */
#define KRPG_PROF_ETREE 2       /* eigenvector-stage tree construction   */
#define KRPG_PROF_DRAWS 3       /* batched root-to-leaf descent          */
#define KRPG_PROF_PROB 4        /* probability epilogue                  */
#define KRPG_PROF_UPDATE 5      /* incremental updates                   */
#define KRPG_PROF_OTHER 6       /* fills, gathers, conversions           */
#define KRPG_PROF_STS 7         /* STS-CP solve: weights, Grams, fiber scatter, row solve, normalise */
/* finer split of KRPG_PROF_DRAWS for the grouped descent (only timed when
 * KRPG_OPT_PROFILE_DETAIL is set; their launches are counted under DRAWS) */
#define KRPG_PROF_D_ROOT 8       /* normaliser passes (root of E / Z trees) */
#define KRPG_PROF_D_LEVEL_CTA 9  /* shallow levels, cooperative CTA kernel */
#define KRPG_PROF_D_LEVEL_WARP 10 /* deep levels, per-warp kernel          */
#define KRPG_PROF_D_REGROUP 11   /* child-run scatter                      */
#define KRPG_PROF_D_LEAF 12      /* leaf scan + h update                   */
#define KRPG_PROF_D_MISC 13      /* stage init, z formation                */
#define KRPG_PROF_STS_SCATTER 14 /* STS-CP: fiber lookup + scatter of the sampled right-hand side */
#define KRPG_PROF_N 16
int krpg_profile_enable(krpg_t h, int on);
/* ms and launches: arrays of KRPG_PROF_N (nullable); reset != 0 zeroes them */
int krpg_profile_read(krpg_t h, double* ms, uint64_t* launches, int reset);

/* ---- options ----
 * KRPG_OPT_GROUPED_DESCENT (default 1): use the level-synchronous, node-grouped
 * DMMA descent (R = 8..64, multiple of 8, two-stage mode); 0 forces the
 * per-draw-warp descent (the path used for every other rank / mode). */
#define KRPG_OPT_GROUPED_DESCENT 1
#define KRPG_OPT_PROFILE_DETAIL 2 /* per-kernel-type event timing inside the descent */
#define KRPG_OPT_FUSED_DEEP 3     /* default 1: deep levels + leaf scan in one warp-local pass;
                                     0: per-level global regrouping down to the leaves */
/* KRPG_OPT_ASYNC (default 0): krpg_sample_device returns once the call's work is
 * enqueued on the handle's stream, without a host synchronisation, so the host
 * setup of the next call (R x R eigensolves) overlaps this call's kernels. A
 * degenerate-distribution error raised by any such call is reported by the next
 * krpg_sync (or krpg_sample) on the handle; profiling events are resolved by
 * krpg_profile_read. */
#define KRPG_OPT_ASYNC 4
/* KRPG_OPT_SLICES (default 1, 1..8): the grouped descent splits the J draws into this
 * many slices run on concurrent streams (results are identical for any value; on
 * config 2 one slice measured fastest). */
#define KRPG_OPT_SLICES 5
#define KRPG_OPT_HOST_TRACE 6 /* host-side phase times of krpg_sample on stderr */
/* Kernel-variant / tuning options of the grouped descent (defaults = measured best).
 * EVAL_REG (1), POS0_TABLES (1), DEEP_THRESHOLD (0: by rank, 16 at R <= 32 else 32), DEEP_CHUNK (0: chosen from J, 8 .. 32; or 1 .. 32) give bit-identical
 * samples; EVAL_SPLIT (16: R = 128 only; 1: also R = 64; 0: off), DEEP_DMMA_MIN (1) and
 * LEAF_PAR (8) change last-bit rounding when moved off their defaults. */
#define KRPG_OPT_EVAL_REG 16
#define KRPG_OPT_POS0_TABLES 17
#define KRPG_OPT_DEEP_THRESHOLD 18
#define KRPG_OPT_DEEP_CHUNK 19
#define KRPG_OPT_EVAL_SPLIT 20
#define KRPG_OPT_DEEP_DMMA_MIN 21
#define KRPG_OPT_LEAF_PAR 22
/* krpg_sample into page-locked host buffers: the last position runs as this many draw
 * slices, each copied out while the next computes (default 2, 1..4; same bits) */
#define KRPG_OPT_OUT_SLICES 23
/* krpg_sts_solve: 1 (default) the row-ordered, atomic-free scatter and block-ordered column
 * norms (bit-reproducible factor updates); 0 the fp64-atomic fiber scatter (faster on
 * large tensors, sums in run-dependent order) */
#define KRPG_OPT_STS_DETERMINISTIC 25
/* R <= 64: the levels >= 1 of a sampling stage run in ONE cooperatively launched kernel with
 * grid barriers between the levels (default 1; 0: one launch per level; same bits) */
#define KRPG_OPT_EVAL_ML 26
int krpg_set_option(krpg_t h, int option, int64_t value);
/* 1 for the bounds-checked library (make CHECKED=1, device asserts), 0 for production */
int krpg_is_checked_build(void);

/* ---- STS-CP solve slice ----
 * A device-resident sparse tensor: SparseTensorCoo::from_entries (tensor.cpp:34-75)
 * semantics -- coordinates validated, duplicates summed, entries sorted
 * lexicographically; fiber indexes (SparseTensorCoo::fiber_index, tensor.cpp:104-129)
 * are built on the device on first use. Requires prod(dims) <= 2^64, nnz < 2^32, N <= 8. */
typedef struct krpg_tensor* krpg_tensor_t;
int krpg_tensor_create(const uint64_t* dims, uint32_t N, const uint32_t* coords, const double* values,
                       uint64_t nnz, int device, krpg_tensor_t* out);
/* Same as krpg_tensor_create from device-resident COO arrays (nnz x N uint32 coordinates,
 * nnz doubles, on `device`; read only, the caller keeps ownership). Coordinates are
 * range-checked on the device; norm_sq is summed in a fixed blocked order (the host
 * entry sums sequentially). For tensors too large to stage through host memory. */
int krpg_tensor_create_device(const uint64_t* dims, uint32_t N, const uint32_t* d_coords, const double* d_values,
                              uint64_t nnz, int device, krpg_tensor_t* out);
int krpg_tensor_destroy(krpg_tensor_t t);
int krpg_tensor_info(krpg_tensor_t t, uint64_t* nnz, double* norm_sq);
/* deduplicated, sorted entries (host): coords nnz x N, values nnz (each nullable) */
int krpg_tensor_entries(krpg_tensor_t t, uint32_t* coords, double* values);
/* One STS-CP factor update of mode j, the StsCp branch of cp_als.cpp:279-313:
 * batch = sample(j, J, seed); w = 1/sqrt(J q) (make_sampling_weights, sketch.cpp:36-52);
 * SA = w o rows; SB = w o sampled_rhs_rows(T, j, batch) (cp_als.cpp:122-145, formed as a
 * sparse scatter, never the dense J x I_j block); U_j = (pinv_psd(gram(SA)) gram_cross(SA, SB))^T;
 * normalize_columns (cp_als.cpp:39-52) -> sigma (R, host, nullable); update_factor(j, U_j).
 * The factor of the handle is replaced and its tree rebuilt on the device. */
int krpg_sts_solve(krpg_t h, krpg_tensor_t T, uint32_t j, uint64_t J, uint64_t seed, double* sigma);
/* statistics of the last krpg_sts_solve (3 values): draws whose fiber holds a nonzero,
 * distinct sampled fibers, tensor entries visited by the scatter */
int krpg_sts_last_stats(krpg_t h, uint64_t* stats);

/* ---- CP-ARLS-LEV product-of-leverage sampler (sketch.cpp:86-149, §8(f) rank 3) ----
 * Each included factor drawn independently from its own normalised leverage scores
 * p_i = u_i^T pinv(G_k) u_i (cumulative-table inversion, draw_from_cumulative
 * :19-26, CounterRng(seed, draw_offset + d), one uniform per included factor in
 * order); probability = product of the p; rows = Hadamard of the drawn rows.
 * idx: J x N (excluded column 0xFFFFFFFF); prob J; rows J x R; margin (nullable) J:
 * smallest |cum - target| (normalised) over every pick. The handle form uses the
 * resident factors and their cached Grams; the _factors form takes host factors
 * (fp64, row-major) and forms gram(U) on the device, as the reference's free
 * function does. */
int krpg_product_lev_sample(krpg_t h, int64_t excluded, uint64_t J, uint64_t seed, uint64_t draw_offset,
                            uint32_t* idx, double* prob, double* rows, double* margin);
int krpg_product_lev_sample_factors(const double* const* factors, const uint64_t* I, uint32_t N, uint32_t R,
                                    int64_t excluded, uint64_t J, uint64_t seed, int device, uint32_t* idx,
                                    double* prob, double* rows, double* margin);
/* unnormalised leverage scores u_i^T pinv(G_j) u_i of every row of factor j (out: I_j) */
int krpg_leverage_scores(krpg_t h, uint32_t j, double* out);

/* ---- standalone segment tree (SegmentTreeSampler, segment_tree_sampler.hpp:26-139) ----
 * The tree over U (I x R, host, row-major) with leaf capacity F and a fixed PSD Y,
 * rank-1 (y, R) or general (Y, R x R): give exactly one. Device build identical to
 * the sampler's (compact layout). */
typedef struct krpg_segtree* krpg_segtree_t;
int krpg_segtree_create(const double* U, uint64_t I, uint32_t R, uint64_t F, const double* Y,
                        const double* y, int device, krpg_segtree_t* out);
/* The same tree over an explicit row partition: leaf l (in order) holds rows
 * [leaf_offsets[l], leaf_offsets[l+1]), L leaves, offsets[0] = 0, offsets[L] = I,
 * strictly ascending (init_tree's leaf_segments, segment_tree_sampler.cpp:111-149).
 * from_sparse (:67-109) builds its greedy nnz partition on the host and calls this. */
int krpg_segtree_create_segments(const double* U, uint64_t I, uint32_t R, const uint64_t* leaf_offsets,
                                 uint64_t L, const double* Y, const double* y, int device,
                                 krpg_segtree_t* out);
/* leaf offsets of a tree (leaf_count + 1 values) and the rows of heap node v (node_segment) */
int krpg_segtree_leaf_offsets(krpg_segtree_t t, uint64_t* offsets);
int krpg_segtree_node_rows(krpg_segtree_t t, uint64_t v, uint64_t* first, uint64_t* last);
int krpg_segtree_destroy(krpg_segtree_t t);
/* device copy of a tree (the reference SegmentTreeSampler has value semantics) */
int krpg_segtree_clone(krpg_segtree_t t, krpg_segtree_t* out);
int krpg_segtree_shape(krpg_segtree_t t, uint64_t* leaf_count, uint64_t* node_count);
/* node_gram(node) (:79): stored nodes (root, left children) only */
int krpg_segtree_node_gram(krpg_segtree_t t, uint64_t node, double* out /* R x R */);
/* Batched row_sample (:258-293): draw d walks with history H[d] (J x R, host) and the
 * uniform CounterRng(seed, stream0 + d) at `counter` (a fresh CounterRng's first
 * uniform is counter 1). out: J row indices; margin (nullable): boundary margins. */
int krpg_segtree_sample(krpg_segtree_t t, const double* H, uint64_t J, uint64_t seed, uint64_t stream0,
                        uint64_t counter, uint64_t* out, double* margin);
/* Same with a CounterRng key and counter per draw (keys = the generator's mixed
 * stream key, rng.hpp:16-18) -- what the C++ drop-in's row_sample(h, rng) uses. */
int krpg_segtree_sample_keyed(krpg_segtree_t t, const double* H, uint64_t J, const uint64_t* keys,
                              const uint64_t* counters, uint64_t* out, double* margin);
/* analytic_probabilities(h) (:310-323): q_{h,U,Y} for every row (out: I) */
int krpg_segtree_probabilities(krpg_segtree_t t, const double* h, double* out);
/* update_entry(r, c, value) (:358-409) */
int krpg_segtree_update_entry(krpg_segtree_t t, uint64_t r, uint32_t c, double value);

/* ---- row-partitioned construction (multi-GPU) ----
 * The tree over I rows splits into parts = 2^g subtrees (the nodes of level g);
 * subtree `part` covers the contiguous rows krpg_partition_rows(...). A rank that
 * holds (at least) those rows of U_j in its handle builds the subtree's stored
 * nodes with krpg_build_partition, which also returns the subtree root Gram
 * (P doubles, device). After the stored slots (per tree level, each partition's
 * range is contiguous, see sharding.partition_slots) and the subtree roots are
 * exchanged (e.g. NCCL all-gather), krpg_finish_partitions computes levels
 * g-1 .. 0 identically on every rank. Replaces the single-process build_grams
 * (segment_tree_sampler.cpp:151-191); results are bit-identical to it. */
int krpg_tree_device(krpg_t h, uint32_t j, double** d_tree, uint64_t* slots);
int krpg_factor_device(krpg_t h, uint32_t j, void** d_U);
int krpg_build_partition(krpg_t h, uint32_t j, uint32_t parts, uint32_t part, double* d_subroot);
int krpg_finish_partitions(krpg_t h, uint32_t j, uint32_t parts, const double* d_subroots);
int krpg_partition_rows(uint64_t I, uint32_t R, uint32_t parts, uint32_t part, uint64_t* first,
                        uint64_t* last);

/* ---- host-only test support (no device needed) ---- */
/* Row range [first, last) of heap node v of the complete tree over I rows with
 * leaf capacity F (SegmentTreeSampler::node_segment, segment_tree_sampler.hpp:74-76). */
int krpg_topology_node_rows(uint64_t I, uint64_t F, uint64_t v, uint64_t* first, uint64_t* last,
                            uint64_t* leaf_count, uint64_t* node_count);
/* The host eigensolver used per sample call (values descending, vectors as columns). */
int krpg_host_eigh(const double* G, uint32_t n, double* vectors, double* values);

#ifdef __cplusplus
}
#endif
#endif
