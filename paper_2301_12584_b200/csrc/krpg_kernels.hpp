// Internal launch interface between the C-ABI host layer (krpg_api.cpp) and
// the CUDA kernels (tree_build.cu, descent.cu, update.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace krpg {

// ---- tree construction (segment_tree_sampler.cpp:111-191 on device) ----
struct TreeBuildArgs {
    const void* U;       // I x R row-major, fp64 or fp32 (storage)
    uint32_t storage;    // 0 = f64, 1 = f32
    uint64_t I;
    uint32_t R;
    double* compact;     // L x P stored Grams (slot order)
    double* tbuf_a;      // transient level buffers, see tree_transient_doubles
    double* tbuf_b;
    cudaStream_t stream;
    int force_generic;   // test hook: use the scalar kernel
    uint64_t F = 0;      // leaf capacity (0: F = R, the KrpSampler trees)
    const uint64_t* segs = nullptr;  // variable leaf segments (L + 1 device offsets; host copy in segs_h)
    const uint64_t* segs_h = nullptr;
    uint64_t nleaves = 0;
    uint32_t parts = 1;  // > 1: build only subtree `part` of `parts` (a power of two)
    uint32_t part = 0;
    double* subroot = nullptr;  // partitioned build: receives the subtree root Gram (P)
    int leaf_variant = 0;       // 1: the direct-store leaf kernel at every rank (A/B in tools/microbench/leaf_bench.cu)
};
// doubles needed for (tbuf_a, tbuf_b)
void tree_transient_doubles(uint64_t I, uint32_t R, uint64_t* a, uint64_t* b, uint64_t F = 0, uint64_t nleaves = 0);
// leaf / first-pair level (DMMA) then the remaining levels; returns #launches (< 0: CUDA error)
int launch_tree_leaves(const TreeBuildArgs& a);
int launch_tree_levels(const TreeBuildArgs& a);
// partitioned build: levels above the parts subtree roots (parts x P on device)
int launch_tree_top(const TreeBuildArgs& a, const double* subroots);
// positions (level d-1 nodes) of the tree over I rows with leaf capacity R
uint64_t tree_positions(uint64_t I, uint32_t R);
// rows [first, last) under subtree `part` of `parts`
void tree_partition_rows(uint64_t I, uint32_t R, uint32_t parts, uint32_t part, uint64_t* first, uint64_t* last);

// ---- E-tree (eigenvector stage) construction, krp_sampler.cpp:118-123 ----
// Q[slot] = (sum_{u in node} lambda_u V[:,u] V[:,u]^T) o G_k, packed.
void launch_etree_build(const double* V, const double* lam, const double* gk_packed, uint32_t R,
                        double* Q, cudaStream_t s);

// ---- batched draws ----
struct DrawArgs {
    uint32_t R, N, k, pos, mode;  // mode 0 two-stage, 1 one-stage; standalone segment tree
                                  // (SegmentTreeSampler::row_sample): 2 rank-1 y, 3 general Y
    uint64_t J, seed, draw_offset;
    double* H;          // J x R running Hadamard history (also the output rows)
    uint32_t* idx;      // J x N or null
    double* margin;     // J or null
    const double* Q;    // E-tree compact (two-stage)
    const double* V;    // R x R eigenvectors of G_{>k} (two-stage)
    const double* Y;    // packed G_{>k} (one-stage)
    const double* Z;    // factor k tree compact
    const void* U;      // factor k rows
    uint32_t storage;
    uint64_t I;         // rows of factor k
    int* err;           // device error flag
    cudaStream_t stream;
    // modes 2 / 3: leaf capacity, the uniform's counter, rank-1 y, index output
    uint64_t F = 0;
    uint64_t counter = 1;
    const double* yv = nullptr;
    uint64_t* idx64 = nullptr;
    const uint64_t* segs = nullptr;      // variable leaf segments (L + 1 offsets, device), nullable
    uint64_t nleaves = 0;
    const uint64_t* keys = nullptr;      // per-draw CounterRng keys (nullable: derive from seed)
    const uint64_t* counters = nullptr;  // per-draw counters (nullable: `counter`)
};
void launch_draws(const DrawArgs& a);
// SegmentTreeSampler::analytic_probabilities numerators (out[0..I)) and normaliser (out[I])
void launch_segtree_masses(const double* U, uint64_t I, uint32_t R, const double* h, const double* yv,
                           const double* Y, const double* root, double* out, cudaStream_t s);

// ---- grouped (level-synchronous, DMMA) two-stage descent, descent_v2.cu ----
// Kernel-variant / tuning choices of the grouped descent (set per handle through
// krpg_set_option; the defaults are the measured best). The first four give
// bit-identical samples (same arithmetic, tests/test_gpu_kernel_variants.py);
// eval_split == 1 (split summation order at R = 64), deep_dmma_min > 1 (CUDA-core
// forms for small runs) and leaf_par < 8 change last-bit rounding.
struct Tuning {
    int eval_reg = 1;          // R <= 64 shallow levels: register-resident kernel (0: CTA kernel)
    int pos0_tables = 1;       // first included position from (node, component) tables
    int deep_threshold = 0;    // a level is "deep" below this many draws per node on average (0: by rank, 16 / 32)
    int deep_chunk = 0;        // sorted draws per warp work unit of the fused deep pass (1..32; 0: chosen from J)
    int eval_split = 16;       // split-Gram level kernel: 16 = R 128 only, 1 = R 64 and 128, 0 = off
    int deep_dmma_min = 1;     // deep-pass runs with fewer draws use CUDA-core forms
    int leaf_par = 8;          // leaf runs with at most this many draws scan warp-parallel
    int sts_deterministic = 1; // STS-CP scatter: 1 row-ordered (bit-reproducible), 0 fp64 atomics (faster)
    int eval_ml = 1;           // R <= 64: a stage's levels >= 1 in one cooperative launch with grid barriers
    int out_slices = 2;        // krpg_sample into page-locked host memory: draw slices of the
                               // last position whose copies overlap the following slices (1..4)
};

struct GroupedArgs {
    uint32_t R, N, k, pos, storage;
    uint64_t J, seed, draw_offset, I;
    double* H;           // J x R history / output rows
    double* Zb;          // J x R scratch (z = h o V[:,u])
    uint32_t* idx;       // J x N or null
    double* margin;      // J or null
    const double* Q;     // E-tree compact
    const double* V;     // eigenvectors of G_{>k}
    const double* Z;     // factor tree compact
    const void* U;       // factor rows
    uint32_t *perm_a, *perm_b, *node, *rank, *gstart, *gend, *cntL, *cntR;
    uint32_t *nsort_a, *nsort_b;  // node per sorted position (level kernels), nullable
    double *low, *invc, *ud;
    int* err;
    cudaStream_t stream;
    void (*mark)(void* ctx, int cat);  // optional per-launch timing hook
    void* mark_ctx;
    int fused_deep;                    // deep levels + leaf in one warp-local pass
    int h_ones;                        // H is all ones (first included position): table shortcut
    double* pos0_tab;                  // scratch for the first-position tables (pos0_tab_doubles(R)), nullable
    uint32_t* gbar;                    // grid-barrier counter of the multi-level level kernel (zeroed per stage), nullable
    Tuning tune;
    int final_rows;                    // fused deep pass forms h o= U_k[pick] itself (no k_apply_pick)
    double* host_rows;                 // with final_rows: device-mapped page-locked output rows, nullable
    int one_stage;                     // mode 1: M = hh^T o Y on the factor tree directly
    const double* W;                   // one-stage: packed Y = G_{>k} of this position (device)
};
// doubles of scratch the first-position tables need at rank R (E-tree masses, factor-tree
// masses per (node, component) for the top levels, per-node counters)
inline uint64_t pos0_tab_doubles(uint32_t R) { return 2ull * R + 8 + 128ull * R + 256; }
bool grouped_supported(uint32_t R, uint32_t mode);
int launch_position_grouped(const GroupedArgs& g);
void launch_probabilities_grouped(const double* H, const double* gp_packed, uint32_t R, uint64_t J,
                                  double rank, double* prob, cudaStream_t s);

// q_d = h_d^T G+ h_d / rank  (krp_sampler.cpp:143-149)
void launch_probabilities(const double* H, const double* gp_packed, uint32_t R, uint64_t J,
                          double rank, double* prob, cudaStream_t s);
void launch_fill(double* p, double v, uint64_t n, cudaStream_t s);
void launch_fill_u32(uint32_t* p, uint32_t v, uint64_t n, cudaStream_t s);
void launch_set_excluded_column(uint32_t* idx, uint64_t J, uint32_t N, uint32_t col, cudaStream_t s);

// ---- STS-CP gather (cp_als.cpp:284-289) ----
void launch_gather_sa(const double* prob, const double* rows, uint64_t J, uint32_t R, double* w,
                      double* sa, int* err, cudaStream_t s);

// ---- conditional distribution (krp_sampler.cpp:153-196) ----
// HT[u,:] = h o V[:,u]; norms[u] += sum_t (U[t,:] . HT[u,:])^2 (norms zeroed by caller)
void launch_conditional_norms(const void* U, uint32_t storage, uint64_t I, uint32_t R,
                              const double* HT, double* norms, cudaStream_t s);
// probs[t] = sum_u w[u] * (U[t,:] . HT[u,:])^2 / norms[u]  (w[u]=0 skips)
void launch_conditional_probs(const void* U, uint32_t storage, uint64_t I, uint32_t R,
                              const double* HT, const double* w, const double* norms,
                              double* probs, cudaStream_t s);

// ---- updates (segment_tree_sampler.cpp:358-409) ----
// for each touched row: patch u'u'^T - uu^T into every stored node on its path
// Deterministic batched tree patch (update_entry, segment_tree_sampler.cpp:358-409, for a
// batch of distinct rows): every touched node v gets G_v += Delta_v with
// Delta_v = sum over its touched rows of u'u'^T - u u^T, reduced bottom-up in a fixed
// order (a leaf sums its rows in ascending order, a parent adds left + right), one warp
// per node and no atomics, so the patched tree is bit-reproducible run to run.
// Items of one tree depth: leaf items carry the row range [rb, re) of their rows in
// the (ascending) row arrays; internal items the indices of their touched children in
// the previous (deeper) depth's item list (-1 = untouched).
struct PatchItem {
    uint64_t node;
    int64_t lc, rc;
    uint32_t rb, re;
};
void launch_tree_patch_level(double* compact, uint32_t R, const PatchItem* items, uint64_t nitems,
                             const double* delta_prev, double* delta_cur, const double* old_rows,
                             const double* new_rows, cudaStream_t s);
void launch_row_deltas(double* compact, uint64_t I, uint32_t R, uint64_t F, const uint64_t* segs, uint64_t nleaves,
                       uint64_t nrows,
                       const uint64_t* rows, const double* old_rows, const double* new_rows,
                       cudaStream_t s);
void launch_scatter_rows(void* U, uint32_t storage, uint32_t R, uint64_t nrows,
                         const uint64_t* rows, const double* new_rows, cudaStream_t s);
void launch_gather_rows(const void* U, uint32_t storage, uint32_t R, uint64_t nrows,
                        const uint64_t* rows, double* out, cudaStream_t s);
void launch_convert_f64_to_f32(const double* in, float* out, uint64_t n, cudaStream_t s);
void launch_convert_f32_to_f64(const float* in, double* out, uint64_t n, cudaStream_t s);

// fresh Gram of a whole factor (validate): out R x R
// (DMMA for R = 8..64 step 8, else scalar; deterministic ordered reduction of
// per-CTA partials held in work: full_gram_work_doubles(R) doubles)
void launch_full_gram(const void* U, uint32_t storage, uint64_t I, uint32_t R, double* out, double* work,
                      cudaStream_t s);
size_t full_gram_work_doubles(uint32_t R);

// ---- STS-CP solve slice (sts.cu; cp_als.cpp:282-313) ----
// dedup + lexicographic sort of COO entries (tensor.cpp:34-75); returns nnz after
// dedup, *_out allocated with cudaMalloc (caller frees)
// device-resident COO input (krpg_tensor_create_device): every coordinate < its mode's
// size; sum of squared values in a fixed, reproducible order
bool coords_in_range(const uint32_t* d_coords, uint64_t nnz, uint32_t N, const uint64_t* dims, cudaStream_t s);
double sum_of_squares(const double* d_v, uint64_t n, cudaStream_t s);
uint64_t tensor_ingest(const uint32_t* d_coords, const double* d_vals, uint64_t nnz, uint32_t N, const uint64_t* dims,
                       uint32_t** d_coords_out, double** d_vals_out, cudaStream_t s);
// fiber index of mode j (tensor.cpp:104-129): distinct keys, CSR offsets, and the
// (coordinate j, value) of every entry in fiber order
struct FiberIndexDev {
    uint64_t G = 0, nnz = 0, I = 0;
    uint64_t* keys = nullptr;    // G distinct matricization columns, ascending
    uint64_t* fptr = nullptr;    // G + 1
    uint32_t* fcoord = nullptr;  // nnz
    double* fval = nullptr;      // nnz
};
void fiber_index_build(const uint32_t* d_coords, const double* d_vals, uint64_t nnz, uint32_t N, const uint64_t* dims,
                       uint32_t j, FiberIndexDev* out, cudaStream_t s);
void fiber_index_free(FiberIndexDev& f);
// device scratch for one step, and where its statistics live (4 u64: draws with a
// nonzero fiber, distinct sampled fibers, entries visited, unused)
size_t sts_work_bytes(uint64_t J, uint32_t R);
const void* sts_stats_ptr(void* work, uint64_t J, uint32_t R);
// M (I_j x R) = (SA^T SB)^T from the batch: draws -> fibers, per distinct fiber
// S = sum w^2 rows, entries scattered v S (M zeroed here)
void launch_sts_rhs(const uint32_t* idx, uint64_t J, uint32_t N, uint32_t j, const uint64_t* dims, const double* prob,
                    const double* rows, uint32_t R, const FiberIndexDev& F, void* work, double* M, int* err,
                    cudaStream_t s, bool deterministic = true);
// U = (pinv M^T)^T row by row into Utmp, column norms -> nrm (R), then the
// normalised columns (cp_als.cpp:39-52) stored into Uout (storage 0 f64, 1 f32)
void launch_solve_normalize(const double* M, uint64_t I, uint32_t R, const double* pinv, double* Utmp, double* nrm,
                            void* Uout, uint32_t storage, cudaStream_t s);
// U_out = Utmp / nrm column-wise in the storage dtype (normalize_columns' store)
void launch_normalize_store(const double* Utmp, uint64_t I, uint32_t R, const double* nrm, void* Uout,
                            uint32_t storage, cudaStream_t s);

// ---- CP-ARLS-LEV product sampler (productlev.cu; sketch.cpp:86-149) ----
// p_i = u_i^T G+ u_i for every row (DMMA for R % 8 == 0, R <= 160 from the packed
// G+; otherwise the dense G_full, R <= 256)
void launch_row_leverage(const void* U, uint32_t storage, uint64_t I, uint32_t R, const double* Gp_packed,
                         const double* G_full, double* out, cudaStream_t s);
size_t lev_scan_work_bytes(uint64_t I);
int launch_lev_scan(const double* p, double* cum, uint64_t I, void* work, size_t work_bytes, cudaStream_t s);
constexpr uint32_t LEV_MAX_FACTORS = 16;
struct LevDrawArgs {
    uint32_t N = 0, ninc = 0, R = 0, storage = 0;
    uint64_t J = 0, seed = 0, draw_offset = 0;
    uint32_t inc[LEV_MAX_FACTORS];        // included factor ids, in order
    const double* p[LEV_MAX_FACTORS];     // unnormalised masses per included factor
    const double* cum[LEV_MAX_FACTORS];   // their inclusive prefix sums
    const void* U[LEV_MAX_FACTORS];       // factor rows (storage dtype)
    uint64_t I[LEV_MAX_FACTORS];
    uint32_t* idx = nullptr;  // J x N (excluded column 0xFFFFFFFF)
    double* prob = nullptr;   // J (nullable)
    double* rows = nullptr;   // J x R (nullable)
    double* margin = nullptr; // J (nullable): min |cum - target| / cum_last over every pick
};
int launch_lev_draws(const LevDrawArgs& a, cudaStream_t s);

}  // namespace krpg
