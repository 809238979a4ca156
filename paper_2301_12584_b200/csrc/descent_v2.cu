// Batched descent, version 2: level-synchronous, node-grouped, GEMM-shaped.
//
// The reference walks every draw independently (segment_tree_sampler.cpp:258-293):
// per level one packed inner product <G_left, M_d> read straight from DRAM.
// Here all J draws of one factor position advance one tree level per pass:
//
//   * draws are kept sorted by their current node (perm[]): every node's draws
//     are one contiguous run, so a node Gram is read once per run instead of
//     once per draw;
//   * a run's masses x_d^T G x_d (M = x x^T, fold_weights :193-211) are
//     computed on the FP64 tensor cores: for 8 draws X (8 x R) the warp forms
//     Y = X * Gfold with mma.sync m8n8k4 (DMMA), using only the upper-triangle
//     8x8 tiles of the symmetric Gram (off-diagonal tiles doubled, like the
//     reference's folded weights), then mass_d = sum_j X[d,j] Y[d,j]. Gram
//     fragments are gathered straight from the reference's packed layout into
//     registers and reused by every 8-draw block of the run;
//   * after the branch decision (cutoff >= u goes left, :270-276) each draw
//     takes a slot in its child's run with one warp-aggregated atomic per
//     block, and a light scatter pass rewrites perm[] for the next level;
//   * the leaf scan (:281-292) of a run is one DMMA GEMM U_leaf (F x R) x Z^T
//     (R x 8 draws), masses squared into shared memory, then each draw's
//     sequential cumulative scan and the h *= U[t] update.
//
// Used for R = 8, 16, ..., 64 (NB = R/8 column blocks); other ranks use the
// per-draw kernel (descent.cu).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "krpg_device.cuh"
#include "krpg_kernels.hpp"
#include "launch_util.hpp"
#include "ptx.cuh"
#include "qf_dmma.cuh"

namespace krpg {
namespace v2 {

constexpr int CHUNK = 32;  // sorted positions per warp
constexpr int WPB = 4;     // warps per block

enum { EV_ROOT = 0, EV_LEVEL = 1, EV_PROB = 2, EV_LEVEL0 = 3 };

template <int NB>
struct Tiles {
    static constexpr int R = 8 * NB;
    static constexpr int NT = NB * (NB + 1) / 2;
    __host__ __device__ static constexpr int t(int p, int q) { return p * NB - (p * (p - 1)) / 2 + (q - p); }
};

struct EvalArgs {
    uint64_t J;
    const uint32_t* perm;   // sorted position -> draw (nullptr: identity)
    uint32_t* node;         // per draw current node
    uint32_t* rank;         // per draw slot in its child run
    double* low;            // per draw running offset
    double* invc;           // per draw 1/C
    const double* ud;       // per draw uniform of this stage
    double* margin;         // per draw (nullable)
    uint32_t* cntL;         // per node counters (level passes)
    uint32_t* cntR;
    const double* X;        // J x R (indexed by draw id)
    const double* tree;     // compact tree (level passes) or the single matrix
    Topo topo;
    int* err;
    double* prob;           // EV_PROB output
    double rank_div;        // EV_PROB: numerical rank
    uint32_t* perm_out;     // level passes: next level's sorted order
    const uint32_t* nsort_in;  // node of each sorted position (nullable: read node[perm[i]])
    uint32_t* nsort_out;       // node of each position of perm_out
    uint32_t* GS;           // per node position range [GS, GE) at its level
    uint32_t* GE;
    const double* W;        // one-stage mode: packed Y = G_{>k}; node masses use G_v o Y (nullable)
#ifdef KRPG_LEVEL_BENCH
    int fake;               // microbenchmark only (tools/microbench/level_bench.cu): 1 skip the DMMA, 2 also the loads
#endif
    unsigned long long* trace;  // timing experiments only: per-warp phase timestamps (nullable)
};

// timing-experiment switch of the level microbenchmark; always 0 in the library
#ifdef KRPG_LEVEL_BENCH
__device__ int g_ml_dbg = 0;  // multi-level kernel: 1 skip the tiles of levels >= 1, 2 skip the grid barrier
#define EV_FAKE(a) ((a).fake)
#else
#define EV_FAKE(a) 0
#endif


__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

using qf::FragAddr;
using qf::block_qf_packed;

constexpr int CWARPS = 4;        // warps per CTA in the cooperative variant (8 measured slower)
constexpr int CB = CWARPS * 32;  // positions per CTA in the cooperative variant

// Gram buffers per CTA: two (next run prefetched) while they are small; one for
// R > 64 so that 3 CTAs share an SM (the root-fused level 0 always needs two).
template <int NB, bool ROOT0>
__host__ __device__ constexpr int cta_nbuf() { return (ROOT0 || NB <= 8) ? 2 : 1; }

template <int NB, int MODE, bool ROOT0 = false>
__global__ void __launch_bounds__(CB) k_eval_cta(EvalArgs a, uint32_t range) {
    constexpr int R = 8 * NB;
    constexpr uint32_t P = uint32_t(R) * (R + 1) / 2;
    constexpr int NBUF = cta_nbuf<NB, ROOT0>();
    extern __shared__ __align__(128) double sG[];  // [2][P]
    __shared__ uint32_t s_d[CB], s_v[CB], s_rank[CB];
    __shared__ uint8_t s_left[CB];
    __shared__ int s_rs[CB + 1];
    __shared__ int s_nruns;
    __shared__ uint32_t s_cnt[2], s_base[2], s_gs, s_ge;
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // PDL: the next level's grid may launch now; this grid waits for the previous
    // one (its perm / node / counters) before touching global state
    griddep_launch_dependents();
    griddep_wait();
    const uint64_t base = uint64_t(blockIdx.x) * range;  // range <= CB positions per CTA
    const int cnt = a.J - base < uint64_t(range) ? int(a.J - base) : int(range);
    if (tid < cnt) {
        const uint32_t d = a.perm ? a.perm[base + tid] : uint32_t(base + tid);
        s_d[tid] = d;
        s_v[tid] = (MODE == EV_LEVEL && !ROOT0) ? (a.nsort_in ? a.nsort_in[base + tid] : a.node[d]) : 0u;
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    {  // run boundaries -> compact list s_rs
        const bool flag = tid < cnt && (tid == 0 || s_v[tid] != s_v[tid - 1]);
        const unsigned bal = __ballot_sync(0xffffffffu, flag);
        __shared__ int wcount[CWARPS];
        if (lane == 0) wcount[warp] = __popc(bal);
        __syncthreads();
        int off = 0;
        for (int w = 0; w < warp; ++w) off += wcount[w];
        if (flag) s_rs[off + __popc(bal & ((1u << lane) - 1u))] = tid;
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < CWARPS; ++w) tot += wcount[w];
            s_nruns = tot;
            s_rs[tot] = cnt;
        }
        __syncthreads();
    }
    const int nruns = s_nruns;
    auto gsrc = [&](int r) -> const double* {
        if (MODE != EV_LEVEL) return a.tree;
        const uint32_t v = s_v[s_rs[r]];
        if (is_leaf(a.topo, v)) return nullptr;
        return a.tree + slot_of(2ull * v + 1) * uint64_t(P);
    };
    if (tid == 0 && nruns > 0) {
        const double* g0 = gsrc(0);
        if (g0) {
            mbar_arrive_expect_tx(&bar[0], P * 8);
            tma_load_1d(sG, g0, P * 8, &bar[0]);
        }
        if (ROOT0) {  // root Gram (slot 0) for the normaliser, second buffer
            mbar_arrive_expect_tx(&bar[1], P * 8);
            tma_load_1d(sG + P, a.tree, P * 8, &bar[1]);
        }
    }
    const FragAddr<NB> fa(lane);
    uint32_t phase[2] = {0u, 0u};
    for (int r = 0; r < nruns; ++r) {
        const int buf = NBUF == 2 ? (r & 1) : 0;
        if (NBUF == 2 && !ROOT0 && tid == 0 && r + 1 < nruns) {  // prefetch the next run's Gram
            const double* g1 = gsrc(r + 1);
            if (g1) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&bar[buf ^ 1], P * 8);
                tma_load_1d(sG + (buf ^ 1) * P, g1, P * 8, &bar[buf ^ 1]);
            }
        }
        if (NBUF == 1 && tid == 0 && r > 0) {  // single buffer: load after the previous run
            const double* g1 = gsrc(r);
            if (g1) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&bar[0], P * 8);
                tma_load_1d(sG, g1, P * 8, &bar[0]);
            }
        }
        const int rs = s_rs[r], re = s_rs[r + 1];
        const double* gr = gsrc(r);
        if (!gr) {  // draws parked at a leaf one level up keep their positions
            if (MODE == EV_LEVEL)
                for (int t = rs + tid; t < re; t += CB) {
                    a.perm_out[base + t] = s_d[t];
                    if (a.nsort_out) a.nsort_out[base + t] = s_v[t];
                }
            continue;
        }
        mbar_wait(&bar[buf], phase[buf]);
        phase[buf] ^= 1u;
        if (ROOT0) mbar_wait(&bar[1], 0u);
        const uint32_t v = s_v[rs];
        if (tid < 2) s_cnt[tid] = 0;
        if (MODE == EV_LEVEL && tid == 0) {  // this node's position range, from its parent's
            uint32_t gs = 0, ge = uint32_t(a.J);
            if (v != 0) {
                const uint32_t p = (v - 1) >> 1;
                const uint32_t gl = a.GS[p] + a.cntL[p];
                gs = (v & 1u) ? a.GS[p] : gl;
                ge = (v & 1u) ? gl : a.GE[p];
            }
            s_gs = gs;
            s_ge = ge;
            a.GS[v] = gs;
            a.GE[v] = ge;
        }
        __syncthreads();
        const double* G = sG + buf * P;
        const int nblk = (re - rs + 7) >> 3;
        for (int b = warp; b < nblk; b += CWARPS) {
            const int b0 = rs + 8 * b;
            const int n = min(8, re - b0);
            const int m = lane >> 2;
            const bool valid = m < n;
            const uint32_t dd = valid ? s_d[b0 + m] : 0u;
            const double* xrow = valid ? a.X + uint64_t(dd) * R : nullptr;
            const bool owner = valid && (lane & 3) == 0;
            // decision inputs requested before the DMMA chain (independent loads in flight)
            double u_pre = 0.0, ic_pre = 0.0, low_pre = 0.0;
            if (MODE == EV_LEVEL && owner) {
                u_pre = a.ud[dd];
                if (!ROOT0) {
                    ic_pre = a.invc[dd];
                    low_pre = a.low[dd];
                }
            }
            const double mass = block_qf_packed<NB>(G, fa, xrow, lane);
            if (MODE == EV_ROOT) {
                if (owner) {
                    if (!isfinite(mass) || mass <= 0.0) atomicExch(a.err, 1);
                    a.invc[dd] = 1.0 / mass;
                }
            } else if (MODE == EV_PROB) {
                if (owner) a.prob[dd] = mass / a.rank_div;
            } else {
                double croot = 0.0;
                if (ROOT0) croot = block_qf_packed<NB>(sG + P, fa, xrow, lane);
                bool left = false;
                double cutoff = 0.0;
                if (owner) {
                    const double u = u_pre;
                    double ic;
                    if (ROOT0) {
                        if (!isfinite(croot) || croot <= 0.0) atomicExch(a.err, 1);
                        ic = 1.0 / croot;
                        a.invc[dd] = ic;
                        cutoff = 0.0 + ic * mass;
                    } else {
                        ic = ic_pre;
                        cutoff = low_pre + ic * mass;
                    }
                    left = cutoff >= u;
                    if (a.margin) a.margin[dd] = fmin(a.margin[dd], fabs(cutoff - u));
                }
                const unsigned lm = __ballot_sync(0xffffffffu, owner && left);
                const unsigned rm = __ballot_sync(0xffffffffu, owner && !left);
                uint32_t bl = 0, br = 0;
                if (lane == 0) {
                    if (lm) bl = atomicAdd(&s_cnt[0], uint32_t(__popc(lm)));
                    if (rm) br = atomicAdd(&s_cnt[1], uint32_t(__popc(rm)));
                }
                bl = __shfl_sync(0xffffffffu, bl, 0);
                br = __shfl_sync(0xffffffffu, br, 0);
                if (owner) {
                    const unsigned below = (1u << lane) - 1u;
                    const int slot = b0 + m;
                    s_left[slot] = left ? 1 : 0;
                    if (left) {
                        a.node[dd] = 2 * v + 1;
                        s_rank[slot] = bl + __popc(lm & below);
                    } else {
                        a.node[dd] = 2 * v + 2;
                        s_rank[slot] = br + __popc(rm & below);
                        a.low[dd] = cutoff;
                    }
                }
            }
        }
        __syncthreads();
        if (MODE == EV_LEVEL) {
            if (tid == 0) {
                s_base[0] = s_cnt[0] ? atomicAdd(a.cntL + v, s_cnt[0]) : 0u;
                s_base[1] = s_cnt[1] ? atomicAdd(a.cntR + v, s_cnt[1]) : 0u;
            }
            __syncthreads();
            for (int t = rs + tid; t < re; t += CB) {
                const uint32_t pos = s_left[t] ? s_gs + s_base[0] + s_rank[t] : s_ge - 1u - (s_base[1] + s_rank[t]);
                a.perm_out[pos] = s_d[t];
                if (a.nsort_out) a.nsort_out[pos] = 2 * v + (s_left[t] ? 1u : 2u);
            }
            __syncthreads();
        }
    }
}

// ---- register-resident Gram variant (R <= 64) -----------------------------
// Same decisions, bit-identical masses (the DMMA chain and the epilogue run in
// exactly block_qf_packed's order), different data movement. k_eval_cta
// re-gathers every B fragment of the packed Gram from shared memory for every
// 8-draw block (72 dependent LDS per 72 DMMA), which held the FP64 tensor pipe
// near 45%. Here each warp owns a contiguous range of sorted positions (at most
// 64, sized so that the whole level is one wave of 2 CTAs x 4 warps per SM) and
// holds ALL B fragments of its current run's Gram in registers (NB(NB+1)
// doubles per lane, 144 registers at R = 64), loaded once per run straight from
// global memory / L2. The draws' rows (A fragments and the epilogue) stream
// into a per-warp 3-slot shared-memory ring by cp.async two blocks ahead, row
// stride R + 4 doubles so the A-fragment loads are bank-conflict free. Child
// slots are claimed with one pair of atomics per (warp, run) at the run's end.
constexpr int RW = 4;         // warps per CTA
constexpr int RSLOTS = 3;     // x-row ring slots per warp (8 rows each)
constexpr int RRANGE = 64;    // max sorted positions per warp
constexpr int RMAXBLK = RRANGE / 8 + RRANGE;  // full blocks + one partial per run

template <int NB>
struct RegCfg {
    static constexpr int R = 8 * NB;
    static constexpr int XS = R + 4;               // doubles per staged row
    static constexpr int SLOT = 8 * XS;            // doubles per ring slot
    static constexpr int NFR = NB * (NB + 1);      // B-fragment doubles per lane
    // per warp: row ring | decision inputs u, 1/C, low, margin, root mass (f64 x RRANGE each) |
    // per-position info, per-run node / parent range / counts / claims (u32) | block list (u16)
    static constexpr int WARP_D = RSLOTS * SLOT + 6 * RRANGE;
    static constexpr int WARP_U32 = 7 * RRANGE;
    static constexpr size_t WARP_BYTES = size_t(WARP_D) * 8 + WARP_U32 * 4 + RMAXBLK * 2;
    static constexpr size_t WARP_STRIDE = (WARP_BYTES + 15) / 16 * 16;
    static constexpr size_t SMEM = RW * WARP_STRIDE;
};

// fragment (p, s, q >= p) of the register-resident Gram
template <int NB>
__host__ __device__ constexpr int rfrag(int p, int s, int q) {
    return 2 * (p * NB - (p * (p - 1)) / 2) + s * (NB - p) + (q - p);
}

// WGT (one-stage mode, north_star's M = G+ o hh^T o G_{>k}): the B operand is the
// elementwise product G_v o Y, so <G_v, hh^T o Y> = h^T (G_v o Y) h is the same
// GEMM-shaped quadratic form over the draws' h rows (segment_tree_sampler.cpp:193-218)
template <int NB, bool WGT = false>
__device__ __forceinline__ void load_gram_frags(double (&gf)[NB * (NB + 1)], const double* __restrict__ G,
                                                const double* __restrict__ W, int lane) {
    constexpr int R = 8 * NB;
    const int r4 = lane & 3, cq = lane >> 2;
#pragma unroll
    for (int p = 0; p < NB; ++p)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int row = 8 * p + 4 * s + r4;
            const int col = 8 * p + cq;
            const int rowoff = row * R - (row * (row - 1)) / 2 - row;
            const int diag = row <= col ? rowoff + col : col * R - (col * (col - 1)) / 2 - col + row;
            gf[rfrag<NB>(p, s, p)] = WGT ? __ldg(G + diag) * __ldg(W + diag) : __ldg(G + diag);
            // off-diagonal tiles count twice (folded weights); a (2g) == (2a) g exactly, so
            // the doubling is applied once per run here instead of per block to the A fragment
#pragma unroll
            for (int q = p + 1; q < NB; ++q) {
                const double g = WGT ? __ldg(G + rowoff + 8 * q + cq) * __ldg(W + rowoff + 8 * q + cq)
                                     : __ldg(G + rowoff + 8 * q + cq);
                gf[rfrag<NB>(p, s, q)] = g + g;
            }
        }
}

// block_qf_packed with the B fragments in registers (off-diagonal ones doubled) and
// the rows in shared memory (xs = the block's 8 staged rows, row m valid iff valid);
// same operation order, bit-identical result
template <int NB, bool PRED = true>
__device__ __forceinline__ double block_qf_regs(const double (&gf)[NB * (NB + 1)], const double* xs, bool valid,
                                                int lane) {
    constexpr int XS = RegCfg<NB>::XS;
    const int r4 = lane & 3, m = lane >> 2;
    const double* xr = xs + m * XS;
    double y[NB][2];
#pragma unroll
    for (int q = 0; q < NB; ++q) y[q][0] = y[q][1] = 0.0;
#pragma unroll
    for (int p = 0; p < NB; ++p) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const double av = (!PRED || valid) ? xr[8 * p + 4 * s + r4] : 0.0;
            dmma_884(y[p][0], y[p][1], av, gf[rfrag<NB>(p, s, p)]);
#pragma unroll
            for (int q = p + 1; q < NB; ++q) dmma_884(y[q][0], y[q][1], av, gf[rfrag<NB>(p, s, q)]);
        }
    }
    double part = 0.0;
    if (!PRED || valid) {
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const double2 xv = *reinterpret_cast<const double2*>(xr + 8 * q + 2 * r4);
            part = fma(xv.x, y[q][0], part);
            part = fma(xv.y, y[q][1], part);
        }
    }
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    return part;
}

// Everything a warp needs besides the quadratic forms is brought in with ONE
// latency at the start (cp.async into the warp's shared memory: positions'
// decision inputs, the parents' position ranges of its runs); the draws' rows
// stream into a 3-slot ring by 1-D TMA (one bulk copy per row, lanes 0-7,
// completing on the slot's mbarrier); the block loop does nothing but the DMMA
// chain and a store of the 8 masses, so the two warps of an SM sub-partition
// keep the FP64 tensor pipe busy; branch decisions, ranks, slot claims and the
// next level's order are then computed for all of the warp's positions at once
// (two per lane, run membership from ballot masks).
// One warp's tile of a level: the sorted positions [p0, p0 + cnt), cnt <= RRANGE. `wsmem` is
// the warp's shared-memory area (RegCfg::WARP_STRIDE bytes), `bar` its RSLOTS mbarriers
// (initialised by the kernel, count 1) and `phase` their parities (bit sl: parity of slot
// sl's next completion; 0 after the initialisation, carried from tile to tile).
template <int NB, int MODE, bool ROOT0, bool WGT>
__device__ __forceinline__ void eval_reg_tile(const EvalArgs& a, const uint64_t p0, const int cnt,
                                              unsigned char* wsmem, uint64_t* bar, uint32_t& phase,
                                              unsigned long long* tr) {
    constexpr int R = 8 * NB;
    constexpr uint64_t P = uint64_t(R) * (R + 1) / 2;
    using C = RegCfg<NB>;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr bool LEVEL = MODE == EV_LEVEL;
    const int lane = threadIdx.x & 31;
    if (tr && lane == 0) tr[0] = gtimer();
    double* ring = reinterpret_cast<double*>(wsmem);
    double* s_u = ring + RSLOTS * C::SLOT;
    double* s_ic = s_u + RRANGE;
    double* s_lo = s_ic + RRANGE;
    double* s_mg = s_lo + RRANGE;
    double* s_root = s_mg + RRANGE;
    double* s_mass = s_root + RRANGE;
    uint32_t* s_rs = reinterpret_cast<uint32_t*>(s_mass + RRANGE);  // per run: first position
    uint32_t* s_rv = s_rs + RRANGE;     // per run: node
    uint32_t* s_pgs = s_rv + RRANGE;    // parent's GS / cntL / GE
    uint32_t* s_pcl = s_pgs + RRANGE;
    uint32_t* s_pge = s_pcl + RRANGE;
    uint32_t* s_bl = s_pge + RRANGE;    // claimed bases of the run's left / right part
    uint32_t* s_br = s_bl + RRANGE;
    uint16_t* s_blk = reinterpret_cast<uint16_t*>(s_br + RRANGE);

    // the warp's sorted positions p0 + lane (A) and p0 + 32 + lane (B)
    uint32_t dA = 0, dB = 0, vA = 0xFFFFFFFFu, vB = 0xFFFFFFFFu;
    if (lane < cnt) {
        dA = a.perm ? a.perm[p0 + lane] : uint32_t(p0 + lane);
        vA = (LEVEL && !ROOT0) ? (a.nsort_in ? a.nsort_in[p0 + lane] : a.node[dA]) : 0u;
    }
    if (lane + 32 < cnt) {
        dB = a.perm ? a.perm[p0 + 32 + lane] : uint32_t(p0 + 32 + lane);
        vB = (LEVEL && !ROOT0) ? (a.nsort_in ? a.nsort_in[p0 + 32 + lane] : a.node[dB]) : 0u;
    }
    const uint32_t upA = __shfl_up_sync(FULL, vA, 1), lastA = __shfl_sync(FULL, vA, 31);
    const uint32_t upB = __shfl_up_sync(FULL, vB, 1);
    const bool stA = lane < cnt && (lane == 0 || vA != upA);
    const bool stB = lane + 32 < cnt && vB != (lane == 0 ? lastA : upB);
    const uint64_t starts = uint64_t(__ballot_sync(FULL, stA)) | (uint64_t(__ballot_sync(FULL, stB)) << 32);
    const int nruns = __popcll(static_cast<long long>(starts));
    if (tr && lane == 0) tr[1] = gtimer();
    auto pos_d = [&](int t) {  // every lane participates; t may differ per lane
        const uint32_t x = __shfl_sync(FULL, dA, t & 31), y = __shfl_sync(FULL, dB, t & 31);
        return t < 32 ? x : y;
    };
    auto pos_v = [&](int t) {
        const uint32_t x = __shfl_sync(FULL, vA, t & 31), y = __shfl_sync(FULL, vB, t & 31);
        return t < 32 ? x : y;
    };
    auto run_of = [&](int t) { return __popcll(static_cast<long long>(starts & ((2ull << t) - 1ull))) - 1; };
    auto parked = [&](uint32_t v) { return LEVEL && !ROOT0 && is_leaf(a.topo, v); };

    // the first run's Gram (root Gram for the normaliser pass) is requested now, so
    // its latency overlaps the input staging and the block list
    double gf[C::NFR];
    uint32_t gv_first = 0xFFFFFFFFu;
    {
        const uint32_t v0 = __shfl_sync(FULL, vA, 0);
        if (EV_FAKE(a) < 2 && !parked(v0)) {
            KRPG_DCHECK(!(LEVEL && !ROOT0) || (v0 < a.topo.n && slot_of(2ull * v0 + 1) < a.topo.L));
            const double* G = (LEVEL && !ROOT0) ? a.tree + slot_of(2ull * v0 + 1) * P : a.tree;
            load_gram_frags<NB, WGT>(gf, G, a.W, lane);
            gv_first = v0;
        }
    }
    if (tr && lane == 0) tr[8] = gtimer();
    // block 0's rows (positions [0, min(8, first run end))) requested right away as well
    bool pre0 = false;
    {
        const uint32_t v0 = __shfl_sync(FULL, vA, 0);
        if (EV_FAKE(a) < 2 && !parked(v0)) {
            const uint64_t mk = starts & ~1ull;
            const int re0 = mk ? __ffsll(static_cast<long long>(mk)) - 1 : cnt;
            const int n0 = re0 < 8 ? re0 : 8;
            const uint32_t dr = __shfl_sync(FULL, dA, lane & 7);
            if (lane == 0) mbar_arrive_expect_tx(&bar[0], uint32_t(n0) * R * 8);
            __syncwarp();
            if (lane < n0) tma_load_1d(ring + lane * C::XS, a.X + uint64_t(dr) * R, R * 8, &bar[0]);
            pre0 = true;
        }
    }
    if (tr && lane == 0) tr[9] = gtimer();
    // decision inputs of every position and the parents' ranges of every run: one group
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int t = lane + 32 * h;
        const uint32_t d = h ? dB : dA;
        if (LEVEL && t < cnt) {
            cp_async8(s_u + t, a.ud + d);
            if (!ROOT0) {
                cp_async8(s_ic + t, a.invc + d);
                cp_async8(s_lo + t, a.low + d);
            }
            if (a.margin) cp_async8(s_mg + t, a.margin + d);
        }
        if (h ? stB : stA) {
            const uint32_t v = h ? vB : vA;
            const int r = run_of(t);
            s_rs[r] = uint32_t(t);
            s_rv[r] = v;
            if (LEVEL && v != 0 && !parked(v)) {
                const uint32_t pp = (v - 1) >> 1;
                cp_async4(s_pgs + r, a.GS + pp);
                cp_async4(s_pcl + r, a.cntL + pp);
                cp_async4(s_pge + r, a.GE + pp);
            }
        }
    }
    cp_async_commit();
    if (tr && lane == 0) tr[10] = gtimer();

    // block list: (b0, n) of every 8-draw block of every non-parked run
    int nblk = 0;
    {
        uint64_t st = starts;
        while (st) {
            const int rs = __ffsll(static_cast<long long>(st)) - 1;
            st &= st - 1;
            const int re = st ? __ffsll(static_cast<long long>(st)) - 1 : cnt;
            if (parked(pos_v(rs))) continue;
            for (int b0 = rs; b0 < re; b0 += 8) {
                if (lane == 0) s_blk[nblk] = uint16_t(b0 | (min(8, re - b0) << 8));
                ++nblk;
            }
        }
    }
    __syncwarp();
    KRPG_DCHECK(nblk <= RMAXBLK && nruns <= RRANGE && cnt <= RRANGE);
    if (tr && lane == 0) tr[2] = gtimer();

    auto issue = [&](int i) {  // rows of block i -> ring slot i % RSLOTS (1-D TMA, one copy per row)
        if (i >= nblk || EV_FAKE(a) >= 2) return;
        const uint32_t e = s_blk[i];
        const int b0 = e & 0xff, n = e >> 8;
        const int sl = i % RSLOTS;
        KRPG_DCHECK(n >= 1 && n <= 8 && b0 + n <= cnt);
        const uint32_t dr = pos_d(b0 + (lane & 7) < cnt ? b0 + (lane & 7) : b0);
        KRPG_DCHECK(dr < a.J || a.perm == nullptr);
        if (lane == 0) {
            fence_proxy_async();
            mbar_arrive_expect_tx(&bar[sl], uint32_t(n) * R * 8);
        }
        __syncwarp();
        if (lane < n) tma_load_1d(ring + sl * C::SLOT + lane * C::XS, a.X + uint64_t(dr) * R, R * 8, &bar[sl]);
    };

    // one sweep over the warp's blocks: masses into s_mass (root_pass: s_root)
    auto sweep = [&](bool root_pass, uint32_t gv) {
        double* out = root_pass ? s_root : s_mass;
#pragma unroll
        for (int i = (pre0 ? 1 : 0); i < RSLOTS; ++i) issue(i);
        pre0 = false;
        for (int i = 0; i < nblk; ++i) {
            const int sl = i % RSLOTS;
            const uint32_t e = s_blk[i];
            const int b0 = e & 0xff, n = e >> 8;
            const uint32_t v = pos_v(b0);
            if (v != gv && EV_FAKE(a) < 2) {
                const double* G = a.tree;
                if (LEVEL && !root_pass) G = a.tree + slot_of(2ull * v + 1) * P;
                KRPG_DCHECK(!(LEVEL && !root_pass) || (v < a.topo.n && slot_of(2ull * v + 1) < a.topo.L));
                load_gram_frags<NB, WGT>(gf, G, a.W, lane);
                gv = v;
            }
            if (EV_FAKE(a) < 2) {
                mbar_wait(&bar[sl], (phase >> sl) & 1u);
                phase ^= 1u << sl;
                if (n < 8) {  // partial block: zero the unused rows, so the chain needs no predicates
                    double* zr = ring + sl * C::SLOT + n * C::XS;
                    for (int e = lane; e < (8 - n) * C::XS; e += 32) zr[e] = 0.0;
                    fence_proxy_async();
                    __syncwarp();
                }
            }
            if (tr && lane == 0 && i == 0 && !root_pass) tr[6] = gtimer();
            const int m = lane >> 2;
            const bool valid = m < n;
            double mass;
            if (EV_FAKE(a)) {  // timing experiment: pseudo-random branch, no quadratic form
                const uint32_t hsh = (pos_d(b0 + m < cnt ? b0 + m : b0) * 2654435761u) ^ (v * 40503u);
                mass = ((hsh >> 13) & 1u) ? 1e300 : 0.0;
                if (!(LEVEL && !root_pass)) mass = 1.0;
            } else {
                mass = block_qf_regs<NB, false>(gf, ring + sl * C::SLOT, valid, lane);
            }
            if (valid && (lane & 3) == 0) out[b0 + m] = mass;
            if (tr && lane == 0 && i == 0 && !root_pass) tr[7] = gtimer();
            __syncwarp();
            issue(i + RSLOTS);
        }
        __syncwarp();
    };
    cp_async_wait_all();  // decision inputs (needed by the root pass only for the error check: none)
    __syncwarp();
    if (tr && lane == 0) tr[11] = gtimer();
    if (ROOT0) {
        sweep(true, gv_first);
        sweep(false, 0xFFFFFFFFu);
    } else {
        sweep(false, gv_first);
    }
    if (tr && lane == 0) tr[3] = gtimer();

    // decisions for all positions (two per lane)
    bool lf[2] = {false, false}, mv[2] = {false, false};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int t = lane + 32 * h;
        if (t >= cnt) continue;
        const uint32_t d = h ? dB : dA, v = h ? vB : vA;
        if (parked(v)) continue;
        const double mass = s_mass[t];
        if (MODE == EV_ROOT) {
            if (!isfinite(mass) || mass <= 0.0) atomicExch(a.err, 1);
            a.invc[d] = 1.0 / mass;
        } else if (MODE == EV_PROB) {
            a.prob[d] = mass / a.rank_div;
        } else {
            const double u = s_u[t];
            double ic, cutoff;
            if (ROOT0) {
                const double croot = s_root[t];
                if (!isfinite(croot) || croot <= 0.0) atomicExch(a.err, 1);
                ic = 1.0 / croot;
                a.invc[d] = ic;
                cutoff = 0.0 + ic * mass;
            } else {
                ic = s_ic[t];
                cutoff = s_lo[t] + ic * mass;
            }
            const bool left = cutoff >= u;
            if (a.margin) a.margin[d] = fmin(s_mg[t], fabs(cutoff - u));
            if (left) {
                a.node[d] = 2 * v + 1;
            } else {
                a.node[d] = 2 * v + 2;
                a.low[d] = cutoff;
            }
            lf[h] = left;
            mv[h] = true;
        }
    }
    if (!LEVEL) return;
    const uint64_t Lm = uint64_t(__ballot_sync(FULL, lf[0])) | (uint64_t(__ballot_sync(FULL, lf[1])) << 32);
    const uint64_t Mm = uint64_t(__ballot_sync(FULL, mv[0])) | (uint64_t(__ballot_sync(FULL, mv[1])) << 32);
    const uint64_t Rm = Mm & ~Lm;
    auto bits = [](int lo, int hi) {  // [lo, hi) of a 64-bit mask
        const uint64_t up = hi >= 64 ? ~0ull : ((1ull << hi) - 1ull);
        return up & ~((1ull << lo) - 1ull);
    };
    // claim child slots for every run at once (one atomic round trip)
    for (int r = lane; r < nruns; r += 32) {
        const uint32_t v = s_rv[r];
        if (parked(v)) continue;
        const int rs = int(s_rs[r]), re = r + 1 < nruns ? int(s_rs[r + 1]) : cnt;
        const uint64_t rb = bits(rs, re);
        uint32_t gs = 0, ge = uint32_t(a.J);
        if (v != 0) {
            const uint32_t gl = s_pgs[r] + s_pcl[r];
            gs = (v & 1u) ? s_pgs[r] : gl;
            ge = (v & 1u) ? gl : s_pge[r];
        }
        a.GS[v] = gs;
        a.GE[v] = ge;
        const uint32_t nl = __popcll(static_cast<long long>(Lm & rb)), nr = __popcll(static_cast<long long>(Rm & rb));
        const uint32_t bl = nl ? atomicAdd(a.cntL + v, nl) : 0u;
        const uint32_t br = nr ? atomicAdd(a.cntR + v, nr) : 0u;
        s_bl[r] = gs + bl;
        s_br[r] = ge - 1u - br;
    }
    __syncwarp();
    if (tr && lane == 0) tr[4] = gtimer();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int t = lane + 32 * h;
        if (t < cnt) {
            const uint32_t d = h ? dB : dA, v = h ? vB : vA;
            if (parked(v)) {
                a.perm_out[p0 + t] = d;
                if (a.nsort_out) a.nsort_out[p0 + t] = v;
            } else {
                const int r = run_of(t);
                const uint64_t before = bits(int(s_rs[r]), t);
                const uint32_t pos = lf[h] ? s_bl[r] + __popcll(static_cast<long long>(Lm & before))
                                           : s_br[r] - __popcll(static_cast<long long>(Rm & before));
                KRPG_DCHECK(pos < a.J && 2ull * v + 2 < a.topo.n);
                a.perm_out[pos] = d;
                if (a.nsort_out) a.nsort_out[pos] = 2 * v + (lf[h] ? 1u : 2u);
            }
        }
    }
    if (tr && lane == 0) tr[5] = gtimer();
}

template <int NB, int MODE, bool ROOT0, bool WGT = false>
__global__ void __launch_bounds__(RW * 32, 2) k_eval_reg(EvalArgs a, uint32_t range) {
    using C = RegCfg<NB>;
    extern __shared__ __align__(16) unsigned char smem_regb[];
    __shared__ __align__(8) uint64_t s_bar[RW][RSLOTS];
    const int warp = threadIdx.x >> 5;
    griddep_launch_dependents();
    griddep_wait();
    const uint64_t p0 = (uint64_t(blockIdx.x) * RW + warp) * range;
    if (p0 >= a.J) return;
    const int cnt = int(a.J - p0 < uint64_t(range) ? a.J - p0 : uint64_t(range));
    unsigned long long* tr = a.trace ? a.trace + ((uint64_t(blockIdx.x) * RW + warp) * 16) : nullptr;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int sl = 0; sl < RSLOTS; ++sl) mbar_init(&s_bar[warp][sl], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t phase = 0;
    eval_reg_tile<NB, MODE, ROOT0, WGT>(a, p0, cnt, smem_regb + warp * C::WARP_STRIDE, s_bar[warp], phase, tr);
}

// Grid-wide barrier of a cooperatively launched (fully resident) grid: the pattern of
// cooperative groups' grid.sync() on a caller-provided counter that starts at zero
// (the n-th barrier waits for n * gridDim.x arrivals): release arrival after the CTA barrier,
// acquire polling (which invalidates the SM's L1) before it, so plain loads see the other CTAs' data.
__device__ __forceinline__ void grid_barrier(uint32_t* ctr, uint32_t target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t seen;
        asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(seen) : "l"(ctr) : "memory");
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(ctr) : "memory");
        } while (seen < target);
    }
    __syncthreads();
}

// Several consecutive levels in ONE cooperative launch (levels >= 1 of a stage): the same
// per-warp tile routine, a grid barrier where the kernel boundary was, the sorted-order
// buffers swapped in place. Same arithmetic, bit-identical draws; saves the launch, drain
// and ramp of a kernel boundary per level (the level kernels are latency bound, DESIGN 3).
// Warp w takes tiles w, w + #warps, ...; the launcher only uses it while the level is one
// resident wave (one tile per warp).
template <int NB, bool WGT>
__global__ void __launch_bounds__(RW * 32, 2) k_eval_reg_ml(EvalArgs a, uint32_t range, uint32_t nlev, uint32_t* gbar) {
    using C = RegCfg<NB>;
    extern __shared__ __align__(16) unsigned char smem_regb[];
    __shared__ __align__(8) uint64_t s_bar[RW][RSLOTS];
    const int warp = threadIdx.x >> 5;
    griddep_launch_dependents();
    griddep_wait();
    const uint64_t nwarps = uint64_t(gridDim.x) * RW, gw = uint64_t(blockIdx.x) * RW + warp;
    const uint64_t ntiles = (a.J + range - 1) / range;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int sl = 0; sl < RSLOTS; ++sl) mbar_init(&s_bar[warp][sl], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t phase = 0;
    for (uint32_t li = 0;; ++li) {
        for (uint64_t t = gw; t < ntiles; t += nwarps) {
            const uint64_t p0 = t * range;
            const int cnt = int(a.J - p0 < uint64_t(range) ? a.J - p0 : uint64_t(range));
#ifdef KRPG_LEVEL_BENCH
            if (g_ml_dbg == 1 && li > 0) continue;
#endif
            eval_reg_tile<NB, EV_LEVEL, false, WGT>(a, p0, cnt, smem_regb + warp * C::WARP_STRIDE, s_bar[warp], phase,
                                                    nullptr);
            __syncwarp();
        }
        if (li + 1 == nlev) break;
#ifdef KRPG_LEVEL_BENCH
        if (g_ml_dbg != 2)
#endif
        grid_barrier(gbar, (li + 1) * gridDim.x);
        const uint32_t* pn = a.perm_out;
        a.perm_out = const_cast<uint32_t*>(a.perm);
        a.perm = pn;
        if (a.nsort_in) {
            const uint32_t* nn = a.nsort_out;
            a.nsort_out = const_cast<uint32_t*>(a.nsort_in);
            a.nsort_in = nn;
        }
    }
}

// ---- R = 64 / 128: the Gram split over the 4 warps of a CTA (register-resident) ----
// A CTA's 4 warps share every 8-draw block of the CTA's <= 64 positions: warp w
// holds the upper-triangle tiles of the column-block pairs {q, NB-1-q} for
// q = w + 4c (c < NB/8), NB+1 tiles per pair (9 at R = 64, 2 x 17 at R = 128), off-
// diagonal ones pre-doubled, and computes those columns' share of x_d^T G x_d for
// all blocks; the four partial masses are summed in warp order after ONE CTA
// barrier per sweep. Every pair's tiles are listed as entries k = 0..NB of a fixed
// shape (k <= q: tile (k, q), else tile (k-q-1, NB-1-q)) so the fragment registers
// are indexed at compile time for any w. The CTA's rows arrive by one 1-D TMA copy
// per row at the start; decisions, ranks, slot claims and the next level's order
// follow k_eval_reg. qf_split_order computes the same sum in one warp (first-position
// tables), so both give bit-identical masses.
constexpr int SPW = 4;   // warps per CTA
constexpr int SPR = 64;  // max positions per CTA
template <int NB>
struct SplitCfg {
    static constexpr int R = 8 * NB;
    static constexpr int PP = NB / 8;       // column-block pairs per warp
    static constexpr int NE = NB + 1;       // tiles per pair
    static constexpr int XS = R + 4;        // doubles per staged row
    static constexpr size_t ROWS = size_t(SPR) * XS * 8;
    static constexpr size_t PART = size_t(2) * SPW * SPR * 8;  // root and node partial masses
    static constexpr size_t DBL = size_t(4) * SPR * 8;         // u, 1/C, low, margin
    static constexpr size_t U32 = size_t(2) * SPR * 4 + size_t(7) * SPR * 4;
    static constexpr size_t SMEM = ROWS + PART + DBL + U32 + SPR * 2 + 64;
};

template <int NB>
__device__ __forceinline__ void split_entry(int q, int k, int& p, int& col) {
    p = k <= q ? k : k - q - 1;
    col = k <= q ? q : NB - 1 - q;
}

template <int NB, bool WGT = false>
__device__ __forceinline__ void split_load(double (&g)[NB / 8][NB + 1][2], const double* __restrict__ G, int w,
                                           int lane, const double* __restrict__ W = nullptr) {
    constexpr int R = 8 * NB;
    const int r4 = lane & 3, cq = lane >> 2;
#pragma unroll
    for (int c = 0; c < NB / 8; ++c) {
        const int qa = w + 4 * c;
#pragma unroll
        for (int k = 0; k <= NB; ++k) {
            int p, q;  // tile (p, q) of column block q
            split_entry<NB>(qa, k, p, q);
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int row = 8 * p + 4 * s + r4;
                const int rowoff = row * R - (row * (row - 1)) / 2 - row;
                if (p == q) {
                    const int cc = 8 * p + cq;
                    const int diag = row <= cc ? rowoff + cc : cc * R - (cc * (cc - 1)) / 2 - cc + row;
                    g[c][k][s] = WGT ? __ldg(G + diag) * __ldg(W + diag) : __ldg(G + diag);
                } else {
                    const double x = WGT ? __ldg(G + rowoff + 8 * q + cq) * __ldg(W + rowoff + 8 * q + cq)
                                         : __ldg(G + rowoff + 8 * q + cq);
                    g[c][k][s] = x + x;
                }
            }
        }
    }
}

// warp w's columns' share of the masses of the 8 rows xs (row stride xs_stride; row m valid iff valid)
template <int NB>
__device__ __forceinline__ double split_block(const double (&g)[NB / 8][NB + 1][2], const double* xs, int xs_stride,
                                              bool valid, int w, int lane) {
    const int r4 = lane & 3, m = lane >> 2;
    const double* xr = xs + m * xs_stride;
    double y[NB / 8][2][2];  // [pair][first / second column][c0, c1]
#pragma unroll
    for (int c = 0; c < NB / 8; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) y[c][h][0] = y[c][h][1] = 0.0;
#pragma unroll
    for (int c = 0; c < NB / 8; ++c) {
        const int qa = w + 4 * c;
#pragma unroll
        for (int k = 0; k <= NB; ++k) {
            int p, col;
            split_entry<NB>(qa, k, p, col);
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const double av = valid ? xr[8 * p + 4 * s + r4] : 0.0;
                if (k <= qa)
                    dmma_884(y[c][0][0], y[c][0][1], av, g[c][k][s]);
                else
                    dmma_884(y[c][1][0], y[c][1][1], av, g[c][k][s]);
            }
        }
    }
    double part = 0.0;
    if (valid) {
#pragma unroll
        for (int c = 0; c < NB / 8; ++c) {
            const int qa = w + 4 * c;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int q = h == 0 ? qa : NB - 1 - qa;
                const double2 xv = *reinterpret_cast<const double2*>(xr + 8 * q + 2 * r4);
                part = fma(xv.x, y[c][h][0], part);
                part = fma(xv.y, y[c][h][1], part);
            }
        }
    }
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    return part;
}

// the split-order mass of 8 rows in ONE warp: the four warps' partials in turn,
// summed in warp order (bit-identical to k_eval_split; row stride xs_stride)
template <int NB>
__device__ __forceinline__ double qf_split_order(const double* __restrict__ G, const double* xs, int xs_stride,
                                                 bool valid, int lane) {
    double part[SPW];
#pragma unroll 1
    for (int w = 0; w < SPW; ++w) {
        double g[NB / 8][NB + 1][2];
        split_load<NB>(g, G, w, lane);
        part[w] = split_block<NB>(g, xs, xs_stride, valid, w, lane);
    }
    return ((part[0] + part[1]) + part[2]) + part[3];
}

template <int NB, int MODE, bool ROOT0, bool WGT = false>
__global__ void __launch_bounds__(SPW * 32, NB <= 8 ? 4 : 2) k_eval_split(EvalArgs a, uint32_t range) {
    using SC = SplitCfg<NB>;
    constexpr int R = 8 * NB;
    constexpr int SPXS = SC::XS;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr bool LEVEL = MODE == EV_LEVEL;
    extern __shared__ __align__(16) unsigned char sp_smem[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ int s_nruns, s_nblk;
    __shared__ uint64_t s_lm[2], s_mm[2];
    double* rows = reinterpret_cast<double*>(sp_smem);
    double* part = rows + SPR * SPXS;                 // [2][SPW][SPR]
    double* s_u = part + 2 * SPW * SPR;
    double* s_ic = s_u + SPR;
    double* s_lo = s_ic + SPR;
    double* s_mg = s_lo + SPR;
    uint32_t* s_d = reinterpret_cast<uint32_t*>(s_mg + SPR);
    uint32_t* s_v = s_d + SPR;
    uint32_t* s_rs = s_v + SPR;  // per run (SPR + 1)
    uint32_t* s_rv = s_rs + SPR + 1;
    uint32_t* s_gs = s_rv + SPR;
    uint32_t* s_ge = s_gs + SPR;
    uint32_t* s_bl = s_ge + SPR;
    uint32_t* s_br = s_bl + SPR;
    uint16_t* s_blk = reinterpret_cast<uint16_t*>(s_br + SPR);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    griddep_launch_dependents();
    griddep_wait();
    const uint64_t c0 = uint64_t(blockIdx.x) * range;  // range <= SPR positions per CTA
    if (c0 >= a.J) return;
    const int cnt = int(a.J - c0 < uint64_t(range) ? a.J - c0 : uint64_t(range));
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
    }
    if (tid < cnt) {
        const uint32_t d = a.perm ? a.perm[c0 + tid] : uint32_t(c0 + tid);
        s_d[tid] = d;
        s_v[tid] = (LEVEL && !ROOT0) ? (a.nsort_in ? a.nsort_in[c0 + tid] : a.node[d]) : 0u;
        if (LEVEL) {
            s_u[tid] = a.ud[d];
            if (!ROOT0) {
                s_ic[tid] = a.invc[d];
                s_lo[tid] = a.low[d];
            }
            if (a.margin) s_mg[tid] = a.margin[d];
        }
    }
    __syncthreads();
    if (warp == 0) {  // rows (one bulk copy each), runs, block list
        if (lane == 0) mbar_arrive_expect_tx(&s_bar, uint32_t(cnt) * R * 8);
        __syncwarp();
        for (int t = lane; t < cnt; t += 32)
            tma_load_1d(rows + t * SPXS, a.X + uint64_t(s_d[t]) * R, R * 8, &s_bar);
        int nr = 0;
        for (int tb = 0; tb < cnt; tb += 32) {
            const int t = tb + lane;
            const bool start = t < cnt && (t == 0 || s_v[t] != s_v[t - 1]);
            const unsigned bal = __ballot_sync(FULL, start);
            if (start) {
                const int r = nr + __popc(bal & ((1u << lane) - 1u));
                s_rs[r] = uint32_t(t);
                s_rv[r] = s_v[t];
            }
            nr += __popc(bal);
        }
        if (lane == 0) {
            s_rs[nr] = uint32_t(cnt);
            int nb = 0;
            for (int r = 0; r < nr; ++r) {
                const int rs = int(s_rs[r]), re = int(s_rs[r + 1]);
                if (LEVEL && !ROOT0 && is_leaf(a.topo, s_rv[r])) continue;
                for (int b0 = rs; b0 < re; b0 += 8) s_blk[nb++] = uint16_t(b0 | (min(8, re - b0) << 8));
            }
            s_nruns = nr;
            s_nblk = nb;
        }
    }
    __syncthreads();
    const int nruns = s_nruns, nblk = s_nblk;
    if (LEVEL)  // the parents' ranges of every run
        for (int r = tid; r < nruns; r += SPW * 32) {
            const uint32_t v = s_rv[r];
            if (!ROOT0 && is_leaf(a.topo, v)) continue;
            uint32_t gs = 0, ge = uint32_t(a.J);
            if (v != 0) {
                const uint32_t pp = (v - 1) >> 1;
                const uint32_t gl = a.GS[pp] + a.cntL[pp];
                gs = (v & 1u) ? a.GS[pp] : gl;
                ge = (v & 1u) ? gl : a.GE[pp];
            }
            s_gs[r] = gs;
            s_ge[r] = ge;
            a.GS[v] = gs;
            a.GE[v] = ge;
        }
    mbar_wait(&s_bar, 0);
    auto sweep = [&](bool node_gram, double* pbuf) {
        double* pw = pbuf + warp * SPR;
        constexpr uint64_t P = uint64_t(R) * (R + 1) / 2;
        double g[NB / 8][NB + 1][2];
        uint32_t gv = 0xFFFFFFFFu;
        for (int i = 0; i < nblk; ++i) {
            const uint32_t e = s_blk[i];
            const int b0 = e & 0xff, n = e >> 8;
            const uint32_t v = s_v[b0];
            if (v != gv) {
                split_load<NB, WGT>(g, node_gram ? a.tree + slot_of(2ull * v + 1) * P : a.tree, warp, lane, a.W);
                gv = v;
            }
            const int m = lane >> 2;
            const double pm = split_block<NB>(g, rows + b0 * SPXS, SPXS, m < n, warp, lane);
            if ((lane & 3) == 0 && m < n) pw[b0 + m] = pm;
        }
    };
    if (ROOT0) sweep(false, part + SPW * SPR);
    sweep(LEVEL && true, part);
    __syncthreads();
    // decisions (positions t = tid < cnt: warps 0 and 1)
    bool lf = false, mv = false;
    if (tid < cnt) {
        const int t = tid;
        const uint32_t d = s_d[t], v = s_v[t];
        const bool parked = LEVEL && !ROOT0 && is_leaf(a.topo, v);
        if (!parked) {
            const double mass = ((part[t] + part[SPR + t]) + part[2 * SPR + t]) + part[3 * SPR + t];
            if (MODE == EV_PROB) {
                a.prob[d] = mass / a.rank_div;
            } else if (MODE == EV_ROOT) {
                if (!isfinite(mass) || mass <= 0.0) atomicExch(a.err, 1);
                a.invc[d] = 1.0 / mass;
            } else {
                const double u = s_u[t];
                double ic, cutoff;
                if (ROOT0) {
                    const double* pr = part + SPW * SPR;
                    const double croot = ((pr[t] + pr[SPR + t]) + pr[2 * SPR + t]) + pr[3 * SPR + t];
                    if (!isfinite(croot) || croot <= 0.0) atomicExch(a.err, 1);
                    ic = 1.0 / croot;
                    a.invc[d] = ic;
                    cutoff = 0.0 + ic * mass;
                } else {
                    ic = s_ic[t];
                    cutoff = s_lo[t] + ic * mass;
                }
                const bool left = cutoff >= u;
                if (a.margin) a.margin[d] = fmin(s_mg[t], fabs(cutoff - u));
                if (left) {
                    a.node[d] = 2 * v + 1;
                } else {
                    a.node[d] = 2 * v + 2;
                    a.low[d] = cutoff;
                }
                lf = left;
                mv = true;
            }
        }
    }
    if (!LEVEL) return;
    if (warp < 2) {
        const unsigned l = __ballot_sync(FULL, lf), mm = __ballot_sync(FULL, mv);
        if (lane == 0) {
            s_lm[warp] = l;
            s_mm[warp] = mm;
        }
    }
    __syncthreads();
    const uint64_t Lm = s_lm[0] | (s_lm[1] << 32), Mm = s_mm[0] | (s_mm[1] << 32), Rm = Mm & ~Lm;
    auto bits = [](int lo, int hi) {
        const uint64_t up = hi >= 64 ? ~0ull : ((1ull << hi) - 1ull);
        return up & ~((1ull << lo) - 1ull);
    };
    for (int r = tid; r < nruns; r += SPW * 32) {
        const uint32_t v = s_rv[r];
        if (!ROOT0 && is_leaf(a.topo, v)) continue;
        const uint64_t rb = bits(int(s_rs[r]), int(s_rs[r + 1]));
        const uint32_t nl = __popcll(static_cast<long long>(Lm & rb)), nr = __popcll(static_cast<long long>(Rm & rb));
        s_bl[r] = s_gs[r] + (nl ? atomicAdd(a.cntL + v, nl) : 0u);
        s_br[r] = s_ge[r] - 1u - (nr ? atomicAdd(a.cntR + v, nr) : 0u);
    }
    __syncthreads();
    if (tid < cnt) {
        const int t = tid;
        const uint32_t d = s_d[t], v = s_v[t];
        if (!ROOT0 && is_leaf(a.topo, v)) {
            a.perm_out[c0 + t] = d;
            if (a.nsort_out) a.nsort_out[c0 + t] = v;
        } else {
            int r = 0;  // run of position t (runs are few: linear search from the run starts)
            while (r + 1 < nruns && int(s_rs[r + 1]) <= t) ++r;
            const uint64_t before = bits(int(s_rs[r]), t);
            const uint32_t pos = lf ? s_bl[r] + __popcll(static_cast<long long>(Lm & before))
                                    : s_br[r] - __popcll(static_cast<long long>(Rm & before));
            a.perm_out[pos] = d;
            if (a.nsort_out) a.nsort_out[pos] = 2 * v + (lf ? 1u : 2u);
        }
    }
}

// ---- first position (h = ones): per-draw quadratic forms become tables ----
// Before the first included factor the history h is all ones (krp_sampler.cpp
// two-stage loop), so (a) every draw's E-tree mass at node v is the same number
// 1^T Q_v 1, and (b) a draw's factor-tree vector z = h o V[:, u] = V[:, u]
// depends only on its eigen-component u (R possibilities). The masses of the
// E-tree and of the top L0 factor-tree levels are therefore computed once per
// (node, u) -- with block_qf_packed, i.e. exactly the arithmetic the per-draw
// kernels apply to the identical row, so every decision is bit-identical -- and
// each draw walks those levels with table lookups. The draws are then placed in
// node order for level L0 (counting sort) and the level kernels take over.
constexpr int kPos0Levels = 7;  // factor-tree levels served from the table (64 x 127 masses at R = 64)

template <int NB>
__global__ void __launch_bounds__(256) k_pos0_tables(const double* __restrict__ Q, Topo te, const double* __restrict__ Zt,
                                                     uint32_t L0, const double* __restrict__ V, double* __restrict__ etab,
                                                     double* __restrict__ ztab, int* err, int split) {
    constexpr int R = 8 * NB;
    constexpr uint64_t P = uint64_t(R) * (R + 1) / 2;
    __shared__ __align__(16) double s_vt[R * R + R];  // V^T rows (z of component u) + a ones row
    griddep_launch_dependents();
    griddep_wait();
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < R * R; i += blockDim.x) {
        const int u = i / R, c = i - u * R;
        s_vt[i] = 1.0 * V[uint64_t(c) * R + u];  // h o V[:, u] with h = 1 (k_make_z)
    }
    for (int i = tid; i < R; i += blockDim.x) s_vt[R * R + i] = 1.0;
    __syncthreads();
    const FragAddr<NB> fa(lane);
    const uint32_t nz = (1u << L0);  // internal nodes of levels < L0, plus the root normaliser
    const uint64_t ne = te.n + 1;     // E-tree: a mass per node (left child), plus the root
    const uint64_t items = ne + uint64_t(nz) * NB;
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + tid) >> 5, nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t it = gw; it < items; it += nw) {
        const int m = lane >> 2;
        if (it < ne) {  // E-tree node (x = h = ones for all 8 rows)
            const uint64_t v = it;
            const double* G;
            if (v == te.n) G = Q;  // root
            else if (!is_leaf(te, v)) G = Q + slot_of(2 * v + 1) * P;
            else continue;
            double mass;
            if constexpr (NB == 8) {  // the level kernel's arithmetic: split order when it is the split kernel
                mass = split ? qf_split_order<NB>(G, s_vt + R * R, 0, true, lane) : block_qf_packed<NB>(G, fa, s_vt + R * R, lane);
            } else {
                mass = block_qf_packed<NB>(G, fa, s_vt + R * R, lane);
            }
            if (lane == 0) etab[v] = mass;
        } else {
            const uint64_t j = it - ne;
            const uint32_t vi = uint32_t(j / NB), ub = uint32_t(j % NB);
            const double* G = vi == nz - 1 ? Zt : Zt + slot_of(2ull * vi + 1) * P;  // last row: root
            const uint32_t u = ub * 8 + m;
            double mass;
            if constexpr (NB == 8) {
                mass = split ? qf_split_order<NB>(G, s_vt + ub * 8 * R, R, true, lane) : block_qf_packed<NB>(G, fa, s_vt + u * R, lane);
            } else {
                mass = block_qf_packed<NB>(G, fa, s_vt + u * R, lane);
            }
            if ((lane & 3) == 0) {
                ztab[uint64_t(vi) * R + u] = mass;
                if (vi == nz - 1 && (!isfinite(mass) || mass <= 0.0)) atomicExch(err, 1);
            }
        }
    }
}

// E-tree walk of every draw with the node masses of the table (F = 1 leaves)
__global__ void k_pos0_ewalk(const double* __restrict__ etab, Topo te, uint64_t J, const double* __restrict__ ud,
                             double* __restrict__ margin, uint32_t* __restrict__ node, uint32_t* __restrict__ comp,
                             uint32_t* __restrict__ zero, uint32_t nzero, int* err) {
    griddep_launch_dependents();
    griddep_wait();
    const uint64_t i0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (uint64_t i = i0; i < nzero; i += uint64_t(gridDim.x) * blockDim.x) zero[i] = 0;
    const double croot = etab[te.n];
    if (i0 == 0 && (!isfinite(croot) || croot <= 0.0)) atomicExch(err, 1);
    const double ic = 1.0 / croot;
    for (uint64_t d = i0; d < J; d += uint64_t(gridDim.x) * blockDim.x) {
        const double u = ud[d];
        double mg = margin ? margin[d] : 0.0;
        uint64_t v = 0;
        double low = 0.0;
        bool first = true;
        while (!is_leaf(te, v)) {
            const double cutoff = first ? 0.0 + ic * etab[v] : low + ic * etab[v];
            first = false;
            const bool left = cutoff >= u;
            mg = fmin(mg, fabs(cutoff - u));
            if (left) {
                v = 2 * v + 1;
            } else {
                v = 2 * v + 2;
                low = cutoff;
            }
        }
        node[d] = uint32_t(v);
        comp[d] = uint32_t(leaf_index(te, v));
        if (margin) margin[d] = mg;
    }
}

// factor-tree levels [0, L0) of every draw from the table; counts per level-L0 node
__global__ void k_pos0_zwalk(const double* __restrict__ ztab, uint32_t L0, const uint32_t* __restrict__ comp, uint32_t R,
                             uint64_t J, const double* __restrict__ ud, double* __restrict__ margin,
                             uint32_t* __restrict__ node, double* __restrict__ low_out, double* __restrict__ invc,
                             uint32_t* __restrict__ hist) {
    griddep_launch_dependents();
    griddep_wait();
    const uint32_t nz = 1u << L0;
    for (uint64_t d = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; d < J; d += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t u = comp[d];
        const double ic = 1.0 / ztab[uint64_t(nz - 1) * R + u];
        const double uu = ud[d];
        double mg = margin ? margin[d] : 0.0;
        uint32_t v = 0;
        double low = 0.0;
        for (uint32_t l = 0; l < L0; ++l) {
            const double m = ztab[uint64_t(v) * R + u];
            const double cutoff = l == 0 ? 0.0 + ic * m : low + ic * m;
            const bool left = cutoff >= uu;
            mg = fmin(mg, fabs(cutoff - uu));
            if (left) {
                v = 2 * v + 1;
            } else {
                v = 2 * v + 2;
                low = cutoff;
            }
        }
        node[d] = v;
        low_out[d] = low;
        invc[d] = ic;
        if (margin) margin[d] = mg;
        atomicAdd(hist + (v - (nz - 1)), 1u);
    }
}

// counting-sort placement into level-L0 node order; the level L0-1 nodes get the
// position ranges the level kernels derive their children's ranges from
__global__ void __launch_bounds__(256) k_pos0_place(uint32_t L0, uint64_t J, const uint32_t* __restrict__ node,
                                                    const uint32_t* __restrict__ hist, uint32_t* __restrict__ cursor,
                                                    uint32_t* __restrict__ perm, uint32_t* __restrict__ nsort,
                                                    uint32_t* __restrict__ GS, uint32_t* __restrict__ GE,
                                                    uint32_t* __restrict__ cntL) {
    __shared__ uint32_t s_off[1u << kPos0Levels];
    griddep_launch_dependents();
    griddep_wait();
    const uint32_t nl = 1u << L0, first = nl - 1;
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t i = 0; i < nl; ++i) {
            s_off[i] = acc;
            acc += hist[i];
        }
    }
    __syncthreads();
    if (blockIdx.x == 0)
        for (uint32_t i = threadIdx.x; i < nl / 2; i += blockDim.x) {
            const uint32_t p = (first - 1) / 2 + i;  // level L0-1 node; children 2p+1, 2p+2
            const uint32_t c = 2 * p + 1 - first;
            GS[p] = s_off[c];
            cntL[p] = hist[c];
            GE[p] = s_off[c + 1] + hist[c + 1];
        }
    for (uint64_t d = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; d < J; d += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = node[d], c = v - first;
        const uint32_t pos = s_off[c] + atomicAdd(cursor + c, 1u);
        perm[pos] = uint32_t(d);
        nsort[pos] = v;
    }
}

// ---- ranks whose Gram does not fit shared memory (R > 160) ----------------
// Same CTA / run / decision structure as k_eval_cta, but each run's packed
// Gram is streamed HBM/L2 -> shared memory in chunks of whole 8-row tile-rows
// through a 3-stage TMA ring, and the quadratic form is reorganised by
// tile-row so that nothing but a scalar survives between chunks:
//   x^T G x = sum_p x_p . t_p,  t_p = G_pp x_p + 2 sum_{q>p} G_pq x_q,
// t_p for 8 draws = one DMMA chain over q >= p (A = the draws' x_q fragments,
// held in registers for the whole Gram; B = tile-row p of G). A warp carries
// SB_BW 8-draw blocks through one pass over the Gram; runs longer than one
// wave (CWARPS * SB_BW blocks) stream the Gram again (an L2 hit).
constexpr int SB_BW = 2;
constexpr int SB_STAGES = 3;
constexpr int SB_CHD = 3072;  // doubles per ring stage (24 KB) >= the largest tile-row at R <= 256

template <int NB>
__device__ __forceinline__ int tile_row_off(int p) {  // pack_index(8p, 8p)
    constexpr int R = 8 * NB;
    const int r = 8 * p;
    return r * R - (r * (r - 1)) / 2;
}

template <int NB, int MODE>
__global__ void __launch_bounds__(CB) k_eval_stream(EvalArgs a, uint32_t range) {
    constexpr int R = 8 * NB;
    constexpr uint32_t P = uint32_t(R) * (R + 1) / 2;
    static_assert(8 * R <= SB_CHD, "tile-row larger than a ring stage");
    constexpr int BW = NB >= 28 ? 1 : SB_BW;  // register budget: x fragments of BW blocks
    extern __shared__ __align__(128) double ring[];  // [SB_STAGES][SB_CHD]
    __shared__ uint32_t s_d[CB], s_v[CB], s_rank[CB];
    __shared__ uint8_t s_left[CB];
    __shared__ int s_rs[CB + 1];
    __shared__ int s_nruns;
    __shared__ int s_cb[NB + 1];  // chunk c = tile-rows [s_cb[c], s_cb[c+1])
    __shared__ int s_nch;
    __shared__ uint32_t s_cnt[2], s_base[2], s_gs, s_ge;
    __shared__ __align__(8) uint64_t bar[SB_STAGES];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t base = uint64_t(blockIdx.x) * range;  // range <= CB positions per CTA
    const int cnt = a.J - base < uint64_t(range) ? int(a.J - base) : int(range);
    if (tid < cnt) {
        const uint32_t d = a.perm ? a.perm[base + tid] : uint32_t(base + tid);
        s_d[tid] = d;
        s_v[tid] = MODE == EV_LEVEL ? (a.nsort_in ? a.nsort_in[base + tid] : a.node[d]) : 0u;
    }
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < SB_STAGES; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        int nc = 0, p0 = 0;
        while (p0 < NB) {  // greedy: whole tile-rows while they fit one stage
            int p1 = p0 + 1;
            while (p1 < NB && (p1 + 1 < NB ? tile_row_off<NB>(p1 + 1) : int(P)) - tile_row_off<NB>(p0) <= SB_CHD) ++p1;
            s_cb[nc++] = p0;
            p0 = p1;
        }
        s_cb[nc] = NB;
        s_nch = nc;
    }
    __syncthreads();
    {  // run boundaries -> compact list s_rs
        const bool flag = tid < cnt && (tid == 0 || s_v[tid] != s_v[tid - 1]);
        const unsigned bal = __ballot_sync(0xffffffffu, flag);
        __shared__ int wcount[CWARPS];
        if (lane == 0) wcount[warp] = __popc(bal);
        __syncthreads();
        int off = 0;
        for (int w = 0; w < warp; ++w) off += wcount[w];
        if (flag) s_rs[off + __popc(bal & ((1u << lane) - 1u))] = tid;
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < CWARPS; ++w) tot += wcount[w];
            s_nruns = tot;
            s_rs[tot] = cnt;
        }
        __syncthreads();
    }
    const int nruns = s_nruns, nch = s_nch;
    constexpr int WAVE = CWARPS * BW;
    auto gsrc = [&](int r) -> const double* {
        if (MODE != EV_LEVEL) return a.tree;
        const uint32_t v = s_v[s_rs[r]];
        if (is_leaf(a.topo, v)) return nullptr;
        return a.tree + slot_of(2ull * v + 1) * uint64_t(P);
    };
    // producer (thread 0): the sequence run -> wave -> chunk, skipping leaf runs
    int pr = 0, pw = 0, pc = 0;
    uint32_t issued = 0;
    const double* pg = nullptr;
    auto pseek = [&]() {  // advance pr to the next run with a Gram
        while (pr < nruns && !(pg = gsrc(pr))) ++pr;
    };
    auto produce = [&]() {
        if (tid != 0 || pr >= nruns) return;
        const int st = int(issued % SB_STAGES);
        const int o0 = tile_row_off<NB>(s_cb[pc]);
        const int o1 = s_cb[pc + 1] < NB ? tile_row_off<NB>(s_cb[pc + 1]) : int(P);
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[st], uint32_t(o1 - o0) * 8u);
        tma_load_1d(ring + st * SB_CHD, pg + o0, uint32_t(o1 - o0) * 8u, &bar[st]);
        ++issued;
        if (++pc == nch) {
            pc = 0;
            const int nblk = (s_rs[pr + 1] - s_rs[pr] + 7) >> 3;
            if (++pw * WAVE >= nblk) {
                pw = 0;
                ++pr;
                pseek();
            }
        }
    };
    if (tid == 0) {
        pseek();
        for (int s = 0; s < SB_STAGES - 1; ++s) produce();
    }
    uint32_t consumed = 0;
    const int r4 = lane & 3, cq = lane >> 2, m = lane >> 2;
    for (int r = 0; r < nruns; ++r) {
        const int rs = s_rs[r], re = s_rs[r + 1];
        if (!gsrc(r)) {  // draws parked at a leaf one level up keep their positions
            if (MODE == EV_LEVEL)
                for (int t = rs + tid; t < re; t += CB) {
                    a.perm_out[base + t] = s_d[t];
                    if (a.nsort_out) a.nsort_out[base + t] = s_v[t];
                }
            continue;
        }
        const uint32_t v = s_v[rs];
        if (tid < 2) s_cnt[tid] = 0;
        if (MODE == EV_LEVEL && tid == 0) {  // this node's position range, from its parent's
            uint32_t gs = 0, ge = uint32_t(a.J);
            if (v != 0) {
                const uint32_t p = (v - 1) >> 1;
                const uint32_t gl = a.GS[p] + a.cntL[p];
                gs = (v & 1u) ? a.GS[p] : gl;
                ge = (v & 1u) ? gl : a.GE[p];
            }
            s_gs = gs;
            s_ge = ge;
            a.GS[v] = gs;
            a.GE[v] = ge;
        }
        __syncthreads();
        const int nblk = (re - rs + 7) >> 3;
        for (int w0 = 0; w0 < nblk; w0 += WAVE) {
            // this warp's blocks of the wave: x fragments for the whole pass
            double av[BW][NB][2];
            double part[BW];
            bool bval[BW];
            const double* xr[BW];
#pragma unroll
            for (int j = 0; j < BW; ++j) {
                const int b = w0 + warp + CWARPS * j;
                bval[j] = b < nblk;
                const int b0 = rs + 8 * b;
                const bool valid = bval[j] && b0 + m < re;
                xr[j] = valid ? a.X + uint64_t(s_d[b0 + m]) * R : nullptr;
                part[j] = 0.0;
#pragma unroll
                for (int q = 0; q < NB; ++q)
#pragma unroll
                    for (int s = 0; s < 2; ++s) av[j][q][s] = xr[j] ? xr[j][8 * q + 4 * s + r4] : 0.0;
            }
            for (int c = 0; c < nch; ++c, ++consumed) {
                produce();
                const int st = int(consumed % SB_STAGES);
                mbar_wait(&bar[st], (consumed / SB_STAGES) & 1u);
                const double* Gc = ring + st * SB_CHD - tile_row_off<NB>(s_cb[c]);
                const int pa = s_cb[c], pb = s_cb[c + 1];
#pragma unroll
                for (int p = 0; p < NB; ++p) {
                    if (p < pa || p >= pb) continue;
                    const int row = 8 * p + cq;
                    const int roff = row * R - (row * (row - 1)) / 2 - row;  // pack_index(row, col) = roff + col
                    double d0[BW][2], d1[BW][2];  // two chains (even / odd q)
#pragma unroll
                    for (int j = 0; j < BW; ++j) d0[j][0] = d0[j][1] = d1[j][0] = d1[j][1] = 0.0;
#pragma unroll
                    for (int q = p; q < NB; ++q)
#pragma unroll
                        for (int s = 0; s < 2; ++s) {
                            const int col = 8 * q + 4 * s + r4;
                            // off-diagonal tiles count twice: (2a) g == a (2g) exactly
                            const double g = (q > p || col >= row) ? Gc[roff + col]
                                                                   : Gc[col * R - (col * (col - 1)) / 2 - col + row];
#pragma unroll
                            for (int j = 0; j < BW; ++j) {
                                const double x = q > p ? av[j][q][s] + av[j][q][s] : av[j][q][s];
                                if ((q & 1) == 0)
                                    dmma_884(d0[j][0], d0[j][1], x, g);
                                else
                                    dmma_884(d1[j][0], d1[j][1], x, g);
                            }
                        }
#pragma unroll
                    for (int j = 0; j < BW; ++j)
                        if (xr[j]) {
                            const double2 xv = *reinterpret_cast<const double2*>(xr[j] + 8 * p + 2 * r4);
                            part[j] = fma(xv.x, d0[j][0] + d1[j][0], part[j]);
                            part[j] = fma(xv.y, d0[j][1] + d1[j][1], part[j]);
                        }
                }
                __syncthreads();  // stage free for the producer
            }
#pragma unroll
            for (int j = 0; j < BW; ++j) {
                double mass = part[j];
                mass += __shfl_xor_sync(0xffffffffu, mass, 1);
                mass += __shfl_xor_sync(0xffffffffu, mass, 2);
                if (!bval[j]) continue;  // warp-uniform
                const int b0 = rs + 8 * (w0 + warp + CWARPS * j);
                const int n = min(8, re - b0);
                const bool valid = m < n;
                const uint32_t dd = valid ? s_d[b0 + m] : 0u;
                const bool owner = valid && r4 == 0;
                if (MODE == EV_ROOT) {
                    if (owner) {
                        if (!isfinite(mass) || mass <= 0.0) atomicExch(a.err, 1);
                        a.invc[dd] = 1.0 / mass;
                    }
                } else if (MODE == EV_PROB) {
                    if (owner) a.prob[dd] = mass / a.rank_div;
                } else {
                    bool left = false;
                    double cutoff = 0.0;
                    if (owner) {
                        const double u = a.ud[dd];
                        cutoff = a.low[dd] + a.invc[dd] * mass;
                        left = cutoff >= u;
                        if (a.margin) a.margin[dd] = fmin(a.margin[dd], fabs(cutoff - u));
                    }
                    const unsigned lm = __ballot_sync(0xffffffffu, owner && left);
                    const unsigned rm = __ballot_sync(0xffffffffu, owner && !left);
                    uint32_t bl = 0, br = 0;
                    if (lane == 0) {
                        if (lm) bl = atomicAdd(&s_cnt[0], uint32_t(__popc(lm)));
                        if (rm) br = atomicAdd(&s_cnt[1], uint32_t(__popc(rm)));
                    }
                    bl = __shfl_sync(0xffffffffu, bl, 0);
                    br = __shfl_sync(0xffffffffu, br, 0);
                    if (owner) {
                        const unsigned below = (1u << lane) - 1u;
                        const int slot = b0 + m;
                        s_left[slot] = left ? 1 : 0;
                        if (left) {
                            a.node[dd] = 2 * v + 1;
                            s_rank[slot] = bl + __popc(lm & below);
                        } else {
                            a.node[dd] = 2 * v + 2;
                            s_rank[slot] = br + __popc(rm & below);
                            a.low[dd] = cutoff;
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (MODE == EV_LEVEL) {
            if (tid == 0) {
                s_base[0] = s_cnt[0] ? atomicAdd(a.cntL + v, s_cnt[0]) : 0u;
                s_base[1] = s_cnt[1] ? atomicAdd(a.cntR + v, s_cnt[1]) : 0u;
            }
            __syncthreads();
            for (int t = rs + tid; t < re; t += CB) {
                const uint32_t pos = s_left[t] ? s_gs + s_base[0] + s_rank[t] : s_ge - 1u - (s_base[1] + s_rank[t]);
                a.perm_out[pos] = s_d[t];
                if (a.nsort_out) a.nsort_out[pos] = 2 * v + (s_left[t] ? 1u : 2u);
            }
            __syncthreads();
        }
    }
}

// stage init: identity order, everyone at the root, this stage's uniform
__global__ void k_stage_init(uint32_t* perm, uint32_t* node, double* low, double* ud, uint32_t* gstart,
                             uint64_t J, uint64_t seed, uint64_t off, uint64_t counter, double* margin,
                             int reset_margin, uint32_t* cntL, uint32_t* cntR, uint64_t nnodes, uint32_t* zero1,
                             uint32_t* zero2) {
    griddep_launch_dependents();
    griddep_wait();
    if (zero1 && blockIdx.x == 0 && threadIdx.x == 0) *zero1 = 0;
    if (zero2 && blockIdx.x == 0 && threadIdx.x == 0) *zero2 = 0;
    for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < nnodes; v += uint64_t(gridDim.x) * blockDim.x) {
        cntL[v] = 0;
        cntR[v] = 0;
    }
    for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < J; d += uint64_t(gridDim.x) * blockDim.x) {
        perm[d] = uint32_t(d);
        node[d] = 0;
        low[d] = 0.0;
        ud[d] = rng_uniform(rng_key(seed, off + d), counter);
        if (margin && reset_margin) margin[d] = HUGE_VAL;
        if (d == 0) gstart[0] = 0;
    }
}

// z_d = h_d o V[:, u_d], u_d = the E-tree leaf reached (F = 1 -> row = leaf index)
__global__ void k_make_z(const double* __restrict__ H, const double* __restrict__ V, const uint32_t* __restrict__ node,
                         Topo te, uint32_t R, uint64_t J, double* __restrict__ Z) {
    griddep_launch_dependents();
    griddep_wait();
    // a warp per draw row (no per-element 64-bit division): coalesced H / Z rows; for
    // R <= 64 the CTA first transposes V into shared memory (column u contiguous)
    extern __shared__ double s_vt[];
    const uint32_t lane = threadIdx.x & 31;
    const bool tr = R <= 64;
    if (tr) {
        for (uint32_t i = threadIdx.x; i < R * R; i += blockDim.x) {
            const uint32_t c = i / R, u = i - c * R;
            s_vt[u * (R + 1) + c] = V[i];
        }
        __syncthreads();
    }
    const uint64_t w0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t d = w0; d < J; d += nw) {
        const uint64_t u = leaf_index(te, node[d]);
        if (tr) {
            for (uint32_t c = lane; c < R; c += 32) Z[d * R + c] = H[d * R + c] * s_vt[u * (R + 1) + c];
        } else {
            for (uint32_t c = lane; c < R; c += 32) Z[d * R + c] = H[d * R + c] * V[uint64_t(c) * R + u];
        }
    }
}

struct LeafArgs {
    uint64_t J;
    uint32_t N, k;
    const uint32_t* perm;
    const uint32_t* node;
    const double* low;
    const double* invc;
    const double* ud;
    double* margin;
    const double* Z;    // J x R
    double* H;          // J x R history (updated)
    uint32_t* idx;      // J x N (nullable)
    const void* U;
    Topo topo;          // Z topology (F = R)
};

// Leaf scan, streaming version: each warp streams the rows of its runs' leaves
// HBM -> shared memory through a 3-stage 1-D TMA ring (16 rows per stage, rows
// padded for conflict-light fragment reads), computes the 16 x 8 mass tile of
// every 8-draw block on DMMA, and lets each draw's lane continue its sequential
// cumulative scan (segment_tree_sampler.cpp:284-292) over those 16 rows. Scan
// state (cum, pick, last nonzero, margin) lives in the lane that owns the draw's
// sorted position, so no per-leaf mass buffer is needed.
template <int NB, typename T>
struct LeafCfg2 {
    static constexpr int R = 8 * NB;
    static constexpr int CH = NB <= 8 ? 16 : 8;  // rows per stage (smem: 4 warps x 3 stages)
    static constexpr int STAGES = 3;
    static constexpr int ROWB = R * int(sizeof(T));
    // rows padded by 16 bytes (one bulk copy per row): unpadded 1 KB rows put the 8 rows of
    // a DMMA A fragment on the same banks (8-way conflicts, 22 % short-scoreboard at R = 128)
    static constexpr int RS = ROWB + 16;
    static constexpr int CHB = CH * RS;
    static constexpr int WARP_BYTES = (STAGES * CHB + CH * 8 * 8 + STAGES * 8 + 127) / 128 * 128;
    static constexpr int SMEM = WPB * WARP_BYTES;
};

template <int NB, typename T>
__global__ void __launch_bounds__(WPB * 32) k_leaf2(LeafArgs a) {
    using C = LeafCfg2<NB, T>;
    constexpr int R = 8 * NB;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* ring = smem_raw + warp * C::WARP_BYTES;
    double* msm = reinterpret_cast<double*>(ring + C::STAGES * C::CHB);  // [CH][8]
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + C::STAGES * C::CHB + C::CH * 8 * 8);
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t base = (uint64_t(blockIdx.x) * WPB + warp) * CHUNK;
    if (base >= a.J) return;
    const int cnt = a.J - base < uint64_t(CHUNK) ? int(a.J - base) : CHUNK;
    const bool live = lane < cnt;
    const uint32_t dl = live ? a.perm[base + lane] : 0u;
    const uint32_t vl = live ? a.node[dl] : 0xFFFFFFFFu;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, vl, 1);
    const uint32_t starts0 = __ballot_sync(0xffffffffu, live && (lane == 0 || vl != prev));
    // lane-owned scan state of the draw at sorted position base + lane
    double cum = 0.0, ic = 0.0, u = 0.0, mg = 0.0;
    if (live) {
        cum = a.low[dl];
        ic = a.invc[dl];
        u = a.ud[dl];
        mg = a.margin ? a.margin[dl] : 0.0;
    }
    uint64_t pick = ~uint64_t{0}, last_nz = ~uint64_t{0};
    const T* U = static_cast<const T*>(a.U);

    auto run_rows = [&](uint32_t v, uint64_t& first, uint64_t& last) {
        const uint64_t l = leaf_index(a.topo, v);
        first = l * a.topo.F;
        last = first + a.topo.F < a.topo.I ? first + a.topo.F : a.topo.I;
    };
    // producer cursor: current run (bit set of remaining run starts) and row
    uint32_t pstarts = starts0;
    uint64_t prow = 0, plast = 0;
    bool pmore = pstarts != 0;
    if (pmore) {
        const int rs = __ffs(pstarts) - 1;
        pstarts &= pstarts - 1;
        run_rows(__shfl_sync(0xffffffffu, vl, rs), prow, plast);
    }
    uint32_t issued = 0;
    auto produce = [&]() {
        if (!pmore) return;
        const int st = int(issued % C::STAGES);
        const uint64_t left = plast - prow;
        const uint32_t nrows = left < uint64_t(C::CH) ? uint32_t(left) : uint32_t(C::CH);
        if (lane == 0) {
            mbar_arrive_expect_tx(&bars[st], nrows * C::ROWB);
            if (C::RS == C::ROWB)  // one contiguous bulk copy per chunk
                tma_load_1d(ring + st * C::CHB, U + prow * R, nrows * C::ROWB, &bars[st]);
        }
        __syncwarp();
        if (C::RS != C::ROWB && uint32_t(lane) < nrows)
            tma_load_1d(ring + st * C::CHB + lane * C::RS, U + (prow + lane) * R, C::ROWB, &bars[st]);
        ++issued;
        prow += C::CH;
        if (prow >= plast) {
            if (pstarts) {
                const int rs = __ffs(pstarts) - 1;
                pstarts &= pstarts - 1;
                run_rows(__shfl_sync(0xffffffffu, vl, rs), prow, plast);
            } else {
                pmore = false;
            }
        }
    };
    for (int s = 0; s < C::STAGES - 1; ++s) produce();

    const int r4 = lane & 3, m8 = lane >> 2;
    uint32_t cstarts = starts0;
    uint32_t chunk_i = 0;
    while (cstarts) {
        const int rs = __ffs(cstarts) - 1;
        cstarts &= cstarts - 1;
        const int re = cstarts ? __ffs(cstarts) - 1 : cnt;
        uint64_t first, last;
        run_rows(__shfl_sync(0xffffffffu, vl, rs), first, last);
        // z fragments of the run's first 8-draw block, loaded once for all of the leaf's
        // chunks (re-reading them per chunk put one global-latency load in front of every
        // DMMA: 75 % long-scoreboard stalls at R = 128)
        double zfirst[2 * NB];
        {
            const int n0 = min(8, re - rs);
            const uint32_t dd0 = __shfl_sync(0xffffffffu, dl, (rs + m8) & 31);
#pragma unroll
            for (int s = 0; s < 2 * NB; ++s) zfirst[s] = m8 < n0 ? a.Z[uint64_t(dd0) * R + 4 * s + r4] : 0.0;
        }
        for (uint64_t r0 = first; r0 < last; r0 += C::CH, ++chunk_i) {
            produce();
            const int st = int(chunk_i % C::STAGES);
            mbar_wait(&bars[st], (chunk_i / C::STAGES) & 1u);
            const int nr = last - r0 < uint64_t(C::CH) ? int(last - r0) : C::CH;
            const unsigned char* buf = ring + st * C::CHB;
            for (int b0 = rs; b0 < re; b0 += 8) {
                const int n = min(8, re - b0);
                const bool valid = m8 < n;
                const uint32_t dd = __shfl_sync(0xffffffffu, dl, (b0 + m8) & 31);
                double zb[2 * NB];
#pragma unroll
                for (int s = 0; s < 2 * NB; ++s)
                    zb[s] = b0 == rs ? zfirst[s] : (valid ? a.Z[uint64_t(dd) * R + 4 * s + r4] : 0.0);
#pragma unroll
                for (int mt = 0; mt < C::CH / 8; ++mt) {
                    const int row = 8 * mt + m8;
                    const bool rv = row < nr;
                    const T* up = reinterpret_cast<const T*>(buf + (rv ? row : 0) * C::RS) + r4;
                    // NC independent DMMA chains over k (a single chain of 2*NB dependent
                    // DMMAs is latency bound at large R)
                    constexpr int NC = NB >= 8 ? 4 : (NB >= 2 ? 2 : 1);
                    double c0[NC], c1[NC];
#pragma unroll
                    for (int c = 0; c < NC; ++c) c0[c] = c1[c] = 0.0;
#pragma unroll
                    for (int s = 0; s < 2 * NB; ++s)
                        dmma_884(c0[s % NC], c1[s % NC], rv ? static_cast<double>(up[4 * s]) : 0.0, zb[s]);
#pragma unroll
                    for (int c = 1; c < NC; ++c) {
                        c0[0] += c0[c];
                        c1[0] += c1[c];
                    }
                    const double acc0 = c0[0], acc1 = c1[0];
                    msm[(8 * mt + m8) * 8 + 2 * r4] = acc0 * acc0;
                    msm[(8 * mt + m8) * 8 + 2 * r4 + 1] = acc1 * acc1;
                }
                __syncwarp();
                if (lane >= b0 && lane < b0 + n && pick == ~uint64_t{0}) {
                    const int col = lane - b0;
                    for (int i = 0; i < nr; ++i) {
                        const double mm = ic * msm[i * 8 + col];
                        if (mm > 0.0) last_nz = r0 + i;
                        cum += mm;
                        mg = fmin(mg, fabs(cum - u));
                        if (cum >= u) {
                            pick = r0 + i;
                            break;
                        }
                    }
                }
                __syncwarp();
            }
            fence_proxy_async();
            __syncwarp();
        }
        // finalize the run's draws (fallback :292), index, margin
        const bool mine = lane >= rs && lane < re;
        if (mine) {
            if (pick == ~uint64_t{0}) pick = last_nz != ~uint64_t{0} ? last_nz : last - 1;
            if (a.margin) a.margin[dl] = mg;
            if (a.idx) a.idx[uint64_t(dl) * a.N + a.k] = uint32_t(pick);
        }
        // h *= U[pick]  (krp_sampler.cpp:137-138): every load of a group of 4 draws issued first
        constexpr int CPL = (R + 31) / 32;
        for (int t0 = rs; t0 < re; t0 += 4) {
            double hv[4][CPL], uv[4][CPL];
            uint32_t dt[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int t = t0 + q < re ? t0 + q : rs;
                dt[q] = __shfl_sync(0xffffffffu, dl, t);
                const uint64_t pt = __shfl_sync(0xffffffffu, pick, t);
#pragma unroll
                for (int cc = 0; cc < CPL; ++cc) {
                    const int c = lane + 32 * cc;
                    hv[q][cc] = c < R ? a.H[uint64_t(dt[q]) * R + c] : 0.0;
                    uv[q][cc] = c < R ? static_cast<double>(U[pt * R + c]) : 0.0;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int cc = 0; cc < CPL; ++cc) {
                    const int c = lane + 32 * cc;
                    if (t0 + q < re && c < R) a.H[uint64_t(dt[q]) * R + c] = hv[q][cc] * uv[q][cc];
                }
        }
    }
}

struct DeepArgs {
    uint64_t J;
    uint32_t N, k, level0;
    const uint32_t* perm;
    const uint32_t* node;
    const double* low;
    const double* invc;
    const double* ud;
    double* margin;
    const double* X;   // z rows (J x R)
    double* H;         // history rows (updated with the drawn row)
    uint32_t* idx;
    uint32_t* pick;    // per draw picked row (for the h update pass)
    const void* U;
    const double* tree;
    Topo topo;
    uint32_t chunk;    // sorted draws per warp (<= 32)
    int leaf_par;      // leaf runs with at most this many draws scan warp-parallel
    int dmma_min;      // internal-level runs with at least this many draws use DMMA
    uint32_t* work;    // chunk counter (zeroed before the launch) for persistent warps, nullable
    int final_rows;    // apply h o= U_k[pick] here (last position of a host-output call)
    double* host_rows; // with final_rows: the call's page-locked host rows (device-mapped), nullable
};


template <int NB, typename T>
struct DeepCfg {
    static constexpr int R = 8 * NB;
    static constexpr int P = R * (R + 1) / 2;
    static constexpr int GB = (P * 8 + 15) / 16 * 16;
    static constexpr int LROWS = 32;
    static constexpr int ROWB = R * int(sizeof(T));
    static constexpr int RSP = ROWB + 16;  // padded leaf row stride (conflict-light fragments)
    static constexpr int LB = LROWS * RSP;
    static constexpr int BUF = ((GB > LB ? GB : LB) + 127) / 128 * 128;
    static constexpr int XS = 3 * R * 8;
    static constexpr int WARP_BYTES = BUF + XS + 128 + 32;  // + perm scratch + 3 mbarriers
    static constexpr int SMEM = WPB * WARP_BYTES;
};

// small runs (<= 3 draws) from a shared-memory Gram: lane b owns x_b
template <int NB, int ND>
__device__ __forceinline__ void small_qf(const double* Gs, const double* x2s, const double (&xr)[3][(8 * NB + 31) / 32],
                                         int lane, double (&mass)[3]) {
    constexpr int R = 8 * NB;
    constexpr int S = (R + 31) / 32;
    // two partial accumulators (even / odd rows) halve the dependent DFMA chains
    double acc[ND][S], acc1[ND][S];
#pragma unroll
    for (int t = 0; t < ND; ++t)
#pragma unroll
        for (int s = 0; s < S; ++s) acc[t][s] = acc1[t][s] = 0.0;
    int off = 0;
#pragma unroll
    for (int kb = 0; kb < S; ++kb) {
        const int a_end = R < 32 * (kb + 1) ? R : 32 * (kb + 1);  // even: R is a multiple of 8
#pragma unroll 2
        for (int ar = 32 * kb; ar < a_end; ar += 2) {
            const int off1 = off + R - ar;  // row ar + 1
            double g[S], h[S];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int b = lane + 32 * s;
                if (s < kb) {
                    g[s] = 0.0;
                    h[s] = 0.0;
                } else if (s == kb) {
                    g[s] = (b >= ar && b < R) ? Gs[off + b - ar] : 0.0;
                    h[s] = (b >= ar + 1 && b < R) ? Gs[off1 + b - ar - 1] : 0.0;
                } else {
                    g[s] = b < R ? Gs[off + b - ar] : 0.0;
                    h[s] = b < R ? Gs[off1 + b - ar - 1] : 0.0;
                }
            }
#pragma unroll
            for (int t = 0; t < ND; ++t) {
                const double xa2 = x2s[t * R + ar];
                const double xb2 = x2s[t * R + ar + 1];
#pragma unroll
                for (int s = kb; s < S; ++s) {
                    acc[t][s] = fma(g[s], xa2, acc[t][s]);
                    acc1[t][s] = fma(h[s], xb2, acc1[t][s]);
                }
            }
            off = off1 + R - ar - 1;
        }
    }
#pragma unroll
    for (int t = 0; t < ND; ++t)
#pragma unroll
        for (int s = 0; s < S; ++s) acc[t][s] += acc1[t][s];
    double gbb[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int b = lane + 32 * s;
        gbb[s] = b < R ? Gs[b * R - (b * (b - 1)) / 2] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < ND; ++t) {
        double p = 0.0;
#pragma unroll
        for (int s = 0; s < S; ++s) p = fma(xr[t][s], acc[t][s] - gbb[s] * xr[t][s], p);
        mass[t] = warp_sum(p);
    }
}

template <int NB, typename T>
__global__ void __launch_bounds__(WPB * 32) k_deep2(DeepArgs a) {
    using C = DeepCfg<NB, T>;
    constexpr int R = 8 * NB;
    constexpr int S = (R + 31) / 32;
    constexpr uint64_t P = uint64_t(R) * (R + 1) / 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    griddep_launch_dependents();
    griddep_wait();
    unsigned char* wbase = smem_raw + warp * C::WARP_BYTES;
    unsigned char* buf = wbase;
    double* xs = reinterpret_cast<double*>(wbase + C::BUF);
    uint32_t* perm_sm = reinterpret_cast<uint32_t*>(wbase + C::BUF + C::XS);
    // 1-D TMA completion barriers: [0] node Gram, [1], [2] leaf-row half buffers
    uint64_t* wbar = reinterpret_cast<uint64_t*>(wbase + C::BUF + C::XS + 128);
    if (lane == 0) {
        mbar_init(&wbar[0], 1);
        mbar_init(&wbar[1], 1);
        mbar_init(&wbar[2], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t gph = 0, lph = 0, lpend = 0;
    // persistent warps take chunks of sorted positions from a counter (no ragged last
    // wave); a chunk's result does not depend on which warp processes it
    for (uint32_t it = 0;; ++it) {
    uint64_t ci;
    if (a.work) {
        uint32_t c = 0;
        if (lane == 0) c = atomicAdd(a.work, 1u);
        ci = __shfl_sync(0xffffffffu, c, 0);
    } else {
        if (it > 0) break;
        ci = uint64_t(blockIdx.x) * WPB + warp;
    }
    const uint64_t base = ci * a.chunk;
    if (base >= a.J) break;
    const int cnt = a.J - base < uint64_t(a.chunk) ? int(a.J - base) : int(a.chunk);
    const bool live = lane < cnt;
    uint32_t d = live ? a.perm[base + lane] : 0u;
    uint32_t v = live ? a.node[d] : 0xFFFFFFFFu;
    double lo = 0.0, ic = 0.0, uu = 0.0, mg = 0.0;
    if (live) {
        lo = a.low[d];
        ic = a.invc[d];
        uu = a.ud[d];
        mg = a.margin ? a.margin[d] : 0.0;
    }
    const FragAddr<NB> fa(lane);
    const unsigned below = (1u << lane) - 1u;
    const double* Gs = reinterpret_cast<const double*>(buf);
    const int r4d = lane & 3;

    for (uint32_t lev = a.level0; lev < a.topo.d; ++lev) {
        const uint32_t prevv = __shfl_up_sync(0xffffffffu, v, 1);
        const uint32_t starts = __ballot_sync(0xffffffffu, live && (lane == 0 || v != prevv));
        double mine = 0.0;
        uint32_t st = starts;
        while (st) {
            const int rs = __ffs(st) - 1;
            st &= st - 1;
            const int re = st ? __ffs(st) - 1 : cnt;
            const uint32_t vr = __shfl_sync(0xffffffffu, v, rs);
            if (is_leaf(a.topo, vr)) continue;
            {  // stage this run's Gram, warm L2 with the next one
                KRPG_DCHECK(vr < a.topo.n && slot_of(2ull * vr + 1) < a.topo.L);
                const double* g = a.tree + slot_of(2ull * vr + 1) * P;
                if (lane == 0) {  // one bulk copy (TMA) of the packed Gram
                    fence_proxy_async();
                    mbar_arrive_expect_tx(&wbar[0], uint32_t(P * 8));
                    tma_load_1d(buf, g, uint32_t(P * 8), &wbar[0]);
                }
                if (st) {
                    const uint32_t vn = __shfl_sync(0xffffffffu, v, __ffs(st) - 1);
                    if (!is_leaf(a.topo, vn)) {
                        const char* gn = reinterpret_cast<const char*>(a.tree + slot_of(2ull * vn + 1) * P);
                        for (int o = lane * 128; o < C::GB; o += 32 * 128)
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(gn + o));
                    }
                }
            }
            const int n = re - rs;
            if (n >= a.dmma_min) {
                // the first block's A fragments are requested before waiting on the Gram
                const int m = lane >> 2;
                double av0[NB][2];
                {
                    const uint32_t dd = __shfl_sync(0xffffffffu, d, (rs + m) & 31);
                    const double* xr = a.X + uint64_t(dd) * R;
                    const bool valid = m < min(8, n);
#pragma unroll
                    for (int p = 0; p < NB; ++p)
#pragma unroll
                        for (int s = 0; s < 2; ++s) av0[p][s] = valid ? xr[8 * p + 4 * s + r4d] : 0.0;
                }
                mbar_wait(&wbar[0], gph);
                gph ^= 1u;
                __syncwarp();
                for (int b0 = rs; b0 < re; b0 += 8) {
                    const int nb = min(8, re - b0);
                    const uint32_t dd = __shfl_sync(0xffffffffu, d, (b0 + m) & 31);
                    const double* xr = m < nb ? a.X + uint64_t(dd) * R : nullptr;
                    const double mass = b0 == rs ? qf::block_qf_packed_pre<NB>(Gs, fa, av0, xr, lane)
                                                 : block_qf_packed<NB>(Gs, fa, xr, lane);
                    const double mj = __shfl_sync(0xffffffffu, mass, (4 * (lane - b0)) & 31);
                    if (lane >= b0 && lane < b0 + nb) mine = mj;
                }
            } else {
                double xr[3][S];
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    const uint32_t dt = __shfl_sync(0xffffffffu, d, (rs + t) & 31);
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const uint32_t b = lane + 32u * s;
                        const double x = (t < n && b < uint32_t(R)) ? a.X[uint64_t(dt) * R + b] : 0.0;
                        xr[t][s] = x;
                        if (b < uint32_t(R)) xs[t * R + b] = x + x;
                    }
                }
                mbar_wait(&wbar[0], gph);
                gph ^= 1u;
                __syncwarp();
                double ms[3] = {0.0, 0.0, 0.0};
                if (n == 1)
                    small_qf<NB, 1>(Gs, xs, xr, lane, ms);
                else if (n == 2)
                    small_qf<NB, 2>(Gs, xs, xr, lane, ms);
                else
                    small_qf<NB, 3>(Gs, xs, xr, lane, ms);
#pragma unroll
                for (int t = 0; t < 3; ++t)
                    if (lane == rs + t && t < n) mine = ms[t];
            }
            __syncwarp();
        }
        const bool moved = live && !is_leaf(a.topo, v);
        bool left = false;
        if (moved) {
            const double cutoff = lo + ic * mine;
            left = cutoff >= uu;
            mg = fmin(mg, fabs(cutoff - uu));
            if (!left) lo = cutoff;
        }
        const uint32_t leftm = __ballot_sync(0xffffffffu, moved && left);
        const uint32_t movedm = __ballot_sync(0xffffffffu, moved);
        int newpos = lane;
        if (moved) {
            const uint32_t le = starts & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
            const int rs = 31 - __clz(le);
            const uint32_t gt = starts & ~(lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
            const int re = gt ? __ffs(gt) - 1 : cnt;
            const uint32_t runm = (re == 32 ? 0xffffffffu : ((1u << re) - 1u)) & ~((1u << rs) - 1u);
            const int nl = __popc(leftm & runm);
            newpos = left ? rs + __popc(leftm & runm & below) : rs + nl + __popc(movedm & ~leftm & runm & below);
            v = left ? 2 * v + 1 : 2 * v + 2;
        }
        perm_sm[newpos] = uint32_t(lane);
        __syncwarp();
        const int src = live ? int(perm_sm[lane]) : lane;
        __syncwarp();
        d = __shfl_sync(0xffffffffu, d, src);
        v = __shfl_sync(0xffffffffu, v, src);
        lo = __shfl_sync(0xffffffffu, lo, src);
        ic = __shfl_sync(0xffffffffu, ic, src);
        uu = __shfl_sync(0xffffffffu, uu, src);
        mg = __shfl_sync(0xffffffffu, mg, src);
    }

    // ---------------- leaf scan (segment_tree_sampler.cpp:281-292) ----------------
    const T* U = static_cast<const T*>(a.U);
    const int r4 = lane & 3, m8 = lane >> 2;
    const uint32_t prevv = __shfl_up_sync(0xffffffffu, v, 1);
    uint32_t st = __ballot_sync(0xffffffffu, live && (lane == 0 || v != prevv));
    uint64_t pick = ~uint64_t{0}, last_nz = ~uint64_t{0};
    double cum = lo;
    constexpr int PIECES = C::ROWB / 16;  // 16-byte pieces per row
    while (st) {
        const int rs = __ffs(st) - 1;
        st &= st - 1;
        const int re = st ? __ffs(st) - 1 : cnt;
        const uint32_t vr = __shfl_sync(0xffffffffu, v, rs);
        KRPG_DCHECK(vr < a.topo.n && is_leaf(a.topo, vr));
        const uint64_t l = leaf_index(a.topo, vr);
        const uint64_t first = l * a.topo.F;
        const uint64_t last = first + a.topo.F < a.topo.I ? first + a.topo.F : a.topo.I;
        KRPG_DCHECK(l < a.topo.L && first < last && last <= a.topo.I);
        const bool in_run = lane >= rs && lane < re;
        // z fragments of the run's first 8-draw block, loaded once for all its chunks
        double zfirst[2 * NB];
        {
            const int nb0 = min(8, re - rs);
            const uint32_t dd0 = __shfl_sync(0xffffffffu, d, (rs + m8) & 31);
#pragma unroll
            for (int s = 0; s < 2 * NB; ++s) zfirst[s] = m8 < nb0 ? a.X[uint64_t(dd0) * R + 4 * s + r4] : 0.0;
        }
        // rows stream through two half-buffers of PR rows: piece k+1 is in flight
        // while piece k is scanned
        constexpr int PR = C::LROWS / 2;
        auto issue = [&](uint64_t c0, int slot) {  // one 1-D TMA copy per row (padded stride)
            const int nrow = last - c0 < uint64_t(PR) ? int(last - c0) : PR;
            const char* src = reinterpret_cast<const char*>(U + c0 * R);
            unsigned char* dst = buf + slot * PR * C::RSP;
            if (lane == 0) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&wbar[1 + slot], uint32_t(nrow * C::ROWB));
            }
            __syncwarp();
            if (lane < nrow) tma_load_1d(dst + lane * C::RSP, src + uint64_t(lane) * C::ROWB, C::ROWB, &wbar[1 + slot]);
            lpend |= 1u << slot;
        };
        auto wait_piece = [&](int slot) {
            mbar_wait(&wbar[1 + slot], (lph >> slot) & 1u);
            lph ^= 1u << slot;
            lpend &= ~(1u << slot);
        };
        issue(first, 0);
        if (st) {  // warm L2 with the first rows of the next run's leaf
            const uint32_t vn = __shfl_sync(0xffffffffu, v, __ffs(st) - 1);
            const uint64_t fn = leaf_index(a.topo, vn) * a.topo.F;
            const uint64_t ln = fn + a.topo.F < a.topo.I ? fn + a.topo.F : a.topo.I;
            const uint64_t bytes = (ln - fn < uint64_t(C::LROWS) ? ln - fn : uint64_t(C::LROWS)) * C::ROWB;
            const char* pn = reinterpret_cast<const char*>(U + fn * R);
            for (uint64_t o = uint64_t(lane) * 128; o < bytes; o += 32 * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pn + o));
        }
        int slot = 0;
        for (uint64_t c0 = first; c0 < last; c0 += PR, slot ^= 1) {
            if (!__any_sync(0xffffffffu, in_run && pick == ~uint64_t{0})) break;  // every draw picked
            const int nrow = last - c0 < uint64_t(PR) ? int(last - c0) : PR;
            if (c0 + PR < last) issue(c0 + PR, slot ^ 1);
            wait_piece(slot);
            __syncwarp();
            const unsigned char* pbuf = buf + slot * PR * C::RSP;
            for (int b0 = rs; b0 < re; b0 += 8) {
                const int nb = min(8, re - b0);
                const bool mine_lane = lane >= b0 && lane < b0 + nb;
                const int jj = (lane - b0) & 7;
                const uint32_t dd = __shfl_sync(0xffffffffu, d, (b0 + m8) & 31);
                double zb[2 * NB];
#pragma unroll
                for (int s = 0; s < 2 * NB; ++s)
                    zb[s] = b0 == rs ? zfirst[s] : (m8 < nb ? a.X[uint64_t(dd) * R + 4 * s + r4] : 0.0);
                // all tiles of the piece first: 2 x NTL independent DMMA chains (even / odd k)
                constexpr int NTL = PR / 8;
                double qa[NTL][2];
#pragma unroll
                for (int tt = 0; tt < NTL; ++tt) {
                    const int row = 8 * tt + m8;
                    const bool rv = row < nrow;
                    const T* up = reinterpret_cast<const T*>(pbuf + (rv ? row : 0) * C::RSP) + r4;
                    double e0 = 0.0, e1 = 0.0, o0 = 0.0, o1 = 0.0;
#pragma unroll
                    for (int s = 0; s < 2 * NB; s += 2) {
                        dmma_884(e0, e1, rv ? static_cast<double>(up[4 * s]) : 0.0, zb[s]);
                        if (s + 1 < 2 * NB) dmma_884(o0, o1, rv ? static_cast<double>(up[4 * s + 4]) : 0.0, zb[s + 1]);
                    }
                    const double acc0 = e0 + o0, acc1 = e1 + o1;
                    qa[tt][0] = acc0 * acc0;
                    qa[tt][1] = acc1 * acc1;
                }
                if (nb <= a.leaf_par) {
                    // each draw's scan over the piece's rows is spread over a half warp
                    // (lane 16h + i = row i of draw j + h): masses gathered from the tile,
                    // inclusive prefix sum by shuffles, first crossing by ballot; two draws
                    // per step. A draw's result does not depend on the other draws of its run.
                    static_assert(NTL == 2, "leaf piece of 16 rows");
                    const int half = lane >> 4, i = lane & 15;
                    for (int j = 0; j < nb; j += 2) {
                        const int jj = j + half;
                        const bool dv = jj < nb;
                        const int own = b0 + (dv ? jj : j);
                        const bool act = __shfl_sync(0xffffffffu, pick == ~uint64_t{0} ? 1 : 0, own) != 0;
                        const double icj = __shfl_sync(0xffffffffu, ic, own);
                        const double uj = __shfl_sync(0xffffffffu, uu, own);
                        const double cj = __shfl_sync(0xffffffffu, cum, own);
                        const int src = (i & 7) * 4 + (jj >> 1);
                        const double v00 = __shfl_sync(0xffffffffu, qa[0][0], src);
                        const double v01 = __shfl_sync(0xffffffffu, qa[0][1], src);
                        const double v10 = __shfl_sync(0xffffffffu, qa[1][0], src);
                        const double v11 = __shfl_sync(0xffffffffu, qa[1][1], src);
                        const double q = i < 8 ? ((jj & 1) ? v01 : v00) : ((jj & 1) ? v11 : v10);
                        const bool rowok = dv && act && i < nrow;
                        const double mm = rowok ? icj * q : 0.0;
                        double sc = mm;
#pragma unroll
                        for (int o = 1; o < 16; o <<= 1) {
                            const double t = __shfl_up_sync(0xffffffffu, sc, o, 16);
                            if (i >= o) sc += t;
                        }
                        const double ci = cj + sc;
                        const unsigned hb = __ballot_sync(0xffffffffu, rowok && ci >= uj);
                        const unsigned hit = (hb >> (16 * half)) & 0xffffu;
                        const int first = hit ? __ffs(hit) - 1 : nrow - 1;
                        double dm = (rowok && i <= first) ? fabs(ci - uj) : HUGE_VAL;
#pragma unroll
                        for (int o = 8; o > 0; o >>= 1) dm = fmin(dm, __shfl_xor_sync(0xffffffffu, dm, o));
                        const unsigned nzb = __ballot_sync(0xffffffffu, rowok && i <= first && mm > 0.0);
                        const unsigned nz = (nzb >> (16 * half)) & 0xffffu;
                        const double cend = __shfl_sync(0xffffffffu, ci, 16 * half + first);
                        // results of half h live in its lanes; hand them to the draw's own lane
                        const int h_of_me = lane - b0 - j;  // 0 or 1 if this lane owns draw j or j + 1
                        const bool mine_here = h_of_me == 0 || (h_of_me == 1 && j + 1 < nb);
                        const int from = 16 * (h_of_me == 1 ? 1 : 0);
                        const double dm_r = __shfl_sync(0xffffffffu, dm, from);
                        const double ce_r = __shfl_sync(0xffffffffu, cend, from);
                        const unsigned hit_r = (hb >> from) & 0xffffu;
                        const unsigned nz_r = (nzb >> from) & 0xffffu;
                        if (mine_here && pick == ~uint64_t{0}) {
                            mg = fmin(mg, dm_r);
                            if (nz_r) last_nz = c0 + uint64_t(31 - __clz(nz_r));
                            cum = ce_r;
                            if (hit_r) pick = c0 + uint64_t(__ffs(hit_r) - 1);
                        }
                    }
                } else {
#pragma unroll
                    for (int tt = 0; tt < NTL; ++tt) {
                        if (8 * tt >= nrow) break;
                        const double q0 = qa[tt][0], q1 = qa[tt][1];
                        const uint64_t rb = c0 + 8 * tt;
#pragma unroll
                        for (int rr = 0; rr < 8; ++rr) {
                            const double w0 = __shfl_sync(0xffffffffu, q0, rr * 4 + (jj >> 1));
                            const double w1 = __shfl_sync(0xffffffffu, q1, rr * 4 + (jj >> 1));
                            if (mine_lane && pick == ~uint64_t{0} && rb + rr < last) {
                                const double mm = ic * ((jj & 1) ? w1 : w0);
                                if (mm > 0.0) last_nz = rb + rr;
                                cum += mm;
                                mg = fmin(mg, fabs(cum - uu));
                                if (cum >= uu) pick = rb + rr;
                            }
                        }
                    }
                }
            }
            __syncwarp();
        }
        if (lpend & 1u) wait_piece(0);  // drain a piece issued before an early exit
        if (lpend & 2u) wait_piece(1);
        __syncwarp();
        if (in_run) {
            if (pick == ~uint64_t{0}) pick = last_nz != ~uint64_t{0} ? last_nz : last - 1;
            if (a.margin) a.margin[d] = mg;
            KRPG_DCHECK(pick >= first && pick < last && d < a.J);
            if (a.idx) a.idx[uint64_t(d) * a.N + a.k] = uint32_t(pick);
            a.pick[d] = uint32_t(pick);
        }
    }
    if (a.final_rows) {
        // last position of a host-output call (krp_sampler.cpp:137-138): the chunk's final
        // rows h o= U_k[pick] are formed here and stored to HBM and, over PCIe, straight into
        // the caller's page-locked rows, so the 33.5 MB output copy overlaps the deep pass
        // instead of following it
        __syncwarp();
        const unsigned own = __ballot_sync(0xffffffffu, live);
        constexpr int CPL = (R + 31) / 32;
        for (unsigned mm = own; mm;) {
            uint32_t dd[8];
            uint64_t pk[8];
            int nd = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int src = mm ? __ffs(mm) - 1 : 0;
                dd[q] = __shfl_sync(0xffffffffu, d, src);
                pk[q] = __shfl_sync(0xffffffffu, pick, src);
                if (mm) {
                    mm &= mm - 1;
                    nd = q + 1;
                }
            }
            double hv[8][CPL], uv[8][CPL];
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
                for (int cc = 0; cc < CPL; ++cc) {
                    const int c = lane + 32 * cc;
                    const bool ok = q < nd && c < R;
                    hv[q][cc] = ok ? a.H[uint64_t(dd[q]) * R + c] : 0.0;
                    uv[q][cc] = ok ? static_cast<double>(U[pk[q] * R + c]) : 0.0;
                }
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
                for (int cc = 0; cc < CPL; ++cc) {
                    const int c = lane + 32 * cc;
                    if (q < nd && c < R) {
                        const double x = hv[q][cc] * uv[q][cc];
                        a.H[uint64_t(dd[q]) * R + c] = x;
                        if (a.host_rows) a.host_rows[uint64_t(dd[q]) * R + c] = x;
                    }
                }
        }
    }
    }  // chunk loop
}

// h_d *= U_k[pick_d] for every draw (krp_sampler.cpp:137-138): one thread per
// (draw, column pair), fully coalesced, every load independent.
template <typename T>
__global__ void k_apply_pick(double* __restrict__ H, const T* __restrict__ U, const uint32_t* __restrict__ pick,
                             uint64_t J, uint32_t R) {
    griddep_launch_dependents();
    griddep_wait();
    const uint32_t lane = threadIdx.x & 31;  // a warp per draw row
    const uint64_t w0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    if (R == 64) {  // four rows per step, every load of the four issued before any use
        uint64_t d = w0;
        for (; d + 3 * nw < J; d += 4 * nw) {
            double u[4][2], h[4][2];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t dk = d + k * nw;
                const uint64_t row = uint64_t(pick[dk]) * 64;
                u[k][0] = static_cast<double>(U[row + lane]);
                u[k][1] = static_cast<double>(U[row + 32 + lane]);
                h[k][0] = H[dk * 64 + lane];
                h[k][1] = H[dk * 64 + 32 + lane];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t dk = d + k * nw;
                H[dk * 64 + lane] = h[k][0] * u[k][0];
                H[dk * 64 + 32 + lane] = h[k][1] * u[k][1];
            }
        }
        for (; d < J; d += nw) {
            const uint64_t row = uint64_t(pick[d]) * 64;
            H[d * 64 + lane] *= static_cast<double>(U[row + lane]);
            H[d * 64 + 32 + lane] *= static_cast<double>(U[row + 32 + lane]);
        }
        return;
    }
    for (uint64_t d = w0; d < J; d += nw) {
        const uint64_t row = uint64_t(pick[d]) * R;
        for (uint32_t c = lane; c < R; c += 32) H[d * R + c] *= static_cast<double>(U[row + c]);
    }
}

// h-update grid: 8 warps per CTA, ~4 rows per warp
// ---- one-stage leaf (general Y = G_{>k}), R <= 64 --------------------------
// segment_masses' general branch (segment_tree_sampler.cpp:240-251) + the leaf scan
// (:281-292): mass_i = (r_i o h)^T Y (r_i o h) for the rows of the draw's leaf, 8 rows
// at a time as one DMMA quadratic-form block (block_qf_regs) with Y's B fragments
// (off-diagonal doubled) held in registers for the whole kernel -- Y is the same for
// every draw of the position -- and the rows (times h) staged in shared memory, the
// next block's rows loaded into registers while the current block computes. The scan
// runs the reference's sequential cum += inv_c * mass, first cum >= u wins, early exit.
// Persistent warps take sorted positions (draws grouped by leaf) from a counter.
struct LeafOsArgs {
    uint64_t J;
    uint32_t N, k;
    const uint32_t* perm;
    const uint32_t* node;
    const double* low;
    const double* invc;
    const double* ud;
    double* margin;
    const double* H;
    uint32_t* idx;
    uint32_t* pick;
    const void* U;
    const double* W;
    Topo topo;
    uint32_t* work;
};

template <int NB>
struct LeafOsCfg {
    static constexpr int R = 8 * NB;
    static constexpr int XS = RegCfg<NB>::XS;
    static constexpr int PER = 8 * R / 32;  // staged elements per lane per block
    static constexpr size_t WARP_DBL = size_t(8) * XS + R;
    static constexpr size_t SMEM = RW * WARP_DBL * 8;
};

template <int NB, typename T>
__global__ void __launch_bounds__(RW * 32, 2) k_leaf_os(LeafOsArgs a) {
    constexpr int R = 8 * NB;
    using C = LeafOsCfg<NB>;
    extern __shared__ __align__(16) double smem_los[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    griddep_launch_dependents();
    griddep_wait();
    double* xs = smem_los + warp * C::WARP_DBL;
    double* hs = xs + 8 * C::XS;
    const T* U = static_cast<const T*>(a.U);
    double gf[NB * (NB + 1)];
    load_gram_frags<NB>(gf, a.W, nullptr, lane);
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(a.work, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= a.J) break;
        const uint32_t d = a.perm[t];
        KRPG_DCHECK(d < a.J);
        const uint64_t v = a.node[d];
        KRPG_DCHECK(v < a.topo.n && is_leaf(a.topo, v));
        uint64_t f, l;
        leaf_rows(a.topo, leaf_index(a.topo, v), &f, &l);
        KRPG_DCHECK(f < l && l <= a.topo.I);
        const double ic = a.invc[d], u = a.ud[d];
        double cum = a.low[d];
        double mg = a.margin ? a.margin[d] : HUGE_VAL;
        for (int c = lane; c < R; c += 32) hs[c] = a.H[uint64_t(d) * R + c];
        double cur[C::PER];
        auto fetch = [&](uint64_t b0, double (&buf)[C::PER]) {
#pragma unroll
            for (int i = 0; i < C::PER; ++i) {
                const int e = lane + 32 * i, m = e / R, c = e % R;
                buf[i] = b0 + m < l ? static_cast<double>(U[(b0 + m) * R + c]) : 0.0;
            }
        };
        fetch(f, cur);
        __syncwarp();
        uint64_t pick = ~uint64_t{0}, last_nz = ~uint64_t{0};
        for (uint64_t b0 = f; b0 < l; b0 += 8) {
#pragma unroll
            for (int i = 0; i < C::PER; ++i) {
                const int e = lane + 32 * i, m = e / R, c = e % R;
                xs[m * C::XS + c] = cur[i] * hs[c];
            }
            if (b0 + 8 < l) fetch(b0 + 8, cur);
            __syncwarp();
            const double mass = block_qf_regs<NB, false>(gf, xs, true, lane);
            const int n = int(l - b0 < 8 ? l - b0 : 8);
            for (int j = 0; j < n; ++j) {
                const double mj = __shfl_sync(0xffffffffu, mass, 4 * j);
                const double m = ic * mj;
                if (m > 0.0) last_nz = b0 + j;
                cum += m;
                mg = fmin(mg, fabs(cum - u));
                if (cum >= u) {
                    pick = b0 + j;
                    break;
                }
            }
            __syncwarp();
            if (pick != ~uint64_t{0}) break;
        }
        if (pick == ~uint64_t{0}) pick = last_nz != ~uint64_t{0} ? last_nz : l - 1;
        KRPG_DCHECK(pick >= f && pick < l);
        if (lane == 0) {
            if (a.idx) a.idx[uint64_t(d) * a.N + a.k] = uint32_t(pick);
            a.pick[d] = uint32_t(pick);
            if (a.margin) a.margin[d] = mg;
        }
        __syncwarp();
    }
}

template <int NB, typename T>
void launch_leaf_os(const LeafOsArgs& a, cudaStream_t s) {
    using C = LeafOsCfg<NB>;
    const int occ = occupancy(k_leaf_os<NB, T>, RW * 32, C::SMEM);
    const unsigned grid = unsigned(std::min<uint64_t>(uint64_t(sm_count_current()) * occ, (a.J + RW - 1) / RW));
    launch_pdl(k_leaf_os<NB, T>, dim3(std::max(1u, grid)), dim3(RW * 32), C::SMEM, s, a);
}

// ---- one-stage leaf at R = 128: Y's fragments split over the 4 warps of a CTA ----
// (272 B-fragment doubles per lane would not fit one warp): the CTA takes one draw at a
// time, stages 8 rows (times h) in shared memory, every warp computes its column pairs'
// share of the 8 masses (split_block, k_eval_split's order) and the partials are summed
// in warp order after a barrier; warp 0 runs the sequential scan and early exit.
template <int NB>
struct LeafOsSplitCfg {
    static constexpr int R = 8 * NB;
    static constexpr int XS = R + 4;
    static constexpr size_t SMEM = (size_t(8) * XS + R + SPW * 8 + 8) * 8;
};

template <int NB, typename T>
__global__ void __launch_bounds__(SPW * 32, 2) k_leaf_os_split(LeafOsArgs a) {
    constexpr int R = 8 * NB;
    using C = LeafOsSplitCfg<NB>;
    extern __shared__ __align__(16) double smem_lss[];
    double* xs = smem_lss;             // 8 x XS staged rows o h
    double* hs = xs + 8 * C::XS;       // h of the current draw
    double* part = hs + R;             // [SPW][8] partial masses
    double* ctl = part + SPW * 8;      // [0] = picked flag (as double)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    griddep_launch_dependents();
    griddep_wait();
    const T* U = static_cast<const T*>(a.U);
    double g[NB / 8][NB + 1][2];
    split_load<NB>(g, a.W, warp, lane);
    __shared__ uint32_t s_t;
    for (;;) {
        __syncthreads();
        if (tid == 0) s_t = atomicAdd(a.work, 1u);
        __syncthreads();
        const uint32_t t = s_t;
        if (t >= a.J) break;
        const uint32_t d = a.perm[t];
        KRPG_DCHECK(d < a.J);
        const uint64_t v = a.node[d];
        KRPG_DCHECK(v < a.topo.n && is_leaf(a.topo, v));
        uint64_t f, l;
        leaf_rows(a.topo, leaf_index(a.topo, v), &f, &l);
        for (int c = tid; c < R; c += SPW * 32) hs[c] = a.H[uint64_t(d) * R + c];
        const double ic = a.invc[d], u = a.ud[d];
        double cum = a.low[d], mg = a.margin ? a.margin[d] : HUGE_VAL;
        uint64_t pick = ~uint64_t{0}, last_nz = ~uint64_t{0};
        __syncthreads();
        for (uint64_t b0 = f; b0 < l; b0 += 8) {
            for (int e = tid; e < 8 * R; e += SPW * 32) {
                const int m = e / R, c = e - m * R;
                xs[m * C::XS + c] = b0 + m < l ? static_cast<double>(U[(b0 + m) * R + c]) * hs[c] : 0.0;
            }
            __syncthreads();
            const double pm = split_block<NB>(g, xs, C::XS, true, warp, lane);
            if ((lane & 3) == 0) part[warp * 8 + (lane >> 2)] = pm;
            __syncthreads();
            if (warp == 0) {  // sequential scan (segment_tree_sampler.cpp:284-291), uniform in the warp
                const int n = int(l - b0 < 8 ? l - b0 : 8);
                for (int j = 0; j < n; ++j) {
                    const double mass = ((part[j] + part[8 + j]) + part[16 + j]) + part[24 + j];
                    const double mm = ic * mass;
                    if (mm > 0.0) last_nz = b0 + j;
                    cum += mm;
                    mg = fmin(mg, fabs(cum - u));
                    if (cum >= u) {
                        pick = b0 + j;
                        break;
                    }
                }
                if (lane == 0) ctl[0] = pick != ~uint64_t{0} ? 1.0 : 0.0;
            }
            __syncthreads();
            if (ctl[0] != 0.0) break;
        }
        if (tid == 0) {
            if (pick == ~uint64_t{0}) pick = last_nz != ~uint64_t{0} ? last_nz : l - 1;
            KRPG_DCHECK(pick >= f && pick < l);
            if (a.idx) a.idx[uint64_t(d) * a.N + a.k] = uint32_t(pick);
            a.pick[d] = uint32_t(pick);
            if (a.margin) a.margin[d] = mg;
        }
        if (tid == 0) ctl[0] = 0.0;
    }
}

template <typename T>
void dispatch_leaf_os(uint32_t R, const LeafOsArgs& a, cudaStream_t s) {
    if (R == 128) {
        using C = LeafOsSplitCfg<16>;
        const int occ = occupancy(k_leaf_os_split<16, T>, SPW * 32, C::SMEM);
        const unsigned grid = unsigned(std::min<uint64_t>(uint64_t(sm_count_current()) * occ, a.J));
        launch_pdl(k_leaf_os_split<16, T>, dim3(std::max(1u, grid)), dim3(SPW * 32), C::SMEM, s, a);
        return;
    }
    switch (R / 8) {
        case 1: return launch_leaf_os<1, T>(a, s);
        case 2: return launch_leaf_os<2, T>(a, s);
        case 3: return launch_leaf_os<3, T>(a, s);
        case 4: return launch_leaf_os<4, T>(a, s);
        case 5: return launch_leaf_os<5, T>(a, s);
        case 6: return launch_leaf_os<6, T>(a, s);
        case 7: return launch_leaf_os<7, T>(a, s);
        default: return launch_leaf_os<8, T>(a, s);
    }
}

inline unsigned apply_grid(uint64_t J) { return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((J + 31) / 32, 148ull * 16))); }

unsigned grid_for(uint64_t n, unsigned block) {
    return unsigned(std::min<uint64_t>((n + block - 1) / block, 148ull * 64));
}

// launch with programmatic stream serialization (PDL): the kernel may start
// while the previous one drains; every kernel launched this way executes
// griddep_wait() before it touches data the previous kernel produces
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

// positions per CTA (a multiple of 8, at most maxpos) such that the level's CTAs fill whole
// waves of `ctas` resident CTAs: the last wave of a fixed-size tiling is otherwise part empty
// (J = 65536 in 128-position CTAs on 296 slots: 1.73 waves)
inline uint64_t wave_range(uint64_t J, uint64_t ctas, uint64_t maxpos) {
    const uint64_t waves = (J + ctas * maxpos - 1) / (ctas * maxpos);
    const uint64_t range = (J + ctas * waves - 1) / (ctas * waves);
    return std::min<uint64_t>(std::max<uint64_t>((range + 7) / 8 * 8, 8), maxpos);
}

template <int NB, int MODE, bool ROOT0>
void launch_cta(const EvalArgs& a, unsigned, cudaStream_t s) {
    constexpr size_t smem = cta_nbuf<NB, ROOT0>() * sizeof(double) * (8 * NB) * (8 * NB + 1) / 2;
    smem_optin(k_eval_cta<NB, MODE, ROOT0>, smem);
    const uint32_t range = uint32_t(wave_range(
        a.J, uint64_t(sm_count_current()) * occupancy(k_eval_cta<NB, MODE, ROOT0>, CB, smem), CB));
    const unsigned grid = unsigned((a.J + range - 1) / range);
    // launched with programmatic stream serialization: overlaps the previous
    // kernel's tail (k_eval_cta waits on griddepcontrol before reading its inputs)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(CB);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_eval_cta<NB, MODE, ROOT0>, a, range);
}

template <int NB, int MODE>
void launch_stream_mode(const EvalArgs& a, unsigned, cudaStream_t s) {
    constexpr size_t smem = size_t(SB_STAGES) * SB_CHD * sizeof(double);
    smem_optin(k_eval_stream<NB, MODE>, smem);
    const uint32_t range =
        uint32_t(wave_range(a.J, uint64_t(sm_count_current()) * occupancy(k_eval_stream<NB, MODE>, CB, smem), CB));
    const unsigned grid = unsigned((a.J + range - 1) / range);
    k_eval_stream<NB, MODE><<<grid, CB, smem, s>>>(a, range);
}

// R > 160: streamed-Gram kernel; no root-fused level 0 (the host runs EV_ROOT first)
template <int NB>
void launch_stream(int mode, const EvalArgs& a, cudaStream_t s) {
    const unsigned grid = unsigned((a.J + uint64_t(CB) - 1) / uint64_t(CB));
    if (mode == EV_ROOT)
        launch_stream_mode<NB, EV_ROOT>(a, grid, s);
    else if (mode == EV_PROB)
        launch_stream_mode<NB, EV_PROB>(a, grid, s);
    else
        launch_stream_mode<NB, EV_LEVEL>(a, grid, s);
}

template <int NB, int MODE, bool ROOT0, bool WGT = false>
void launch_reg(const EvalArgs& a, cudaStream_t s) {
    using C = RegCfg<NB>;
    const int slots = sm_count_current() * occupancy(k_eval_reg<NB, MODE, ROOT0, WGT>, RW * 32, C::SMEM) * RW;
    // one wave: the level's positions split evenly over the resident warps
    uint64_t range = (a.J + uint64_t(slots) - 1) / uint64_t(slots);
    range = std::min<uint64_t>(std::max<uint64_t>((range + 7) / 8 * 8, 8), RRANGE);
    const unsigned grid = unsigned((a.J + range * RW - 1) / (range * RW));
    launch_pdl(k_eval_reg<NB, MODE, ROOT0, WGT>, dim3(grid), dim3(RW * 32), C::SMEM, s, a, uint32_t(range));
}

// Tuning::eval_split: 0 off, 1 R = 64 and 128, 16 (default) R = 128 only -- at R = 64 the
// register-resident single-warp kernel measured faster (2.41 vs 2.83 ms per config-2 step)
inline bool eval_split_on(const Tuning& t, int NB) { return t.eval_split == 1 || t.eval_split == NB; }

// levels [l, l + nlev) of a stage in one cooperative launch (a.perm / a.perm_out etc. are
// level l's; the kernel swaps them per level). Returns false if the device refuses the launch
// (the caller then launches level by level).
template <int NB, bool WGT>
bool launch_reg_ml(const EvalArgs& a, uint32_t nlev, uint32_t* gbar, cudaStream_t s) {
    using C = RegCfg<NB>;
    auto kern = k_eval_reg_ml<NB, WGT>;
    const int ctas = sm_count_current() * occupancy(kern, RW * 32, C::SMEM);
    const uint64_t slots = uint64_t(ctas) * RW;
    uint64_t range = (a.J + slots - 1) / slots;
    range = std::min<uint64_t>(std::max<uint64_t>((range + 7) / 8 * 8, 8), RRANGE);
    const uint64_t ntiles = (a.J + range - 1) / range;
    // several tiles per warp (J beyond one resident wave): the static tile order of the
    // persistent kernel balances worse than the hardware's CTA scheduling and the launch
    // overhead is amortised anyway (config 3, J = 2^20: 34.2 ms fused against 24.1 ms)
    if (ntiles > slots) return false;
    const unsigned grid = unsigned(std::min<uint64_t>((ntiles + RW - 1) / RW, uint64_t(ctas)));
    EvalArgs arg = a;
    uint32_t r32 = uint32_t(range);
    void* params[] = {&arg, &r32, &nlev, &gbar};
    if (cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(RW * 32), params, C::SMEM,
                                    s) == cudaSuccess)
        return true;
    cudaGetLastError();  // refused (e.g. fewer SMs available than the grid needs): not an error of the call
    return false;
}

template <int NB>
bool launch_eval_ml(const EvalArgs& a, uint32_t nlev, uint32_t* gbar, cudaStream_t s, const Tuning& t) {
    if constexpr (NB <= 8) {
        if (!t.eval_reg || !t.eval_ml || !gbar || nlev < 2) return false;
        if (NB == 8 && eval_split_on(t, NB)) return false;
        if (a.W) return launch_reg_ml<NB, true>(a, nlev, gbar, s);
        return launch_reg_ml<NB, false>(a, nlev, gbar, s);
    }
    return false;
}

bool dispatch_eval_ml(uint32_t R, const EvalArgs& a, uint32_t nlev, uint32_t* gbar, cudaStream_t s, const Tuning& t) {
    if (R % 8 != 0 || R > 64) return false;
    switch (R / 8) {
        case 1: return launch_eval_ml<1>(a, nlev, gbar, s, t);
        case 2: return launch_eval_ml<2>(a, nlev, gbar, s, t);
        case 3: return launch_eval_ml<3>(a, nlev, gbar, s, t);
        case 4: return launch_eval_ml<4>(a, nlev, gbar, s, t);
        case 5: return launch_eval_ml<5>(a, nlev, gbar, s, t);
        case 6: return launch_eval_ml<6>(a, nlev, gbar, s, t);
        case 7: return launch_eval_ml<7>(a, nlev, gbar, s, t);
        default: return launch_eval_ml<8>(a, nlev, gbar, s, t);
    }
}

template <int NB, int MODE, bool ROOT0, bool WGT = false>
void launch_split(const EvalArgs& a, cudaStream_t s) {
    // whole waves: the positions per CTA are sized so that the level fills the last wave too
    // (J = 65536 at R = 128: 1171 CTAs of 56 positions = 3.96 waves of 296 instead of 1024
    // CTAs of 64 = 3.46 waves, the last one half empty)
    const uint64_t ctas = uint64_t(sm_count_current()) *
                          occupancy(k_eval_split<NB, MODE, ROOT0, WGT>, SPW * 32, SplitCfg<NB>::SMEM);
    const uint64_t range = wave_range(a.J, ctas, SPR);
    const unsigned grid = unsigned((a.J + range - 1) / range);
    launch_pdl(k_eval_split<NB, MODE, ROOT0, WGT>, dim3(grid), dim3(SPW * 32), SplitCfg<NB>::SMEM, s, a,
               uint32_t(range));
}

template <int NB>
void launch_eval(int mode, const EvalArgs& a, cudaStream_t s, const Tuning& t) {
    const unsigned grid = unsigned((a.J + uint64_t(CB) - 1) / uint64_t(CB));
    if constexpr (NB <= 8) {
        if (a.W) {  // one-stage mode: every level on the register-resident kernel
            if (mode == EV_LEVEL0) return launch_reg<NB, EV_LEVEL, true, true>(a, s);
            if (mode == EV_LEVEL) return launch_reg<NB, EV_LEVEL, false, true>(a, s);
        }
    }
    if constexpr (NB == 16) {
        if (a.W) {  // one-stage mode at R = 128: the split-Gram kernel with B = G_v o Y
            if (mode == EV_LEVEL0) return launch_split<NB, EV_LEVEL, true, true>(a, s);
            if (mode == EV_LEVEL) return launch_split<NB, EV_LEVEL, false, true>(a, s);
        }
    }
    if constexpr (NB == 8 || NB == 16) {
        if (eval_split_on(t, NB)) {
            if (mode == EV_PROB) return launch_split<NB, EV_PROB, false>(a, s);
            if (mode == EV_LEVEL0) return launch_split<NB, EV_LEVEL, true>(a, s);
            if (mode == EV_LEVEL) return launch_split<NB, EV_LEVEL, false>(a, s);
        }
    }
    if constexpr (NB <= 8) {
        if (t.eval_reg) {
            if (mode == EV_PROB) return launch_reg<NB, EV_PROB, false>(a, s);
            if (mode == EV_LEVEL0) return launch_reg<NB, EV_LEVEL, true>(a, s);
            if (mode == EV_LEVEL) return launch_reg<NB, EV_LEVEL, false>(a, s);
        }
    }
    if (mode == EV_ROOT)
        launch_cta<NB, EV_ROOT, false>(a, grid, s);
    else if (mode == EV_PROB)
        launch_cta<NB, EV_PROB, false>(a, grid, s);
    else if (mode == EV_LEVEL0)
        launch_cta<NB, EV_LEVEL, true>(a, grid, s);
    else
        launch_cta<NB, EV_LEVEL, false>(a, grid, s);
}

void dispatch_eval(uint32_t R, int mode, const EvalArgs& a, cudaStream_t s, const Tuning& t) {
    switch (R / 8) {
        case 1: return launch_eval<1>(mode, a, s, t);
        case 2: return launch_eval<2>(mode, a, s, t);
        case 3: return launch_eval<3>(mode, a, s, t);
        case 4: return launch_eval<4>(mode, a, s, t);
        case 5: return launch_eval<5>(mode, a, s, t);
        case 6: return launch_eval<6>(mode, a, s, t);
        case 7: return launch_eval<7>(mode, a, s, t);
        case 8: return launch_eval<8>(mode, a, s, t);
        case 9: return launch_eval<9>(mode, a, s, t);
        case 10: return launch_eval<10>(mode, a, s, t);
        case 11: return launch_eval<11>(mode, a, s, t);
        case 12: return launch_eval<12>(mode, a, s, t);
        case 13: return launch_eval<13>(mode, a, s, t);
        case 14: return launch_eval<14>(mode, a, s, t);
        case 15: return launch_eval<15>(mode, a, s, t);
        case 16: return launch_eval<16>(mode, a, s, t);
        case 17: return launch_eval<17>(mode, a, s, t);
        case 18: return launch_eval<18>(mode, a, s, t);
        case 19: return launch_eval<19>(mode, a, s, t);
        case 20: return launch_eval<20>(mode, a, s, t);
        case 24: return launch_stream<24>(mode, a, s);
        case 28: return launch_stream<28>(mode, a, s);
        default: return launch_stream<32>(mode, a, s);
    }
}

// draws per warp work unit of the fused deep kernel (Tuning::deep_chunk; 0 = by J): larger
// units share a node's Gram among more draws and fill the 8-draw DMMA blocks better, but the
// kernel holds ~12 warps per SM, so the units must stay numerous enough to balance: about four
// per resident warp (J = 65536: 8 draws, measured best against 4 / 6 / 12 / 16; J = 2^20 at
// R = 32: 32 draws, 21.2 ms per config-3 call against 23.9 ms with 8)
inline uint32_t deep_chunk(const Tuning& t, uint64_t J) {
    if (t.deep_chunk >= 1 && t.deep_chunk <= 32) return uint32_t(t.deep_chunk);
    const uint64_t per = J / (4ull * 12ull * uint64_t(sm_count_current()));
    return uint32_t(std::min<uint64_t>(std::max<uint64_t>(per / 8 * 8, 8), 32));
}

// shallow levels (many draws per node) -> level kernels with global regrouping; deep -> fused pass
// (Tuning::deep_threshold; 0 = by rank: 32 draws per node at R > 32 -- measured against 16 / 64 on
// config 2 --, 16 at R <= 32, where a level-kernel level costs less relative to the deep pass:
// config-4 R = 32 1.256 -> 1.205 ms, R = 16 0.954 -> 0.938 ms per call)
inline bool deep_level(const Tuning& t, uint32_t R, uint64_t J, uint32_t level) {
    return (J >> level) < uint64_t(t.deep_threshold >= 1 ? t.deep_threshold : (R <= 32 ? 16 : 32));
}

template <int NB, typename T>
void launch_deep2(const DeepArgs& a, unsigned grid, cudaStream_t s) {
    using C = DeepCfg<NB, T>;
    const int resident = sm_count_current() * occupancy(k_deep2<NB, T>, WPB * 32, C::SMEM);
    if (a.work) grid = std::min<unsigned>(grid, unsigned(resident));  // persistent: one wave
    launch_pdl(k_deep2<NB, T>, dim3(grid), dim3(WPB * 32), C::SMEM, s, a);
}

template <typename T>
void dispatch_deep(uint32_t R, const DeepArgs& a, unsigned grid, cudaStream_t s) {
    switch (R / 8) {
        case 1: return launch_deep2<1, T>(a, grid, s);
        case 2: return launch_deep2<2, T>(a, grid, s);
        case 3: return launch_deep2<3, T>(a, grid, s);
        case 4: return launch_deep2<4, T>(a, grid, s);
        case 5: return launch_deep2<5, T>(a, grid, s);
        case 6: return launch_deep2<6, T>(a, grid, s);
        case 7: return launch_deep2<7, T>(a, grid, s);
        default: return launch_deep2<8, T>(a, grid, s);
    }
}

template <int NB, typename T>
void launch_leaf2(const LeafArgs& a, cudaStream_t s) {
    using C = LeafCfg2<NB, T>;
    smem_optin(k_leaf2<NB, T>, C::SMEM);
    const unsigned grid = unsigned((a.J + uint64_t(CHUNK) * WPB - 1) / (uint64_t(CHUNK) * WPB));
    k_leaf2<NB, T><<<grid, WPB * 32, C::SMEM, s>>>(a);
}

template <typename T>
void dispatch_leaf(uint32_t R, const LeafArgs& a, cudaStream_t s) {
    switch (R / 8) {
        case 1: return launch_leaf2<1, T>(a, s);
        case 2: return launch_leaf2<2, T>(a, s);
        case 3: return launch_leaf2<3, T>(a, s);
        case 4: return launch_leaf2<4, T>(a, s);
        case 5: return launch_leaf2<5, T>(a, s);
        case 6: return launch_leaf2<6, T>(a, s);
        case 7: return launch_leaf2<7, T>(a, s);
        case 8: return launch_leaf2<8, T>(a, s);
        case 9: return launch_leaf2<9, T>(a, s);
        case 10: return launch_leaf2<10, T>(a, s);
        case 11: return launch_leaf2<11, T>(a, s);
        case 12: return launch_leaf2<12, T>(a, s);
        case 13: return launch_leaf2<13, T>(a, s);
        case 14: return launch_leaf2<14, T>(a, s);
        case 15: return launch_leaf2<15, T>(a, s);
        case 16: return launch_leaf2<16, T>(a, s);
        case 17: return launch_leaf2<17, T>(a, s);
        case 18: return launch_leaf2<18, T>(a, s);
        case 19: return launch_leaf2<19, T>(a, s);
        case 20: return launch_leaf2<20, T>(a, s);
        case 24: return launch_leaf2<24, T>(a, s);
        case 28: return launch_leaf2<28, T>(a, s);
        default: return launch_leaf2<32, T>(a, s);
    }
}

}  // namespace v2

namespace v2 {
template <int NB>
void launch_pos0_tables(const double* Q, Topo te, const double* Z, uint32_t L0, const double* V, double* etab,
                        double* ztab, int* err, cudaStream_t s, int split_order) {
    launch_pdl(k_pos0_tables<NB>, dim3(64), dim3(256), 0, s, Q, te, Z, L0, V, etab, ztab, err,
               int(NB == 8 && split_order));
}

inline void dispatch_pos0_tables(uint32_t R, const double* Q, Topo te, const double* Z, uint32_t L0, const double* V,
                                 double* etab, double* ztab, int* err, cudaStream_t s, const Tuning& t) {
    const int so = eval_split_on(t, 8) ? 1 : 0;
    switch (R / 8) {
        case 1: return launch_pos0_tables<1>(Q, te, Z, L0, V, etab, ztab, err, s, so);
        case 2: return launch_pos0_tables<2>(Q, te, Z, L0, V, etab, ztab, err, s, so);
        case 3: return launch_pos0_tables<3>(Q, te, Z, L0, V, etab, ztab, err, s, so);
        case 4: return launch_pos0_tables<4>(Q, te, Z, L0, V, etab, ztab, err, s, so);
        case 5: return launch_pos0_tables<5>(Q, te, Z, L0, V, etab, ztab, err, s, so);
        case 6: return launch_pos0_tables<6>(Q, te, Z, L0, V, etab, ztab, err, s, so);
        case 7: return launch_pos0_tables<7>(Q, te, Z, L0, V, etab, ztab, err, s, so);
        default: return launch_pos0_tables<8>(Q, te, Z, L0, V, etab, ztab, err, s, so);
    }
}
}  // namespace v2

// R <= 64: CTA levels + fused deep/leaf kernel; 64 < R <= 160: CTA kernel on every
// level (both Gram buffers of a run fit in shared memory) + streaming leaf scan.
// 160 < R <= 256 (R % 32 == 0): streamed-Gram level kernel + streaming leaf scan.
bool grouped_supported(uint32_t R, uint32_t mode) {
    if (mode == 1) return (R % 8 == 0 && R >= 8 && R <= 64) || R == 128;  // one-stage grouped kernels
    return mode == 0 && R % 8 == 0 && R >= 8 && (R <= 160 || (R <= 256 && R % 32 == 0));
}

// One factor position of the one-stage draw (north_star (2)/(3): M = G+ o hh^T o G_{>k}
// per draw, SURVEY 8(c) chain: counter p+1, general-Y tree walk + leaf). Every internal
// level runs the node-grouped register-resident DMMA kernel with B = G_v o Y, then the
// one-stage leaf kernel, then h o= U_k[pick]. Requires a tree of depth >= 1.
static int launch_position_one_stage(const GroupedArgs& g) {
    using namespace v2;
    const uint32_t R = g.R;
    const uint64_t J = g.J;
    const unsigned gs = grid_for(J, 256);
    const Topo tz = make_topo(g.I, R);
    uint32_t* work = reinterpret_cast<uint32_t*>(g.pos0_tab);  // leaf-kernel counter (tables unused here)
    launch_pdl(k_stage_init, dim3(gs), dim3(256), 0, g.stream, g.perm_a, g.node, g.low, g.ud, g.gstart, J, g.seed,
               g.draw_offset, uint64_t(g.pos) + 1, g.margin, int(g.pos == 0), g.cntL, g.cntR, uint64_t(tz.n), work,
               g.gbar);
    int launches = 1;
    EvalArgs e{};
    e.J = J;
    e.node = g.node;
    e.rank = g.rank;
    e.low = g.low;
    e.invc = g.invc;
    e.ud = g.ud;
    e.margin = g.margin;
    e.cntL = g.cntL;
    e.cntR = g.cntR;
    e.err = g.err;
    e.GS = g.gstart;
    e.GE = g.gend;
    e.X = g.H;
    e.tree = g.Z;
    e.topo = tz;
    e.W = g.W;
    uint32_t *pin = g.perm_a, *pout = g.perm_b, *nin = g.nsort_a, *nout = g.nsort_b;
    for (uint32_t l = 0; l < tz.d; ++l) {
        e.perm = l == 0 ? nullptr : pin;
        e.perm_out = pout;
        e.nsort_in = l == 0 ? nullptr : nin;
        e.nsort_out = nout;
        // levels l .. d - 1 in one cooperative launch with grid barriers (R <= 64)
        if (l >= 1 && tz.d - l >= 2 && dispatch_eval_ml(R, e, tz.d - l, g.gbar, g.stream, g.tune)) {
            ++launches;
            if ((tz.d - l) & 1u) {
                std::swap(pin, pout);
                std::swap(nin, nout);
            }
            break;
        }
        dispatch_eval(R, l == 0 ? EV_LEVEL0 : EV_LEVEL, e, g.stream, g.tune);
        ++launches;
        std::swap(pin, pout);
        std::swap(nin, nout);
    }
    LeafOsArgs la{};
    la.J = J;
    la.N = g.N;
    la.k = g.k;
    la.perm = pin;
    la.node = g.node;
    la.low = g.low;
    la.invc = g.invc;
    la.ud = g.ud;
    la.margin = g.margin;
    la.H = g.H;
    la.idx = g.idx;
    la.pick = g.rank;  // rank[] is free after the last level
    la.U = g.U;
    la.W = g.W;
    la.topo = tz;
    la.work = work;
    if (g.storage == 1) {
        dispatch_leaf_os<float>(R, la, g.stream);
        launch_pdl(k_apply_pick<float>, dim3(apply_grid(J)), dim3(256), 0, g.stream, g.H,
                   static_cast<const float*>(g.U), (const uint32_t*)g.rank, J, R);
    } else {
        dispatch_leaf_os<double>(R, la, g.stream);
        launch_pdl(k_apply_pick<double>, dim3(apply_grid(J)), dim3(256), 0, g.stream, g.H,
                   static_cast<const double*>(g.U), (const uint32_t*)g.rank, J, R);
    }
    return launches + 2;
}

// One factor position of the two-stage draw, grouped version. Returns #launches.
int launch_position_grouped(const GroupedArgs& g) {
    using namespace v2;
    if (g.one_stage) return launch_position_one_stage(g);
    const uint32_t R = g.R;
    const uint64_t J = g.J;
    int launches = 0;
    const unsigned gs = grid_for(J, 256);
    auto mark = [&](int cat) {
        if (g.mark) g.mark(g.mark_ctx, cat);
    };
    mark(-1);
    EvalArgs e{};
    e.J = J;
    e.node = g.node;
    e.rank = g.rank;
    e.low = g.low;
    e.invc = g.invc;
    e.ud = g.ud;
    e.margin = g.margin;
    e.cntL = g.cntL;
    e.cntR = g.cntR;
    e.err = g.err;

    // ---------------- stage 1: eigenvector tree (F = 1, Y = G_k) ----------------
    const Topo te = make_topo(R, 1);
    launch_pdl(k_stage_init, dim3(gs), dim3(256), 0, g.stream, g.perm_a, g.node, g.low, g.ud, g.gstart, J, g.seed,
               g.draw_offset, 2ull * g.pos + 1, g.margin, int(g.pos == 0), g.cntL, g.cntR, uint64_t(te.n),
               (uint32_t*)nullptr, g.gbar);
    ++launches;
    mark(13);
    e.GS = g.gstart;
    e.GE = g.gend;
    uint32_t* pin = g.perm_a;
    uint32_t* pout = g.perm_b;
    // CTA-cooperative levels [lstart, lcta) with direct next-level scatter; level 0
    // also computes the normaliser (a separate pass only when lcta == 0); a
    // nonzero lstart continues from draws already placed in node order in
    // perm_a / nsort_a (first-position tables)
    auto cta_levels = [&](uint32_t lcta, uint32_t lstart = 0) {
        pin = g.perm_a;
        pout = g.perm_b;
        if (lcta == 0) {
            e.perm = nullptr;
            dispatch_eval(R, EV_ROOT, e, g.stream, g.tune);
            ++launches;
            mark(8);
            return;
        }
        if (R > 160) {  // streamed kernel: separate normaliser pass
            e.perm = nullptr;
            dispatch_eval(R, EV_ROOT, e, g.stream, g.tune);
            ++launches;
            mark(8);
        }
        uint32_t* nin = g.nsort_a;
        uint32_t* nout = g.nsort_b;
        for (uint32_t l = lstart; l < lcta; ++l) {
            e.perm = l == 0 ? nullptr : pin;
            e.perm_out = pout;
            e.nsort_in = (l == 0 || !nin) ? nullptr : nin;
            e.nsort_out = nout;
            // levels l .. lcta - 1 in one cooperative launch with grid barriers (R <= 64)
            if (l >= 1 && lcta - l >= 2 && dispatch_eval_ml(R, e, lcta - l, g.gbar, g.stream, g.tune)) {
                ++launches;
                mark(9);
                if ((lcta - l) & 1u) {
                    std::swap(pin, pout);
                    std::swap(nin, nout);
                }
                break;
            }
            dispatch_eval(R, (l == 0 && R <= 160) ? EV_LEVEL0 : EV_LEVEL, e, g.stream, g.tune);
            ++launches;
            mark(9);
            std::swap(pin, pout);
            std::swap(nin, nout);
        }
        e.nsort_in = nullptr;
        e.nsort_out = nullptr;
    };
    const Topo tz = make_topo(g.I, R);
    // shallow levels: global regrouping; deep levels + leaf scan: one fused pass (R <= 64).
    // Without the fused pass (R > 64, or fused_deep off) every level runs on the level kernels.
    uint32_t l0 = 0;
    while (l0 < tz.d && (R > 64 || !g.fused_deep || !deep_level(g.tune, R, J, l0))) ++l0;
    // first position: E-tree and the top factor-tree levels from (node, component) tables
    const uint32_t L0 = tz.d >= 2 ? std::min<uint32_t>(kPos0Levels, std::min<uint32_t>(l0, tz.d - 1)) : 0;
    const bool tab0 = g.h_ones && g.pos0_tab && R <= 64 && R % 8 == 0 && L0 >= 1 && g.tune.pos0_tables;
    double* etab = g.pos0_tab;
    double* ztab = etab ? etab + 2 * R + 8 : nullptr;
    uint32_t* hist = etab ? reinterpret_cast<uint32_t*>(ztab + (uint64_t(1) << kPos0Levels) * R) : nullptr;
    // chunk counter of the persistent deep pass (zeroed by the factor-tree stage init)
    uint32_t* deep_work = (hist && g.fused_deep && R <= 64) ? hist + 300 : nullptr;
    e.X = g.H;
    e.tree = g.Q;
    e.topo = te;
    if (tab0) {
        dispatch_pos0_tables(R, g.Q, te, g.Z, L0, g.V, etab, ztab, g.err, g.stream, g.tune);
        launch_pdl(k_pos0_ewalk, dim3(grid_for(J, 256)), dim3(256), 0, g.stream, (const double*)etab, te, J,
                   (const double*)g.ud, g.margin, g.node, g.rank, hist, uint32_t(2u << L0), g.err);
        launches += 2;
        mark(9);
    } else {
        cta_levels(te.d);
    }
    {  // a few CTAs per SM, each transposing V once (R <= 64)
        const size_t zsm = R <= 64 ? size_t(R) * (R + 1) * sizeof(double) : 0;
        const unsigned zg = unsigned(std::min<uint64_t>((J + 7) / 8, 148ull * 4));
        launch_pdl(k_make_z, dim3(zg), dim3(256), zsm, g.stream, (const double*)g.H, g.V, (const uint32_t*)g.node, te, R,
                   J, g.Zb);
    }
    ++launches;
    mark(13);

    // ---------------- stage 2: factor tree, rank-1 M = z z^T ----------------
    launch_pdl(k_stage_init, dim3(gs), dim3(256), 0, g.stream, g.perm_a, g.node, g.low, g.ud, g.gstart, J, g.seed,
               g.draw_offset, 2ull * g.pos + 2, g.margin, 0, g.cntL, g.cntR, uint64_t(tz.n), deep_work, g.gbar);
    ++launches;
    mark(13);
    e.X = g.Zb;
    e.tree = g.Z;
    e.topo = tz;
    if (tab0) {
        launch_pdl(k_pos0_zwalk, dim3(grid_for(J, 256)), dim3(256), 0, g.stream, (const double*)ztab, L0,
                   (const uint32_t*)g.rank, R, J, (const double*)g.ud, g.margin, g.node, g.low, g.invc, hist);
        launch_pdl(k_pos0_place, dim3(grid_for(J, 256)), dim3(256), 0, g.stream, L0, J, (const uint32_t*)g.node,
                   (const uint32_t*)hist, hist + (1u << L0), g.perm_a, g.nsort_a, g.gstart, g.gend, g.cntL);
        launches += 2;
        mark(9);
        cta_levels(l0, L0);
    } else {
        cta_levels(l0);
    }
    if (g.fused_deep && R <= 64) {
        DeepArgs da{};
        da.J = J;
        da.N = g.N;
        da.k = g.k;
        da.level0 = l0;
        da.perm = pin;
        da.node = g.node;
        da.low = g.low;
        da.invc = g.invc;
        da.ud = g.ud;
        da.margin = g.margin;
        da.X = g.Zb;
        da.H = g.H;
        da.idx = g.idx;
        da.pick = g.rank;  // rank[] is free after the last regroup
        da.U = g.U;
        da.tree = g.Z;
        da.topo = tz;
        da.chunk = deep_chunk(g.tune, J);
        da.work = deep_work;
        da.dmma_min = g.tune.deep_dmma_min;
        da.leaf_par = g.tune.leaf_par;
        da.final_rows = g.final_rows;
        da.host_rows = g.host_rows;
        const unsigned grid = unsigned((J + uint64_t(da.chunk) * WPB - 1) / (uint64_t(da.chunk) * WPB));
        if (g.storage == 1)
            dispatch_deep<float>(R, da, grid, g.stream);
        else
            dispatch_deep<double>(R, da, grid, g.stream);
        mark(12);
        if (g.final_rows) return launches + 1;  // h o= U_k[pick] done in the deep pass
        if (g.storage == 1)
            launch_pdl(k_apply_pick<float>, dim3(apply_grid(J)), dim3(256), 0, g.stream, g.H,
                       static_cast<const float*>(g.U), (const uint32_t*)g.rank, J, R);
        else
            launch_pdl(k_apply_pick<double>, dim3(apply_grid(J)), dim3(256), 0, g.stream, g.H,
                       static_cast<const double*>(g.U), (const uint32_t*)g.rank, J, R);
        launches += 2;
        mark(13);
        return launches;
    }
    LeafArgs la{};
    la.J = J;
    la.N = g.N;
    la.k = g.k;
    la.perm = pin;
    la.node = g.node;
    la.low = g.low;
    la.invc = g.invc;
    la.ud = g.ud;
    la.margin = g.margin;
    la.Z = g.Zb;
    la.H = g.H;
    la.idx = g.idx;
    la.U = g.U;
    la.topo = tz;
    if (g.storage == 1)
        dispatch_leaf<float>(R, la, g.stream);
    else
        dispatch_leaf<double>(R, la, g.stream);
    ++launches;
    mark(12);
    return launches;
}

void launch_probabilities_grouped(const double* H, const double* gp_packed, uint32_t R, uint64_t J, double rank,
                                  double* prob, cudaStream_t s) {
    using namespace v2;
    EvalArgs e{};
    e.J = J;
    e.X = H;
    e.tree = gp_packed;
    e.prob = prob;
    e.rank_div = rank;
    dispatch_eval(R, EV_PROB, e, s, Tuning{});
}

}  // namespace krpg
