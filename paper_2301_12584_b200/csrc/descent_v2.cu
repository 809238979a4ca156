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

#include "krpg_device.cuh"
#include "krpg_kernels.hpp"
#include "ptx.cuh"

namespace krpg {
namespace v2 {

constexpr int CHUNK = 32;  // sorted positions per warp
constexpr int WPB = 4;     // warps per block

enum { EV_ROOT = 0, EV_LEVEL = 1, EV_PROB = 2 };

template <int NB>
struct Tiles {
    static constexpr int R = 8 * NB;
    static constexpr int NT = NB * (NB + 1) / 2;
    __host__ __device__ static constexpr int t(int p, int q) { return p * NB - (p * (p - 1)) / 2 + (q - p); }
};

// Gather the DMMA B fragments of a packed symmetric matrix (reference packed
// upper triangle, segment_tree_sampler.hpp:111-115): bf[t(p,q)][s] holds
// c_pq * G[8p + 4s + (lane&3)][8q + (lane>>2)], c = 2 off the diagonal tile.
template <int NB>
__device__ __forceinline__ void load_gfrag(const double* __restrict__ G, int lane,
                                           double (&bf)[Tiles<NB>::NT][2]) {
    constexpr int R = 8 * NB;
    const int r4 = lane & 3, cq = lane >> 2;
#pragma unroll
    for (int p = 0; p < NB; ++p) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int row = 8 * p + 4 * s + r4;
            const int rowoff = row * R - (row * (row - 1)) / 2 - row;  // pack_index(row, col) = rowoff + col
#pragma unroll
            for (int q = p; q < NB; ++q) {
                const int col = 8 * q + cq;
                int idx;
                if (q > p) {
                    idx = rowoff + col;
                } else {
                    idx = row <= col ? rowoff + col : col * R - (col * (col - 1)) / 2 - col + row;
                }
                const double g = __ldg(G + idx);
                bf[Tiles<NB>::t(p, q)][s] = q > p ? g + g : g;
            }
        }
    }
}

// mass_m = x_m^T G x_m for the 8 rows m = lane>>2 of an X block (row pointer xr,
// nullptr = masked row); all 4 lanes of a row end with the same value.
template <int NB>
__device__ __forceinline__ double block_qf(const double (&bf)[Tiles<NB>::NT][2], const double* __restrict__ xr,
                                           int lane) {
    const int r4 = lane & 3;
    double y[NB][2];
#pragma unroll
    for (int q = 0; q < NB; ++q) y[q][0] = y[q][1] = 0.0;
#pragma unroll
    for (int p = 0; p < NB; ++p) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const double a = xr ? xr[8 * p + 4 * s + r4] : 0.0;
#pragma unroll
            for (int q = p; q < NB; ++q) dmma_884(y[q][0], y[q][1], a, bf[Tiles<NB>::t(p, q)][s]);
        }
    }
    double part = 0.0;
    if (xr) {
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
};

template <int NB, int MODE>
__global__ void __launch_bounds__(WPB * 32) k_eval(EvalArgs a) {
    constexpr int R = 8 * NB;
    constexpr uint64_t P = uint64_t(R) * (R + 1) / 2;
    const int lane = threadIdx.x & 31;
    const uint64_t base = (uint64_t(blockIdx.x) * WPB + (threadIdx.x >> 5)) * CHUNK;
    if (base >= a.J) return;
    const int cnt = a.J - base < uint64_t(CHUNK) ? int(a.J - base) : CHUNK;
    const bool live = lane < cnt;
    const uint32_t dl = live ? (a.perm ? a.perm[base + lane] : uint32_t(base + lane)) : 0u;
    uint32_t vl = 0;
    if (MODE == EV_LEVEL) vl = live ? a.node[dl] : 0xFFFFFFFFu;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, vl, 1);
    uint32_t starts = __ballot_sync(0xffffffffu, live && (lane == 0 || vl != prev));

    double bf[Tiles<NB>::NT][2];
    while (starts) {
        const int rs = __ffs(starts) - 1;
        starts &= starts - 1;
        const int re = starts ? __ffs(starts) - 1 : cnt;
        const uint32_t v = __shfl_sync(0xffffffffu, vl, rs);
        const double* G = a.tree;
        if (MODE == EV_LEVEL) {
            if (is_leaf(a.topo, v)) continue;  // reached a leaf one level up (non-perfect tree)
            G = a.tree + slot_of(2ull * v + 1) * P;
        }
        load_gfrag<NB>(G, lane, bf);
        for (int b0 = rs; b0 < re; b0 += 8) {
            const int n = min(8, re - b0);
            const int m = lane >> 2;
            const bool valid = m < n;
            const uint32_t dd = __shfl_sync(0xffffffffu, dl, (b0 + m) & 31);
            const double mass = block_qf<NB>(bf, valid ? a.X + uint64_t(dd) * R : nullptr, lane);
            const bool owner = valid && (lane & 3) == 0;
            if (MODE == EV_ROOT) {
                if (owner) {
                    if (!isfinite(mass) || mass <= 0.0) atomicExch(a.err, 1);
                    a.invc[dd] = 1.0 / mass;
                }
            } else if (MODE == EV_PROB) {
                if (owner) a.prob[dd] = mass / a.rank_div;
            } else {
                bool left = false;
                double lo = 0.0, u = 0.0, cutoff = 0.0;
                if (owner) {
                    lo = a.low[dd];
                    u = a.ud[dd];
                    cutoff = lo + a.invc[dd] * mass;
                    left = cutoff >= u;
                    if (a.margin) a.margin[dd] = fmin(a.margin[dd], fabs(cutoff - u));
                }
                const unsigned lm = __ballot_sync(0xffffffffu, owner && left);
                const unsigned rm = __ballot_sync(0xffffffffu, owner && !left);
                uint32_t bl = 0, br = 0;
                if (lane == 0) {
                    if (lm) bl = atomicAdd(a.cntL + v, uint32_t(__popc(lm)));
                    if (rm) br = atomicAdd(a.cntR + v, uint32_t(__popc(rm)));
                }
                bl = __shfl_sync(0xffffffffu, bl, 0);
                br = __shfl_sync(0xffffffffu, br, 0);
                if (owner) {
                    const unsigned below = (1u << lane) - 1u;
                    if (left) {
                        a.node[dd] = 2 * v + 1;
                        a.rank[dd] = bl + __popc(lm & below);
                    } else {
                        a.node[dd] = 2 * v + 2;
                        a.rank[dd] = br + __popc(rm & below);
                        a.low[dd] = cutoff;
                    }
                }
            }
        }
    }
}

// perm_out for the next level (draws that moved to depth l+1 take their slot in
// the child run; draws parked at a leaf one level up keep their position).
__global__ void k_scatter(const uint32_t* __restrict__ perm_in, uint32_t* __restrict__ perm_out,
                          const uint32_t* __restrict__ node, const uint32_t* __restrict__ rank,
                          uint32_t* __restrict__ gstart, const uint32_t* __restrict__ cntL, uint64_t J,
                          uint32_t first_next) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < J; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t d = perm_in[i];
        const uint32_t c = node[d];
        if (c >= first_next) {
            const uint32_t par = (c - 1) >> 1;
            const bool left = c & 1;
            const uint32_t b = left ? gstart[par] : gstart[par] + cntL[par];
            const uint32_t r = rank[d];
            perm_out[b + r] = d;
            if (r == 0) gstart[c] = b;
        } else {
            perm_out[i] = d;
        }
    }
}

// stage init: identity order, everyone at the root, this stage's uniform
__global__ void k_stage_init(uint32_t* perm, uint32_t* node, double* low, double* ud, uint32_t* gstart,
                             uint64_t J, uint64_t seed, uint64_t off, uint64_t counter, double* margin,
                             int reset_margin) {
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
    const uint64_t total = J * R;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t d = e / R;
        const uint32_t c = uint32_t(e % R);
        const uint64_t u = leaf_index(te, node[d]);
        Z[e] = H[e] * V[uint64_t(c) * R + u];
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

// Leaf scan for runs of draws sharing a leaf: S = U_leaf * Z^T on DMMA, masses
// S^2, per-draw sequential scan (segment_tree_sampler.cpp:281-292), then
// h *= U[t] and the index write (krp_sampler.cpp:136-138).
template <int NB, typename T>
__global__ void __launch_bounds__(WPB * 32) k_leaf(LeafArgs a) {
    constexpr int R = 8 * NB;
    __shared__ double sm[WPB][R][9];  // masses [row][draw], padded
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t base = (uint64_t(blockIdx.x) * WPB + warp) * CHUNK;
    if (base >= a.J) return;
    const int cnt = a.J - base < uint64_t(CHUNK) ? int(a.J - base) : CHUNK;
    const bool live = lane < cnt;
    const uint32_t dl = live ? a.perm[base + lane] : 0u;
    const uint32_t vl = live ? a.node[dl] : 0xFFFFFFFFu;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, vl, 1);
    uint32_t starts = __ballot_sync(0xffffffffu, live && (lane == 0 || vl != prev));
    const T* U = static_cast<const T*>(a.U);
    const int r4 = lane & 3, m8 = lane >> 2;
    while (starts) {
        const int rs = __ffs(starts) - 1;
        starts &= starts - 1;
        const int re = starts ? __ffs(starts) - 1 : cnt;
        const uint32_t v = __shfl_sync(0xffffffffu, vl, rs);
        const uint64_t l = leaf_index(a.topo, v);
        const uint64_t first = l * a.topo.F;
        const uint64_t last = first + a.topo.F < a.topo.I ? first + a.topo.F : a.topo.I;
        const int nrows = int(last - first);
        for (int b0 = rs; b0 < re; b0 += 8) {
            const int n = min(8, re - b0);
            const bool valid = m8 < n;
            const uint32_t dd = __shfl_sync(0xffffffffu, dl, (b0 + m8) & 31);
            // B fragments: Z[draw = lane>>2][4s + (lane&3)]
            double zb[2 * NB];
#pragma unroll
            for (int s = 0; s < 2 * NB; ++s) zb[s] = valid ? a.Z[uint64_t(dd) * R + 4 * s + r4] : 0.0;
            double acc[NB][2];
#pragma unroll
            for (int mt = 0; mt < NB; ++mt) {
                acc[mt][0] = acc[mt][1] = 0.0;
                const int row = 8 * mt + m8;
                const bool rv = row < nrows;
                const T* up = U + (first + (rv ? row : 0)) * R + r4;
#pragma unroll
                for (int s = 0; s < 2 * NB; ++s) {
                    const double av = rv ? static_cast<double>(up[4 * s]) : 0.0;
                    dmma_884(acc[mt][0], acc[mt][1], av, zb[s]);
                }
            }
            __syncwarp();
#pragma unroll
            for (int mt = 0; mt < NB; ++mt) {
                sm[warp][8 * mt + m8][2 * r4] = acc[mt][0] * acc[mt][0];
                sm[warp][8 * mt + m8][2 * r4 + 1] = acc[mt][1] * acc[mt][1];
            }
            __syncwarp();
            uint64_t pick = 0;
            const uint32_t dme = __shfl_sync(0xffffffffu, dl, (b0 + (lane & 7)) & 31);
            if (lane < n) {
                const double ic = a.invc[dme];
                const double u = a.ud[dme];
                double cum = a.low[dme];
                double mg = a.margin ? a.margin[dme] : 0.0;
                uint64_t last_nz = ~uint64_t{0};
                pick = ~uint64_t{0};
                for (int i = 0; i < nrows; ++i) {
                    const double mm = ic * sm[warp][i][lane];
                    if (mm > 0.0) last_nz = first + i;
                    cum += mm;
                    mg = fmin(mg, fabs(cum - u));
                    if (cum >= u) {
                        pick = first + i;
                        break;
                    }
                }
                if (pick == ~uint64_t{0}) pick = last_nz != ~uint64_t{0} ? last_nz : last - 1;
                if (a.margin) a.margin[dme] = mg;
                if (a.idx) a.idx[uint64_t(dme) * a.N + a.k] = uint32_t(pick);
            }
            // h *= U[pick] for the block's draws
            for (int t = 0; t < n; ++t) {
                const uint32_t dt = __shfl_sync(0xffffffffu, dme, t);
                const uint64_t pt = __shfl_sync(0xffffffffu, pick, t);
                for (int c = lane; c < R; c += 32)
                    a.H[uint64_t(dt) * R + c] *= static_cast<double>(U[pt * R + c]);
            }
            __syncwarp();
        }
    }
}

unsigned grid_for(uint64_t n, unsigned block) {
    return unsigned(std::min<uint64_t>((n + block - 1) / block, 148ull * 64));
}

template <int NB>
void launch_eval(int mode, const EvalArgs& a, cudaStream_t s) {
    const unsigned grid = unsigned((a.J + uint64_t(CHUNK) * WPB - 1) / (uint64_t(CHUNK) * WPB));
    if (mode == EV_ROOT)
        k_eval<NB, EV_ROOT><<<grid, WPB * 32, 0, s>>>(a);
    else if (mode == EV_PROB)
        k_eval<NB, EV_PROB><<<grid, WPB * 32, 0, s>>>(a);
    else
        k_eval<NB, EV_LEVEL><<<grid, WPB * 32, 0, s>>>(a);
}

void dispatch_eval(uint32_t R, int mode, const EvalArgs& a, cudaStream_t s) {
    switch (R / 8) {
        case 1: return launch_eval<1>(mode, a, s);
        case 2: return launch_eval<2>(mode, a, s);
        case 3: return launch_eval<3>(mode, a, s);
        case 4: return launch_eval<4>(mode, a, s);
        case 5: return launch_eval<5>(mode, a, s);
        case 6: return launch_eval<6>(mode, a, s);
        case 7: return launch_eval<7>(mode, a, s);
        default: return launch_eval<8>(mode, a, s);
    }
}

template <typename T>
void dispatch_leaf(uint32_t R, const LeafArgs& a, cudaStream_t s) {
    const unsigned grid = unsigned((a.J + uint64_t(CHUNK) * WPB - 1) / (uint64_t(CHUNK) * WPB));
    switch (R / 8) {
        case 1: return k_leaf<1, T><<<grid, WPB * 32, 0, s>>>(a), void();
        case 2: return k_leaf<2, T><<<grid, WPB * 32, 0, s>>>(a), void();
        case 3: return k_leaf<3, T><<<grid, WPB * 32, 0, s>>>(a), void();
        case 4: return k_leaf<4, T><<<grid, WPB * 32, 0, s>>>(a), void();
        case 5: return k_leaf<5, T><<<grid, WPB * 32, 0, s>>>(a), void();
        case 6: return k_leaf<6, T><<<grid, WPB * 32, 0, s>>>(a), void();
        case 7: return k_leaf<7, T><<<grid, WPB * 32, 0, s>>>(a), void();
        default: return k_leaf<8, T><<<grid, WPB * 32, 0, s>>>(a), void();
    }
}

}  // namespace v2

bool grouped_supported(uint32_t R, uint32_t mode) { return mode == 0 && R % 8 == 0 && R >= 8 && R <= 64; }

// One factor position of the two-stage draw, grouped version. Returns #launches.
int launch_position_grouped(const GroupedArgs& g) {
    using namespace v2;
    const uint32_t R = g.R;
    const uint64_t J = g.J;
    int launches = 0;
    const unsigned gs = grid_for(J, 256);
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
    k_stage_init<<<gs, 256, 0, g.stream>>>(g.perm_a, g.node, g.low, g.ud, g.gstart, J, g.seed, g.draw_offset,
                                            2ull * g.pos + 1, g.margin, g.pos == 0);
    cudaMemsetAsync(g.cntL, 0, sizeof(uint32_t) * te.n, g.stream);
    cudaMemsetAsync(g.cntR, 0, sizeof(uint32_t) * te.n, g.stream);
    ++launches;
    e.X = g.H;
    e.tree = g.Q;
    e.topo = te;
    e.perm = nullptr;
    dispatch_eval(R, EV_ROOT, e, g.stream);
    ++launches;
    uint32_t* pin = g.perm_a;
    uint32_t* pout = g.perm_b;
    for (uint32_t l = 0; l < te.d; ++l) {
        e.perm = pin;
        dispatch_eval(R, EV_LEVEL, e, g.stream);
        k_scatter<<<gs, 256, 0, g.stream>>>(pin, pout, g.node, g.rank, g.gstart, g.cntL, J, (2u << l) - 1);
        launches += 2;
        std::swap(pin, pout);
    }
    k_make_z<<<grid_for(J * R, 256), 256, 0, g.stream>>>(g.H, g.V, g.node, te, R, J, g.Zb);
    ++launches;

    // ---------------- stage 2: factor tree, rank-1 M = z z^T ----------------
    const Topo tz = make_topo(g.I, R);
    k_stage_init<<<gs, 256, 0, g.stream>>>(g.perm_a, g.node, g.low, g.ud, g.gstart, J, g.seed, g.draw_offset,
                                            2ull * g.pos + 2, g.margin, 0);
    cudaMemsetAsync(g.cntL, 0, sizeof(uint32_t) * tz.n, g.stream);
    cudaMemsetAsync(g.cntR, 0, sizeof(uint32_t) * tz.n, g.stream);
    ++launches;
    e.X = g.Zb;
    e.tree = g.Z;
    e.topo = tz;
    e.perm = nullptr;
    dispatch_eval(R, EV_ROOT, e, g.stream);
    ++launches;
    pin = g.perm_a;
    pout = g.perm_b;
    for (uint32_t l = 0; l < tz.d; ++l) {
        e.perm = pin;
        dispatch_eval(R, EV_LEVEL, e, g.stream);
        k_scatter<<<gs, 256, 0, g.stream>>>(pin, pout, g.node, g.rank, g.gstart, g.cntL, J, (2u << l) - 1);
        launches += 2;
        std::swap(pin, pout);
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
    dispatch_eval(R, EV_PROB, e, s);
}

}  // namespace krpg
