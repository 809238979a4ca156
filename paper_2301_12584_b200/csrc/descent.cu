// Batched draws: the reference's KrpSampler::sample hot loop
// (/root/reference/proj/src/krp_sampler.cpp:113-149) and
// SegmentTreeSampler::row_sample (segment_tree_sampler.cpp:258-293) on device.
//
// Version 1 (per-draw warps): one warp owns one draw for one factor position.
// It walks the eigenvector tree E_k (two-stage mode) and the factor tree Z_k
// root -> leaf, evaluating each node mass <G_v, M> = sum_{a<=b} c_ab G_ab x_a x_b
// as a lane-parallel packed quadratic form (lane b owns x_b; rows of the
// packed triangle are contiguous in memory, so every row is one coalesced
// load), then scans the leaf's rows and multiplies the drawn row into the
// running Hadamard history h. Uniforms are the reference CounterRng evaluated
// in closed form: stream = draw id, counters 2p+1 (E) / 2p+2 (Z) for included
// position p (one-stage: p+1), so results are identical for any sharding.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "krpg_device.cuh"
#include "krpg_kernels.hpp"

namespace krpg {

namespace {

constexpr int kWarpsPerBlock = 8;

// sum_{a<=b} c_ab G_ab [W_ab] x_a x_b with c = 1 on the diagonal, 2 off it.
// xs: the warp's shared copy of x (broadcast reads); xr[s] = x[lane + 32 s].
template <int S, bool WEIGHTED>
__device__ __forceinline__ double packed_qf(const double* __restrict__ G, const double* __restrict__ W,
                                            const double* xs, const double (&xr)[S], uint32_t R,
                                            int lane) {
    double acc[S];
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = 0.0;
    // Rows are processed in batches of RB with all loads issued before any use,
    // so each lane keeps RB*S independent loads in flight (memory-level parallelism).
    constexpr int RB = 8;
    for (uint32_t a0 = 0; a0 < R; a0 += RB) {
        double g[RB][S];
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            const uint32_t a = a0 + j;
            const uint32_t off = a * R - (a * (a - 1)) / 2;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const uint32_t b = uint32_t(lane) + 32u * s;
                const bool ok = a < R && b >= a && b < R;
                double v = ok ? __ldg(G + off + (b - a)) : 0.0;
                if (WEIGHTED) v *= ok ? __ldg(W + off + (b - a)) : 0.0;
                g[j][s] = v;
            }
        }
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            const uint32_t a = a0 + j;
            const double xa = a < R ? xs[a] : 0.0;
            const double xa2 = xa + xa;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const uint32_t b = uint32_t(lane) + 32u * s;
                acc[s] = fma(g[j][s], b == a ? xa : xa2, acc[s]);
            }
        }
    }
    double t = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) t = fma(acc[s], xr[s], t);
    return warp_sum(t);
}

// Root -> leaf walk of one tree (row_sample :259-277). Returns false on a
// degenerate / non-finite normaliser (the reference throws runtime_error).
template <int S, bool WEIGHTED>
__device__ __forceinline__ bool walk(const double* __restrict__ tree, const double* __restrict__ W,
                                     const Topo& t, uint64_t P, const double* xs, const double (&xr)[S],
                                     uint32_t R, int lane, double u, double& inv_c, double& low,
                                     uint64_t& node, double& margin) {
    const double C = packed_qf<S, WEIGHTED>(tree, W, xs, xr, R, lane);
    if (!isfinite(C) || C <= 0.0) return false;
    inv_c = 1.0 / C;
    node = 0;
    low = 0.0;
    while (!is_leaf(t, node)) {
        const uint64_t left = 2 * node + 1;
        const double cutoff = low + inv_c * packed_qf<S, WEIGHTED>(tree + slot_of(left) * P, W, xs, xr, R, lane);
        margin = fmin(margin, fabs(cutoff - u));
        if (cutoff >= u) {
            node = left;
        } else {
            low = cutoff;
            node = left + 1;
        }
    }
    return true;
}

template <int S, typename T, int MODE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_draws(DrawArgs a) {
    extern __shared__ double xs_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t d = uint64_t(blockIdx.x) * kWarpsPerBlock + warp;
    if (d >= a.J) return;
    const uint32_t R = a.R;
    const uint64_t P = uint64_t(R) * (R + 1) / 2;
    double* xs = xs_all + warp * R;
    const T* U = static_cast<const T*>(a.U);
    const uint64_t key = a.keys ? a.keys[d] : rng_key(a.seed, a.draw_offset + d);

    constexpr bool STANDALONE = MODE >= 2;  // SegmentTreeSampler::row_sample on a single tree
    double hr[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const uint32_t b = lane + 32u * s;
        hr[s] = b < R ? ((a.pos == 0 && !STANDALONE) ? 1.0 : a.H[d * R + b]) : 0.0;
    }
    double margin = (a.pos == 0 || STANDALONE || !a.margin) ? HUGE_VAL : a.margin[d];
    const Topo tz = a.segs ? make_topo_segments(a.I, a.nleaves, a.segs) : make_topo(a.I, a.F ? a.F : R);

    double zr[S];
    double inv_c, low, u;
    uint64_t node;
    if (MODE == 0) {
        // ---- stage 1: eigenvector u of G_{>k} (E-tree, F = 1, Y = G_k) ----
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (lane + 32 * s < int(R)) xs[lane + 32 * s] = hr[s];
        __syncwarp();
        const Topo te = make_topo(R, 1);
        u = rng_uniform(key, 2ull * a.pos + 1);
        if (!walk<S, false>(a.Q, nullptr, te, P, xs, hr, R, lane, u, inv_c, low, node, margin)) {
            if (lane == 0) atomicExch(a.err, 1);
            return;
        }
        // F = 1: the leaf holds exactly one row and the scan always returns it.
        const uint64_t ev = leaf_index(te, node);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const uint32_t b = lane + 32u * s;
            zr[s] = b < R ? hr[s] * __ldg(a.V + uint64_t(b) * R + ev) : 0.0;
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (lane + 32 * s < int(R)) xs[lane + 32 * s] = zr[s];
        __syncwarp();
        // ---- stage 2: row of U_k under the rank-1 M = h~ h~^T (Z-tree, y = ones) ----
        u = rng_uniform(key, 2ull * a.pos + 2);
        if (!walk<S, false>(a.Z, nullptr, tz, P, xs, zr, R, lane, u, inv_c, low, node, margin)) {
            if (lane == 0) atomicExch(a.err, 1);
            return;
        }
    } else if (MODE == 2) {
        // ---- rank-1 Y = y y^T: z = h o y, M = z z^T (fold_weights :197-204) ----
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const uint32_t b = lane + 32u * s;
            zr[s] = b < R ? hr[s] * __ldg(a.yv + b) : 0.0;
            if (b < R) xs[b] = zr[s];
        }
        __syncwarp();
        u = rng_uniform(key, a.counters ? a.counters[d] : a.counter);
        if (!walk<S, false>(a.Z, nullptr, tz, P, xs, zr, R, lane, u, inv_c, low, node, margin)) {
            if (lane == 0) atomicExch(a.err, 1);
            return;
        }
    } else if (MODE == 3) {
        // ---- general Y: M = hh^T o Y ----
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (lane + 32 * s < int(R)) xs[lane + 32 * s] = hr[s];
        __syncwarp();
        u = rng_uniform(key, a.counters ? a.counters[d] : a.counter);
        if (!walk<S, true>(a.Z, a.Y, tz, P, xs, hr, R, lane, u, inv_c, low, node, margin)) {
            if (lane == 0) atomicExch(a.err, 1);
            return;
        }
    } else {
        // ---- one-stage: M = hh^T o G_{>k} on the factor tree directly ----
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (lane + 32 * s < int(R)) xs[lane + 32 * s] = hr[s];
        __syncwarp();
        u = rng_uniform(key, uint64_t(a.pos) + 1);
        if (!walk<S, true>(a.Z, a.Y, tz, P, xs, hr, R, lane, u, inv_c, low, node, margin)) {
            if (lane == 0) atomicExch(a.err, 1);
            return;
        }
    }

    // ---- leaf scan (:281-292): first row whose running mass reaches u ----
    uint64_t first, last;
    {
        leaf_rows(tz, leaf_index(tz, node), &first, &last);
    }
    double cum = low;
    uint64_t pick = ~uint64_t{0}, last_nz = ~uint64_t{0};
    if (MODE == 0 || MODE == 2) {
        // rank-1 leaf masses (U[i,:] . z)^2, 8 rows per batch: loads of the whole
        // batch are in flight together, then the sequential scan (:284-291).
        constexpr int LB = 8;
        for (uint64_t i0 = first; i0 < last && pick == ~uint64_t{0}; i0 += LB) {
            double part[LB];
#pragma unroll
            for (int j = 0; j < LB; ++j) {
                const uint64_t i = i0 + j;
                double p = 0.0;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const uint32_t b = lane + 32u * s;
                    const double u_ib = (i < last && b < R) ? static_cast<double>(U[i * R + b]) : 0.0;
                    p = fma(u_ib, zr[s], p);
                }
                part[j] = p;
            }
#pragma unroll
            for (int j = 0; j < LB; ++j) part[j] = warp_sum(part[j]);
#pragma unroll
            for (int j = 0; j < LB; ++j) {
                const uint64_t i = i0 + j;
                if (i >= last || pick != ~uint64_t{0}) continue;
                const double m = inv_c * (part[j] * part[j]);
                if (m > 0.0) last_nz = i;
                cum += m;
                margin = fmin(margin, fabs(cum - u));
                if (cum >= u) pick = i;
            }
        }
    }
    for (uint64_t i = first; (MODE == 1 || MODE == 3) && i < last; ++i) {
        double mass;
        {
            // general leaf mass: (h o r)^T G_{>k} (h o r), packed
            double xr[S];
            __syncwarp();
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const uint32_t b = lane + 32u * s;
                xr[s] = b < R ? hr[s] * static_cast<double>(U[i * R + b]) : 0.0;
                if (b < R) xs[b] = xr[s];
            }
            __syncwarp();
            mass = packed_qf<S, false>(a.Y, nullptr, xs, xr, R, lane);
        }
        const double m = inv_c * mass;
        if (m > 0.0) last_nz = i;
        cum += m;
        margin = fmin(margin, fabs(cum - u));
        if (cum >= u) {
            pick = i;
            break;
        }
    }
    if (pick == ~uint64_t{0}) pick = last_nz != ~uint64_t{0} ? last_nz : last - 1;

    if (STANDALONE) {
        if (lane == 0) {
            a.idx64[d] = pick;
            if (a.margin) a.margin[d] = margin;
        }
        return;
    }
    // ---- outputs: index, h *= U_k[pick] (:136-138) ----
    if (a.idx && lane == 0) a.idx[d * a.N + a.k] = static_cast<uint32_t>(pick);
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const uint32_t b = lane + 32u * s;
        if (b < R) a.H[d * R + b] = hr[s] * static_cast<double>(U[pick * R + b]);
    }
    if (a.margin && lane == 0) a.margin[d] = margin;
}

// q_{h,U,Y}[i] numerators for every row (SegmentTreeSampler::analytic_probabilities,
// segment_tree_sampler.cpp:310-323): one warp per row; rank-1 (U_i . (h o y))^2, or
// (h o U_i)^T Y (h o U_i) for general Y (packed); row 0 of `out` ... I-1, and
// out[I] = the normaliser C (root Gram).
template <int S>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_segtree_masses(const double* __restrict__ U, uint64_t I, uint32_t R, const double* __restrict__ h,
                     const double* __restrict__ yv, const double* __restrict__ Y, const double* __restrict__ root,
                     double* __restrict__ out) {
    extern __shared__ double xs_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* xs = xs_all + warp * R;
    const uint64_t nw = uint64_t(gridDim.x) * kWarpsPerBlock;
    for (uint64_t i = uint64_t(blockIdx.x) * kWarpsPerBlock + warp; i <= I; i += nw) {
        double xr[S];
        __syncwarp();
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const uint32_t b = lane + 32u * s;
            double x = 0.0;
            if (b < R) {
                if (i == I)
                    x = yv ? h[b] * yv[b] : h[b];  // normaliser: x = z (rank-1) or h (general)
                else
                    x = yv ? U[i * R + b] * h[b] * yv[b] : h[b] * U[i * R + b];
            }
            xr[s] = x;
            if (b < R) xs[b] = x;
        }
        __syncwarp();
        double m;
        if (i == I) {
            m = yv ? packed_qf<S, false>(root, nullptr, xs, xr, R, lane) : packed_qf<S, true>(root, Y, xs, xr, R, lane);
        } else if (yv) {
            double p = 0.0;
#pragma unroll
            for (int s = 0; s < S; ++s) p += xr[s];
            p = warp_sum(p);
            m = p * p;
        } else {
            m = packed_qf<S, false>(Y, nullptr, xs, xr, R, lane);
        }
        if (lane == 0) out[i] = m;
    }
}

void launch_segtree_masses_s(const double* U, uint64_t I, uint32_t R, const double* h, const double* yv,
                             const double* Y, const double* root, double* out, cudaStream_t s) {
    const unsigned grid = unsigned(std::min<uint64_t>((I + 1 + kWarpsPerBlock - 1) / kWarpsPerBlock, 148ull * 16));
    const size_t smem = size_t(kWarpsPerBlock) * R * sizeof(double);
    switch ((R + 31) / 32) {
        case 1: k_segtree_masses<1><<<grid, kWarpsPerBlock * 32, smem, s>>>(U, I, R, h, yv, Y, root, out); break;
        case 2: k_segtree_masses<2><<<grid, kWarpsPerBlock * 32, smem, s>>>(U, I, R, h, yv, Y, root, out); break;
        case 3: k_segtree_masses<3><<<grid, kWarpsPerBlock * 32, smem, s>>>(U, I, R, h, yv, Y, root, out); break;
        case 4: k_segtree_masses<4><<<grid, kWarpsPerBlock * 32, smem, s>>>(U, I, R, h, yv, Y, root, out); break;
        case 5: k_segtree_masses<5><<<grid, kWarpsPerBlock * 32, smem, s>>>(U, I, R, h, yv, Y, root, out); break;
        case 6: k_segtree_masses<6><<<grid, kWarpsPerBlock * 32, smem, s>>>(U, I, R, h, yv, Y, root, out); break;
        case 7: k_segtree_masses<7><<<grid, kWarpsPerBlock * 32, smem, s>>>(U, I, R, h, yv, Y, root, out); break;
        default: k_segtree_masses<8><<<grid, kWarpsPerBlock * 32, smem, s>>>(U, I, R, h, yv, Y, root, out); break;
    }
}

template <int S, typename T>
void launch_draws_t(const DrawArgs& a) {
    const unsigned grid = unsigned((a.J + kWarpsPerBlock - 1) / kWarpsPerBlock);
    const size_t smem = size_t(kWarpsPerBlock) * a.R * sizeof(double);
    if (a.mode == 0)
        k_draws<S, T, 0><<<grid, kWarpsPerBlock * 32, smem, a.stream>>>(a);
    else if (a.mode == 1)
        k_draws<S, T, 1><<<grid, kWarpsPerBlock * 32, smem, a.stream>>>(a);
    else if (a.mode == 2)
        k_draws<S, T, 2><<<grid, kWarpsPerBlock * 32, smem, a.stream>>>(a);
    else
        k_draws<S, T, 3><<<grid, kWarpsPerBlock * 32, smem, a.stream>>>(a);
}

template <typename T>
void launch_draws_s(const DrawArgs& a) {
    const uint32_t S = (a.R + 31) / 32;
    switch (S) {
        case 1: return launch_draws_t<1, T>(a);
        case 2: return launch_draws_t<2, T>(a);
        case 3: return launch_draws_t<3, T>(a);
        case 4: return launch_draws_t<4, T>(a);
        case 5: return launch_draws_t<5, T>(a);
        case 6: return launch_draws_t<6, T>(a);
        case 7: return launch_draws_t<7, T>(a);
        default: return launch_draws_t<8, T>(a);
    }
}

// ---------------------------------------------------------------------------
// E-tree: Q[slot] = (sum_{u in node} lambda_u V[:,u] V[:,u]^T) o G_k (packed)
// ---------------------------------------------------------------------------
// One thread per (stored node, packed entry): grid (ceil(P/128), R), so
// every entry's sum over the node's eigenvectors runs in parallel.
__global__ void __launch_bounds__(128) k_etree2(const double* __restrict__ V, const double* __restrict__ lam,
                                                const double* __restrict__ gk, uint32_t R, double* __restrict__ Q) {
    const uint32_t P = R * (R + 1) / 2;
    const uint32_t k = blockIdx.x * 128 + threadIdx.x;
    if (k >= P) return;
    const uint64_t s = blockIdx.y;
    const Topo te = make_topo(R, 1);
    const uint64_t v = s == 0 ? 0 : 2 * s - 1;
    uint64_t u0, u1;
    node_rows(te, v, &u0, &u1);
    uint32_t a, b;
    unpack_pair(R, k, a, b);
    const double g = __ldg(gk + k);
    const double* va = V + uint64_t(a) * R;
    const double* vb = V + uint64_t(b) * R;
    double acc = 0.0;
#pragma unroll 8
    for (uint64_t u = u0; u < u1; ++u) acc = fma(__ldg(lam + u) * __ldg(va + u), __ldg(vb + u), acc);
    Q[s * P + k] = acc * g;
}

template <int S>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_probabilities(const double* __restrict__ H, const double* __restrict__ gp, uint32_t R, uint64_t J,
                    double rank, double* __restrict__ prob) {
    extern __shared__ double xs_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t d = uint64_t(blockIdx.x) * kWarpsPerBlock + warp;
    if (d >= J) return;
    double* xs = xs_all + warp * R;
    double xr[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const uint32_t b = lane + 32u * s;
        xr[s] = b < R ? H[d * R + b] : 0.0;
        if (b < R) xs[b] = xr[s];
    }
    __syncwarp();
    const double q = packed_qf<S, false>(gp, nullptr, xs, xr, R, lane);
    if (lane == 0) prob[d] = q / rank;
}

__global__ void k_fill(double* p, double v, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}
__global__ void k_fill_u32(uint32_t* p, uint32_t v, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}
__global__ void k_set_col(uint32_t* idx, uint64_t J, uint32_t N, uint32_t col) {
    for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < J; d += uint64_t(gridDim.x) * blockDim.x)
        idx[d * N + col] = 0xFFFFFFFFu;
}

// STS-CP gather: w_d = 1/sqrt(J q_d) (sketch.cpp:36-52), SA = diag(w) rows (cp_als.cpp:287-289)
__global__ void k_gather_sa(const double* __restrict__ prob, const double* __restrict__ rows, uint64_t J,
                            uint32_t R, double* __restrict__ w, double* __restrict__ sa, int* err) {
    const uint64_t total = J * R;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t d = e / R;
        const double q = prob[d];
        if (!(q > 0.0) || !isfinite(q)) {
            atomicExch(err, 1);
            continue;
        }
        const double wd = 1.0 / sqrt(static_cast<double>(J) * q);
        if (e % R == 0 && w) w[d] = wd;
        sa[e] = wd * rows[e];
    }
}

// conditional: norms[u] = sum_t (U[t,:] . HT[u,:])^2, HT[u,c] = h_c V[c,u]
template <typename T>
__global__ void k_cond_norms(const T* __restrict__ U, uint64_t I, uint32_t R, const double* __restrict__ HT,
                             double* __restrict__ norms) {
    const uint32_t u = blockIdx.y;
    __shared__ double red[32];
    double part = 0.0;
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < I; t += uint64_t(gridDim.x) * blockDim.x) {
        double dot = 0.0;
        for (uint32_t c = 0; c < R; ++c) dot = fma(static_cast<double>(U[t * R + c]), HT[uint64_t(u) * R + c], dot);
        part = fma(dot, dot, part);
    }
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) atomicAdd(norms + u, v);
    }
}

template <typename T>
__global__ void k_cond_probs(const T* __restrict__ U, uint64_t I, uint32_t R, const double* __restrict__ HT,
                             const double* __restrict__ w, const double* __restrict__ norms,
                             double* __restrict__ probs) {
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < I; t += uint64_t(gridDim.x) * blockDim.x) {
        double p = 0.0;
        for (uint32_t u = 0; u < R; ++u) {
            if (w[u] == 0.0) continue;
            double dot = 0.0;
            for (uint32_t c = 0; c < R; ++c) dot = fma(static_cast<double>(U[t * R + c]), HT[uint64_t(u) * R + c], dot);
            p += w[u] * (dot * dot) / norms[u];
        }
        probs[t] = p;
    }
}

unsigned grid_for(uint64_t n, unsigned block) {
    return unsigned(std::min<uint64_t>((n + block - 1) / block, 148ull * 32));
}

}  // namespace

void launch_segtree_masses(const double* U, uint64_t I, uint32_t R, const double* h, const double* yv,
                           const double* Y, const double* root, double* out, cudaStream_t s) {
    launch_segtree_masses_s(U, I, R, h, yv, Y, root, out, s);
}

void launch_draws(const DrawArgs& a) {
    if (a.storage == 1)
        launch_draws_s<float>(a);
    else
        launch_draws_s<double>(a);
}

void launch_etree_build(const double* V, const double* lam, const double* gk_packed, uint32_t R, double* Q,
                        cudaStream_t s) {
    const uint32_t P = R * (R + 1) / 2;
    k_etree2<<<dim3((P + 127) / 128, R), 128, 0, s>>>(V, lam, gk_packed, R, Q);
}

void launch_probabilities(const double* H, const double* gp_packed, uint32_t R, uint64_t J, double rank,
                          double* prob, cudaStream_t s) {
    const unsigned grid = unsigned((J + kWarpsPerBlock - 1) / kWarpsPerBlock);
    const size_t smem = size_t(kWarpsPerBlock) * R * sizeof(double);
    switch ((R + 31) / 32) {
        case 1: k_probabilities<1><<<grid, kWarpsPerBlock * 32, smem, s>>>(H, gp_packed, R, J, rank, prob); break;
        case 2: k_probabilities<2><<<grid, kWarpsPerBlock * 32, smem, s>>>(H, gp_packed, R, J, rank, prob); break;
        case 3: k_probabilities<3><<<grid, kWarpsPerBlock * 32, smem, s>>>(H, gp_packed, R, J, rank, prob); break;
        case 4: k_probabilities<4><<<grid, kWarpsPerBlock * 32, smem, s>>>(H, gp_packed, R, J, rank, prob); break;
        case 5: k_probabilities<5><<<grid, kWarpsPerBlock * 32, smem, s>>>(H, gp_packed, R, J, rank, prob); break;
        case 6: k_probabilities<6><<<grid, kWarpsPerBlock * 32, smem, s>>>(H, gp_packed, R, J, rank, prob); break;
        case 7: k_probabilities<7><<<grid, kWarpsPerBlock * 32, smem, s>>>(H, gp_packed, R, J, rank, prob); break;
        default: k_probabilities<8><<<grid, kWarpsPerBlock * 32, smem, s>>>(H, gp_packed, R, J, rank, prob); break;
    }
}

void launch_fill(double* p, double v, uint64_t n, cudaStream_t s) {
    if (n) k_fill<<<grid_for(n, 256), 256, 0, s>>>(p, v, n);
}
void launch_fill_u32(uint32_t* p, uint32_t v, uint64_t n, cudaStream_t s) {
    if (n) k_fill_u32<<<grid_for(n, 256), 256, 0, s>>>(p, v, n);
}
void launch_set_excluded_column(uint32_t* idx, uint64_t J, uint32_t N, uint32_t col, cudaStream_t s) {
    if (J) k_set_col<<<grid_for(J, 256), 256, 0, s>>>(idx, J, N, col);
}

void launch_gather_sa(const double* prob, const double* rows, uint64_t J, uint32_t R, double* w, double* sa,
                      int* err, cudaStream_t s) {
    k_gather_sa<<<grid_for(J * R, 256), 256, 0, s>>>(prob, rows, J, R, w, sa, err);
}

void launch_conditional_norms(const void* U, uint32_t storage, uint64_t I, uint32_t R, const double* HT,
                              double* norms, cudaStream_t s) {
    dim3 grid(std::min<uint64_t>((I + 255) / 256, 1024), R);
    if (storage == 1)
        k_cond_norms<float><<<grid, 256, 0, s>>>(static_cast<const float*>(U), I, R, HT, norms);
    else
        k_cond_norms<double><<<grid, 256, 0, s>>>(static_cast<const double*>(U), I, R, HT, norms);
}

void launch_conditional_probs(const void* U, uint32_t storage, uint64_t I, uint32_t R, const double* HT,
                              const double* w, const double* norms, double* probs, cudaStream_t s) {
    if (storage == 1)
        k_cond_probs<float><<<grid_for(I, 256), 256, 0, s>>>(static_cast<const float*>(U), I, R, HT, w, norms, probs);
    else
        k_cond_probs<double><<<grid_for(I, 256), 256, 0, s>>>(static_cast<const double*>(U), I, R, HT, w, norms, probs);
}

}  // namespace krpg
