// Segment-tree construction on device: the reference's build_grams
// (/root/reference/proj/src/segment_tree_sampler.cpp:151-191) for the Z-trees
// (leaf capacity F = R, krp_sampler.cpp:53), B200-first:
//
//  * k_leaf_dmma: leaf Grams on the FP64 tensor cores (mma.sync m8n8k4 ->
//    DMMA.8x8x4), U rows streamed HBM -> shared memory by 1-D TMA bulk copies
//    (cp.async.bulk -> UBLKCP) through a per-warp 4-stage mbarrier ring. One
//    warp owns one "position" (a node on level d-1: a pair of leaves, or a
//    single leaf of a non-perfect tree) and accumulates its full upper-triangle
//    tile set in registers: after the left leaf's rows the accumulators are the
//    left leaf's Gram (stored: it is a left child), after the right leaf's rows
//    they are the parent's Gram. So the first reduction level costs nothing.
//  * k_subtree_reduce: the remaining levels, up to 5 per pass: a block owns a
//    subtree, each thread one packed entry of all its nodes (parent = left + right,
//    :180-186), writing only the stored nodes (root and left children, :142) into
//    the compact array; the transient position level is read once.
//  * k_leaf_generic: scalar fallback for ranks the DMMA path does not cover.
#include <algorithm>
#include <cstdio>
#include <stdexcept>

#include "krpg_device.cuh"
#include "krpg_kernels.hpp"
#include "launch_util.hpp"
#include "ptx.cuh"

namespace krpg {

namespace {

// timing-experiment switch of the leaf microbenchmark (tools/microbench/leaf_bench.cu);
// always false in the library
#ifdef KRPG_LEAF_BENCH
__device__ int g_leaf_exp = 0;
#define LEAF_EXP(x) (g_leaf_exp == (x))
#else
#define LEAF_EXP(x) false
#endif

struct PosGeom {
    uint64_t I, F, npos, hb, pos_node0, left_slot0;
    uint64_t p0, p1;  // positions processed by this launch: [p0, p1) (a partition's subtree)
    uint32_t R, P;
    // 1: the transient position level holds only the right children (odd positions, at index
    // j >> 1); a left child is read back from its compact slot by the first level pass, so it
    // is written once instead of twice
    uint32_t tr_half;
    const uint64_t* seg;  // variable leaf segments (device, L + 1 offsets) or null
};

// where a finished position Gram goes: d0 (and d1, nullable)
__device__ __forceinline__ void pos_dest(const PosGeom& g, uint64_t j, double* compact, double* tout, double*& d0,
                                         double*& d1) {
    const uint64_t v = g.pos_node0 + j;
    if (g.tr_half) {
        d0 = stored(v) ? compact + slot_of(v) * g.P : tout + (j >> 1) * g.P;
        d1 = nullptr;
        return;
    }
    d0 = tout ? tout + j * g.P : nullptr;
    d1 = stored(v) ? compact + slot_of(v) * g.P : nullptr;
    if (!d0) {
        d0 = d1;
        d1 = nullptr;
    }
}

__host__ __device__ __forceinline__ void pos_rows(const PosGeom& g, uint64_t j, uint64_t& r0,
                                                  uint64_t& rs, uint64_t& r1) {
    if (g.seg) {  // in-order leaves: bottom pairs first, then the singles one level up
        if (j < g.hb) {
            r0 = g.seg[2 * j];
            rs = g.seg[2 * j + 1];
            r1 = g.seg[2 * j + 2];
        } else {
            r0 = g.seg[j + g.hb];
            rs = ~uint64_t{0};
            r1 = g.seg[j + g.hb + 1];
        }
        return;
    }
    if (j < g.hb) {  // pair of bottom-level leaves 2j, 2j+1
        r0 = 2 * j * g.F;
        rs = r0 + g.F;
        r1 = r0 + 2 * g.F < g.I ? r0 + 2 * g.F : g.I;
    } else {  // single leaf one level up
        r0 = (j + g.hb) * g.F;
        rs = ~uint64_t{0};
        r1 = r0 + g.F < g.I ? r0 + g.F : g.I;
    }
}

PosGeom make_geom(uint64_t I, uint32_t R, uint64_t F = 0, uint64_t nleaves = 0, const uint64_t* seg = nullptr) {
    if (!F) F = R;
    const Topo t = nleaves ? make_topo_segments(I, nleaves, seg) : make_topo(I, F);
    PosGeom g;
    g.seg = nleaves ? seg : nullptr;
    g.I = I;
    g.F = F;
    g.R = R;
    g.P = R * (R + 1) / 2;
    const uint32_t D = t.d ? t.d - 1 : 0;
    g.npos = uint64_t{1} << D;
    g.hb = t.bottom / 2;
    g.pos_node0 = t.d ? (uint64_t{1} << D) - 1 : 0;
    g.left_slot0 = t.d ? (uint64_t{1} << (t.d - 1)) : 0;  // slot of node 2^d-1+2j is 2^(d-1)+j
    g.p0 = 0;
    g.p1 = g.npos;
    g.tr_half = 0;
    return g;
}

// MINB resident CTAs of WPC warps per SM (register budget 64K / (MINB * WPC * 32)),
// STAGES-deep TMA ring per warp
template <int NB, typename T, int MINB = 2, int STAGES_ = 4>
struct LeafCfg {
    static constexpr int R = 8 * NB;
    static constexpr int NT = NB * (NB + 1) / 2;  // upper-triangle 8x8 tiles
    static constexpr int CH = 8;                  // rows per TMA chunk (2 k-steps)
    static constexpr int STAGES = STAGES_;
    static constexpr int ROWB = R * int(sizeof(T));
    static constexpr int RS = ROWB + 16;  // padded row stride: conflict-free fragment reads
    static constexpr int CHB = CH * RS;
    static constexpr int WPC = 4;  // warps per CTA (independent pipelines)
    static constexpr int SMEM = WPC * STAGES * CHB + WPC * STAGES * 8;
};

// Fragment loader: lane reads NB consecutive elements of one staged row.
template <int NB, typename T>
__device__ __forceinline__ void load_frag(const unsigned char* rowp, double (&x)[NB]) {
    const T* p = reinterpret_cast<const T*>(rowp);
    if constexpr (sizeof(T) == 8 && NB % 2 == 0) {
#pragma unroll
        for (int i = 0; i < NB; i += 2) {
            const double2 v = *reinterpret_cast<const double2*>(p + i);
            x[i] = v.x;
            x[i + 1] = v.y;
        }
    } else if constexpr (sizeof(T) == 4 && NB % 4 == 0) {
#pragma unroll
        for (int i = 0; i < NB; i += 4) {
            const float4 v = *reinterpret_cast<const float4*>(p + i);
            x[i] = v.x;
            x[i + 1] = v.y;
            x[i + 2] = v.z;
            x[i + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < NB; ++i) x[i] = static_cast<double>(p[i]);
    }
}

// Scatter the warp's accumulator tiles into packed upper-triangle Gram(s).
// Lane l holds tile (p,q) elements (m, n) = (l>>2, 2(l&3)+i), i.e. G[a][b]
// with a = m*NB + p, b = n*NB + q (strided column blocks).
template <int NB>
__device__ __forceinline__ void store_tiles(const double (&acc)[NB * (NB + 1) / 2][2], int lane,
                                            double* dst0, double* dst1) {
    constexpr int R = 8 * NB;
    const int m = lane >> 2;
    int t = 0;
#pragma unroll
    for (int p = 0; p < NB; ++p) {
#pragma unroll
        for (int q = p; q < NB; ++q, ++t) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int n = 2 * (lane & 3) + i;
                if (p == q && m > n) continue;
                const uint32_t a = m * NB + p, b = n * NB + q;
                const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
                const uint32_t idx = pack_index(R, lo, hi);
                dst0[idx] = acc[t][i];
                if (dst1) dst1[idx] = acc[t][i];
            }
        }
    }
}

template <int NB, typename T, int MINB = 2, int STAGES = 4>
__global__ void __launch_bounds__(LeafCfg<NB, T, MINB, STAGES>::WPC * 32, MINB)
    k_leaf_dmma(const T* __restrict__ U, PosGeom g, double* __restrict__ compact,
                double* __restrict__ tout) {
    using C = LeafCfg<NB, T, MINB, STAGES>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* ring = smem + warp * (C::STAGES * C::CHB);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::WPC * C::STAGES * C::CHB) + warp * C::STAGES;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();

    const uint64_t nw = uint64_t(gridDim.x) * C::WPC;
    const uint64_t gw = g.p0 + uint64_t(blockIdx.x) * C::WPC + warp;
    if (gw >= g.p1) return;
    const uint64_t P = g.P;

    // producer cursor (runs STAGES-1 chunks ahead)
    uint64_t pj = gw, prow, prs, pr1;
    pos_rows(g, pj, prow, prs, pr1);
    uint64_t issued = 0;
    auto produce = [&]() {
        if (pj >= g.p1) return;
        const int st = int(issued % C::STAGES);
        const uint64_t left = pr1 - prow;
        const uint32_t nrows = left < uint64_t(C::CH) ? uint32_t(left) : uint32_t(C::CH);
        if (lane == 0) mbar_arrive_expect_tx(&bars[st], nrows * C::ROWB);
        __syncwarp();
        if (uint32_t(lane) < nrows)
            tma_load_1d(ring + st * C::CHB + lane * C::RS, U + (prow + lane) * C::R, C::ROWB, &bars[st]);
        ++issued;
        prow += C::CH;
        if (prow >= pr1) {
            pj += nw;
            if (pj < g.p1) pos_rows(g, pj, prow, prs, pr1);
        }
    };
    for (int s = 0; s < C::STAGES - 1; ++s) produce();

    uint64_t cj = gw, crow, crs, cr1;
    pos_rows(g, cj, crow, crs, cr1);
    double acc[C::NT][2];
#pragma unroll
    for (int t = 0; t < C::NT; ++t) acc[t][0] = acc[t][1] = 0.0;

    const int frow = lane & 3;
    const int fcol = (lane >> 2) * NB * int(sizeof(T));
    for (uint64_t i = 0; cj < g.p1; ++i) {
        produce();
        const int st = int(i % C::STAGES);
        mbar_wait(&bars[st], uint32_t((i / C::STAGES) & 1));
        const uint64_t left = cr1 - crow;
        const int nvalid = left < uint64_t(C::CH) ? int(left) : C::CH;
        const unsigned char* buf = ring + st * C::CHB;
#pragma unroll
        for (int ks = 0; ks < C::CH / 4; ++ks) {
            const int row = ks * 4 + frow;
            double x[NB];
            if (row < nvalid) {
                load_frag<NB, T>(buf + row * C::RS + fcol, x);
            } else {
#pragma unroll
                for (int p = 0; p < NB; ++p) x[p] = 0.0;
            }
            int t = 0;
#pragma unroll
            for (int p = 0; p < NB; ++p)
#pragma unroll
                for (int q = p; q < NB; ++q, ++t) dmma_884(acc[t][0], acc[t][1], x[p], x[q]);
        }
        fence_proxy_async();
        __syncwarp();
        crow += C::CH;
        if (crow == crs && !LEAF_EXP(1)) {  // left leaf of a pair complete: it is a left child -> stored
            store_tiles<NB>(acc, lane, compact + (g.left_slot0 + cj) * P, nullptr);
        }
        if (crow >= cr1) {
            double *d0, *d1;
            pos_dest(g, cj, compact, tout, d0, d1);
            if (d0 && !LEAF_EXP(1)) store_tiles<NB>(acc, lane, d0, d1);
#pragma unroll
            for (int t = 0; t < C::NT; ++t) acc[t][0] = acc[t][1] = 0.0;
            cj += nw;
            if (cj < g.p1) pos_rows(g, cj, crow, crs, cr1);
        }
    }
}

// ---- staged-store variant -------------------------------------------------
// k_leaf_dmma's accumulator layout (strided column blocks) scatters every Gram as
// 8-byte stores over the whole packed triangle: each one occupies a 32-byte L2 sector
// slot, and the 1.6 GB of Grams per config-2 factor cost as much L2 write bandwidth as
// 6.5 GB would (measured: 1.17 ms with the stores, 0.65 ms without). Here a finished
// Gram is first laid out packed in a shared-memory staging buffer (NSTG per CTA, taken
// with a shared-memory lock for the ~0.5 us a store lasts) and leaves as ONE bulk
// shared -> global copy per destination (TMA store: full lines, one instruction).
template <int NB, typename T, int CH_, int STAGES_, int NSTG_>
struct LeafCfgS {
    static constexpr int R = 8 * NB;
    static constexpr int NT = NB * (NB + 1) / 2;
    static constexpr int P = R * (R + 1) / 2;
    static constexpr int CH = CH_;
    static constexpr int STAGES = STAGES_;
    static constexpr int NSTG = NSTG_;
    static constexpr int ROWB = R * int(sizeof(T));
    static constexpr int RS = ROWB + 16;
    static constexpr int CHB = CH * RS;
    static constexpr int WPC = 4;
    static constexpr int STGB = (P * 8 + 127) / 128 * 128;  // staging buffer bytes
    static constexpr int OFF_BARS = WPC * STAGES * CHB;
    static constexpr int OFF_STG = (OFF_BARS + WPC * STAGES * 8 + 127) / 128 * 128;
    static constexpr int OFF_LOCK = OFF_STG + NSTG * STGB;
    static constexpr int SMEM = OFF_LOCK + 16 * ((NSTG + 3) / 4);
    static_assert((P * 8) % 16 == 0, "bulk copies move multiples of 16 bytes");
};

template <int NB, typename T, int CH, int STAGES, int NSTG>
__global__ void __launch_bounds__(128, 2)
    k_leaf_dmma_s(const T* __restrict__ U, PosGeom g, double* __restrict__ compact, double* __restrict__ tout) {
    using C = LeafCfgS<NB, T, CH, STAGES, NSTG>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* ring = smem + warp * (C::STAGES * C::CHB);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BARS) + warp * C::STAGES;
    int* lock = reinterpret_cast<int*>(smem + C::OFF_LOCK);
    if (threadIdx.x < C::NSTG) lock[threadIdx.x] = 0;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint64_t nw = uint64_t(gridDim.x) * C::WPC;
    const uint64_t gw = g.p0 + uint64_t(blockIdx.x) * C::WPC + warp;
    if (gw >= g.p1) return;
    constexpr uint64_t P = C::P;

    // producer cursor (runs STAGES-1 chunks ahead)
    uint64_t pj = gw, prow, prs, pr1;
    pos_rows(g, pj, prow, prs, pr1);
    uint32_t issued = 0;
    auto produce = [&]() {
        if (pj >= g.p1) return;
        const uint64_t left = pr1 - prow;
        const uint32_t nrows = left < uint64_t(C::CH) ? uint32_t(left) : uint32_t(C::CH);
        // one lane per row (measured faster than one elected lane issuing all rows: 0.77 vs 0.79 ms)
        const int st = int(issued % C::STAGES);
        if (lane == 0) mbar_arrive_expect_tx(&bars[st], nrows * C::ROWB);
        __syncwarp();
        if (uint32_t(lane) < nrows)
            tma_load_1d(ring + st * C::CHB + lane * C::RS, U + (prow + lane) * C::R, C::ROWB, &bars[st]);
        ++issued;
        prow += C::CH;
        if (prow >= pr1) {
            pj += nw;
            if (pj < g.p1) pos_rows(g, pj, prow, prs, pr1);
        }
    };
    for (int s = 0; s < C::STAGES - 1; ++s) produce();

    uint64_t cj = gw, crow, crs, cr1;
    pos_rows(g, cj, crow, crs, cr1);
    double acc[C::NT][2];
#pragma unroll
    for (int t = 0; t < C::NT; ++t) acc[t][0] = acc[t][1] = 0.0;

    // the finished Gram in `acc` -> d0 (and d1): staged packed in shared memory, bulk-stored
    auto emit = [&](double* d0, double* d1) {
        int b = -1;
        if (lane == 0) {
            for (;;) {
#pragma unroll
                for (int k = 0; k < C::NSTG; ++k)
                    if (b < 0 && atomicCAS(&lock[k], 0, 1) == 0) b = k;
                if (b >= 0) break;
                __nanosleep(100);
            }
        }
        b = __shfl_sync(0xffffffffu, b, 0);
        double* stg = reinterpret_cast<double*>(smem + C::OFF_STG + b * C::STGB);
        store_tiles<NB>(acc, lane, stg, nullptr);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            tma_store_1d(d0, stg, uint32_t(P * 8));
            if (d1) tma_store_1d(d1, stg, uint32_t(P * 8));
            tma_store_commit();
            tma_store_wait_read();  // the buffer has been read: hand it back
            __threadfence_block();
            atomicExch(&lock[b], 0);
        }
        __syncwarp();
    };

    const int frow = lane & 3;
    const int fcol = (lane >> 2) * NB * int(sizeof(T));
    for (uint32_t i = 0; cj < g.p1; ++i) {
        produce();
        const int st = int(i % C::STAGES);
        mbar_wait(&bars[st], (i / C::STAGES) & 1u);
        const uint64_t left = cr1 - crow;
        const int nvalid = left < uint64_t(C::CH) ? int(left) : C::CH;
        const unsigned char* buf = ring + st * C::CHB;
#pragma unroll
        for (int ks = 0; ks < C::CH / 4; ++ks) {
            const int row = ks * 4 + frow;
            double x[NB];
            if (row < nvalid) {
                load_frag<NB, T>(buf + row * C::RS + fcol, x);
            } else {
#pragma unroll
                for (int p = 0; p < NB; ++p) x[p] = 0.0;
            }
            int t = 0;
#pragma unroll
            for (int p = 0; p < NB; ++p)
#pragma unroll
                for (int q = p; q < NB; ++q, ++t) dmma_884(acc[t][0], acc[t][1], x[p], x[q]);
        }
        fence_proxy_async();
        __syncwarp();
        crow += C::CH;
        // left leaf of a pair complete: it is a left child -> stored
        if (crow == crs && !LEAF_EXP(1)) emit(compact + (g.left_slot0 + cj) * P, nullptr);
        if (crow >= cr1) {
            double *d0, *d1;
            pos_dest(g, cj, compact, tout, d0, d1);
            if (d0 && !LEAF_EXP(1)) emit(d0, d1);
#pragma unroll
            for (int t = 0; t < C::NT; ++t) acc[t][0] = acc[t][1] = 0.0;
            cj += nw;
            if (cj < g.p1) pos_rows(g, cj, crow, crs, cr1);
        }
    }
    if (lane == 0) tma_store_wait_all();
}

// ---- large ranks (R = 96 .. 256, R % 32 == 0): one CTA per position ------
// The upper-triangle 8x8 tile set no longer fits one warp's registers, so it
// is split into 4x4-tile super-blocks (32 columns x 32 columns); warp w owns
// super-blocks w and w + NW (at most 32 tiles = 64 accumulator registers).
// Rows are staged once per CTA by TMA (warp 0 issues one bulk copy per row
// through a 4-stage ring) and read by every warp. Columns use the contiguous
// fragment layout (block p = columns 8p .. 8p+7, lane m -> column 8p+m) with
// rows padded by 8 elements, so each fragment load is bank-conflict free.
template <int R_, typename T>
struct BigCfg {
    static constexpr int R = R_;
    static constexpr int NB = R / 8;
    static constexpr int NBS = NB / 4;                // super-blocks per dimension
    static constexpr int S = NBS * (NBS + 1) / 2;     // upper-triangle super-blocks
    // Register budget: one SM cannot hold R=256's 528 tiles (67k accumulator
    // registers), so from R=192 the super-blocks are split over SPLIT CTAs
    // (gridDim.y) that read the same rows (the repeat reads are L2 hits when
    // the group runs concurrently; these ranks are FP64-pipe bound anyway).
    static constexpr int SPLIT = R >= 256 ? 3 : (R >= 192 ? 2 : 1);
    // super-blocks per warp: one from R = 192 (registers) and at R = 128 (10 warps per CTA keep the
    // DMMA pipe busier than 5: 1.41 -> 1.06 ms per 2^20-row factor; at R = 96 / 160 two measured better)
    static constexpr int SBW = (R >= 192 || R == 128) ? 1 : 2;
    static constexpr int SS = (S + SPLIT - 1) / SPLIT;  // super-blocks per CTA
    static constexpr int NW = (SS + SBW - 1) / SBW;     // warps per CTA
    static constexpr int CH = 8;                      // rows per chunk (2 k-steps)
    static constexpr int STAGES = 4;
    static constexpr int ROWB = R * int(sizeof(T));
    static constexpr int RS = ROWB + 8 * int(sizeof(T));
    static constexpr int CHB = CH * RS;
    static constexpr int SMEM = STAGES * CHB + STAGES * 8;
    static_assert(R % 32 == 0, "large-rank leaf kernel needs R % 32 == 0");
};

template <int R>
__device__ __forceinline__ void store_superblock(const double (&acc)[16][2], int P0, int Q0, int lane,
                                                 double* dst0, double* dst1) {
    const int m = lane >> 2;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int p = 4 * P0 + i, q = 4 * Q0 + j;
            if (q < p) continue;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t a = 8 * p + m, b = 8 * q + 2 * (lane & 3) + e;
                if (a > b) continue;
                const uint32_t idx = pack_index(R, a, b);
                dst0[idx] = acc[4 * i + j][e];
                if (dst1) dst1[idx] = acc[4 * i + j][e];
            }
        }
}

template <int R_, typename T>
__global__ void __launch_bounds__(BigCfg<R_, T>::NW * 32, 1)
    k_leaf_cta(const T* __restrict__ U, PosGeom g, double* __restrict__ compact, double* __restrict__ tout) {
    using C = BigCfg<R_, T>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::CHB);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    int sp[C::SBW], sq[C::SBW];
    bool has[C::SBW];
#pragma unroll
    for (int k = 0; k < C::SBW; ++k) {
        const int sl = warp + k * C::NW;
        const int s = int(blockIdx.y) * C::SS + sl;
        has[k] = sl < C::SS && s < C::S;
        if (s < C::NBS) {
            sp[k] = sq[k] = s;
        } else {
            int o = s - C::NBS, p = 0, len = C::NBS - 1;
            while (len > 0 && o >= len) {
                o -= len;
                ++p;
                --len;
            }
            sp[k] = p;
            sq[k] = p + 1 + o;
        }
    }

    const uint64_t P = g.P;
    if (g.p0 + blockIdx.x >= g.p1) return;
    // producer cursor: warp 0 only (runs STAGES-1 chunks ahead of the consumers)
    uint64_t pj = g.p0 + blockIdx.x, prow = 0, prs, pr1 = 0, issued = 0;
    if (warp == 0) pos_rows(g, pj, prow, prs, pr1);
    auto produce = [&]() {
        if (warp != 0 || pj >= g.p1) return;
        const int st = int(issued % C::STAGES);
        const uint64_t left = pr1 - prow;
        const uint32_t nrows = left < uint64_t(C::CH) ? uint32_t(left) : uint32_t(C::CH);
        if (lane == 0) mbar_arrive_expect_tx(&bars[st], nrows * C::ROWB);
        __syncwarp();
        if (uint32_t(lane) < nrows)
            tma_load_1d(smem + st * C::CHB + lane * C::RS, U + (prow + lane) * C::R, C::ROWB, &bars[st]);
        ++issued;
        prow += C::CH;
        if (prow >= pr1) {
            pj += gridDim.x;
            if (pj < g.p1) pos_rows(g, pj, prow, prs, pr1);
        }
    };
    for (int s = 0; s < C::STAGES - 1; ++s) produce();

    uint64_t cj = g.p0 + blockIdx.x, crow, crs, cr1;
    pos_rows(g, cj, crow, crs, cr1);
    double acc[C::SBW][16][2];
#pragma unroll
    for (int k = 0; k < C::SBW; ++k)
#pragma unroll
        for (int t = 0; t < 16; ++t) acc[k][t][0] = acc[k][t][1] = 0.0;

    const int m = lane >> 2;
    for (uint32_t i = 0; cj < g.p1; ++i) {
        produce();
        const int st = int(i % C::STAGES);
        mbar_wait(&bars[st], (i / C::STAGES) & 1);
        const uint64_t left = cr1 - crow;
        const int nvalid = left < uint64_t(C::CH) ? int(left) : C::CH;
        const T* buf = reinterpret_cast<const T*>(smem + st * C::CHB);
#pragma unroll
        for (int ks = 0; ks < C::CH / 4; ++ks) {
            const int row = ks * 4 + (lane & 3);
            const bool valid = row < nvalid;
            const T* rp = buf + row * (C::RS / int(sizeof(T))) + m;
#pragma unroll
            for (int k = 0; k < C::SBW; ++k) {
                if (!has[k]) continue;
                double xa[4], xb[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    xa[u] = valid ? static_cast<double>(rp[8 * (4 * sp[k] + u)]) : 0.0;
                    xb[u] = valid ? static_cast<double>(rp[8 * (4 * sq[k] + u)]) : 0.0;
                }
                if (sp[k] == sq[k]) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = u; v < 4; ++v) dmma_884(acc[k][4 * u + v][0], acc[k][4 * u + v][1], xa[u], xb[v]);
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) dmma_884(acc[k][4 * u + v][0], acc[k][4 * u + v][1], xa[u], xb[v]);
                }
            }
        }
        fence_proxy_async();
        __syncthreads();
        crow += C::CH;
        if (crow == crs) {  // left leaf of a pair complete: it is a left child -> stored
            double* dst = compact + (g.left_slot0 + cj) * P;
#pragma unroll
            for (int k = 0; k < C::SBW; ++k)
                if (has[k]) store_superblock<C::R>(acc[k], sp[k], sq[k], lane, dst, nullptr);
        }
        if (crow >= cr1) {
            double *d0, *d1;
            pos_dest(g, cj, compact, tout, d0, d1);
#pragma unroll
            for (int k = 0; k < C::SBW; ++k) {
                if (has[k] && d0) store_superblock<C::R>(acc[k], sp[k], sq[k], lane, d0, d1);
#pragma unroll
                for (int t = 0; t < 16; ++t) acc[k][t][0] = acc[k][t][1] = 0.0;
            }
            cj += gridDim.x;
            if (cj < g.p1) pos_rows(g, cj, crow, crs, cr1);
        }
    }
}

template <typename T>
__global__ void k_leaf_generic(const T* __restrict__ U, PosGeom g, double* __restrict__ compact,
                               double* __restrict__ tout) {
    const uint32_t R = g.R;
    const uint64_t P = g.P;
    for (uint64_t j = g.p0 + blockIdx.x; j < g.p1; j += gridDim.x) {
        uint64_t r0, rs, r1;
        pos_rows(g, j, r0, rs, r1);
        for (uint32_t k = threadIdx.x; k < P; k += blockDim.x) {
            uint32_t a, b;
            unpack_pair(R, k, a, b);
            double acc = 0.0;
            for (uint64_t i = r0; i < r1; ++i) {
                acc += static_cast<double>(U[i * R + a]) * static_cast<double>(U[i * R + b]);
                if (i + 1 == rs) compact[(g.left_slot0 + j) * P + k] = acc;
            }
            double *d0, *d1;
            pos_dest(g, j, compact, tout, d0, d1);
            if (d0) d0[k] = acc;
            if (d1) d1[k] = acc;
        }
    }
}

__global__ void k_level_reduce(const double* __restrict__ child, double* __restrict__ parent,
                               double* __restrict__ compact, uint64_t j0, uint64_t nj, uint64_t P, uint64_t node0) {
    for (uint64_t j = j0 + blockIdx.x; j < nj; j += gridDim.x) {
        const double* c0 = child + 2 * j * P;
        const double* c1 = c0 + P;
        const uint64_t v = node0 + j;
        double* cp = stored(v) ? compact + slot_of(v) * P : nullptr;
        double* pp = parent ? parent + j * P : nullptr;
        for (uint64_t k = threadIdx.x; k < P; k += blockDim.x) {
            const double s = c0[k] + c1[k];
            if (pp) pp[k] = s;
            if (cp) cp[k] = s;
        }
    }
}

// K levels at once (:180-186, parent = left + right in the same order as k_level_reduce,
// so the tree is bit-identical): block b owns the subtree of 2^K consecutive child-level
// nodes under parent-level-(c-K) node j0 + b; thread e reads packed entry e of all 2^K
// children (2^K independent loads in flight, coalesced across the warp), sums pairs K
// times in registers, writes every stored node's entry, and the subtree root's entry to
// `top` (next pass's child level; null at the root). One pass replaces K launches and
// reads the transient level once.
// HALF (first pass after a tr_half leaf pass): the child level holds the right children only
// (index >> 1); the left children are read from their compact slots.
template <int K, bool HALF>
__global__ void __launch_bounds__(256) k_subtree_reduce(const double* __restrict__ child, double* __restrict__ top,
                                                        double* compact, uint32_t c, uint64_t j0,
                                                        uint64_t nj, uint64_t P) {
    constexpr int W = 1 << K;
    // last subtrees first: the child level was just written in ascending order, so its tail
    // is what the L2 still holds
    const uint64_t j = nj - 1 - blockIdx.x;  // parent-level (c - K) index in [j0, nj)
    if (j < j0 || j >= nj) return;
    for (uint64_t e = threadIdx.x; e < P; e += blockDim.x) {
        double v[W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint64_t ci = j * W + i;
            if (HALF)
                v[i] = (i & 1) ? child[(ci >> 1) * P + e] : compact[slot_of(((uint64_t{1} << c) - 1) + ci) * P + e];
            else
                v[i] = child[ci * P + e];
        }
#pragma unroll
        for (int l = 1; l <= K; ++l) {
            const uint32_t lev = c - l;  // level of the nodes formed now
#pragma unroll
            for (int i = 0; i < (W >> l); ++i) {
                v[i] = v[2 * i] + v[2 * i + 1];
                const uint64_t node = ((uint64_t{1} << lev) - 1) + (j << (K - l)) + i;
                if (stored(node)) compact[slot_of(node) * P + e] = v[i];
            }
        }
        if (top) top[j * P + e] = v[0];
    }
}

template <int K>
void launch_subtree(const double* child, double* top, double* compact, uint32_t c, uint64_t j0, uint64_t nj,
                    uint64_t P, bool half, cudaStream_t s) {
    if (half)
        k_subtree_reduce<K, true><<<unsigned(nj - j0), 256, 0, s>>>(child, top, compact, c, j0, nj, P);
    else
        k_subtree_reduce<K, false><<<unsigned(nj - j0), 256, 0, s>>>(child, top, compact, c, j0, nj, P);
}

// the leaf pass of this launch writes the halved transient level (at least one level pass follows)
bool transient_half(const PosGeom& g) { return g.p1 - g.p0 >= 2; }

int sm_count() { return sm_count_current(); }


template <int NB, typename T, int MINB, int STAGES>
void launch_dmma_v(const T* U, const PosGeom& g, double* compact, double* tout, cudaStream_t s) {
    using C = LeafCfg<NB, T, MINB, STAGES>;
    auto kern = k_leaf_dmma<NB, T, MINB, STAGES>;
    smem_optin(kern, C::SMEM);
    const int occ = occupancy(kern, C::WPC * 32, C::SMEM);
    const uint64_t need = (g.p1 - g.p0 + C::WPC - 1) / C::WPC;
    const uint64_t grid = std::min<uint64_t>(need, uint64_t(sm_count()) * occ);
    kern<<<unsigned(grid), C::WPC * 32, C::SMEM, s>>>(U, g, compact, tout);
}

// ring depth of the staged-store kernel: as deep as lets two CTAs share an SM (2..4 stages)
template <int NB, typename T, int CH>
constexpr int staged_stages() {
    constexpr int R = 8 * NB;
    constexpr int stage = 4 * CH * (R * int(sizeof(T)) + 16);
    constexpr int stg = 2 * ((R * (R + 1) / 2 * 8 + 127) / 128 * 128);
    constexpr int fit = (110 * 1024 - stg) / stage;
    return fit < 2 ? 2 : (fit > 4 ? 4 : fit);
}

template <int NB, typename T, int CH, int STAGES, int NSTG>
void launch_dmma_s(const T* U, const PosGeom& g, double* compact, double* tout, cudaStream_t s) {
    using C = LeafCfgS<NB, T, CH, STAGES, NSTG>;
    auto kern = k_leaf_dmma_s<NB, T, CH, STAGES, NSTG>;
    smem_optin(kern, C::SMEM);
    const int occ = occupancy(kern, C::WPC * 32, C::SMEM);
    const uint64_t need = (g.p1 - g.p0 + C::WPC - 1) / C::WPC;
    const uint64_t grid = std::min<uint64_t>(need, uint64_t(sm_count()) * occ);
    kern<<<unsigned(grid), C::WPC * 32, C::SMEM, s>>>(U, g, compact, tout);
}

// 2 CTAs x 4 warps per SM with 4-stage rings: forcing 3 CTAs (168 registers, 3 stages) or
// 4 CTAs (128 registers, 2 stages) spills accumulators and measured 1.59 / 2.71 ms per
// config-2 leaf build against 1.19 ms (profiles/r02_tree_variants.jsonl)
template <int NB, typename T>
void launch_dmma(const T* U, const PosGeom& g, double* compact, double* tout, cudaStream_t s, int variant) {
    // small Grams (R <= 16: at most 1 KB) are cheaper to scatter straight from the registers
    // than to stage (measured per 2^22-row factor, staged / direct: R = 8 0.245 / 0.168 ms,
    // 16 0.204 / 0.189, 24 0.247 / 0.351, 32 0.400 / 0.426, 48 0.53 / 0.88, 64 0.79 / 1.17)
    if (variant == 1 || NB <= 2) return launch_dmma_v<NB, T, 2, 4>(U, g, compact, tout, s);
    // 16-row chunks when the leaf boundary (a multiple of F) falls on a chunk boundary
    if (g.F % 16 == 0) return launch_dmma_s<NB, T, 16, staged_stages<NB, T, 16>(), 2>(U, g, compact, tout, s);
    launch_dmma_s<NB, T, 8, staged_stages<NB, T, 8>(), 2>(U, g, compact, tout, s);
}

template <int R_, typename T>
void launch_big(const T* U, const PosGeom& g, double* compact, double* tout, cudaStream_t s) {
    using C = BigCfg<R_, T>;
    auto kern = k_leaf_cta<R_, T>;
    smem_optin(kern, C::SMEM);
    const int occ = occupancy(kern, C::NW * 32, C::SMEM);
    const uint64_t grid = std::min<uint64_t>(g.p1 - g.p0, std::max<uint64_t>(1, uint64_t(sm_count()) * occ / C::SPLIT));
    kern<<<dim3(unsigned(grid), C::SPLIT), C::NW * 32, C::SMEM, s>>>(U, g, compact, tout);
}

template <typename T>
void launch_leaf(const T* U, const PosGeom& g, double* compact, double* tout, cudaStream_t s,
                 bool generic, int variant) {
    if (g.F % 8 != 0 || g.seg) generic = true;  // the DMMA kernels stream uniform leaves in 8-row chunks
    if (!generic) {
        switch (g.R) {
            case 96: return launch_big<96, T>(U, g, compact, tout, s);
            case 128: return launch_big<128, T>(U, g, compact, tout, s);
            case 160: return launch_big<160, T>(U, g, compact, tout, s);
            case 192: return launch_big<192, T>(U, g, compact, tout, s);
            case 224: return launch_big<224, T>(U, g, compact, tout, s);
            case 256: return launch_big<256, T>(U, g, compact, tout, s);
            case 8: return launch_dmma<1, T>(U, g, compact, tout, s, variant);
            case 16: return launch_dmma<2, T>(U, g, compact, tout, s, variant);
            case 24: return launch_dmma<3, T>(U, g, compact, tout, s, variant);
            case 32: return launch_dmma<4, T>(U, g, compact, tout, s, variant);
            case 40: return launch_dmma<5, T>(U, g, compact, tout, s, variant);
            case 48: return launch_dmma<6, T>(U, g, compact, tout, s, variant);
            case 56: return launch_dmma<7, T>(U, g, compact, tout, s, variant);
            case 64: return launch_dmma<8, T>(U, g, compact, tout, s, variant);
            default: break;
        }
    }
    const uint64_t grid = std::min<uint64_t>(g.p1 - g.p0, uint64_t(sm_count()) * 16);
    k_leaf_generic<T><<<unsigned(grid), 256, 0, s>>>(U, g, compact, tout);
}

}  // namespace

uint64_t tree_positions(uint64_t I, uint32_t R) { return make_geom(I, R).npos; }

void tree_partition_rows(uint64_t I, uint32_t R, uint32_t parts, uint32_t part, uint64_t* first, uint64_t* last) {
    const PosGeom g = make_geom(I, R);
    const uint64_t span = g.npos / parts;
    uint64_t r0, rs, r1;
    pos_rows(g, uint64_t(part) * span, r0, rs, r1);
    *first = r0;
    pos_rows(g, uint64_t(part + 1) * span - 1, r0, rs, r1);
    *last = r1;
}

void tree_transient_doubles(uint64_t I, uint32_t R, uint64_t* a, uint64_t* b, uint64_t F, uint64_t nleaves) {
    const PosGeom g = make_geom(I, R, F, nleaves);
    *a = g.npos > 1 ? g.npos * g.P : 0;
    *b = g.npos > 2 ? (g.npos / 2) * g.P : 0;
}

int launch_tree_leaves(const TreeBuildArgs& a) {
    PosGeom g = make_geom(a.I, a.R, a.F, a.nleaves, a.segs);
    if (a.parts > 1) {  // one partition's subtree: positions [part, part+1) * npos / parts
        const uint64_t span = g.npos / a.parts;
        g.p0 = uint64_t(a.part) * span;
        g.p1 = g.p0 + span;
    }
    double* tout = g.npos > 1 ? a.tbuf_a : nullptr;
    g.tr_half = transient_half(g) ? 1 : 0;
    if (a.storage == 1)
        launch_leaf<float>(static_cast<const float*>(a.U), g, a.compact, tout, a.stream, a.force_generic,
                           a.leaf_variant);
    else
        launch_leaf<double>(static_cast<const double*>(a.U), g, a.compact, tout, a.stream, a.force_generic,
                            a.leaf_variant);
    return 1;
}

// Levels above the positions, bottom-up (:180-186). Whole tree: down to the
// root. One partition (parts = 2^gl > 1): only the partition's own nodes on
// levels D-1 .. gl, and its subtree root Gram (level gl) is copied to a.subroot.
int launch_tree_levels(const TreeBuildArgs& a) {
    const PosGeom g = make_geom(a.I, a.R, a.F, a.nleaves, a.segs);
    uint32_t D = 0;
    while ((uint64_t{1} << D) < g.npos) ++D;
    uint32_t gl = 0;
    while ((1u << gl) < a.parts) ++gl;
    double* cur = a.tbuf_a;
    double* nxt = a.tbuf_b;
    int launches = 0;
    bool half = false;  // the position level as the leaf pass left it (launch_tree_leaves)
    {
        PosGeom gp = g;
        if (a.parts > 1) {
            const uint64_t span = g.npos / a.parts;
            gp.p0 = uint64_t(a.part) * span;
            gp.p1 = gp.p0 + span;
        }
        half = transient_half(gp);
    }
    // passes of up to 5 levels each (k_subtree_reduce): level c -> c - k
    for (int c = int(D); c > int(gl);) {
        const int k = std::min(5, c - int(gl));
        const int l = c - k;  // parent level of this pass
        const uint64_t nj = uint64_t{1} << l;
        const uint64_t span = nj >> gl;
        const uint64_t j0 = a.parts > 1 ? uint64_t(a.part) * span : 0;
        const uint64_t j1 = a.parts > 1 ? j0 + span : nj;
        double* parent = (l > 0 || a.parts > 1) ? nxt : nullptr;
        switch (k) {
            case 1: launch_subtree<1>(cur, parent, a.compact, uint32_t(c), j0, j1, g.P, half, a.stream); break;
            case 2: launch_subtree<2>(cur, parent, a.compact, uint32_t(c), j0, j1, g.P, half, a.stream); break;
            case 3: launch_subtree<3>(cur, parent, a.compact, uint32_t(c), j0, j1, g.P, half, a.stream); break;
            case 4: launch_subtree<4>(cur, parent, a.compact, uint32_t(c), j0, j1, g.P, half, a.stream); break;
            default: launch_subtree<5>(cur, parent, a.compact, uint32_t(c), j0, j1, g.P, half, a.stream); break;
        }
        ++launches;
        half = false;
        std::swap(cur, nxt);
        c = l;
    }
    if (a.parts > 1 && a.subroot) {  // cur holds level gl
        if (cudaMemcpyAsync(a.subroot, cur + uint64_t(a.part) * g.P, sizeof(double) * g.P,
                            cudaMemcpyDeviceToDevice, a.stream) != cudaSuccess)
            return -1;
    }
    return launches;
}

// Top of a partitioned build: the parts = 2^gl subtree roots (parts x P, in
// subtree order) are level gl; stores the stored ones and reduces to the root.
int launch_tree_top(const TreeBuildArgs& a, const double* subroots) {
    const PosGeom g = make_geom(a.I, a.R, a.F, a.nleaves, a.segs);
    uint32_t gl = 0;
    while ((1u << gl) < a.parts) ++gl;
    int launches = 0;
    for (uint32_t i = 0; i < a.parts; i += 2) {  // even i = left children (odd heap ids) -> stored
        const uint64_t v = (uint64_t{1} << gl) - 1 + i;
        if (cudaMemcpyAsync(a.compact + slot_of(v) * g.P, subroots + uint64_t(i) * g.P,
                            sizeof(double) * g.P, cudaMemcpyDeviceToDevice, a.stream) != cudaSuccess)
            return -1;
    }
    const double* cur = subroots;
    double* bufs[2] = {a.tbuf_a, a.tbuf_b};
    int which = 0;
    for (int l = int(gl) - 1; l >= 0; --l) {
        const uint64_t nj = uint64_t{1} << l;
        double* parent = l > 0 ? bufs[which] : nullptr;
        k_level_reduce<<<unsigned(nj), 256, 0, a.stream>>>(cur, parent, a.compact, 0, nj, g.P, nj - 1);
        ++launches;
        cur = parent;
        which ^= 1;
    }
    return launches;
}

}  // namespace krpg
