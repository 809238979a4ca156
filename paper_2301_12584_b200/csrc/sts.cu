// STS-CP solve slice on device: the sparse-tensor side of
// one sketched ALS factor update, cp_als.cpp:282-313 with solver StsCp.
//
//  * tensor ingestion (SparseTensorCoo::from_entries, tensor.cpp:34-75):
//    entries sorted by their mixed-radix linear index (mode 0 slowest =
//    lexicographic coordinate order), duplicates summed (CUB radix sort +
//    reduce-by-key, both stable);
//  * fiber index of mode j (SparseTensorCoo::fiber_index, tensor.cpp:104-129):
//    entries sorted by their mode-j matricization column (lowest mode
//    fastest), distinct keys + CSR offsets; the fiber's (coordinate j, value)
//    pairs are stored contiguously in key order;
//  * sampled right-hand side (sampled_rhs_rows, cp_als.cpp:122-145) without
//    the dense J x I_j block: each draw's fiber is found by binary search,
//    draws are sorted by fiber, and every distinct sampled fiber g gets
//    S_g = sum_{d -> g} w_d^2 rows_d (a deterministic segmented sum), so a
//    fiber drawn many times is visited once; its nonzeros then add v_e S_g
//    into row coord_j(e) of M = (SA^T SB)^T, in fixed-size chunks of entries
//    per warp (load-balanced across huge Zipf fibers);
//  * the solve U_j[i] = pinv(SA^T SA) M[i] row by row (gram_cross + matmul +
//    transpose, dense_kernels.cpp:44-56, 209-223), column norms on the way,
//    then normalize_columns (cp_als.cpp:39-52) fused with the store into U_j.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>
#include <cmath>
#include <stdexcept>
#include <string>

#include "krpg_device.cuh"
#include "krpg_kernels.hpp"
#include "launch_util.hpp"
#include "ptx.cuh"

namespace krpg {

namespace {

#define STS_CK(call)                                                                                       \
    do {                                                                                                   \
        cudaError_t e_ = (call);                                                                           \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct Scratch {  // CUB temporary storage
    void* p = nullptr;
    size_t n = 0;
    void* get(size_t want) {
        if (want > n) {
            if (p) cudaFree(p);
            p = nullptr;
            STS_CK(cudaMalloc(&p, want));
            n = want;
        }
        return p;
    }
    ~Scratch() {
        if (p) cudaFree(p);
    }
};

struct Radix {  // mixed-radix strides, up to 8 modes
    uint64_t stride[8];
    uint32_t N;
};

constexpr uint32_t SCHUNK = 128;  // entries per scatter work item
constexpr uint32_t NONE = 0xFFFFFFFFu;

unsigned grid_of(uint64_t n) { return unsigned(std::min<uint64_t>((n + 255) / 256, 148ull * 32)); }

int bits_for(uint64_t top) { return top ? 64 - __builtin_clzll(top) : 1; }

__global__ void k_linear_keys(const uint32_t* __restrict__ coords, uint64_t nnz, Radix rx, uint64_t* __restrict__ key,
                              uint64_t* __restrict__ id) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < nnz; e += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t k = 0;
        for (uint32_t m = 0; m < rx.N; ++m) k += uint64_t(coords[e * rx.N + m]) * rx.stride[m];
        key[e] = k;
        if (id) id[e] = e;
    }
}

__global__ void k_decode(const uint64_t* __restrict__ key, uint64_t n, Radix rx, uint32_t* __restrict__ coords) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n; e += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t k = key[e];
        for (uint32_t m = 0; m < rx.N; ++m) {
            coords[e * rx.N + m] = uint32_t(k / rx.stride[m]);
            k %= rx.stride[m];
        }
    }
}

__global__ void k_gather_fiber(const uint64_t* __restrict__ order, const uint32_t* __restrict__ coords,
                               const double* __restrict__ vals, uint64_t nnz, uint32_t N, uint32_t j,
                               uint32_t* __restrict__ fcoord, double* __restrict__ fval) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < nnz; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t e = order[p];
        fcoord[p] = coords[e * N + j];
        fval[p] = vals[e];
    }
}

// per draw: the fiber (index into the sorted distinct keys) its drawn
// coordinates select, NONE if that fiber has no nonzero; checks q > 0
__global__ void k_draw_fibers(const uint32_t* __restrict__ idx, uint64_t J, uint32_t N, Radix colrx,
                              const double* __restrict__ prob, const uint64_t* __restrict__ keys, uint64_t G,
                              uint32_t* __restrict__ gdraw, uint32_t* __restrict__ did, int* err) {
    for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < J; d += uint64_t(gridDim.x) * blockDim.x) {
        const double q = prob[d];
        if (!(q > 0.0) || !isfinite(q)) atomicExch(err, 1);  // make_sampling_weights (sketch.cpp:44-47)
        // flat index, RowOrder::Reversed (first included factor fastest) = the
        // mode-j matricization column of the drawn coordinates (tensor.cpp:20-32)
        uint64_t u = 0;
        for (uint32_t k = 0; k < N; ++k) u += uint64_t(idx[d * N + k]) * colrx.stride[k];
        uint64_t lo = 0, hi = G;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (keys[mid] < u)
                lo = mid + 1;
            else
                hi = mid;
        }
        gdraw[d] = (lo < G && keys[lo] == u) ? uint32_t(lo) : NONE;
        did[d] = uint32_t(d);
    }
}

// one warp per sampled fiber (segment of the fiber-sorted draws):
// S[sg] = sum_d (w_d rows_d) w_d in draw order; chunk count of its entries
__global__ void k_fiber_sums(const uint32_t* __restrict__ ug, const uint32_t* __restrict__ cnt,
                             const uint32_t* __restrict__ start, const uint32_t* __restrict__ nseg,
                             const uint32_t* __restrict__ dsorted, const double* __restrict__ prob,
                             const double* __restrict__ rows, uint64_t J, uint32_t R,
                             const uint64_t* __restrict__ fptr, double* __restrict__ S, uint32_t* __restrict__ wcnt) {
    const int lane = threadIdx.x & 31;
    const uint32_t n = *nseg;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t sg = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); sg < J; sg += warps) {
        if (sg >= n) {  // unused segment slots take no scatter work
            if (lane == 0) wcnt[sg] = 0;
            continue;
        }
        const uint32_t g = ug[sg];
        if (g == NONE) {  // draws whose fiber holds no nonzero (all-zero SB row)
            if (lane == 0) wcnt[sg] = 0;
            continue;
        }
        if (lane == 0) wcnt[sg] = uint32_t((fptr[g + 1] - fptr[g] + SCHUNK - 1) / SCHUNK);
        for (uint32_t c = lane; c < R; c += 32) {
            double acc = 0.0;
            for (uint32_t t = start[sg]; t < start[sg] + cnt[sg]; ++t) {
                const uint32_t d = dsorted[t];
                const double w = 1.0 / sqrt(static_cast<double>(J) * prob[d]);
                acc += (w * rows[uint64_t(d) * R + c]) * w;
            }
            S[sg * R + c] = acc;
        }
    }
}

// step statistics: draws with a nonzero fiber, distinct sampled fibers, entries visited
__global__ void k_sts_stats(const uint32_t* __restrict__ ug, const uint32_t* __restrict__ cnt,
                            const uint32_t* __restrict__ nseg, const uint64_t* __restrict__ fptr,
                            unsigned long long* __restrict__ stats) {
    const uint32_t n = *nseg;
    unsigned long long a = 0, b = 0, c = 0;
    for (uint32_t sg = blockIdx.x * blockDim.x + threadIdx.x; sg < n; sg += gridDim.x * blockDim.x) {
        const uint32_t g = ug[sg];
        if (g == NONE) continue;
        a += cnt[sg];
        b += 1;
        c += fptr[g + 1] - fptr[g];
    }
    atomicAdd(stats + 0, a);
    atomicAdd(stats + 1, b);
    atomicAdd(stats + 2, c);
}

// one warp per work item (SCHUNK entries of one sampled fiber):
// M[coord_j(e), :] += v_e S[sg] (the products of gram_cross(sa, sb), regrouped)
__global__ void k_fiber_scatter(const uint32_t* __restrict__ ug, const uint32_t* __restrict__ wstart,
                                const uint32_t* __restrict__ nseg, uint64_t J, const uint64_t* __restrict__ fptr,
                                const uint32_t* __restrict__ fcoord, const double* __restrict__ fval,
                                const double* __restrict__ S, uint32_t R, double* __restrict__ M) {
    const int lane = threadIdx.x & 31;
    const uint32_t n = *nseg;
    if (n == 0) return;
    const uint64_t total = wstart[J];  // exclusive scan over J slots, J + 1 entries
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t it = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); it < total; it += warps) {
        uint32_t lo = 0, hi = n;  // last segment with wstart <= it (it has work, so it is a fiber)
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (wstart[mid] <= it)
                lo = mid;
            else
                hi = mid;
        }
        const uint32_t sg = lo, g = ug[sg];
        const uint64_t p0 = fptr[g] + (it - wstart[sg]) * SCHUNK;
        const uint64_t p1 = p0 + SCHUNK < fptr[g + 1] ? p0 + SCHUNK : fptr[g + 1];
        const double* Sg = S + uint64_t(sg) * R;
        double sv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) sv[t] = (lane + 32 * t < int(R)) ? Sg[lane + 32 * t] : 0.0;
        for (uint64_t p = p0; p < p1; ++p) {
            const uint64_t i = fcoord[p];
            const double v = fval[p];
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (lane + 32 * t < int(R)) atomicAdd(M + i * R + lane + 32 * t, v * sv[t]);
        }
    }
}

// ---- deterministic row-ordered scatter (replaces the atomic fiber scatter) ----
// gram_cross(SA, SB) of cp_als.cpp:290-294 without the dense J x I_j SB block (:128):
// M[i] = sum over the sampled fibers' entries with coordinate i of v_e S[sg_e], in the
// fixed order (fiber slot sg ascending, entry ascending): every visited entry gets its
// position e in that order, a stable radix sort by row groups them, and each row is summed
// by one warp in pieces of at most RPIECE entries (partial rows of multi-piece rows summed
// in piece order), so M -- and the solved factor -- are bit-reproducible run to run.
constexpr uint32_t RPIECE = 1024;

__global__ void k_seg_len(const uint32_t* __restrict__ ug, const uint32_t* __restrict__ nseg,
                          const uint64_t* __restrict__ fptr, uint64_t J, uint32_t* __restrict__ len) {
    const uint32_t n = *nseg;
    for (uint64_t sg = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; sg <= J; sg += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t L = 0;
        if (sg < n && ug[sg] != NONE) L = uint32_t(fptr[ug[sg] + 1] - fptr[ug[sg]]);
        len[sg] = L;
    }
}

// one warp per work item (SCHUNK entries of one sampled fiber): row key, order position
__global__ void k_visit(const uint32_t* __restrict__ ug, const uint32_t* __restrict__ wstart,
                        const uint32_t* __restrict__ nseg, uint64_t J, const uint64_t* __restrict__ fptr,
                        const uint32_t* __restrict__ fcoord, const double* __restrict__ fval,
                        const uint32_t* __restrict__ eoff, uint32_t* __restrict__ key, uint32_t* __restrict__ ord,
                        double* __restrict__ pv, uint32_t* __restrict__ psg) {
    const int lane = threadIdx.x & 31;
    const uint32_t n = *nseg;
    if (n == 0) return;
    const uint64_t total = wstart[J];
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t it = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); it < total; it += warps) {
        uint32_t lo = 0, hi = n;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (wstart[mid] <= it)
                lo = mid;
            else
                hi = mid;
        }
        const uint32_t sg = lo, g = ug[sg];
        const uint64_t f0 = fptr[g];
        const uint64_t p0 = f0 + (it - wstart[sg]) * SCHUNK;
        const uint64_t p1 = p0 + SCHUNK < fptr[g + 1] ? p0 + SCHUNK : fptr[g + 1];
        for (uint64_t p = p0 + lane; p < p1; p += 32) {
            const uint32_t e = eoff[sg] + uint32_t(p - f0);
            key[e] = fcoord[p];
            ord[e] = e;
            pv[e] = fval[p];
            psg[e] = sg;
        }
    }
}

__global__ void k_row_pieces(const uint32_t* __restrict__ rcnt, const uint32_t* __restrict__ nrows, uint64_t cap,
                             uint32_t* __restrict__ np, uint32_t* __restrict__ mp) {
    const uint32_t n = *nrows;
    for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r <= cap; r += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t k = 0;
        if (r < n) k = (rcnt[r] + RPIECE - 1) / RPIECE;
        np[r] = k;
        mp[r] = k > 1 ? k : 0;  // partial-row slots only for multi-piece rows
    }
}

// (value, fiber slot) of every visited entry in row-sorted order (coalesced for the sums)
__global__ void k_gather_sorted(const uint32_t* __restrict__ ord, const double* __restrict__ pv,
                                const uint32_t* __restrict__ psg, uint64_t E, double* __restrict__ vs,
                                uint32_t* __restrict__ ss) {
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < E; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t e = ord[t];
        vs[t] = pv[e];
        ss[t] = psg[e];
    }
}

// one warp per piece: lane owns columns lane + 32 c (R <= 256); the piece's (v, slot) pairs
// are read 32 at a time by the lanes and broadcast, so every S-row load is independent
__global__ void k_piece_sums(const uint32_t* __restrict__ urow, const uint32_t* __restrict__ rcnt,
                             const uint32_t* __restrict__ roff, const uint32_t* __restrict__ poff,
                             const uint32_t* __restrict__ moff, const uint32_t* __restrict__ nrows,
                             const double* __restrict__ vs, const uint32_t* __restrict__ ss,
                             const double* __restrict__ S, uint32_t R, double* __restrict__ M,
                             double* __restrict__ pbuf) {
    const int lane = threadIdx.x & 31;
    const uint32_t nr = *nrows;
    if (nr == 0) return;
    const uint64_t npieces = poff[nr];
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t q = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); q < npieces; q += warps) {
        uint32_t lo = 0, hi = nr;  // last row with poff <= q
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (poff[mid] <= q)
                lo = mid;
            else
                hi = mid;
        }
        const uint32_t r = lo, k = uint32_t(q - poff[r]);
        const uint32_t b = roff[r] + k * RPIECE;
        const uint32_t e1 = min(roff[r] + rcnt[r], b + RPIECE);
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t t0 = b; t0 < e1; t0 += 32) {
            const uint32_t nt = min(32u, e1 - t0);
            const double myv = lane < int(nt) ? vs[t0 + lane] : 0.0;
            const uint32_t mys = lane < int(nt) ? ss[t0 + lane] : 0u;
#pragma unroll 8
            for (uint32_t j = 0; j < nt; ++j) {  // entries in order: the sum is order-fixed
                const double v = __shfl_sync(0xffffffffu, myv, int(j));
                const double* Sg = S + uint64_t(__shfl_sync(0xffffffffu, mys, int(j))) * R;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (lane + 32 * c < int(R)) acc[c] = fma(v, Sg[lane + 32 * c], acc[c]);
            }
        }
        const bool multi = poff[r + 1] - poff[r] > 1;
        double* dst = multi ? pbuf + (uint64_t(moff[r]) + k) * R : M + uint64_t(urow[r]) * R;
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (lane + 32 * c < int(R)) dst[lane + 32 * c] = acc[c];
    }
}

// rows split into several pieces: their partial rows summed in piece order
__global__ void k_piece_merge(const uint32_t* __restrict__ urow, const uint32_t* __restrict__ poff,
                              const uint32_t* __restrict__ moff, const uint32_t* __restrict__ nrows,
                              const double* __restrict__ pbuf, uint32_t R, double* __restrict__ M) {
    const int lane = threadIdx.x & 31;
    const uint32_t nr = *nrows;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t r = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); r < nr; r += warps) {
        const uint32_t k = poff[r + 1] - poff[r];
        if (k <= 1) continue;
        for (uint32_t c = lane; c < R; c += 32) {
            double acc = 0.0;
            for (uint32_t t = 0; t < k; ++t) acc += pbuf[(uint64_t(moff[r]) + t) * R + c];
            M[uint64_t(urow[r]) * R + c] = acc;
        }
    }
}

// U[i, a] = sum_k pinv[a, k] M[i, k] (matmul(pinv, gram_cross) transposed,
// dense_kernels.cpp:209-223), one warp per row; pinv staged transposed in shared
// memory so lanes (= output columns) read consecutive words. The column sums of
// squares for normalize_columns are accumulated on the way (colsq, R).
__global__ void k_solve_rows(const double* __restrict__ M, uint64_t I, uint32_t R, const double* __restrict__ pinv,
                             double* __restrict__ U, double* __restrict__ colsq, int staged) {
    extern __shared__ double smem_p[];  // pinv^T, R x R, when it fits shared memory
    __shared__ double s_sq[256];
    for (uint32_t e = threadIdx.x; e < R; e += blockDim.x) s_sq[e] = 0.0;
    if (staged)
        for (uint32_t e = threadIdx.x; e < R * R; e += blockDim.x) smem_p[(e % R) * R + e / R] = pinv[e];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    double sq[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // R <= 256: lane owns columns lane + 32 t
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < I; i += warps) {
        const double* m = M + i * R;
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        bool nz = false;  // rows no sampled fiber touched are zero: skip the product
#pragma unroll
        for (int t = 0; t < 8; ++t)
            if (lane + 32 * t < int(R)) nz |= m[lane + 32 * t] != 0.0;
        if (__any_sync(0xffffffffu, nz))
        for (uint32_t k = 0; k < R; ++k) {
            const double mk = m[k];
            if (mk == 0.0) continue;  // untouched rows / zero entries (matmul skips them too)
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const uint32_t a = lane + 32 * t;
                if (a < R) acc[t] = fma(staged ? smem_p[k * R + a] : pinv[a * R + k], mk, acc[t]);
            }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const uint32_t a = lane + 32 * t;
            if (a < R) {
                U[i * R + a] = acc[t];
                sq[t] = fma(acc[t], acc[t], sq[t]);
            }
        }
    }
    // column sums of squares, reproducibly: warps in order within the block, blocks in
    // order in k_colsq_finish (colsq = this block's partial row of the grid x R buffer)
    const int warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int w = 0; w < nwarp; ++w) {
        if (warp == w)
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const uint32_t a = lane + 32 * t;
                if (a < R) s_sq[a] += sq[t];
            }
        __syncthreads();
    }
    for (uint32_t e = threadIdx.x; e < R; e += blockDim.x) colsq[uint64_t(blockIdx.x) * R + e] = s_sq[e];
}

// Same solve on the FP64 tensor cores: a warp takes 8 rows, D (8 rows x 8 cols of
// U) = sum over k-steps of M[rows, 4s..4s+3] (A) x pinv^T[4s..4s+3, 8q..8q+7] (B);
// pinv staged in shared memory with rows padded to R + 4 doubles (conflict-free
// B fragments). All-zero 8-row blocks (rows no sampled fiber touched) skip the MMA.
template <int NB>
__global__ void __launch_bounds__(256) k_solve_rows_dmma(const double* __restrict__ M, uint64_t I,
                                                         const double* __restrict__ pinv, double* __restrict__ U,
                                                         double* __restrict__ colsq) {
    constexpr int R = 8 * NB, KS = R / 4, LD = R + 4;
    extern __shared__ double sp[];  // R x LD
    __shared__ double s_sq[R];
    for (int e = threadIdx.x; e < R; e += blockDim.x) s_sq[e] = 0.0;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) sp[(e / R) * LD + e % R] = pinv[e];
    __syncthreads();
    const int lane = threadIdx.x & 31, m = lane >> 2, kq = lane & 3;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    double sq[NB][2];
#pragma unroll
    for (int q = 0; q < NB; ++q) sq[q][0] = sq[q][1] = 0.0;
    const uint64_t nblk = (I + 7) / 8;
    for (uint64_t b = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); b < nblk; b += warps) {
        const uint64_t row = 8 * b + m;
        const bool rv = row < I;
        double a[KS];
        bool nz = false;
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            a[t] = rv ? M[row * R + 4 * t + kq] : 0.0;
            nz |= a[t] != 0.0;
        }
        double d[NB][2];
#pragma unroll
        for (int q = 0; q < NB; ++q) d[q][0] = d[q][1] = 0.0;
        if (__any_sync(0xffffffffu, nz)) {
#pragma unroll
            for (int t = 0; t < KS; ++t)
#pragma unroll
                for (int q = 0; q < NB; ++q) dmma_884(d[q][0], d[q][1], a[t], sp[(8 * q + m) * LD + 4 * t + kq]);
        }
        if (rv) {
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                *reinterpret_cast<double2*>(U + row * R + 8 * q + 2 * kq) = make_double2(d[q][0], d[q][1]);
                sq[q][0] = fma(d[q][0], d[q][0], sq[q][0]);
                sq[q][1] = fma(d[q][1], d[q][1], sq[q][1]);
            }
        }
    }
    // reduce over the 8 row-lanes sharing (lane & 3), then per block, then global
#pragma unroll
    for (int q = 0; q < NB; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double v = sq[q][e];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            sq[q][e] = v;
        }
    // warps in order within the block, blocks in order in k_colsq_finish
    const int warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int w = 0; w < nwarp; ++w) {
        if (warp == w && m == 0)
#pragma unroll
            for (int q = 0; q < NB; ++q)
#pragma unroll
                for (int e = 0; e < 2; ++e) s_sq[8 * q + 2 * kq + e] += sq[q][e];
        __syncthreads();
    }
    for (int e = threadIdx.x; e < R; e += blockDim.x) colsq[uint64_t(blockIdx.x) * R + e] = s_sq[e];
}

__global__ void k_colsq_finish(const double* __restrict__ part, int nblocks, uint32_t R, double* __restrict__ nrm) {
    for (uint32_t a = threadIdx.x; a < R; a += blockDim.x) {
        double t = 0.0;
        for (int b = 0; b < nblocks; ++b) t += part[uint64_t(b) * R + a];
        nrm[a] = sqrt(t);
    }
}

__global__ void k_sqrt_inplace(double* x, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = sqrt(x[i]);
}

// normalize_columns (cp_als.cpp:39-52) fused with the store into the factor's
// storage type
template <typename T>
__global__ void k_normalize_store(const double* __restrict__ U, uint64_t I, uint32_t R, const double* __restrict__ nrm,
                                  T* __restrict__ out) {
    const uint64_t total = I * R;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = uint32_t(e % R);
        const double n = nrm[c];
        double x = U[e];
        if (n > 0.0)
            x /= n;
        else if (e / R == c % I)  // zero column: deterministic unit basis vector
            x = 1.0;
        out[e] = static_cast<T>(x);
    }
}

struct StsWork {  // views into the per-step scratch (sts_work_bytes)
    double* S;
    unsigned long long* stats;
    uint32_t *gdraw, *gsort, *did, *dsort, *ug, *cnt, *wcnt, *start, *wstart, *nseg;
    void* cub;
    StsWork(void* work, uint64_t J, uint32_t R) {
        char* w = static_cast<char*>(work);
        S = reinterpret_cast<double*>(w);
        stats = reinterpret_cast<unsigned long long*>(w + 8 * J * R);
        gdraw = reinterpret_cast<uint32_t*>(stats + 4);
        gsort = gdraw + J;
        did = gsort + J;
        dsort = did + J;
        ug = dsort + J;
        cnt = ug + J;
        wcnt = cnt + J;  // J + 1 (the last slot stays 0)
        start = wcnt + J + 1;
        wstart = start + J + 1;
        nseg = wstart + J + 1;
        cub = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(nseg + 1) + 255) & ~uintptr_t(255));
    }
};

constexpr size_t kCubBytes = size_t(1) << 20;

}  // namespace

// ---- ingestion ----
uint64_t tensor_ingest(const uint32_t* d_coords, const double* d_vals, uint64_t nnz, uint32_t N, const uint64_t* dims,
                       uint32_t** d_coords_out, double** d_vals_out, cudaStream_t s) {
    Radix rx{};
    rx.N = N;
    uint64_t st = 1;
    for (int m = int(N) - 1; m >= 0; --m) {  // mode 0 slowest: lexicographic order
        rx.stride[m] = st;
        st *= dims[m];
    }
    // the unsorted keys' buffer is reused for the distinct keys (4 x 8 B per entry of scratch)
    uint64_t *key = nullptr, *key2 = nullptr, *nrun = nullptr;
    double *val2 = nullptr, *uval = nullptr;
    STS_CK(cudaMallocAsync(&key, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&key2, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&val2, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&uval, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&nrun, 8, s));
    uint64_t* ukey = key;
    k_linear_keys<<<grid_of(nnz), 256, 0, s>>>(d_coords, nnz, rx, key, nullptr);
    Scratch tmp;
    size_t need = 0;
    const int bits = bits_for(st - 1);
    STS_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, d_vals, val2, nnz, 0, bits, s));
    STS_CK(cub::DeviceRadixSort::SortPairs(tmp.get(need), need, key, key2, d_vals, val2, nnz, 0, bits, s));
    need = 0;
    STS_CK(cub::DeviceReduce::ReduceByKey(nullptr, need, key2, ukey, val2, uval, nrun, cub::Sum(), nnz, s));
    STS_CK(cub::DeviceReduce::ReduceByKey(tmp.get(need), need, key2, ukey, val2, uval, nrun, cub::Sum(), nnz, s));
    uint64_t n = 0;
    STS_CK(cudaMemcpyAsync(&n, nrun, 8, cudaMemcpyDeviceToHost, s));
    STS_CK(cudaStreamSynchronize(s));
    STS_CK(cudaMalloc(d_coords_out, 4 * std::max<uint64_t>(n, 1) * N));
    STS_CK(cudaMalloc(d_vals_out, 8 * std::max<uint64_t>(n, 1)));
    k_decode<<<grid_of(n), 256, 0, s>>>(ukey, n, rx, *d_coords_out);
    STS_CK(cudaMemcpyAsync(*d_vals_out, uval, 8 * n, cudaMemcpyDeviceToDevice, s));
    for (void* p : {static_cast<void*>(key), static_cast<void*>(key2), static_cast<void*>(val2),
                    static_cast<void*>(uval), static_cast<void*>(nrun)})
        STS_CK(cudaFreeAsync(p, s));
    STS_CK(cudaStreamSynchronize(s));
    return n;
}

// ---- device-resident input: coordinate range check, sum of squares ----
__global__ void k_check_coords(const uint32_t* __restrict__ coords, uint64_t nnz, uint32_t N, Radix lim,
                               int* __restrict__ bad) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < nnz * N;
         e += uint64_t(gridDim.x) * blockDim.x)
        if (coords[e] >= lim.stride[e % N]) atomicExch(bad, 1);
}

constexpr int kNormBlocks = 1184;
// per-block partial sums over a fixed contiguous split (block b sums [b*chunk, ...) in
// thread-strided order + a fixed tree), so the total is run-to-run reproducible
__global__ void __launch_bounds__(256) k_sumsq_partials(const double* __restrict__ v, uint64_t n,
                                                        double* __restrict__ part) {
    const uint64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t b0 = blockIdx.x * chunk, b1 = b0 + chunk < n ? b0 + chunk : n;
    double acc = 0.0;
    for (uint64_t e = b0 + threadIdx.x; e < b1; e += blockDim.x) acc = fma(v[e], v[e], acc);
    __shared__ double red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (int(threadIdx.x) < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

bool coords_in_range(const uint32_t* d_coords, uint64_t nnz, uint32_t N, const uint64_t* dims, cudaStream_t s) {
    Radix lim{};
    lim.N = N;
    for (uint32_t m = 0; m < N; ++m) lim.stride[m] = dims[m];
    int* bad = nullptr;
    STS_CK(cudaMallocAsync(&bad, sizeof(int), s));
    STS_CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
    if (nnz) k_check_coords<<<grid_of(nnz * N), 256, 0, s>>>(d_coords, nnz, N, lim, bad);
    int h = 0;
    STS_CK(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    STS_CK(cudaFreeAsync(bad, s));
    STS_CK(cudaStreamSynchronize(s));
    return h == 0;
}

double sum_of_squares(const double* d_v, uint64_t n, cudaStream_t s) {
    if (!n) return 0.0;
    double* part = nullptr;
    STS_CK(cudaMallocAsync(&part, 8 * kNormBlocks, s));
    k_sumsq_partials<<<kNormBlocks, 256, 0, s>>>(d_v, n, part);
    std::vector<double> h(kNormBlocks);
    STS_CK(cudaMemcpyAsync(h.data(), part, 8 * kNormBlocks, cudaMemcpyDeviceToHost, s));
    STS_CK(cudaFreeAsync(part, s));
    STS_CK(cudaStreamSynchronize(s));
    double t = 0.0;
    for (double x : h) t += x;
    return t;
}

// ---- fiber index of mode j ----
void fiber_index_build(const uint32_t* d_coords, const double* d_vals, uint64_t nnz, uint32_t N, const uint64_t* dims,
                       uint32_t j, FiberIndexDev* out, cudaStream_t s) {
    Radix rx{};
    rx.N = N;
    uint64_t st = 1;
    for (uint32_t m = 0; m < N; ++m) {  // lowest mode fastest, mode j skipped (tensor.cpp:20-32)
        rx.stride[m] = m == j ? 0 : st;
        if (m != j) st *= dims[m];
    }
    const uint64_t n1 = std::max<uint64_t>(nnz, 1);
    uint64_t *key = nullptr, *key2 = nullptr, *id = nullptr, *id2 = nullptr, *cnt = nullptr, *nrun = nullptr;
    STS_CK(cudaMallocAsync(&key, 8 * n1, s));
    STS_CK(cudaMallocAsync(&key2, 8 * n1, s));
    STS_CK(cudaMallocAsync(&id, 8 * n1, s));
    STS_CK(cudaMallocAsync(&id2, 8 * n1, s));
    STS_CK(cudaMallocAsync(&cnt, 8 * (n1 + 1), s));
    STS_CK(cudaMallocAsync(&nrun, 8, s));
    k_linear_keys<<<grid_of(nnz), 256, 0, s>>>(d_coords, nnz, rx, key, id);
    const int bits = bits_for(st - 1);
    Scratch tmp;
    size_t need = 0;
    STS_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, id, id2, nnz, 0, bits, s));
    STS_CK(cub::DeviceRadixSort::SortPairs(tmp.get(need), need, key, key2, id, id2, nnz, 0, bits, s));
    need = 0;
    STS_CK(cub::DeviceRunLengthEncode::Encode(nullptr, need, key2, key, cnt, nrun, nnz, s));
    STS_CK(cub::DeviceRunLengthEncode::Encode(tmp.get(need), need, key2, key, cnt, nrun, nnz, s));
    uint64_t G = 0;
    STS_CK(cudaMemcpyAsync(&G, nrun, 8, cudaMemcpyDeviceToHost, s));
    STS_CK(cudaStreamSynchronize(s));
    out->G = G;
    out->nnz = nnz;
    out->I = dims[j];
    STS_CK(cudaMalloc(&out->keys, 8 * std::max<uint64_t>(G, 1)));
    STS_CK(cudaMalloc(&out->fptr, 8 * (G + 1)));
    STS_CK(cudaMalloc(&out->fcoord, 4 * n1));
    STS_CK(cudaMalloc(&out->fval, 8 * n1));
    STS_CK(cudaMemcpyAsync(out->keys, key, 8 * G, cudaMemcpyDeviceToDevice, s));
    STS_CK(cudaMemsetAsync(cnt + G, 0, 8, s));
    need = 0;
    STS_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, out->fptr, G + 1, s));
    STS_CK(cub::DeviceScan::ExclusiveSum(tmp.get(need), need, cnt, out->fptr, G + 1, s));
    k_gather_fiber<<<grid_of(nnz), 256, 0, s>>>(id2, d_coords, d_vals, nnz, N, j, out->fcoord, out->fval);
    for (void* p : {static_cast<void*>(key), static_cast<void*>(key2), static_cast<void*>(id), static_cast<void*>(id2),
                    static_cast<void*>(cnt), static_cast<void*>(nrun)})
        STS_CK(cudaFreeAsync(p, s));
    STS_CK(cudaStreamSynchronize(s));
}

void fiber_index_free(FiberIndexDev& f) {
    for (void* p : {static_cast<void*>(f.keys), static_cast<void*>(f.fptr), static_cast<void*>(f.fcoord),
                    static_cast<void*>(f.fval)})
        if (p) cudaFree(p);
    f = FiberIndexDev{};
}

// ---- one STS-CP step's device work ----
// layout: S (J x R doubles) | stats (4 u64) | gdraw gsort did dsort ug cnt (J u32 each)
//         | wcnt start wstart (J+1 each) | nseg | CUB scratch (256-aligned)
size_t sts_work_bytes(uint64_t J, uint32_t R) { return 8 * J * R + 32 + 4 * (9 * J + 4) + 512 + kCubBytes; }

const void* sts_stats_ptr(void* work, uint64_t J, uint32_t R) { return StsWork(work, J, R).stats; }

void launch_sts_rhs(const uint32_t* idx, uint64_t J, uint32_t N, uint32_t j, const uint64_t* dims, const double* prob,
                    const double* rows, uint32_t R, const FiberIndexDev& F, void* work, double* M, int* err,
                    cudaStream_t s, bool deterministic) {
    Radix colrx{};
    colrx.N = N;
    uint64_t st = 1;
    for (uint32_t m = 0; m < N; ++m) {
        colrx.stride[m] = m == j ? 0 : st;
        if (m != j) st *= dims[m];
    }
    StsWork W(work, J, R);
    auto cub_check = [&](size_t need) {
        if (need > kCubBytes) throw std::runtime_error("sts: CUB scratch too small");
    };
    k_draw_fibers<<<grid_of(J), 256, 0, s>>>(idx, J, N, colrx, prob, F.keys, F.G, W.gdraw, W.did, err);
    size_t need = 0;
    STS_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, W.gdraw, W.gsort, W.did, W.dsort, J, 0, 32, s));
    cub_check(need);
    STS_CK(cub::DeviceRadixSort::SortPairs(W.cub, need, W.gdraw, W.gsort, W.did, W.dsort, J, 0, 32, s));
    need = 0;
    STS_CK(cub::DeviceRunLengthEncode::Encode(nullptr, need, W.gsort, W.ug, W.cnt, W.nseg, J, s));
    cub_check(need);
    STS_CK(cub::DeviceRunLengthEncode::Encode(W.cub, need, W.gsort, W.ug, W.cnt, W.nseg, J, s));
    need = 0;
    STS_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, W.cnt, W.start, J, s));
    cub_check(need);
    STS_CK(cub::DeviceScan::ExclusiveSum(W.cub, need, W.cnt, W.start, J, s));
    const unsigned wgrid = unsigned(std::min<uint64_t>((J + 7) / 8, 148ull * 16));
    k_fiber_sums<<<wgrid, 256, 0, s>>>(W.ug, W.cnt, W.start, W.nseg, W.dsort, prob, rows, J, R, F.fptr, W.S, W.wcnt);
    STS_CK(cudaMemsetAsync(W.wcnt + J, 0, 4, s));  // wstart[J] = total work items
    need = 0;
    STS_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, W.wcnt, W.wstart, J + 1, s));
    cub_check(need);
    STS_CK(cub::DeviceScan::ExclusiveSum(W.cub, need, W.wcnt, W.wstart, J + 1, s));
    STS_CK(cudaMemsetAsync(W.stats, 0, 32, s));
    k_sts_stats<<<64, 256, 0, s>>>(W.ug, W.cnt, W.nseg, F.fptr, W.stats);
    STS_CK(cudaMemsetAsync(M, 0, 8 * F.I * R, s));
    if (!deterministic) {  // fp64 atomics: faster, sums in run-dependent order
        k_fiber_scatter<<<148 * 16, 256, 0, s>>>(W.ug, W.wstart, W.nseg, J, F.fptr, F.fcoord, F.fval, W.S, R, M);
        return;
    }
    // deterministic row-ordered scatter (k_visit -> stable sort by row -> per-row pieces);
    // its E-sized buffers come from the stream-ordered pool, kept cached between steps
    // (the default release threshold 0 would hand them back to the driver at every sync)
    {
        static bool pool_set[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev >= 0 && dev < 64 && !pool_set[dev]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t keep = ~uint64_t{0};
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            pool_set[dev] = true;
        }
    }
    uint32_t* len = nullptr;
    uint32_t* eoff = nullptr;
    STS_CK(cudaMallocAsync(&len, 4 * (J + 1), s));
    STS_CK(cudaMallocAsync(&eoff, 4 * (J + 1), s));
    k_seg_len<<<grid_of(J + 1), 256, 0, s>>>(W.ug, W.nseg, F.fptr, J, len);
    Scratch tmp;
    need = 0;
    STS_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, len, eoff, J + 1, s));
    STS_CK(cub::DeviceScan::ExclusiveSum(tmp.get(need), need, len, eoff, J + 1, s));
    uint32_t E = 0;
    STS_CK(cudaMemcpyAsync(&E, eoff + J, 4, cudaMemcpyDeviceToHost, s));
    STS_CK(cudaStreamSynchronize(s));
    if (E > 0) {
        const uint64_t E1 = E;
        uint32_t *key, *key2, *ord, *ord2, *psg, *ss, *urow, *rcnt, *roff, *nrows, *np, *poff, *mp, *moff;
        double *pv, *vs;
        for (uint32_t** b : {&key, &key2, &ord, &ord2, &psg, &ss}) STS_CK(cudaMallocAsync(b, 4 * E1, s));
        for (double** b : {&pv, &vs}) STS_CK(cudaMallocAsync(b, 8 * E1, s));
        for (uint32_t** b : {&urow, &rcnt, &roff, &np, &poff, &mp, &moff}) STS_CK(cudaMallocAsync(b, 4 * (E1 + 1), s));
        STS_CK(cudaMallocAsync(&nrows, 4, s));
        k_visit<<<148 * 16, 256, 0, s>>>(W.ug, W.wstart, W.nseg, J, F.fptr, F.fcoord, F.fval, eoff, key, ord, pv, psg);
        const int bits = bits_for(F.I > 1 ? F.I - 1 : 1);
        need = 0;
        STS_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, ord, ord2, E1, 0, bits, s));
        STS_CK(cub::DeviceRadixSort::SortPairs(tmp.get(need), need, key, key2, ord, ord2, E1, 0, bits, s));
        k_gather_sorted<<<grid_of(E1), 256, 0, s>>>(ord2, pv, psg, E1, vs, ss);
        need = 0;
        STS_CK(cub::DeviceRunLengthEncode::Encode(nullptr, need, key2, urow, rcnt, nrows, E1, s));
        STS_CK(cub::DeviceRunLengthEncode::Encode(tmp.get(need), need, key2, urow, rcnt, nrows, E1, s));
        need = 0;
        STS_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, rcnt, roff, E1, s));
        STS_CK(cub::DeviceScan::ExclusiveSum(tmp.get(need), need, rcnt, roff, E1, s));
        k_row_pieces<<<grid_of(E1 + 1), 256, 0, s>>>(rcnt, nrows, E1, np, mp);
        need = 0;
        STS_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, np, poff, E1 + 1, s));
        STS_CK(cub::DeviceScan::ExclusiveSum(tmp.get(need), need, np, poff, E1 + 1, s));
        need = 0;
        STS_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, mp, moff, E1 + 1, s));
        STS_CK(cub::DeviceScan::ExclusiveSum(tmp.get(need), need, mp, moff, E1 + 1, s));
        // partial rows: at most E / RPIECE + (rows with > RPIECE entries) pieces in multi-piece rows
        const uint64_t pmax = 2 * (E1 / RPIECE) + 2;
        double* pbuf = nullptr;
        STS_CK(cudaMallocAsync(&pbuf, 8 * pmax * R, s));
        k_piece_sums<<<148 * 16, 256, 0, s>>>(urow, rcnt, roff, poff, moff, nrows, vs, ss, W.S, R, M, pbuf);
        k_piece_merge<<<148 * 8, 256, 0, s>>>(urow, poff, moff, nrows, pbuf, R, M);
        for (void* b : {static_cast<void*>(key), static_cast<void*>(key2), static_cast<void*>(ord),
                        static_cast<void*>(ord2), static_cast<void*>(pv), static_cast<void*>(psg),
                        static_cast<void*>(vs), static_cast<void*>(ss),
                        static_cast<void*>(urow), static_cast<void*>(rcnt), static_cast<void*>(roff),
                        static_cast<void*>(np), static_cast<void*>(poff), static_cast<void*>(mp),
                        static_cast<void*>(moff), static_cast<void*>(nrows), static_cast<void*>(pbuf)})
            STS_CK(cudaFreeAsync(b, s));
    }
    STS_CK(cudaFreeAsync(len, s));
    STS_CK(cudaFreeAsync(eoff, s));
    STS_CK(cudaStreamSynchronize(s));  // the CUB scratch (tmp) is freed on return
}

void launch_solve_normalize(const double* M, uint64_t I, uint32_t R, const double* pinv, double* Utmp, double* nrm,
                            void* Uout, uint32_t storage, cudaStream_t s) {
    const size_t need = sizeof(double) * R * R;
    const bool staged = need <= 160 * 1024;  // R <= 144; larger pinv is read through L1/L2
    const size_t smem = staged ? need : 0;
    smem_optin(k_solve_rows, smem);
    // per-block column partials (grid x R), summed in block order by k_colsq_finish
    double* part = nullptr;
    STS_CK(cudaMallocAsync(&part, sizeof(double) * 148ull * 8 * R, s));
    int nblocks = 0;
    if (R % 8 == 0 && R <= 128) {  // FP64 tensor-core path (padded pinv fits shared memory)
        const size_t dsm = sizeof(double) * R * (R + 4);
        const unsigned grid = unsigned(std::min<uint64_t>((I + 63) / 64, 148ull * 8));
        nblocks = int(grid);
        auto launch = [&](auto kern) {
            smem_optin(kern, dsm);
            kern<<<grid, 256, dsm, s>>>(M, I, pinv, Utmp, part);
        };
        switch (R / 8) {
            case 1: launch(k_solve_rows_dmma<1>); break;
            case 2: launch(k_solve_rows_dmma<2>); break;
            case 3: launch(k_solve_rows_dmma<3>); break;
            case 4: launch(k_solve_rows_dmma<4>); break;
            case 5: launch(k_solve_rows_dmma<5>); break;
            case 6: launch(k_solve_rows_dmma<6>); break;
            case 7: launch(k_solve_rows_dmma<7>); break;
            case 8: launch(k_solve_rows_dmma<8>); break;
            case 12: launch(k_solve_rows_dmma<12>); break;
            case 16: launch(k_solve_rows_dmma<16>); break;
            default: {
                const unsigned g2 = unsigned(std::min<uint64_t>((I + 7) / 8, 148ull * 8));
                nblocks = int(g2);
                k_solve_rows<<<g2, 256, smem, s>>>(M, I, R, pinv, Utmp, part, staged ? 1 : 0);
            }
        }
    } else {
        const unsigned grid = unsigned(std::min<uint64_t>((I + 7) / 8, 148ull * 8));
        nblocks = int(grid);
        k_solve_rows<<<grid, 256, smem, s>>>(M, I, R, pinv, Utmp, part, staged ? 1 : 0);
    }
    k_colsq_finish<<<1, 256, 0, s>>>(part, nblocks, R, nrm);
    STS_CK(cudaFreeAsync(part, s));
    if (Uout) launch_normalize_store(Utmp, I, R, nrm, Uout, storage, s);
}

void launch_normalize_store(const double* Utmp, uint64_t I, uint32_t R, const double* nrm, void* Uout,
                            uint32_t storage, cudaStream_t s) {
    if (storage == 1)
        k_normalize_store<float><<<grid_of(I * R), 256, 0, s>>>(Utmp, I, R, nrm, static_cast<float*>(Uout));
    else
        k_normalize_store<double><<<grid_of(I * R), 256, 0, s>>>(Utmp, I, R, nrm, static_cast<double*>(Uout));
}

}  // namespace krpg
