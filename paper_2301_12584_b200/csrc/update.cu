// Incremental tree updates and small factor utilities.
//
// SegmentTreeSampler::update_entry (/root/reference/proj/src/segment_tree_sampler.cpp:358-409)
// patches row/column c of every stored partial Gram on the root->leaf path of
// row r with delta*U[r,b] (b != c) and 2*delta*old + delta^2 (b == c). A batch
// of such updates applied in order changes every node containing row r by
// exactly u'u'^T - u u^T (u: the row before the batch, u': after), so the
// device applies one warp per touched row with that net rank-2 patch:
//   D_ab = u_a (u'_b - u_b) + (u'_a - u_a) u'_b     (exact identity; diagonal
//   gives 2 delta old + delta^2 like :398), atomically added along the path.
#include <algorithm>

#include "krpg_device.cuh"
#include "krpg_kernels.hpp"
#include "launch_util.hpp"
#include "ptx.cuh"

namespace krpg {

namespace {

unsigned grid_for(uint64_t n, unsigned block) {
    return unsigned(std::min<uint64_t>((n + block - 1) / block, 148ull * 32));
}

__global__ void k_row_deltas(double* __restrict__ compact, Topo t, uint32_t R, uint64_t nrows,
                             const uint64_t* __restrict__ rows, const double* __restrict__ oldr,
                             const double* __restrict__ newr) {
    const int lane = threadIdx.x & 31;
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= nrows) return;
    const uint64_t r = rows[w];
    const double* u0 = oldr + w * R;
    const double* u1 = newr + w * R;
    const uint64_t P = uint64_t(R) * (R + 1) / 2;
    uint64_t node = 0;
    for (;;) {
        if (stored(node)) {
            double* g = compact + slot_of(node) * P;
            for (uint32_t c = 0; c < R; ++c) {
                const double dc = u1[c] - u0[c];
                if (dc == 0.0) continue;  // warp-uniform
                for (uint32_t b = lane; b < R; b += 32) {
                    const double db = u1[b] - u0[b];
                    if (db != 0.0 && b < c) continue;  // pair (b, c) handled when c' = b
                    // entry (b, c): u_b dc + db u'_c  ==  u'_b u'_c - u_b u_c
                    const double D = fma(u0[b], dc, db * u1[c]);
                    if (D == 0.0) continue;
                    const uint32_t lo = b < c ? b : c, hi = b < c ? c : b;
                    atomicAdd(g + pack_index(R, lo, hi), D);
                }
            }
        }
        if (is_leaf(t, node)) break;
        uint64_t f, l;
        node_rows(t, 2 * node + 1, &f, &l);
        node = r < l ? 2 * node + 1 : 2 * node + 2;
    }
}

template <typename T>
__global__ void k_scatter_rows(T* __restrict__ U, uint32_t R, uint64_t nrows, const uint64_t* __restrict__ rows,
                               const double* __restrict__ vals) {
    const uint64_t total = nrows * R;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total; e += uint64_t(gridDim.x) * blockDim.x)
        U[rows[e / R] * R + e % R] = static_cast<T>(vals[e]);
}
template <typename T>
__global__ void k_gather_rows(const T* __restrict__ U, uint32_t R, uint64_t nrows, const uint64_t* __restrict__ rows,
                              double* __restrict__ out) {
    const uint64_t total = nrows * R;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total; e += uint64_t(gridDim.x) * blockDim.x)
        out[e] = static_cast<double>(U[rows[e / R] * R + e % R]);
}
__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = static_cast<float>(in[i]);
}
__global__ void k_f32_to_f64(const float* __restrict__ in, double* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = static_cast<double>(in[i]);
}

// Fresh Gram U^T U on the FP64 tensor cores (gram, dense_kernels.cpp:19-42), R = 8 NB <= 64:
// each warp streams 8-row blocks through registers into its own padded smem rows and
// accumulates the NT upper-triangle 8x8 tiles (A = X_p^T, B = X_q share one fragment
// load per column block); warps of a CTA are summed in order into one partial per
// CTA, partials in CTA order by k_gram_finish -- deterministic run to run.
constexpr int GRAM_WARPS = 4;
constexpr int GRAM_PARTS = 148 * 4;  // generic kernel: row chunks (partials)
template <int NB, typename T>
__global__ void __launch_bounds__(GRAM_WARPS * 32)
    k_gram_dmma(const T* __restrict__ U, uint64_t I, double* __restrict__ partial) {
    constexpr int R = 8 * NB, RS = R + 4, NT = NB * (NB + 1) / 2, EPL = R / 4;
    __shared__ __align__(16) double xs_all[GRAM_WARPS * 8 * RS];
    __shared__ double red[NT * 64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r4 = lane & 3, cq = lane >> 2;
    double* xs = xs_all + warp * 8 * RS;
    double acc[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
    const uint64_t nblk = (I + 7) / 8, lim = I * R;
    const uint64_t stride = uint64_t(gridDim.x) * GRAM_WARPS;
    double v[EPL];
    auto load = [&](uint64_t blk) {
        const uint64_t base = blk * 8 * R;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
            const uint64_t e = base + lane + 32 * i;
            v[i] = e < lim ? static_cast<double>(U[e]) : 0.0;
        }
    };
    uint64_t b = uint64_t(blockIdx.x) * GRAM_WARPS + warp;
    if (b < nblk) load(b);
    while (b < nblk) {
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
            const int e = lane + 32 * i;
            xs[(e / R) * RS + (e % R)] = v[i];
        }
        __syncwarp();
        const uint64_t bn = b + stride;
        if (bn < nblk) load(bn);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            double f[NB];
#pragma unroll
            for (int p = 0; p < NB; ++p) f[p] = xs[(4 * s + r4) * RS + 8 * p + cq];
            int t = 0;
#pragma unroll
            for (int p = 0; p < NB; ++p)
#pragma unroll
                for (int q = p; q < NB; ++q, ++t) dmma_884(acc[t][0], acc[t][1], f[p], f[q]);
        }
        __syncwarp();
        b = bn;
    }
    for (int w = 0; w < GRAM_WARPS; ++w) {  // warps summed in a fixed order
        if (warp == w) {
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int e = t * 64 + cq * 8 + 2 * r4 + j;
                    red[e] = (w == 0) ? acc[t][j] : red[e] + acc[t][j];
                }
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < NT * 64; e += blockDim.x) partial[uint64_t(blockIdx.x) * NT * 64 + e] = red[e];
}

// out (R x R) = sum of the CTA partials in CTA order, mirrored to the lower triangle
template <int NB>
__global__ void k_gram_finish(const double* __restrict__ partial, int nparts, double* __restrict__ out) {
    constexpr int R = 8 * NB, NT = NB * (NB + 1) / 2;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= NT * 64) return;
    double acc = 0.0;
    for (int c = 0; c < nparts; ++c) acc += partial[uint64_t(c) * NT * 64 + e];
    int t = e / 64, p = 0;
    while (t >= NB - p) t -= NB - p++;
    const int q = p + t, m = (e % 64) / 8, n = e % 8;
    const int a = 8 * p + m, bcol = 8 * q + n;
    out[a * R + bcol] = acc;
    if (p != q) out[bcol * R + a] = acc;
}

// generic R: per block one partial (P packed pairs), then an ordered sum
template <typename T>
__global__ void k_full_gram_part(const T* __restrict__ U, uint64_t I, uint32_t R, uint64_t rows_per_block,
                                 double* __restrict__ partial) {
    const uint64_t r0 = blockIdx.x * rows_per_block;
    const uint64_t r1 = r0 + rows_per_block < I ? r0 + rows_per_block : I;
    const uint32_t P = R * (R + 1) / 2;
    for (uint32_t k = threadIdx.x; k < P; k += blockDim.x) {
        uint32_t a, b;
        unpack_pair(R, k, a, b);
        double acc = 0.0;
        for (uint64_t i = r0; i < r1; ++i)
            acc = fma(static_cast<double>(U[i * R + a]), static_cast<double>(U[i * R + b]), acc);
        partial[uint64_t(blockIdx.x) * P + k] = acc;
    }
}
__global__ void k_full_gram_finish(const double* __restrict__ partial, int nparts, uint32_t R, double* __restrict__ out) {
    const uint32_t P = R * (R + 1) / 2;
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= P) return;
    double acc = 0.0;
    for (int c = 0; c < nparts; ++c) acc += partial[uint64_t(c) * P + k];
    uint32_t a, b;
    unpack_pair(R, k, a, b);
    out[uint64_t(a) * R + b] = acc;
    out[uint64_t(b) * R + a] = acc;
}

int sm_count_upd() { return sm_count_current(); }

template <int NB, typename T>
void launch_gram_dmma(const T* U, uint64_t I, double* out, double* partial, cudaStream_t s) {
    constexpr int NT = NB * (NB + 1) / 2;
    const uint64_t nblk = (I + 7) / 8;
    const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>((nblk + GRAM_WARPS - 1) / GRAM_WARPS,
                                                                   uint64_t(sm_count_upd()) * 4)));
    k_gram_dmma<NB, T><<<grid, GRAM_WARPS * 32, 0, s>>>(U, I, partial);
    k_gram_finish<NB><<<(NT * 64 + 255) / 256, 256, 0, s>>>(partial, grid, out);
}

template <typename T>
void launch_gram_any(const T* U, uint64_t I, uint32_t R, double* out, double* partial, cudaStream_t s) {
    switch (R) {
        case 8: return launch_gram_dmma<1, T>(U, I, out, partial, s);
        case 16: return launch_gram_dmma<2, T>(U, I, out, partial, s);
        case 24: return launch_gram_dmma<3, T>(U, I, out, partial, s);
        case 32: return launch_gram_dmma<4, T>(U, I, out, partial, s);
        case 40: return launch_gram_dmma<5, T>(U, I, out, partial, s);
        case 48: return launch_gram_dmma<6, T>(U, I, out, partial, s);
        case 56: return launch_gram_dmma<7, T>(U, I, out, partial, s);
        case 64: return launch_gram_dmma<8, T>(U, I, out, partial, s);
        default: break;
    }
    const uint64_t rpb = std::max<uint64_t>(64, (I + GRAM_PARTS - 1) / GRAM_PARTS);
    const int grid = int((I + rpb - 1) / rpb);
    const uint32_t P = R * (R + 1) / 2;
    k_full_gram_part<T><<<grid, 256, 0, s>>>(U, I, R, rpb, partial);
    k_full_gram_finish<<<(P + 255) / 256, 256, 0, s>>>(partial, grid, R, out);
}

__global__ void __launch_bounds__(256) k_patch_level(double* __restrict__ compact, uint32_t R,
                                                     const PatchItem* __restrict__ items, uint64_t nitems,
                                                     const double* __restrict__ dprev, double* __restrict__ dcur,
                                                     const double* __restrict__ oldr, const double* __restrict__ newr) {
    const int lane = threadIdx.x & 31;
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= nitems) return;
    const PatchItem it = items[w];
    const uint64_t P = uint64_t(R) * (R + 1) / 2;
    KRPG_DCHECK(it.re >= it.rb && (it.re > it.rb || it.lc >= 0 || it.rc >= 0));
    double* out = dcur + w * P;
    double* g = stored(it.node) ? compact + slot_of(it.node) * P : nullptr;
    if (it.re > it.rb) {  // leaf: its touched rows in ascending order
        for (uint32_t a = 0; a < R; ++a) {
            const uint32_t k0 = pack_index(R, a, a);
            for (uint32_t b = a + lane; b < R; b += 32) {
                double acc = 0.0;
                for (uint32_t r = it.rb; r < it.re; ++r) {
                    const double* u0 = oldr + uint64_t(r) * R;
                    const double* u1 = newr + uint64_t(r) * R;
                    // u'_a u'_b - u_a u_b  ==  u_a (u'_b - u_b) + (u'_a - u_a) u'_b
                    acc += fma(u0[a], u1[b] - u0[b], (u1[a] - u0[a]) * u1[b]);
                }
                const uint32_t k = k0 + (b - a);
                out[k] = acc;
                if (g) g[k] += acc;
            }
        }
        return;
    }
    const double* l = it.lc >= 0 ? dprev + uint64_t(it.lc) * P : nullptr;
    const double* r = it.rc >= 0 ? dprev + uint64_t(it.rc) * P : nullptr;
    for (uint64_t k = lane; k < P; k += 32) {
        const double d = l && r ? l[k] + r[k] : (l ? l[k] : r[k]);
        out[k] = d;
        if (g) g[k] += d;
    }
}

}  // namespace

void launch_tree_patch_level(double* compact, uint32_t R, const PatchItem* items, uint64_t nitems,
                             const double* delta_prev, double* delta_cur, const double* old_rows,
                             const double* new_rows, cudaStream_t s) {
    if (!nitems) return;
    k_patch_level<<<unsigned((nitems * 32 + 255) / 256), 256, 0, s>>>(compact, R, items, nitems, delta_prev,
                                                                    delta_cur, old_rows, new_rows);
}


size_t full_gram_work_doubles(uint32_t R) {
    const size_t P = size_t(R) * (R + 1) / 2;
    const size_t nt64 = size_t((R + 7) / 8) * ((R + 7) / 8 + 1) / 2 * 64;
    return std::max<size_t>(size_t(GRAM_PARTS) * P, size_t(sm_count_upd()) * 4 * nt64);
}

void launch_row_deltas(double* compact, uint64_t I, uint32_t R, uint64_t F, const uint64_t* segs, uint64_t nleaves,
                       uint64_t nrows, const uint64_t* rows, const double* old_rows, const double* new_rows,
                       cudaStream_t s) {
    if (!nrows) return;
    const Topo t = segs ? make_topo_segments(I, nleaves, segs) : make_topo(I, F ? F : R);
    const uint64_t threads = nrows * 32;
    k_row_deltas<<<unsigned((threads + 255) / 256), 256, 0, s>>>(compact, t, R, nrows, rows, old_rows, new_rows);
}

void launch_scatter_rows(void* U, uint32_t storage, uint32_t R, uint64_t nrows, const uint64_t* rows,
                         const double* new_rows, cudaStream_t s) {
    if (!nrows) return;
    if (storage == 1)
        k_scatter_rows<float><<<grid_for(nrows * R, 256), 256, 0, s>>>(static_cast<float*>(U), R, nrows, rows, new_rows);
    else
        k_scatter_rows<double><<<grid_for(nrows * R, 256), 256, 0, s>>>(static_cast<double*>(U), R, nrows, rows, new_rows);
}

void launch_gather_rows(const void* U, uint32_t storage, uint32_t R, uint64_t nrows, const uint64_t* rows,
                        double* out, cudaStream_t s) {
    if (!nrows) return;
    if (storage == 1)
        k_gather_rows<float><<<grid_for(nrows * R, 256), 256, 0, s>>>(static_cast<const float*>(U), R, nrows, rows, out);
    else
        k_gather_rows<double><<<grid_for(nrows * R, 256), 256, 0, s>>>(static_cast<const double*>(U), R, nrows, rows, out);
}

void launch_convert_f64_to_f32(const double* in, float* out, uint64_t n, cudaStream_t s) {
    if (n) k_f64_to_f32<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
}
void launch_convert_f32_to_f64(const float* in, double* out, uint64_t n, cudaStream_t s) {
    if (n) k_f32_to_f64<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
}

void launch_full_gram(const void* U, uint32_t storage, uint64_t I, uint32_t R, double* out, double* work,
                      cudaStream_t s) {
    if (storage == 1)
        launch_gram_any<float>(static_cast<const float*>(U), I, R, out, work, s);
    else
        launch_gram_any<double>(static_cast<const double*>(U), I, R, out, work, s);
}

}  // namespace krpg
