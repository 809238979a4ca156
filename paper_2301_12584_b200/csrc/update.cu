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

// fresh Gram (validate support): out (R x R, zeroed) += sum over a row chunk
template <typename T>
__global__ void k_full_gram(const T* __restrict__ U, uint64_t I, uint32_t R, uint64_t rows_per_block,
                            double* __restrict__ out) {
    const uint64_t r0 = blockIdx.x * rows_per_block;
    const uint64_t r1 = r0 + rows_per_block < I ? r0 + rows_per_block : I;
    const uint32_t P = R * (R + 1) / 2;
    for (uint32_t k = threadIdx.x; k < P; k += blockDim.x) {
        uint32_t a, b;
        unpack_pair(R, k, a, b);
        double acc = 0.0;
        for (uint64_t i = r0; i < r1; ++i)
            acc = fma(static_cast<double>(U[i * R + a]), static_cast<double>(U[i * R + b]), acc);
        atomicAdd(out + uint64_t(a) * R + b, acc);
        if (a != b) atomicAdd(out + uint64_t(b) * R + a, acc);
    }
}

}  // namespace

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

void launch_full_gram(const void* U, uint32_t storage, uint64_t I, uint32_t R, double* out, cudaStream_t s) {
    // ~4 blocks per SM whatever I is (each block: one partial Gram, then atomics)
    const uint64_t rpb = std::max<uint64_t>(64, (I + 148 * 4 - 1) / (148 * 4));
    const unsigned grid = unsigned((I + rpb - 1) / rpb);
    cudaMemsetAsync(out, 0, sizeof(double) * R * R, s);
    if (storage == 1)
        k_full_gram<float><<<grid, 256, 0, s>>>(static_cast<const float*>(U), I, R, rpb, out);
    else
        k_full_gram<double><<<grid, 256, 0, s>>>(static_cast<const double*>(U), I, R, rpb, out);
}

}  // namespace krpg
