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
//    pairs are stored contiguously in key order for the scatter;
//  * sampled right-hand side (sampled_rhs_rows, cp_als.cpp:122-145) without
//    the dense J x I_j block: each draw's fiber is found by binary search and
//    its nonzeros scattered straight into M = (SA^T SB)^T (I_j x R):
//    M[i, :] += (w_d rows_d) (w_d v), the products gram_cross forms;
//  * the solve U_j = (pinv(SA^T SA) (SA^T SB))^T row by row, then
//    normalize_columns (cp_als.cpp:39-52).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "krpg_device.cuh"
#include "krpg_kernels.hpp"

namespace krpg {

namespace {

#define STS_CK(call)                                                                          \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
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
    uint64_t dim[8], stride[8];
    uint32_t N;
};

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

unsigned grid_of(uint64_t n) { return unsigned(std::min<uint64_t>((n + 255) / 256, 148ull * 32)); }

// one warp per draw: fiber lookup (lane 0 binary search), then the fiber's
// nonzeros scattered into M with the products of gram_cross(sa, sb)
__global__ void k_sampled_rhs_scatter(const uint32_t* __restrict__ idx, uint64_t J, uint32_t N, Radix colrx,
                                      const double* __restrict__ prob, const double* __restrict__ rows, uint32_t R,
                                      const uint64_t* __restrict__ keys, uint64_t G, const uint64_t* __restrict__ ptr,
                                      const uint32_t* __restrict__ fcoord, const double* __restrict__ fval,
                                      double* __restrict__ M, int* err) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t d = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); d < J; d += warps) {
        const double q = prob[d];
        if (!(q > 0.0) || !isfinite(q)) {  // make_sampling_weights (sketch.cpp:44-47)
            if (lane == 0) atomicExch(err, 1);
            continue;
        }
        const double w = 1.0 / sqrt(static_cast<double>(J) * q);
        int64_t g = -1;
        if (lane == 0) {
            // flat index, RowOrder::Reversed (first included factor fastest) = the
            // mode-j matricization column of the drawn coordinates
            uint64_t u = 0;
            for (uint32_t k = 0; k < N; ++k) u += uint64_t(idx[d * N + k]) * colrx.stride[k];
            uint64_t lo = 0, hi = G;
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (keys[mid] < u) lo = mid + 1; else hi = mid;
            }
            if (lo < G && keys[lo] == u) g = int64_t(lo);
        }
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g < 0) continue;  // all-zero fiber
        for (uint64_t p = ptr[g]; p < ptr[g + 1]; ++p) {
            const uint64_t i = fcoord[p];
            const double sb = w * fval[p];
            for (uint32_t c = lane; c < R; c += 32) atomicAdd(M + i * R + c, (w * rows[d * R + c]) * sb);
        }
    }
}

// U[i, a] = sum_k pinv[a, k] M[i, k] (matmul(pinv, gram_cross) transposed, dense_kernels.cpp:209-223)
__global__ void k_solve_rows(const double* __restrict__ M, uint64_t I, uint32_t R, const double* __restrict__ pinv,
                             double* __restrict__ U, int staged) {
    extern __shared__ double smem_p[];  // R x R when it fits shared memory
    if (staged)
        for (uint32_t e = threadIdx.x; e < R * R; e += blockDim.x) smem_p[e] = pinv[e];
    __syncthreads();
    const double* sp = staged ? smem_p : pinv;
    const int lane = threadIdx.x & 31;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < I; i += warps) {
        const double* m = M + i * R;
        for (uint32_t a = lane; a < R; a += 32) {
            double acc = 0.0;
            for (uint32_t k = 0; k < R; ++k) acc += sp[a * R + k] * m[k];
            U[i * R + a] = acc;
        }
    }
}

__global__ void k_col_sumsq(const double* __restrict__ U, uint64_t I, uint32_t R, uint64_t rows_per_block,
                            double* __restrict__ out) {
    const uint64_t r0 = blockIdx.x * rows_per_block;
    const uint64_t r1 = r0 + rows_per_block < I ? r0 + rows_per_block : I;
    for (uint32_t c = threadIdx.x; c < R; c += blockDim.x) {
        double acc = 0.0;
        for (uint64_t i = r0; i < r1; ++i) acc += U[i * R + c] * U[i * R + c];
        atomicAdd(out + c, acc);
    }
}

__global__ void k_sqrt_inplace(double* x, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = sqrt(x[i]);
}

__global__ void k_normalize(double* __restrict__ U, uint64_t I, uint32_t R, const double* __restrict__ nrm) {
    const uint64_t total = I * R;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = uint32_t(e % R);
        const double n = nrm[c];
        if (n > 0.0)
            U[e] /= n;
        else if (e / R == c % I)  // zero column: deterministic unit basis vector (cp_als.cpp:48-50)
            U[e] = 1.0;
    }
}

}  // namespace

// ---- ingestion ----
uint64_t tensor_ingest(const uint32_t* d_coords, const double* d_vals, uint64_t nnz, uint32_t N, const uint64_t* dims,
                       uint32_t** d_coords_out, double** d_vals_out, cudaStream_t s) {
    Radix rx{};
    rx.N = N;
    uint64_t st = 1;
    for (int m = int(N) - 1; m >= 0; --m) {
        rx.dim[m] = dims[m];
        rx.stride[m] = st;
        st *= dims[m];
    }
    uint64_t *key = nullptr, *key2 = nullptr, *ukey = nullptr;
    double *val2 = nullptr, *uval = nullptr;
    uint64_t* nrun = nullptr;
    STS_CK(cudaMallocAsync(&key, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&key2, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&val2, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&ukey, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&uval, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&nrun, 8, s));
    k_linear_keys<<<grid_of(nnz), 256, 0, s>>>(d_coords, nnz, rx, key, nullptr);
    Scratch tmp;
    size_t need = 0;
    int bits = 64;
    {
        uint64_t top = st - 1;
        bits = top ? 64 - __builtin_clzll(top) : 1;
    }
    STS_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, d_vals, val2, nnz, 0, bits, s));
    STS_CK(cub::DeviceRadixSort::SortPairs(tmp.get(need), need, key, key2, d_vals, val2, nnz, 0, bits, s));
    need = 0;
    STS_CK(cub::DeviceReduce::ReduceByKey(nullptr, need, key2, ukey, val2, uval, nrun, cub::Sum(), nnz, s));
    STS_CK(cub::DeviceReduce::ReduceByKey(tmp.get(need), need, key2, ukey, val2, uval, nrun, cub::Sum(), nnz, s));
    uint64_t n = 0;
    STS_CK(cudaMemcpyAsync(&n, nrun, 8, cudaMemcpyDeviceToHost, s));
    STS_CK(cudaStreamSynchronize(s));
    STS_CK(cudaMalloc(d_coords_out, 4 * n * N));
    STS_CK(cudaMalloc(d_vals_out, 8 * n));
    k_decode<<<grid_of(n), 256, 0, s>>>(ukey, n, rx, *d_coords_out);
    STS_CK(cudaMemcpyAsync(*d_vals_out, uval, 8 * n, cudaMemcpyDeviceToDevice, s));
    for (void* p : {static_cast<void*>(key), static_cast<void*>(key2), static_cast<void*>(val2),
                    static_cast<void*>(ukey), static_cast<void*>(uval), static_cast<void*>(nrun)})
        STS_CK(cudaFreeAsync(p, s));
    STS_CK(cudaStreamSynchronize(s));
    return n;
}

// ---- fiber index of mode j ----
uint64_t fiber_index_build(const uint32_t* d_coords, const double* d_vals, uint64_t nnz, uint32_t N,
                           const uint64_t* dims, uint32_t j, uint64_t** d_keys, uint64_t** d_ptr,
                           uint32_t** d_fcoord, double** d_fval, cudaStream_t s) {
    Radix rx{};
    rx.N = N;
    uint64_t st = 1;
    for (uint32_t m = 0; m < N; ++m) {  // lowest mode fastest, mode j skipped (tensor.cpp:20-32)
        rx.dim[m] = dims[m];
        rx.stride[m] = m == j ? 0 : st;
        if (m != j) st *= dims[m];
    }
    uint64_t *key = nullptr, *key2 = nullptr, *id = nullptr, *id2 = nullptr, *cnt = nullptr, *nrun = nullptr;
    STS_CK(cudaMallocAsync(&key, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&key2, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&id, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&id2, 8 * nnz, s));
    STS_CK(cudaMallocAsync(&cnt, 8 * (nnz + 1), s));
    STS_CK(cudaMallocAsync(&nrun, 8, s));
    k_linear_keys<<<grid_of(nnz), 256, 0, s>>>(d_coords, nnz, rx, key, id);
    int bits = 1;
    {
        const uint64_t top = st - 1;
        bits = top ? 64 - __builtin_clzll(top) : 1;
    }
    Scratch tmp;
    size_t need = 0;
    STS_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, id, id2, nnz, 0, bits, s));
    STS_CK(cub::DeviceRadixSort::SortPairs(tmp.get(need), need, key, key2, id, id2, nnz, 0, bits, s));
    uint64_t* ukeys = key;  // reuse
    need = 0;
    STS_CK(cub::DeviceRunLengthEncode::Encode(nullptr, need, key2, ukeys, cnt, nrun, nnz, s));
    STS_CK(cub::DeviceRunLengthEncode::Encode(tmp.get(need), need, key2, ukeys, cnt, nrun, nnz, s));
    uint64_t G = 0;
    STS_CK(cudaMemcpyAsync(&G, nrun, 8, cudaMemcpyDeviceToHost, s));
    STS_CK(cudaStreamSynchronize(s));
    STS_CK(cudaMalloc(d_keys, 8 * std::max<uint64_t>(G, 1)));
    STS_CK(cudaMalloc(d_ptr, 8 * (G + 1)));
    STS_CK(cudaMalloc(d_fcoord, 4 * std::max<uint64_t>(nnz, 1)));
    STS_CK(cudaMalloc(d_fval, 8 * std::max<uint64_t>(nnz, 1)));
    STS_CK(cudaMemcpyAsync(*d_keys, ukeys, 8 * G, cudaMemcpyDeviceToDevice, s));
    STS_CK(cudaMemsetAsync(cnt + G, 0, 8, s));
    need = 0;
    STS_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, *d_ptr, G + 1, s));
    STS_CK(cub::DeviceScan::ExclusiveSum(tmp.get(need), need, cnt, *d_ptr, G + 1, s));
    // the fiber-ordered (coordinate j, value) pairs, from the sorted entry ids
    k_gather_fiber<<<grid_of(nnz), 256, 0, s>>>(id2, d_coords, d_vals, nnz, N, j, *d_fcoord, *d_fval);
    for (void* p : {static_cast<void*>(key), static_cast<void*>(key2), static_cast<void*>(id), static_cast<void*>(id2),
                    static_cast<void*>(cnt), static_cast<void*>(nrun)})
        STS_CK(cudaFreeAsync(p, s));
    STS_CK(cudaStreamSynchronize(s));
    return G;
}

// ---- one STS-CP step's device work ----
void launch_sampled_rhs(const uint32_t* idx, uint64_t J, uint32_t N, uint32_t j, const uint64_t* dims,
                        const double* prob, const double* rows, uint32_t R, const uint64_t* keys, uint64_t G,
                        const uint64_t* ptr, const uint32_t* fcoord, const double* fval, double* M, int* err,
                        cudaStream_t s) {
    Radix colrx{};
    colrx.N = N;
    uint64_t st = 1;
    for (uint32_t m = 0; m < N; ++m) {
        colrx.stride[m] = m == j ? 0 : st;
        if (m != j) st *= dims[m];
    }
    const unsigned grid = unsigned(std::min<uint64_t>((J + 7) / 8, 148ull * 16));
    k_sampled_rhs_scatter<<<grid, 256, 0, s>>>(idx, J, N, colrx, prob, rows, R, keys, G, ptr, fcoord, fval, M, err);
}

void launch_solve_rows(const double* M, uint64_t I, uint32_t R, const double* pinv, double* U, cudaStream_t s) {
    const size_t need = sizeof(double) * R * R;
    const bool staged = need <= 160 * 1024;  // R <= 144; larger pinv is read through L1/L2
    const size_t smem = staged ? need : 0;
    static size_t configured_for = 0;
    if (smem > 48 * 1024 && configured_for < smem) {
        cudaFuncSetAttribute(k_solve_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        configured_for = smem;
    }
    const unsigned grid = unsigned(std::min<uint64_t>((I + 7) / 8, 148ull * 8));
    k_solve_rows<<<grid, 256, smem, s>>>(M, I, R, pinv, U, staged ? 1 : 0);
}

void launch_normalize_columns(double* U, uint64_t I, uint32_t R, double* nrm, cudaStream_t s) {
    const uint64_t rpb = 256;
    const unsigned grid = unsigned((I + rpb - 1) / rpb);
    cudaMemsetAsync(nrm, 0, sizeof(double) * R, s);
    k_col_sumsq<<<grid, 64, 0, s>>>(U, I, R, rpb, nrm);
    k_sqrt_inplace<<<1, 256, 0, s>>>(nrm, R);
    k_normalize<<<grid_of(I * R), 256, 0, s>>>(U, I, R, nrm);
}

}  // namespace krpg
