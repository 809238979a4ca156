// CP-ARLS-LEV product-of-leverage sampler (sketch.cpp:86-149) on the device.
//
// The reference, per included factor U_k (I_k x R): G+ = pinv_psd(gram(U_k)),
// p_i = u_i^T G+ u_i (quadratic_form), normalised by their sum, a cumulative table
// by a sequential running sum; then per draw d, CounterRng(seed, d) gives one
// uniform per included factor (in order) and t = lower_bound(cum, u * cum.back()),
// clamped to I - 1 (draw_from_cumulative, :19-26); probability = product of the
// p[t], row = Hadamard product of the drawn rows (:133-145).
//
// Here:
//   * k_row_leverage<NB,T>: all I_k quadratic forms on the FP64 tensor cores --
//     8 rows per warp-step (qf::block_qf_packed over the upper-triangle 8x8 tiles of
//     the packed G+, held in shared memory), rows prefetched into registers while
//     the previous block computes. HBM-bound read of U_k once (I*R*elt bytes) plus
//     I*8 bytes of output; DMMA work I*NT*128 flops;
//   * the cumulative table is a CUB inclusive scan of the unnormalised masses; the
//     draw compares cum_i >= u * cum_last (the reference's normalised comparison
//     scaled by the same total) -- equal up to summation order, boundary draws are
//     counted through the reported margin;
//   * k_lev_draws: one thread per draw, binary search per included factor;
//     k_lev_rows: one thread per (draw, column) Hadamard product in the reference's
//     factor order (bit-exact given the indices).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "krpg_device.cuh"
#include "krpg_kernels.hpp"
#include "launch_util.hpp"
#include "qf_dmma.cuh"

namespace krpg {

namespace {

template <int NB>
struct LevCfg {
    static constexpr int R = 8 * NB;
    static constexpr int P = R * (R + 1) / 2;
    static constexpr int RS = R + 4;  // padded staging row: 2 wavefronts per fragment load
    static constexpr int WARPS = NB <= 4 ? 8 : 4;
    static constexpr int EPL = R / 4;  // staged elements per lane per 8-row block
    static constexpr int GOFF = (P + 1) & ~1;
    static constexpr int SMEM = 8 * (GOFF + WARPS * 8 * RS);
};

template <int NB, typename T>
__global__ void __launch_bounds__(LevCfg<NB>::WARPS * 32)
    k_row_leverage(const T* __restrict__ U, uint64_t I, const double* __restrict__ Gp, double* __restrict__ out) {
    using C = LevCfg<NB>;
    constexpr int R = C::R;
    extern __shared__ __align__(16) double sm[];
    double* sG = sm;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* xs = sm + C::GOFF + warp * 8 * C::RS;
    for (int k = threadIdx.x; k < C::P; k += blockDim.x) sG[k] = Gp[k];
    __syncthreads();
    const qf::FragAddr<NB> fa(lane);
    const uint64_t nblk = (I + 7) / 8;
    const uint64_t stride = uint64_t(gridDim.x) * C::WARPS;
    const uint64_t lim = I * R;
    double v[C::EPL];
    auto load = [&](uint64_t blk) {
        const uint64_t base = blk * 8 * R;
#pragma unroll
        for (int i = 0; i < C::EPL; ++i) {
            const uint64_t e = base + lane + 32 * i;
            v[i] = e < lim ? static_cast<double>(U[e]) : 0.0;
        }
    };
    uint64_t b = uint64_t(blockIdx.x) * C::WARPS + warp;
    if (b < nblk) load(b);
    while (b < nblk) {
#pragma unroll
        for (int i = 0; i < C::EPL; ++i) {
            const int e = lane + 32 * i;
            xs[(e / R) * C::RS + (e % R)] = v[i];
        }
        __syncwarp();
        const uint64_t bn = b + stride;
        if (bn < nblk) load(bn);  // in flight while this block computes
        const double mass = qf::block_qf_packed<NB>(sG, fa, xs + (lane >> 2) * C::RS, lane);
        const uint64_t row = b * 8 + (lane >> 2);
        if ((lane & 3) == 0 && row < I) out[row] = mass;
        __syncwarp();
        b = bn;
    }
}

// any R: one warp per row, G+ dense (R x R) from global memory
template <typename T>
__global__ void k_row_leverage_generic(const T* __restrict__ U, uint64_t I, uint32_t R, const double* __restrict__ G,
                                       double* __restrict__ out) {
    constexpr int MAXJ = 8;  // R <= 256
    const int lane = threadIdx.x & 31;
    const uint64_t w0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t i = w0; i < I; i += nw) {
        double xb[MAXJ];
#pragma unroll
        for (int j = 0; j < MAXJ; ++j) {
            const uint32_t c = lane + 32 * j;
            xb[j] = c < R ? static_cast<double>(U[i * R + c]) : 0.0;
        }
        double acc = 0.0;
        for (uint32_t a = 0; a < R; ++a) {
            double t = 0.0;
#pragma unroll
            for (int j = 0; j < MAXJ; ++j) {
                const uint32_t c = lane + 32 * j;
                if (c < R) t = fma(G[size_t(a) * R + c], xb[j], t);
            }
            t = warp_sum(t);
            double xa = 0.0;
#pragma unroll
            for (int j = 0; j < MAXJ; ++j)
                if (int(a >> 5) == j) xa = __shfl_sync(0xffffffffu, xb[j], a & 31);
            acc = fma(xa, t, acc);
        }
        if (lane == 0) out[i] = acc;
    }
}

int sm_count_lev() { return sm_count_current(); }

template <int NB, typename T>
void launch_lev(const T* U, uint64_t I, const double* Gp, double* out, cudaStream_t s) {
    using C = LevCfg<NB>;
    auto kern = k_row_leverage<NB, T>;
    smem_optin(kern, C::SMEM);
    const int occ = occupancy(kern, C::WARPS * 32, C::SMEM);
    const uint64_t nblk = (I + 7) / 8;
    const uint64_t need = (nblk + C::WARPS - 1) / C::WARPS;
    const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(need, uint64_t(sm_count_lev()) * occ));
    kern<<<unsigned(grid), C::WARPS * 32, C::SMEM, s>>>(U, I, Gp, out);
}

template <typename T>
void launch_lev_any(const T* U, uint64_t I, uint32_t R, const double* Gp_packed, const double* G_full, double* out,
                    cudaStream_t s) {
    switch (R) {
#define KRPG_LEV_CASE(nb) \
    case 8 * nb:          \
        return launch_lev<nb, T>(U, I, Gp_packed, out, s);
        KRPG_LEV_CASE(1)
        KRPG_LEV_CASE(2)
        KRPG_LEV_CASE(3)
        KRPG_LEV_CASE(4)
        KRPG_LEV_CASE(5)
        KRPG_LEV_CASE(6)
        KRPG_LEV_CASE(7)
        KRPG_LEV_CASE(8)
        KRPG_LEV_CASE(10)
        KRPG_LEV_CASE(12)
        KRPG_LEV_CASE(16)
        KRPG_LEV_CASE(20)
#undef KRPG_LEV_CASE
        default:
            break;
    }
    const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>((I + 7) / 8, uint64_t(sm_count_lev()) * 8));
    k_row_leverage_generic<T><<<unsigned(grid), 256, 0, s>>>(U, I, R, G_full, out);
}

__global__ void k_lev_draws(LevDrawArgs a) {
    const uint64_t d = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (d >= a.J) return;
    const uint64_t key = rng_key(a.seed, a.draw_offset + d);
    double pr = 1.0, mg = HUGE_VAL;
    for (uint32_t k = 0; k < a.N; ++k) a.idx[d * a.N + k] = 0xFFFFFFFFu;
    for (uint32_t q = 0; q < a.ninc; ++q) {
        const double* c = a.cum[q];
        const uint64_t n = a.I[q];
        const double last = c[n - 1];
        const double target = rng_uniform(key, q + 1) * last;
        uint64_t lo = 0, hi = n;  // first x with c[x] >= target
        while (lo < hi) {
            const uint64_t mid = lo + ((hi - lo) >> 1);
            if (c[mid] < target)
                lo = mid + 1;
            else
                hi = mid;
        }
        const uint64_t t = lo < n - 1 ? lo : n - 1;
        mg = fmin(mg, fabs(c[t] - target) / last);
        if (t > 0) mg = fmin(mg, fabs(c[t - 1] - target) / last);
        pr *= a.p[q][t] / last;
        a.idx[d * a.N + a.inc[q]] = uint32_t(t);
    }
    if (a.prob) a.prob[d] = pr;
    if (a.margin) a.margin[d] = mg;
}

template <typename T>
__global__ void k_lev_rows(LevDrawArgs a) {
    const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= a.J * a.R) return;
    const uint64_t d = e / a.R;
    const uint32_t c = uint32_t(e - d * a.R);
    double h = 1.0;
    for (uint32_t q = 0; q < a.ninc; ++q) {
        const uint64_t t = a.idx[d * a.N + a.inc[q]];
        h *= static_cast<double>(static_cast<const T*>(a.U[q])[t * a.R + c]);
    }
    a.rows[e] = h;
}

}  // namespace

void launch_row_leverage(const void* U, uint32_t storage, uint64_t I, uint32_t R, const double* Gp_packed,
                         const double* G_full, double* out, cudaStream_t s) {
    if (!I) return;
    if (storage == 1)
        launch_lev_any<float>(static_cast<const float*>(U), I, R, Gp_packed, G_full, out, s);
    else
        launch_lev_any<double>(static_cast<const double*>(U), I, R, Gp_packed, G_full, out, s);
}

size_t lev_scan_work_bytes(uint64_t I) {
    size_t need = 0;
    cub::DeviceScan::InclusiveSum(nullptr, need, static_cast<const double*>(nullptr), static_cast<double*>(nullptr),
                                  int64_t(I));
    return need;
}

int launch_lev_scan(const double* p, double* cum, uint64_t I, void* work, size_t work_bytes, cudaStream_t s) {
    return cub::DeviceScan::InclusiveSum(work, work_bytes, p, cum, int64_t(I), s) == cudaSuccess ? 1 : -1;
}

int launch_lev_draws(const LevDrawArgs& a, cudaStream_t s) {
    if (!a.J) return 0;
    k_lev_draws<<<unsigned((a.J + 127) / 128), 128, 0, s>>>(a);
    int launches = 1;
    if (a.rows) {
        const uint64_t n = a.J * a.R;
        if (a.storage == 1)
            k_lev_rows<float><<<unsigned((n + 255) / 256), 256, 0, s>>>(a);
        else
            k_lev_rows<double><<<unsigned((n + 255) / 256), 256, 0, s>>>(a);
        ++launches;
    }
    return launches;
}

}  // namespace krpg
