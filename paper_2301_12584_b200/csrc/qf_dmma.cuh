// FP64 tensor-core (DMMA m8n8k4) quadratic forms x_d^T G x_d of 8 rows at once
// against one packed symmetric matrix (fold_weights + packed_inner semantics,
// segment_tree_sampler.cpp:193-218): shared by the grouped descent
// (descent_v2.cu) and the row-leverage kernel (productlev.cu).
#pragma once

#include "ptx.cuh"

namespace krpg {
namespace qf {

// Per-lane B-fragment addressing into a packed symmetric Gram (same for every
// node): rowoff[p][s] = pack_index(row, 0) - row for row = 8p + 4s + (lane&3);
// diag[p][s] = packed index of the diagonal-tile element (mirrored below the diagonal).
template <int NB>
struct FragAddr {
    int rowoff[NB][2];
    int diag[NB][2];
    __device__ __forceinline__ explicit FragAddr(int lane) {
        constexpr int R = 8 * NB;
        const int r4 = lane & 3, cq = lane >> 2;
#pragma unroll
        for (int p = 0; p < NB; ++p)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int row = 8 * p + 4 * s + r4;
                const int col = 8 * p + cq;
                rowoff[p][s] = row * R - (row * (row - 1)) / 2 - row;
                diag[p][s] = row <= col ? rowoff[p][s] + col : col * R - (col * (col - 1)) / 2 - col + row;
            }
    }
};

// mass of the 8 X rows of a block against a packed Gram G (shared or global
// memory; B fragments are gathered per block, nothing persists in registers).
template <int NB>
__device__ __forceinline__ double block_qf_packed(const double* G, const FragAddr<NB>& fa, const double* xr,
                                                  int lane) {
    const int r4 = lane & 3, cq = lane >> 2;
    double av[NB][2];
#pragma unroll
    for (int p = 0; p < NB; ++p)
#pragma unroll
        for (int s = 0; s < 2; ++s) av[p][s] = xr ? xr[8 * p + 4 * s + r4] : 0.0;
    double y[NB][2];
#pragma unroll
    for (int q = 0; q < NB; ++q) y[q][0] = y[q][1] = 0.0;
#pragma unroll
    for (int p = 0; p < NB; ++p) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const double gd = G[fa.diag[p][s]];
            dmma_884(y[p][0], y[p][1], av[p][s], gd);
            // off-diagonal tiles count twice (folded weights): (2a) g == a (2g)
            // exactly, so the doubling is applied once to the A fragment
            const double a2 = av[p][s] + av[p][s];
#pragma unroll
            for (int q = p + 1; q < NB; ++q) {
                const double g = G[fa.rowoff[p][s] + 8 * q + cq];
                dmma_884(y[q][0], y[q][1], a2, g);
            }
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

// block_qf_packed with the A fragments already in registers (av[p][s] = x[8p+4s+(lane&3)]
// of row lane>>2, zero for invalid rows); xr (the row, nullable) for the epilogue.
// Same operation order, bit-identical result.
template <int NB>
__device__ __forceinline__ double block_qf_packed_pre(const double* G, const FragAddr<NB>& fa, const double (&av)[NB][2],
                                                      const double* xr, int lane) {
    const int r4 = lane & 3, cq = lane >> 2;
    double y[NB][2];
#pragma unroll
    for (int q = 0; q < NB; ++q) y[q][0] = y[q][1] = 0.0;
#pragma unroll
    for (int p = 0; p < NB; ++p) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const double gd = G[fa.diag[p][s]];
            dmma_884(y[p][0], y[p][1], av[p][s], gd);
            const double a2 = av[p][s] + av[p][s];
#pragma unroll
            for (int q = p + 1; q < NB; ++q) {
                const double g = G[fa.rowoff[p][s] + 8 * q + cq];
                dmma_884(y[q][0], y[q][1], a2, g);
            }
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

}  // namespace qf
}  // namespace krpg
