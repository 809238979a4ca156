// DMMA issue rate of the descent's quadratic-form block shapes (R = 64, 8 draws per block):
//   full : all 36 upper-triangle 8x8 tiles of the Gram in registers, 8 accumulator chains
//   half : 18 tiles (column blocks {q, 7-q} for two q), 4 chains (the Gram split over 2 warps)
//   quart: 9 tiles (column blocks {q, 7-q}), 2 chains (the Gram split over 4 warps)
// A fragments come from shared memory as in the kernels. Reports DMMA per SM-cycle
// (peak 4 / 16 = 0.25) vs warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

constexpr int NB = 8, XS = 68;

// column-block sets
template <int V> struct QS;
template <> struct QS<0> { static constexpr int n = 8; __device__ static constexpr int q(int i) { return i; } };
template <> struct QS<1> { static constexpr int n = 4; __device__ static constexpr int q(int i) { return i == 0 ? 0 : i == 1 ? 7 : i == 2 ? 1 : 6; } };
template <> struct QS<2> { static constexpr int n = 2; __device__ static constexpr int q(int i) { return i == 0 ? 0 : 7; } };

template <int V, int MINB>
__global__ void __launch_bounds__(128, MINB) k(int iters, double* out, long long* cyc) {
    using Q = QS<V>;
    __shared__ double xs[4][8 * XS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = lane; i < 8 * XS; i += 32) xs[warp][i] = 1.0 + 1e-3 * i;
    __syncwarp();
    double g[NB][2][Q::n];
#pragma unroll
    for (int p = 0; p < NB; ++p)
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int j = 0; j < Q::n; ++j) g[p][s][j] = 1.0 + 1e-6 * (p * 37 + s * 11 + j + lane);
    const int r4 = lane & 3, m = lane >> 2;
    double acc = 0;
    long long t0 = clock64();
    int ndmma = 0;
    for (int it = 0; it < iters; ++it) {
        const double* xr = xs[warp] + m * XS + 2 * (it & 1);
        double y[Q::n][2];
#pragma unroll
        for (int j = 0; j < Q::n; ++j) y[j][0] = y[j][1] = 0.0;
#pragma unroll
        for (int p = 0; p < NB; ++p)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const double av = xr[8 * p + 4 * s + r4];
#pragma unroll
                for (int j = 0; j < Q::n; ++j)
                    if (Q::q(j) >= p) dmma(y[j][0], y[j][1], av, g[p][s][j]);
            }
        double part = 0;
#pragma unroll
        for (int j = 0; j < Q::n; ++j) {
            const double2 xv = *reinterpret_cast<const double2*>(xr + 8 * Q::q(j) + 2 * r4);
            part = fma(xv.x, y[j][0], part);
            part = fma(xv.y, y[j][1], part);
        }
        acc += part;
    }
    long long t1 = clock64();
#pragma unroll
    for (int p = 0; p < NB; ++p)
#pragma unroll
        for (int j = 0; j < Q::n; ++j)
            if (Q::q(j) >= p) ndmma += 2;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) * 1000 + ndmma;
}

template <int V, int MINB>
void run(int ctas_per_sm) {
    const int blocks = 148 * ctas_per_sm, iters = 2000;
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * blocks * 128);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    k<V, MINB><<<blocks, 128>>>(iters, out, cyc);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(err)); fflush(stdout); return; }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<V, MINB><<<blocks, 128>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c0;
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    const int nd = int(c0 % 1000);
    const double cycles = double(c0 / 1000);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<V, MINB>);
    const double dm = double(blocks) * 4 * iters * nd;
    printf("%-5s regs %3d  warps/SM %2d: %6.1f cyc per block per warp (%d DMMA), %.3f DMMA/SM/cyc, %6.2f TFLOP/s\n",
           V == 0 ? "full" : V == 1 ? "half" : "quart", fa.numRegs, 4 * ctas_per_sm, cycles / iters, nd,
           dm / (ms * 1e-3 * 1.965e9 * 148), dm * 512 / (ms * 1e-3) / 1e12);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) { printf("no device\n"); return 1; }
    printf("start\n"); fflush(stdout);
    run<0, 1>(1);
    run<0, 2>(2);
    run<1, 1>(1);
    run<1, 2>(2);
    run<1, 3>(3);
    run<1, 4>(4);
    run<2, 2>(2);
    run<2, 4>(4);
    run<2, 4>(6);
    run<2, 4>(8);
}
