// DMMA (mma.sync.m8n8k4.f64) latency / issue rate vs independent chains and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int C>
__global__ void k(int iters, double* out, long long* cyc) {
    double c[C][2];
    for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < C; ++i) dmma(c[i][0], c[i][1], a, b);
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
void run(int warps) {
    const int blocks = 148, iters = 4096;
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * blocks * 32 * warps);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    k<C><<<blocks, 32 * warps>>>(iters, out, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<C><<<blocks, 32 * warps>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c0;
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    const double dm = double(blocks) * warps * iters * C;
    printf("chains %d warps/SM %2d: %6.1f cyc per dmma per warp (chain step %6.1f cyc)  %6.2f TFLOP/s\n", C, warps,
           double(c0) / (double(iters) * C), double(c0) / iters, dm * 512 / (ms * 1e-3) / 1e12);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {1, 4, 8, 16}) {
        run<1>(w);
        run<2>(w);
        run<4>(w);
        run<8>(w);
    }
}
