// The leaf-Gram kernel of the tree build in isolation (config-2 shape: 2^22 x 64 fp64):
//   usage: leaf_bench [exp] [variant] [I] [R]   (variant 1: the scattered-store kernel, the comparison reference)
// exp: timing experiments compiled in only here (1: skip the Gram stores).
#define KRPG_LEAF_BENCH 1
#include "../../paper_2301_12584_b200/csrc/tree_build.cu"

#include <cstdio>
#include <vector>

using namespace krpg;

__global__ void k_fill_rand(double* x, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        uint64_t z = i * 0x9E3779B97F4A7C15ull + 12345;
        z ^= z >> 31;
        z *= 0xBF58476D1CE4E5B9ull;
        z ^= z >> 29;
        x[i] = double(int64_t(z >> 11) - (int64_t(1) << 52)) * (1.0 / double(int64_t(1) << 52));
    }
}

int main(int argc, char** argv) {
    const int exp = argc > 1 ? std::atoi(argv[1]) : 0;
    const int variant = argc > 2 ? std::atoi(argv[2]) : 0;
    const uint64_t I = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : (1ull << 22);
    const uint32_t R = argc > 4 ? std::atoi(argv[4]) : 64, P = R * (R + 1) / 2;
    const Topo t = make_topo(I, R);
    double *U, *compact, *ta, *tb, *ref;
    uint64_t na, nb;
    tree_transient_doubles(I, R, &na, &nb, 0, 0);
    cudaMalloc(&U, I * R * 8);
    cudaMalloc(&compact, t.L * P * 8);
    cudaMalloc(&ref, t.L * P * 8);
    cudaMalloc(&ta, (na + 16) * 8);
    cudaMalloc(&tb, (nb + 16) * 8);
    k_fill_rand<<<1024, 256>>>(U, I * R);
    cudaMemcpyToSymbol(g_leaf_exp, &exp, sizeof(int));
    cudaStream_t s;
    cudaStreamCreate(&s);
    TreeBuildArgs a{};
    a.U = U;
    a.storage = 0;
    a.I = I;
    a.R = R;
    a.tbuf_a = ta;
    a.tbuf_b = tb;
    a.stream = s;
    // reference build (variant 0, no experiment)
    {
        const int zero = 0;
        cudaMemcpyToSymbol(g_leaf_exp, &zero, sizeof(int));
        a.compact = ref;
        a.leaf_variant = 1;
        launch_tree_leaves(a);
        launch_tree_levels(a);
        cudaStreamSynchronize(s);
        cudaMemcpyToSymbol(g_leaf_exp, &exp, sizeof(int));
    }
    a.compact = compact;
    a.leaf_variant = variant;
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    double leaf = 0, lev = 0;
    const int K = 5;
    for (int it = 0; it < K + 2; ++it) {
        cudaEventRecord(e0, s);
        launch_tree_leaves(a);
        cudaEventRecord(e1, s);
        launch_tree_levels(a);
        cudaEventRecord(e2, s);
        cudaEventSynchronize(e2);
        float m0, m1;
        cudaEventElapsedTime(&m0, e0, e1);
        cudaEventElapsedTime(&m1, e1, e2);
        if (it >= 2) {
            leaf += m0;
            lev += m1;
        }
    }
    const cudaError_t err = cudaGetLastError();
    // compare with the reference build
    std::vector<double> h0(size_t(t.L) * P), h1(size_t(t.L) * P);
    cudaMemcpy(h0.data(), ref, h0.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h1.data(), compact, h1.size() * 8, cudaMemcpyDeviceToHost);
    size_t diff = 0;
    double maxrel = 0;
    for (size_t i = 0; i < h0.size(); ++i) {
        if (h0[i] != h1[i]) {
            ++diff;
            const double r = std::abs(h0[i] - h1[i]) / (std::abs(h0[i]) + 1e-300);
            if (r > maxrel) maxrel = r;
        }
    }
    printf("{\"exp\": %d, \"variant\": %d, \"leaf_ms\": %.4f, \"levels_ms\": %.4f, \"total_ms\": %.4f, \"differing\": %zu, "
           "\"max_rel\": %.3g, \"err\": \"%s\"}\n",
           exp, variant, leaf / K, lev / K, (leaf + lev) / K, diff, maxrel, cudaGetErrorString(err));
    return 0;
}
