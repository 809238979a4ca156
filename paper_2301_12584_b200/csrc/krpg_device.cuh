// Device-side building blocks shared by the tree-build, descent and update
// kernels of the krpg sampler (sm_100a).
#pragma once

#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

// Checked build (make CHECKED=1 -> lib/libkrpg_checked.so): bounds / invariant checks on
// the kernels' index arithmetic (node ids, stored slots, row ranges, sorted positions,
// ring and block-list capacity). A failed check traps the kernel through a device-side
// assert, so the call returns a CUDA error; the production build compiles them away.
// This stands in for compute-sanitizer's memcheck, which is closed on the GPU pool.
#ifdef KRPG_CHECKED
#include <cassert>
#define KRPG_DCHECK(cond) assert(cond)
#else
#define KRPG_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

namespace krpg {

// ---------------------------------------------------------------------------
// CounterRng, bit-exact with /root/reference/proj/include/krplev/rng.hpp:13-48.
// uniform #c (1-based) of stream s under seed: mix(key + c * golden) >> 11.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t rng_mix(uint64_t z) {
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ull;
    z ^= z >> 33;
    return z;
}
__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t stream) {
    return rng_mix(rng_mix(seed + 0x9e3779b97f4a7c15ull) ^ rng_mix(stream + 0xbf58476d1ce4e5b9ull));
}
__host__ __device__ __forceinline__ double rng_uniform(uint64_t key, uint64_t counter) {
    const uint64_t bits = rng_mix(key + counter * 0x9e3779b97f4a7c15ull);
    return static_cast<double>(bits >> 11) * 0x1.0p-53;
}

// ---------------------------------------------------------------------------
// Complete-tree heap topology, segment_tree_sampler.cpp:111-149.
// n = 2L-1 nodes, depth d = ceil_log2(L), bottom = 2L - 2^d leaves on level d.
// Compact storage: slot 0 = root, slot s >= 1 = node 2s-1 (left children).
// ---------------------------------------------------------------------------
struct Topo {
    uint64_t I;       // rows
    uint64_t F;       // leaf capacity
    uint64_t L;       // leaves
    uint64_t n;       // nodes
    uint32_t d;       // depth
    uint64_t bottom;  // leaves on the deepest level
    const uint64_t* seg = nullptr;  // variable leaf segments: leaf l = rows [seg[l], seg[l+1])
};

__host__ __device__ __forceinline__ uint32_t ceil_log2_u64(uint64_t n) {
    uint32_t d = 0;
    while ((uint64_t{1} << d) < n) ++d;
    return d;
}

__host__ __device__ inline Topo make_topo(uint64_t I, uint64_t F) {
    Topo t;
    t.I = I;
    t.F = F;
    t.L = (I + F - 1) / F;
    t.n = 2 * t.L - 1;
    t.d = ceil_log2_u64(t.L);
    t.bottom = 2 * t.L - (uint64_t{1} << t.d);
    return t;
}

// complete tree over L leaves with explicit row segments (init_tree with arbitrary
// leaf_segments, segment_tree_sampler.cpp:111-149; from_sparse's partition)
__host__ __device__ inline Topo make_topo_segments(uint64_t I, uint64_t L, const uint64_t* seg) {
    Topo t;
    t.I = I;
    t.F = 0;
    t.L = L;
    t.n = 2 * t.L - 1;
    t.d = ceil_log2_u64(t.L);
    t.bottom = 2 * t.L - (uint64_t{1} << t.d);
    t.seg = seg;
    return t;
}

__host__ __device__ __forceinline__ bool is_leaf(const Topo& t, uint64_t v) { return 2 * v + 1 >= t.n; }
__host__ __device__ __forceinline__ uint64_t slot_of(uint64_t v) { return v == 0 ? 0 : (v + 1) / 2; }
__host__ __device__ __forceinline__ bool stored(uint64_t v) { return v == 0 || (v & 1); }

// in-order leaf index of a leaf node
__host__ __device__ __forceinline__ uint64_t leaf_index(const Topo& t, uint64_t v) {
    const uint64_t first_deep = (uint64_t{1} << t.d) - 1;
    return v >= first_deep ? v - first_deep : t.bottom + (v - (t.L - 1));
}
__host__ __device__ __forceinline__ uint64_t leaf_node(const Topo& t, uint64_t l) {
    return l < t.bottom ? (uint64_t{1} << t.d) - 1 + l : t.L - 1 + (l - t.bottom);
}
__host__ __device__ __forceinline__ uint32_t depth_of(uint64_t v) {
    uint32_t dv = 0;
    while ((uint64_t{2} << dv) - 1 <= v) ++dv;  // 2^(dv+1)-1 <= v
    return dv;
}
// row range [first, last) of any node (seg0_/seg1_ of init_tree)
__host__ __device__ inline void node_rows(const Topo& t, uint64_t v, uint64_t* first, uint64_t* last) {
    const uint32_t dv = depth_of(v);
    uint64_t lfirst, llast;
    if (dv == t.d) {
        lfirst = llast = leaf_index(t, v);
    } else {
        const uint32_t s = t.d - dv;
        const uint64_t vl = ((v + 1) << s) - 1;
        const uint64_t vr = ((v + 2) << s) - 2;
        if (vl < t.n) lfirst = vl - ((uint64_t{1} << t.d) - 1);
        else lfirst = leaf_index(t, ((v + 1) << (s - 1)) - 1);
        if (vr < t.n) llast = vr - ((uint64_t{1} << t.d) - 1);
        else llast = leaf_index(t, ((v + 2) << (s - 1)) - 2);
    }
    if (t.seg) {
        *first = t.seg[lfirst];
        *last = t.seg[llast + 1];
        return;
    }
    *first = lfirst * t.F;
    const uint64_t e = (llast + 1) * t.F;
    *last = e < t.I ? e : t.I;
}

// rows [first, last) of the in-order leaf l
__host__ __device__ __forceinline__ void leaf_rows(const Topo& t, uint64_t l, uint64_t* first, uint64_t* last) {
    if (t.seg) {
        *first = t.seg[l];
        *last = t.seg[l + 1];
        return;
    }
    *first = l * t.F;
    *last = *first + t.F < t.I ? *first + t.F : t.I;
}

// packed upper-triangle index, segment_tree_sampler.hpp:111-115 (a <= b)
__host__ __device__ __forceinline__ uint32_t pack_index(uint32_t R, uint32_t a, uint32_t b) {
    return a * R - a * (a - 1) / 2 + (b - a);
}

// inverse of pack_index: packed offset k -> (a, b), a <= b
__host__ __device__ __forceinline__ void unpack_pair(uint32_t R, uint32_t k, uint32_t& a, uint32_t& b) {
    // largest a with a*R - a(a-1)/2 <= k
    const double tr = 2.0 * R + 1.0;
    int aa = int((tr - sqrt(tr * tr - 8.0 * k)) * 0.5);
    if (aa < 0) aa = 0;
    while (aa > 0 && pack_index(R, aa, aa) > k) --aa;
    while (aa + 1 < int(R) && pack_index(R, aa + 1, aa + 1) <= k) ++aa;
    a = uint32_t(aa);
    b = k - pack_index(R, a, a) + a;
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T>
__device__ __forceinline__ double ld_elt(const T* p) {
    return static_cast<double>(__ldg(p));
}

}  // namespace krpg
