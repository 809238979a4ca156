// Host-side launch helpers shared by the kernel files.
//
// The dynamic shared-memory opt-in (cudaFuncAttributeMaxDynamicSharedMemorySize) is a
// per-device-context attribute and occupancy depends on the device, so both are cached
// per (kernel, device) -- a second sampler on another GPU of the same process gets its
// own opt-in -- under a mutex (handles on different host threads may launch at once).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

namespace krpg {

inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

inline int sm_count_current() {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device());
    return n > 0 ? n : 1;
}

namespace detail {
struct LaunchCache {
    std::mutex mu;
    std::map<std::tuple<const void*, int>, int> smem;                  // (kernel, device) -> bytes opted in
    std::map<std::tuple<const void*, int, int, size_t>, int> occ;      // (kernel, device, threads, smem) -> CTAs/SM
};
inline LaunchCache& cache() {
    static LaunchCache c;
    return c;
}
}  // namespace detail

// Opt the kernel in to `bytes` of dynamic shared memory on the current device (once per device).
template <typename... A>
void smem_optin(void (*kern)(A...), size_t bytes) {
    if (bytes <= 48 * 1024) return;
    auto& c = detail::cache();
    const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), current_device());
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.smem.find(key);
    if (it != c.smem.end() && it->second >= int(bytes)) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    c.smem[key] = int(bytes);
}

// Resident CTAs per SM of the kernel on the current device (after the smem opt-in), >= 1.
template <typename... A>
int occupancy(void (*kern)(A...), int threads, size_t smem) {
    smem_optin(kern, smem);
    auto& c = detail::cache();
    const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), current_device(), threads, smem);
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.occ.find(key);
        if (it != c.occ.end()) return it->second;
    }
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, threads, smem);
    bps = bps > 0 ? bps : 1;
    std::lock_guard<std::mutex> lk(c.mu);
    c.occ[key] = bps;
    return bps;
}

}  // namespace krpg
