// C-ABI layer of the B200 KRP leverage sampler (include/krpg.h).
//
// Host orchestration only: argument validation with the reference's error
// classes and messages (krp_sampler.cpp:13-15, 41-72, 84-95), the R x R setup
// math per sample call (Hadamard of Grams, pseudo-inverse, eigendecompositions
// of G_{>k}, krp_sampler.cpp:89-123), device memory ownership, and kernel
// launches on the handle's stream. There is no CPU execution path for any
// per-row or per-draw work: without a CUDA device every entry point fails.
#include "krpg.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "host_linalg.hpp"
#include "krpg_device.cuh"
#include "krpg_kernels.hpp"

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));                   \
    } while (0)

void require(bool c, const char* msg) {
    if (!c) throw std::invalid_argument(msg);
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return KRPG_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return KRPG_INVALID_ARGUMENT;
    } catch (const CudaError& e) {
        g_err = e.what();
        return KRPG_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return KRPG_RUNTIME_ERROR;
    }
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* ensure(size_t n) {
        if (n > bytes) {
            if (p) CK(cudaFree(p));
            p = nullptr;
            bytes = 0;
            CK(cudaMalloc(&p, n));
            bytes = n;
        }
        return p;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct PinBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* ensure(size_t n) {
        if (n > bytes) {
            if (p) CK(cudaFreeHost(p));
            p = nullptr;
            bytes = 0;
            CK(cudaMallocHost(&p, n));
            bytes = n;
        }
        return p;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
};

struct Factor {
    uint64_t I = 0;
    DevBuf U;     // I x R (storage dtype)
    DevBuf tree;  // L x P compact
    std::vector<double> G;  // host copy of the root Gram (R x R)
};

}  // namespace

// Device-resident sparse tensor (SparseTensorCoo, tensor.hpp:18-70): deduplicated,
// lexicographically sorted COO + per-mode fiber indexes built on first use.
struct krpg_tensor {
    int device = 0;
    uint32_t N = 0;
    std::vector<uint64_t> dims;
    uint64_t nnz = 0;
    double norm_sq = 0.0;
    DevBuf coords, values;
    std::vector<krpg::FiberIndexDev> fib;
    std::vector<bool> fib_built;
    cudaStream_t stream = nullptr;
    std::mutex mu;

    const krpg::FiberIndexDev& fiber(uint32_t j) {
        if (!fib_built[j]) {
            krpg::fiber_index_build(coords.as<uint32_t>(), values.as<double>(), nnz, N, dims.data(), j, &fib[j],
                                    stream);
            fib_built[j] = true;
        }
        return fib[j];
    }
    ~krpg_tensor() {
        coords.release();
        values.release();
        for (krpg::FiberIndexDev& F : fib) krpg::fiber_index_free(F);
        if (stream) cudaStreamDestroy(stream);
    }
};

struct krpg_sampler {
    int device = 0;
    uint32_t N = 0, R = 0, storage = 0;
    uint64_t P = 0;
    std::vector<Factor> f;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    float last_build_ms = 0.f;
    std::mutex mu;
    DevBuf tbuf, small, Q, err, sH, sIdx, sProb, sMargin, rowbuf, gstate, zbuf, stswork;
    DevBuf levtab, levwork, levg;  // product_lev_sample: per-factor tables, scan work, pseudo-inverses
    DevBuf gramwork;               // launch_full_gram partials
    double* gram_work() { return static_cast<double*>(gramwork.ensure(8 * krpg::full_gram_work_doubles(R))); }
    uint64_t sts_stats[4] = {0, 0, 0, 0};  // last STS step: draws hitting a nonzero fiber, fibers, entries
    PinBuf up[2], errh;       // operand staging is double-buffered (async calls)
    cudaEvent_t up_ev[2] = {nullptr, nullptr};
    unsigned call_no = 0;
    bool async_mode = false;  // KRPG_OPT_ASYNC: no per-call host sync; errors at krpg_sync
    bool err_zeroed = false;
    bool use_grouped = true;  // level-synchronous DMMA descent where supported
    bool prof_detail = false;  // per-kernel-type timing marks inside the descent
    bool fused_deep = true;    // deep levels + leaf scan fused (descent_v2.cu k_deep)
    uint32_t nslices = 1;      // KRPG_OPT_SLICES: concurrent draw slices of the grouped descent
    bool host_trace = false;   // KRPG_OPT_HOST_TRACE: host-side phase times on stderr
    krpg::Tuning tune;         // kernel-variant / tuning options (KRPG_OPT_EVAL_REG ...)
    // single-entry updates queued by krpg_update_entries (update_factor_entry), per factor,
    // in call order; flushed as one deterministic device patch per factor
    struct PendingEntry {
        uint64_t r;
        uint32_t c;
        double v;
    };
    std::vector<std::vector<PendingEntry>> pending;
    // per-call R x R setup (G+, rank, G_{>k} and its eigenpairs) keyed by (excluded, mode),
    // valid while the included factors' Grams are unchanged (compared bitwise)
    struct SetupEntry {
        bool valid = false;
        std::vector<std::vector<double>> grams;
        krpg::Eig ge;
        size_t rank = 0;
        std::vector<double> gp;
        std::vector<std::vector<double>> Y;
        std::vector<krpg::Eig> ye;
        DevBuf etrees;         // two-stage: the E-tree of every position (npos x R x P), same validity
        bool etrees_ok = false;
    };
    std::map<std::pair<int64_t, uint32_t>, SetupEntry> setup_cache;
    DevBuf patchbuf;
    void flush_updates() {
        for (uint32_t j = 0; j < pending.size(); ++j)
            if (!pending[j].empty()) {
                std::vector<PendingEntry> e;
                e.swap(pending[j]);
                apply_entries(j, e);
            }
    }
    void apply_entries(uint32_t j, const std::vector<PendingEntry>& E);
    std::vector<cudaStream_t> sstreams;
    std::vector<cudaEvent_t> sevents;  // [0] fork, [s] join of slice s
    cudaStream_t slice_stream(int sl) {
        while (int(sstreams.size()) < sl) {
            cudaStream_t x;
            CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
            sstreams.push_back(x);
        }
        return sstreams[sl - 1];
    }
    cudaEvent_t slice_event(int i) {
        while (int(sevents.size()) <= i) {
            cudaEvent_t x;
            CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
            sevents.push_back(x);
        }
        return sevents[i];
    }
    cudaEvent_t fork_ev() { return slice_event(0); }
    cudaEvent_t join_ev(int sl) { return slice_event(sl); }
    cudaEvent_t mark_prev = nullptr;

    // timing hook for the grouped descent: attributes the device time since the
    // previous mark to category `cat` (cat < 0 only sets the reference point)
    static void mark_cb(void* ctx, int cat) {
        auto* self = static_cast<krpg_sampler*>(ctx);
        cudaEvent_t e = self->next_event();
        CK(cudaEventRecord(e, self->stream));
        if (cat >= 0 && self->mark_prev) self->prof_pending.push_back({cat, self->mark_prev, e});
        self->mark_prev = e;
    }

    // ---- instrumentation: launch counts always, event timing when enabled ----
    bool prof_on = false;
    double prof_ms[KRPG_PROF_N] = {};
    uint64_t prof_launches[KRPG_PROF_N] = {};
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct ProfRec {
        int cat;
        cudaEvent_t a, b;
    };
    std::vector<ProfRec> prof_pending;

    cudaEvent_t next_event() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
    cudaEvent_t pbegin() {
        if (!prof_on) return nullptr;
        cudaEvent_t e = next_event();
        CK(cudaEventRecord(e, stream));
        return e;
    }
    void pend(int cat, cudaEvent_t a, int launches) {
        prof_launches[cat] += uint64_t(launches);
        if (!prof_on || !a) return;
        cudaEvent_t b = next_event();
        CK(cudaEventRecord(b, stream));
        prof_pending.push_back({cat, a, b});
    }
    void presolve() {  // call after the stream has been synchronised
        for (const ProfRec& r : prof_pending) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, r.a, r.b));
            prof_ms[r.cat] += ms;
        }
        prof_pending.clear();
        ev_used = 0;
    }

    size_t elt() const { return storage == KRPG_STORE_F32 ? 4 : 8; }

    void set_device() const { CK(cudaSetDevice(device)); }

    void build_tree(uint32_t k) {
        Factor& F = f[k];
        const krpg::Topo t = krpg::make_topo(F.I, R);
        F.tree.ensure(sizeof(double) * t.L * P);
        uint64_t na, nb;
        krpg::tree_transient_doubles(F.I, R, &na, &nb);
        double* base = static_cast<double*>(tbuf.ensure(sizeof(double) * (na + nb) + 16));
        krpg::TreeBuildArgs a{};
        a.U = F.U.p;
        a.storage = storage;
        a.I = F.I;
        a.R = R;
        a.compact = F.tree.as<double>();
        a.tbuf_a = base;
        a.tbuf_b = base + na;
        a.stream = stream;
        a.force_generic = 0;
        CK(cudaEventRecord(ev0, stream));
        cudaEvent_t t0 = pbegin();
        const int nl = krpg::launch_tree_leaves(a);
        pend(KRPG_PROF_TREE_LEAF, t0, nl);
        t0 = pbegin();
        const int nv = krpg::launch_tree_levels(a);
        pend(KRPG_PROF_TREE_LEVELS, t0, nv);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ev1, stream));
        std::vector<double> root(P);
        CK(cudaMemcpyAsync(root.data(), F.tree.p, sizeof(double) * P, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        presolve();
        CK(cudaEventElapsedTime(&last_build_ms, ev0, ev1));
        F.G.assign(size_t(R) * R, 0.0);
        krpg::unpack_upper(root.data(), R, F.G.data());
    }

    // ---- STS-CP factor update (cp_als.cpp:282-313, solver StsCp) ----
    void sts_solve(krpg_tensor& T, uint32_t j, uint64_t J, uint64_t seed, double* sigma_out);

    // ---- row-partitioned construction ----
    krpg::TreeBuildArgs tree_args(uint32_t k) {
        Factor& F = f[k];
        const krpg::Topo t = krpg::make_topo(F.I, R);
        F.tree.ensure(sizeof(double) * t.L * P);
        uint64_t na, nb;
        krpg::tree_transient_doubles(F.I, R, &na, &nb);
        double* base = static_cast<double*>(tbuf.ensure(sizeof(double) * (na + nb) + 16));
        krpg::TreeBuildArgs a{};
        a.U = F.U.p;
        a.storage = storage;
        a.I = F.I;
        a.R = R;
        a.compact = F.tree.as<double>();
        a.tbuf_a = base;
        a.tbuf_b = base + na;
        a.stream = stream;
        return a;
    }
    void check_parts(uint32_t k, uint32_t parts) const {
        require(parts >= 2 && (parts & (parts - 1)) == 0, "krpg_build_partition: parts must be a power of two >= 2");
        require(parts <= krpg::tree_positions(f[k].I, R), "krpg_build_partition: more parts than tree positions");
    }
    // stored nodes of subtree `part` on levels >= log2(parts), from U_k's rows of that subtree
    void build_partition(uint32_t k, uint32_t parts, uint32_t part, double* d_subroot) {
        check_parts(k, parts);
        require(part < parts, "krpg_build_partition: part out of range");
        krpg::TreeBuildArgs a = tree_args(k);
        a.parts = parts;
        a.part = part;
        a.subroot = d_subroot;
        cudaEvent_t t0 = pbegin();
        const int nl = krpg::launch_tree_leaves(a);
        pend(KRPG_PROF_TREE_LEAF, t0, nl);
        t0 = pbegin();
        const int nv = krpg::launch_tree_levels(a);
        if (nv < 0) throw CudaError("krpg_build_partition: device copy failed");
        pend(KRPG_PROF_TREE_LEVELS, t0, nv);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(stream));
    }
    // levels above the parts subtree roots; refreshes the cached root Gram
    void finish_partitions(uint32_t k, uint32_t parts, const double* d_subroots) {
        check_parts(k, parts);
        krpg::TreeBuildArgs a = tree_args(k);
        a.parts = parts;
        cudaEvent_t t0 = pbegin();
        const int nv = krpg::launch_tree_top(a, d_subroots);
        if (nv < 0) throw CudaError("krpg_finish_partitions: device copy failed");
        pend(KRPG_PROF_TREE_LEVELS, t0, nv);
        CK(cudaGetLastError());
        refresh_root(k);
    }
    void refresh_root(uint32_t k) {
        Factor& F = f[k];
        std::vector<double> root(P);
        CK(cudaMemcpyAsync(root.data(), F.tree.p, sizeof(double) * P, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        presolve();
        F.G.assign(size_t(R) * R, 0.0);
        krpg::unpack_upper(root.data(), R, F.G.data());
    }

    void upload_factor(uint32_t k, const double* host, uint64_t I) {
        Factor& F = f[k];
        F.I = I;
        F.U.ensure(elt() * I * R);
        if (storage == KRPG_STORE_F32) {
            std::vector<float> tmp(I * R);
            for (uint64_t e = 0; e < I * R; ++e) tmp[e] = static_cast<float>(host[e]);
            CK(cudaMemcpyAsync(F.U.p, tmp.data(), 4 * I * R, cudaMemcpyHostToDevice, stream));
            CK(cudaStreamSynchronize(stream));
        } else {
            CK(cudaMemcpyAsync(F.U.p, host, 8 * I * R, cudaMemcpyHostToDevice, stream));
            CK(cudaStreamSynchronize(stream));
        }
    }

    std::vector<uint32_t> included(int64_t excluded) const {  // krp_sampler.cpp:64-72
        if (excluded >= 0) require(uint64_t(excluded) < N, "KrpSampler: excluded index out of range");
        std::vector<uint32_t> inc;
        for (uint32_t k = 0; k < N; ++k)
            if (excluded < 0 || uint32_t(excluded) != k) inc.push_back(k);
        require(!inc.empty(), "KrpSampler: no factors left after exclusion");
        return inc;
    }

    std::vector<double> hadamard_of(const std::vector<uint32_t>& ks) const {
        std::vector<double> G(size_t(R) * R, 1.0);
        for (uint32_t k : ks) krpg::hadamard_into(G, f[k].G.data());
        return G;
    }

    void check_zero_krp() const {  // krp_sampler.cpp:55-61
        std::vector<uint32_t> all(N);
        for (uint32_t k = 0; k < N; ++k) all[k] = k;
        const std::vector<double> G = hadamard_of(all);
        double tr = 0.0;
        for (uint32_t r = 0; r < R; ++r) tr += G[size_t(r) * R + r];
        require(tr > 0.0, "KrpSampler: Khatri-Rao product is identically zero");
    }

    // host destinations of krpg_sample: the grouped path copies the last position's
    // draw slices out while the next slice computes (copy stream, stream-ordered events)
    struct HostOut {
        uint32_t* idx;
        double *prob, *rows, *margin;
        bool done;  // set by sample_device when it issued the copies itself
    };
    static bool pinned(const void* p) {
        if (!p) return true;
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    }
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t out_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // [0..3] slices, [4] join
    void copy_out_slice(const HostOut& ho, uint64_t s0, uint64_t s1, const uint32_t* d_idx, const double* d_prob,
                        const double* d_rows, const double* d_margin, int sl, bool rows_done = false) {
        if (!copy_stream) CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
        if (!out_ev[sl]) CK(cudaEventCreateWithFlags(&out_ev[sl], cudaEventDisableTiming));
        CK(cudaEventRecord(out_ev[sl], stream));
        CK(cudaStreamWaitEvent(copy_stream, out_ev[sl], 0));
        const uint64_t n = s1 - s0;
        if (ho.idx) CK(cudaMemcpyAsync(ho.idx + s0 * N, d_idx + s0 * N, 4 * n * N, cudaMemcpyDeviceToHost, copy_stream));
        if (ho.prob) CK(cudaMemcpyAsync(ho.prob + s0, d_prob + s0, 8 * n, cudaMemcpyDeviceToHost, copy_stream));
        if (ho.rows && !rows_done)
            CK(cudaMemcpyAsync(ho.rows + s0 * R, d_rows + s0 * R, 8 * n * R, cudaMemcpyDeviceToHost, copy_stream));
        if (ho.margin) CK(cudaMemcpyAsync(ho.margin + s0, d_margin + s0, 8 * n, cudaMemcpyDeviceToHost, copy_stream));
    }

    void sample_device(int64_t excluded, uint64_t J, uint64_t seed, uint64_t off, uint32_t mode,
                       uint32_t* d_idx, double* d_prob, double* d_rows, double* d_margin,
                       const HostOut* hout = nullptr) {
        require(J >= 1, "KrpSample: sample count must be positive");
        require(mode == KRPG_MODE_TWO_STAGE || mode == KRPG_MODE_ONE_STAGE, "krpg_sample: unknown mode");
        const auto trace_t0 = std::chrono::steady_clock::now();
        const std::vector<uint32_t> inc = included(excluded);
        const size_t RR = size_t(R) * R;

        // ---- R x R setup (krp_sampler.cpp:89-96, 115-122) ----
        // A pure function of the included factors' Grams: cached per (excluded, mode)
        // and reused while those Grams are bitwise unchanged (repeated calls, the
        // per-mode loop of an ALS sweep), so only the first call pays the eigensolves.
        const size_t npos = inc.size();
        SetupEntry& se = setup_cache[{excluded, mode}];
        bool hit = se.valid && se.grams.size() == npos;
        for (size_t p = 0; hit && p < npos; ++p) hit = se.grams[p] == f[inc[p]].G;
        std::vector<std::future<krpg::Eig>> fut(npos);
        if (!hit) {
            se.valid = false;
            se.etrees_ok = false;
            se.grams.clear();
            for (uint32_t k : inc) se.grams.push_back(f[k].G);
            const std::vector<double> G = hadamard_of(inc);
            se.ge = krpg::eigh_psd(G.data(), R);
            se.rank = krpg::numerical_rank(se.ge);
            if (se.rank == 0) throw std::runtime_error("KRPSample: Khatri-Rao product of included factors is zero");
            se.gp = krpg::pinv_from_eigen(se.ge);
            se.Y.assign(npos, {});
            for (size_t p = 0; p < npos; ++p) {  // downstream_gram :74-80
                se.Y[p].assign(RR, 1.0);
                krpg::hadamard_into(se.Y[p], se.gp.data());
                for (size_t q = p + 1; q < npos; ++q) krpg::hadamard_into(se.Y[p], f[inc[q]].G.data());
            }
            se.ye.assign(npos, {});
        }
        const krpg::Eig& ge = se.ge;
        const size_t rank = se.rank;
        const std::vector<double>& gp = se.gp;
        const std::vector<std::vector<double>>& Y = se.Y;
        std::vector<krpg::Eig>& ye = se.ye;
        // Eigendecompositions of G_{>k} (two-stage): position 0 on this thread,
        // the others concurrently; each position's operands are uploaded just
        // before its kernels, so the device starts on position 0 while later
        // eigensolves are still running on the host.
        if (mode == KRPG_MODE_TWO_STAGE && !hit) {
            // the last position's Y is G+ itself (no later factor): its eigenpairs are
            // those of G, inverted and reordered, no eigensolve needed
            const size_t last = npos - 1;
            for (size_t p = 1; p < last; ++p)
                fut[p] = std::async(std::launch::async, [&, p] { return krpg::eigh_psd(Y[p].data(), R); });
            if (last > 0) fut[last] = std::async(std::launch::deferred, [&] { return krpg::eig_of_pinv(ge); });
            ye[0] = last == 0 ? krpg::eig_of_pinv(ge) : krpg::eigh_psd(Y[0].data(), R);
        }

        const size_t per_pos = mode == KRPG_MODE_TWO_STAGE ? RR + R : P;
        const size_t nd = P + npos * per_pos;
        // pinned staging slot: the one used two calls ago, whose uploads have
        // long been consumed (waited on explicitly: calls may be asynchronous)
        const unsigned slot = call_no++ & 1u;
        if (!up_ev[slot]) CK(cudaEventCreateWithFlags(&up_ev[slot], cudaEventDisableTiming));
        else CK(cudaEventSynchronize(up_ev[slot]));
        double* up_h = static_cast<double*>(up[slot].ensure(sizeof(double) * nd));
        double* dsmall = static_cast<double*>(small.ensure(sizeof(double) * nd));
        auto stage_pos = [&](size_t p) {  // fill + upload position p's operands
            double* dst = up_h + P + p * per_pos;
            if (mode == KRPG_MODE_TWO_STAGE) {
                if (p > 0 && fut[p].valid()) ye[p] = fut[p].get();
                std::memcpy(dst, ye[p].vectors.data(), sizeof(double) * RR);
                std::memcpy(dst + RR, ye[p].values.data(), sizeof(double) * R);
            } else {
                const std::vector<double> yp = krpg::pack_upper(Y[p].data(), R);
                std::memcpy(dst, yp.data(), sizeof(double) * P);
            }
            CK(cudaMemcpyAsync(dsmall + P + p * per_pos, dst, sizeof(double) * per_pos, cudaMemcpyHostToDevice,
                               stream));
        };
        {
            const std::vector<double> gpp = krpg::pack_upper(gp.data(), R);
            std::memcpy(up_h, gpp.data(), sizeof(double) * P);
            CK(cudaMemcpyAsync(dsmall, up_h, sizeof(double) * P, cudaMemcpyHostToDevice, stream));
        }
        stage_pos(0);
        if (host_trace)
            std::fprintf(stderr, "krpg_sample host: position-0 operands staged after %.3f ms\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - trace_t0).count());
        struct JoinAll {  // never leave eigensolver threads behind on an exception
            std::vector<std::future<krpg::Eig>>& f;
            ~JoinAll() {
                for (auto& x : f)
                    if (x.valid()) x.wait();
            }
        } join_all{fut};

        double* H = d_rows ? d_rows : static_cast<double*>(sH.ensure(sizeof(double) * J * R));
        int* derr = static_cast<int*>(err.ensure(sizeof(int)));
        if (!async_mode || !err_zeroed) {  // async: the flag is sticky until krpg_sync reads it
            CK(cudaMemsetAsync(derr, 0, sizeof(int), stream));
            err_zeroed = true;
        }
        if (d_idx && excluded >= 0) {
            krpg::launch_set_excluded_column(d_idx, J, N, uint32_t(excluded), stream);
            prof_launches[KRPG_PROF_OTHER] += 1;
        }
        double* dQ = mode == KRPG_MODE_TWO_STAGE ? static_cast<double*>(Q.ensure(sizeof(double) * R * P)) : nullptr;

        bool grouped = use_grouped && krpg::grouped_supported(R, mode);
        if (mode == KRPG_MODE_ONE_STAGE)  // the grouped one-stage path needs trees of depth >= 1
            for (uint32_t k : inc) grouped = grouped && f[k].I > R;
        if (grouped) {
            // ---- level-synchronous grouped descent (descent_v2.cu) ----
            uint64_t nmax = 2ull * R;
            for (uint32_t k : inc) nmax = std::max<uint64_t>(nmax, krpg::make_topo(f[k].I, R).n);
            const size_t Ju = size_t(J);
            // draw slices on concurrent streams: the level kernels of one slice are
            // latency bound, so a second independent slice fills the SMs' idle phases
            const int S = (prof_on && prof_detail) ? 1 : int(std::max<uint64_t>(1, std::min<uint64_t>(nslices, J / 8192)));
            char* st = static_cast<char*>(gstate.ensure(Ju * (4 * 6 + 8 * 3) + S * nmax * 4 * 4 + 1024 * (S + 3) + 128 * S +
                                                        S * (8 * krpg::pos0_tab_doubles(R) + 128)));
            auto carve = [&](size_t bytes) {
                char* p = st;
                st += (bytes + 127) / 128 * 128;
                return p;
            };
            krpg::GroupedArgs g{};
            g.perm_a = reinterpret_cast<uint32_t*>(carve(4 * Ju));
            g.perm_b = reinterpret_cast<uint32_t*>(carve(4 * Ju));
            g.node = reinterpret_cast<uint32_t*>(carve(4 * Ju));
            g.rank = reinterpret_cast<uint32_t*>(carve(4 * Ju));
            g.nsort_a = reinterpret_cast<uint32_t*>(carve(4 * Ju));
            g.nsort_b = reinterpret_cast<uint32_t*>(carve(4 * Ju));
            g.low = reinterpret_cast<double*>(carve(8 * Ju));
            g.invc = reinterpret_cast<double*>(carve(8 * Ju));
            g.ud = reinterpret_cast<double*>(carve(8 * Ju));
            g.gstart = reinterpret_cast<uint32_t*>(carve(4 * nmax * S));
            g.gend = reinterpret_cast<uint32_t*>(carve(4 * nmax * S));
            g.cntL = reinterpret_cast<uint32_t*>(carve(4 * nmax * S));
            g.cntR = reinterpret_cast<uint32_t*>(carve(4 * nmax * S));
            double* pos0_tab = reinterpret_cast<double*>(carve(8 * krpg::pos0_tab_doubles(R) * S));
            g.pos0_tab = pos0_tab;
            g.gbar = reinterpret_cast<uint32_t*>(carve(128 * S));
            g.Zb = static_cast<double*>(zbuf.ensure(sizeof(double) * J * R));
            g.R = R;
            g.N = N;
            g.storage = storage;
            g.J = J;
            g.seed = seed;
            g.draw_offset = off;
            g.H = H;
            g.idx = d_idx;
            g.margin = d_margin;
            g.err = derr;
            g.stream = stream;
            g.fused_deep = fused_deep ? 1 : 0;
            g.tune = tune;
            if (prof_on && prof_detail) {
                g.mark = &krpg_sampler::mark_cb;
                g.mark_ctx = this;
            }
            krpg::launch_fill(H, 1.0, J * R, stream);
            prof_launches[KRPG_PROF_OTHER] += 1;
            // host outputs: the last position runs as SO draw slices one after the other,
            // each slice's probabilities and D2H copies issued as soon as it is done, so
            // all but the last slice's copies overlap the remaining compute
            // host rows written by the last deep pass itself (fused path), else output slices
            double* mapped_rows = nullptr;
            if (hout && hout->rows && S == 1 && mode == KRPG_MODE_TWO_STAGE && R <= 64 && fused_deep &&
                !(prof_on && prof_detail)) {
                if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped_rows), hout->rows, 0) != cudaSuccess) {
                    cudaGetLastError();
                    mapped_rows = nullptr;
                }
            }
            const int SO = (hout && S == 1 && J >= 16384 && !mapped_rows) ? std::max(1, std::min(4, tune.out_slices)) : 1;
            bool copied = false;
            for (size_t p = 0; p < npos; ++p) {
                const uint32_t k = inc[p];
                const double* blk = dsmall + P + p * per_pos;
                if (p > 0) stage_pos(p);
                cudaEvent_t t0 = pbegin();
                if (mode == KRPG_MODE_TWO_STAGE) {  // E-trees are cached with the setup
                    dQ = static_cast<double*>(se.etrees.ensure(sizeof(double) * npos * R * P)) + p * size_t(R) * P;
                    if (!se.etrees_ok) {
                        krpg::launch_etree_build(blk, blk + RR, f[k].tree.as<double>(), R, dQ, stream);
                        pend(KRPG_PROF_ETREE, t0, 1);
                    }
                }
                g.one_stage = mode == KRPG_MODE_ONE_STAGE ? 1 : 0;
                g.W = mode == KRPG_MODE_ONE_STAGE ? blk : nullptr;
                g.k = k;
                g.pos = uint32_t(p);
                g.I = f[k].I;
                g.Q = dQ;
                g.V = blk;
                g.Z = f[k].tree.as<double>();
                g.U = f[k].U.p;
                g.h_ones = p == 0 ? 1 : 0;  // H was just filled with ones
                g.final_rows = (mapped_rows && p + 1 == npos) ? 1 : 0;
                g.host_rows = g.final_rows ? mapped_rows : nullptr;
                t0 = pbegin();
                int nl = 0;
                if (SO > 1 && p + 1 == npos) {
                    for (int sl = 0; sl < SO; ++sl) {
                        const uint64_t s0 = J * uint64_t(sl) / SO, s1 = J * uint64_t(sl + 1) / SO;
                        krpg::GroupedArgs gs = g;
                        gs.J = s1 - s0;
                        gs.draw_offset = off + s0;
                        gs.H = H + s0 * R;
                        gs.Zb = g.Zb + s0 * R;
                        gs.idx = d_idx ? d_idx + s0 * N : nullptr;
                        gs.margin = d_margin ? d_margin + s0 : nullptr;
                        gs.perm_a = g.perm_a + s0;
                        gs.perm_b = g.perm_b + s0;
                        gs.node = g.node + s0;
                        gs.rank = g.rank + s0;
                        gs.nsort_a = g.nsort_a + s0;
                        gs.nsort_b = g.nsort_b + s0;
                        gs.low = g.low + s0;
                        gs.invc = g.invc + s0;
                        gs.ud = g.ud + s0;
                        nl += krpg::launch_position_grouped(gs);
                        if (d_prob) {
                            krpg::launch_probabilities_grouped(H + s0 * R, dsmall, R, s1 - s0, double(rank),
                                                               d_prob + s0, stream);
                            ++nl;
                        }
                        copy_out_slice(*hout, s0, s1, d_idx, d_prob, H, d_margin, sl);
                    }
                    copied = true;
                    pend(KRPG_PROF_DRAWS, t0, nl);
                    continue;
                }
                if (S > 1) CK(cudaEventRecord(fork_ev(), stream));
                for (int sl = 0; sl < S; ++sl) {
                    const uint64_t s0 = J * uint64_t(sl) / S, s1 = J * uint64_t(sl + 1) / S;
                    krpg::GroupedArgs gs = g;
                    gs.J = s1 - s0;
                    gs.draw_offset = off + s0;
                    gs.H = H + s0 * R;
                    gs.Zb = g.Zb + s0 * R;
                    gs.idx = d_idx ? d_idx + s0 * N : nullptr;
                    gs.margin = d_margin ? d_margin + s0 : nullptr;
                    gs.perm_a = g.perm_a + s0;
                    gs.perm_b = g.perm_b + s0;
                    gs.node = g.node + s0;
                    gs.rank = g.rank + s0;
                    gs.nsort_a = g.nsort_a + s0;
                    gs.nsort_b = g.nsort_b + s0;
                    gs.low = g.low + s0;
                    gs.invc = g.invc + s0;
                    gs.ud = g.ud + s0;
                    gs.gstart = g.gstart + sl * nmax;
                    gs.gend = g.gend + sl * nmax;
                    gs.cntL = g.cntL + sl * nmax;
                    gs.cntR = g.cntR + sl * nmax;
                    gs.gbar = g.gbar + sl * 32;
                    gs.pos0_tab = pos0_tab + sl * krpg::pos0_tab_doubles(R);
                    gs.stream = sl == 0 ? stream : slice_stream(sl);
                    if (sl > 0) CK(cudaStreamWaitEvent(gs.stream, fork_ev(), 0));
                    nl += krpg::launch_position_grouped(gs);
                    if (sl > 0) {
                        CK(cudaEventRecord(join_ev(sl), gs.stream));
                        CK(cudaStreamWaitEvent(stream, join_ev(sl), 0));
                    }
                }
                pend(KRPG_PROF_DRAWS, t0, nl);
            }
            CK(cudaEventRecord(up_ev[slot], stream));
            se.valid = true;  // every position's operands are complete
            if (mode == KRPG_MODE_TWO_STAGE) se.etrees_ok = true;
            if (d_prob && !copied) {
                cudaEvent_t t0 = pbegin();
                krpg::launch_probabilities_grouped(H, dsmall, R, J, double(rank), d_prob, stream);
                pend(KRPG_PROF_PROB, t0, 1);
            }
            if (hout && !copied) copy_out_slice(*hout, 0, J, d_idx, d_prob, H, d_margin, 0, mapped_rows != nullptr);
            if (hout) {  // the call's stream joins the copies (sync mode waits for them below)
                const_cast<HostOut*>(hout)->done = true;
                if (!out_ev[4]) CK(cudaEventCreateWithFlags(&out_ev[4], cudaEventDisableTiming));
                CK(cudaEventRecord(out_ev[4], copy_stream));
                CK(cudaStreamWaitEvent(stream, out_ev[4], 0));
            }
            finish_call(derr);
            return;
        }

        for (size_t p = 0; p < npos; ++p) {
            const uint32_t k = inc[p];
            const double* blk = dsmall + P + p * per_pos;
            if (p > 0) stage_pos(p);
            krpg::DrawArgs a{};
            a.R = R;
            a.N = N;
            a.k = k;
            a.pos = uint32_t(p);
            a.mode = mode;
            a.J = J;
            a.seed = seed;
            a.draw_offset = off;
            a.H = H;
            a.idx = d_idx;
            a.margin = d_margin;
            a.Z = f[k].tree.as<double>();
            a.U = f[k].U.p;
            a.storage = storage;
            a.I = f[k].I;
            a.err = derr;
            a.stream = stream;
            if (mode == KRPG_MODE_TWO_STAGE) {
                cudaEvent_t t0 = pbegin();
                krpg::launch_etree_build(blk, blk + RR, f[k].tree.as<double>(), R, dQ, stream);
                pend(KRPG_PROF_ETREE, t0, 1);
                a.Q = dQ;
                a.V = blk;
            } else {
                a.Y = blk;
            }
            cudaEvent_t t0 = pbegin();
            krpg::launch_draws(a);
            pend(KRPG_PROF_DRAWS, t0, 1);
        }
        CK(cudaEventRecord(up_ev[slot], stream));
        se.valid = true;
        if (d_prob) {
            cudaEvent_t t0 = pbegin();
            krpg::launch_probabilities(H, dsmall, R, J, double(rank), d_prob, stream);
            pend(KRPG_PROF_PROB, t0, 1);
        }
        finish_call(derr);
    }

    // end of a sample call: synchronous mode reads the device error flag now;
    // asynchronous mode (KRPG_OPT_ASYNC) leaves it for krpg_sync, and profiling
    // events for krpg_profile_read
    void finish_call(int* derr) {
        CK(cudaGetLastError());
        if (async_mode) return;
        int* eh = static_cast<int*>(errh.ensure(sizeof(int)));
        CK(cudaMemcpyAsync(eh, derr, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        presolve();
        if (*eh) throw std::runtime_error("row_sample: degenerate distribution (C <= 0)");
    }

    // synchronise and surface an error raised by any asynchronous call since the last check
    void sync_check() {
        CK(cudaStreamSynchronize(stream));
        if (!async_mode || !err.p) return;
        int flag = 0;
        CK(cudaMemcpy(&flag, err.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (flag) {
            CK(cudaMemset(err.p, 0, sizeof(int)));
            throw std::runtime_error("row_sample: degenerate distribution (C <= 0)");
        }
    }
};

void krpg_sampler::sts_solve(krpg_tensor& T, uint32_t j, uint64_t J, uint64_t seed, double* sigma_out) {
    require(T.N == N, "sts_solve: tensor order differs from the factor count");
    for (uint32_t k = 0; k < N; ++k) require(T.dims[k] == f[k].I, "sts_solve: tensor dims differ from the factors");
    require(T.device == device, "sts_solve: tensor and sampler on different devices");
    const uint64_t Ij = f[j].I;
    // 1) sampler->sample(j, J, seed) (:279-282)
    uint32_t* di = static_cast<uint32_t*>(sIdx.ensure(4 * J * N));
    double* dp = static_cast<double*>(sProb.ensure(8 * J));
    double* dr = static_cast<double*>(sH.ensure(8 * J * R));
    sample_device(int64_t(j), J, seed, 0, KRPG_MODE_TWO_STAGE, di, dp, dr, nullptr);
    sync_check();  // an asynchronous-mode sample reports its error here
    // 2) weights + SA = w o rows (:283-287, make_sampling_weights sketch.cpp:36-52); gram(sa)
    char* base = static_cast<char*>(rowbuf.ensure(8 * (J * R + J + 2 * size_t(R) * R + R + 2 * Ij * R) + 1024));
    double* sa = reinterpret_cast<double*>(base);
    double* w = sa + J * R;
    double* gs = w + J;
    double* pinv = gs + size_t(R) * R;
    double* nrm = pinv + size_t(R) * R;
    double* M = nrm + R;
    double* Unew = M + Ij * R;
    void* work = stswork.ensure(krpg::sts_work_bytes(J, R));
    int* derr = static_cast<int*>(err.ensure(sizeof(int)));
    CK(cudaMemsetAsync(derr, 0, sizeof(int), stream));
    cudaEvent_t t_sts = pbegin();
    krpg::launch_gather_sa(dp, dr, J, R, w, sa, derr, stream);
    CK(cudaMemsetAsync(gs, 0, 8 * size_t(R) * R, stream));
    krpg::launch_full_gram(sa, KRPG_STORE_F64, J, R, gs, gram_work(), stream);
    pend(KRPG_PROF_STS, t_sts, 3);
    // 3) sampled_rhs_rows + gram_cross(sa, sb), sparse (overlaps the host pinv below)
    CK(cudaStreamSynchronize(T.stream));
    const krpg::FiberIndexDev& F = T.fiber(j);
    t_sts = pbegin();
    krpg::launch_sts_rhs(di, J, N, j, T.dims.data(), dp, dr, R, F, work, M, derr, stream, tune.sts_deterministic != 0);
    pend(KRPG_PROF_STS_SCATTER, t_sts, 9);
    // 4) pinv_psd(gram(sa)) on the host (dense_kernels.cpp:207)
    std::vector<double> gh(size_t(R) * R);
    int eh = 0;
    CK(cudaMemcpyAsync(gh.data(), gs, 8 * gh.size(), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(&eh, derr, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(sts_stats, krpg::sts_stats_ptr(work, J, R), 32, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (eh) throw std::invalid_argument("make_sampling_weights: sampled index has zero probability");
    for (double x : gh) require(std::isfinite(x), "gram: non-finite entries");
    const std::vector<double> ph = krpg::pinv_from_eigen(krpg::eigh_psd(gh.data(), R));
    CK(cudaMemcpyAsync(pinv, ph.data(), 8 * ph.size(), cudaMemcpyHostToDevice, stream));
    // 5) unew = transpose(matmul(pinv, gram_cross)) (:295), normalize_columns (:309)
    // stored into U_j (sampler->update_factor(j, unew), :312-313) only once the column
    // norms are finite (update_factor validates before it mutates), then rebuild
    Factor& Fj = f[j];
    t_sts = pbegin();
    krpg::launch_solve_normalize(M, Ij, R, pinv, Unew, nrm, nullptr, storage, stream);
    std::vector<double> sg(R);
    CK(cudaMemcpyAsync(sg.data(), nrm, 8 * R, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    for (double x : sg) require(std::isfinite(x), "update_factor: invalid factor");
    krpg::launch_normalize_store(Unew, Ij, R, nrm, Fj.U.p, storage, stream);
    pend(KRPG_PROF_STS, t_sts, 4);
    build_tree(j);
    if (sigma_out) std::copy(sg.begin(), sg.end(), sigma_out);
}

// A sequence of update_factor_entry calls on factor j (krp_sampler.cpp:207-228 ->
// segment_tree_sampler.cpp:358-409), applied at once: the touched rows are read back,
// the entries applied to them on the host in call order (the sequential semantics),
// and every node on a touched row's path patched by the net u'u'^T - u u^T of its rows,
// reduced bottom-up in a fixed order (update.cu k_patch_level, no atomics).
void krpg_sampler::apply_entries(uint32_t j, const std::vector<PendingEntry>& E) {
    Factor& F = f[j];
    std::vector<uint64_t> rows;
    rows.reserve(E.size());
    for (const auto& e : E) rows.push_back(e.r);
    std::sort(rows.begin(), rows.end());
    rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
    const uint64_t nr = rows.size();
    // tree items, deepest level first
    const krpg::Topo t = krpg::make_topo(F.I, R);
    std::vector<std::vector<krpg::PatchItem>> lv(t.d + 1);
    for (uint64_t i = 0; i < nr;) {
        const uint64_t leaf = rows[i] / R;
        uint64_t e = i;
        while (e < nr && rows[e] / R == leaf) ++e;
        const uint64_t node = krpg::leaf_node(t, leaf);
        lv[krpg::depth_of(node)].push_back({node, -1, -1, uint32_t(i), uint32_t(e)});
        i = e;
    }
    for (uint32_t dd = t.d; dd >= 1; --dd) {
        auto& cur = lv[dd];
        std::sort(cur.begin(), cur.end(), [](const krpg::PatchItem& a, const krpg::PatchItem& b) { return a.node < b.node; });
        std::vector<krpg::PatchItem> par;
        for (uint64_t i = 0; i < cur.size(); ++i) {
            const uint64_t p = (cur[i].node - 1) / 2;
            if (par.empty() || par.back().node != p) par.push_back({p, -1, -1, 0, 0});
            if (cur[i].node & 1) par.back().lc = int64_t(i);
            else par.back().rc = int64_t(i);
        }
        auto& up = lv[dd - 1];  // may already hold leaves of a ragged tree (distinct nodes)
        up.insert(up.end(), par.begin(), par.end());
    }
    std::sort(lv[0].begin(), lv[0].end(), [](const krpg::PatchItem& a, const krpg::PatchItem& b) { return a.node < b.node; });
    uint64_t nitems = 0, maxl = 0;
    for (auto& l : lv) {
        nitems += l.size();
        maxl = std::max<uint64_t>(maxl, l.size());
    }
    // device scratch: rows, old, new, items, two delta buffers
    const size_t rb = 8 * nr * R;
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t o_old = al(8 * nr), o_new = o_old + al(rb), o_it = o_new + al(rb),
                 o_d0 = o_it + al(sizeof(krpg::PatchItem) * nitems), o_d1 = o_d0 + al(8 * maxl * P),
                 total = o_d1 + al(8 * maxl * P);
    char* d = static_cast<char*>(patchbuf.ensure(total));
    uint64_t* drows = reinterpret_cast<uint64_t*>(d);
    double* dold = reinterpret_cast<double*>(d + o_old);
    double* dnew = reinterpret_cast<double*>(d + o_new);
    krpg::PatchItem* dit = reinterpret_cast<krpg::PatchItem*>(d + o_it);
    double* dl[2] = {reinterpret_cast<double*>(d + o_d0), reinterpret_cast<double*>(d + o_d1)};
    CK(cudaMemcpyAsync(drows, rows.data(), 8 * nr, cudaMemcpyHostToDevice, stream));
    krpg::launch_gather_rows(F.U.p, storage, R, nr, drows, dold, stream);
    std::vector<double> oldh(nr * R);
    CK(cudaMemcpyAsync(oldh.data(), dold, rb, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    std::vector<double> newh = oldh;
    for (const auto& e : E) {  // sequential semantics of update_factor_entry
        const double val = storage == KRPG_STORE_F32 ? double(float(e.v)) : e.v;
        const uint64_t i = uint64_t(std::lower_bound(rows.begin(), rows.end(), e.r) - rows.begin());
        newh[i * R + e.c] = val;
    }
    std::vector<krpg::PatchItem> flat;
    flat.reserve(nitems);
    for (int dd = int(t.d); dd >= 0; --dd) flat.insert(flat.end(), lv[dd].begin(), lv[dd].end());
    // pinned staging would help only huge batches; these copies are stream-ordered
    CK(cudaMemcpyAsync(dnew, newh.data(), rb, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(dit, flat.data(), sizeof(krpg::PatchItem) * nitems, cudaMemcpyHostToDevice, stream));
    cudaEvent_t t0 = pbegin();
    uint64_t off = 0;
    int cur = 0, launches = 0;
    for (int dd = int(t.d); dd >= 0; --dd) {
        const uint64_t m = lv[dd].size();
        krpg::launch_tree_patch_level(F.tree.as<double>(), R, dit + off, m, dl[cur ^ 1], dl[cur], dold, dnew, stream);
        off += m;
        cur ^= 1;
        launches += m ? 1 : 0;
    }
    krpg::launch_scatter_rows(F.U.p, storage, R, nr, drows, dnew, stream);
    pend(KRPG_PROF_UPDATE, t0, launches + 1);
    prof_launches[KRPG_PROF_OTHER] += 1;  // gather of the old rows
    CK(cudaGetLastError());
    std::vector<double> root(P);
    CK(cudaMemcpyAsync(root.data(), F.tree.p, 8 * P, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));  // also keeps newh / flat alive until the copies ran
    presolve();
    krpg::unpack_upper(root.data(), R, F.G.data());
}

// Device SegmentTreeSampler (segment_tree_sampler.hpp:26-139): a standalone tree over
// U (I x R) with leaf capacity F and a fixed PSD Y (rank-1 y y^T or general).
struct krpg_segtree {
    int device = 0;
    uint64_t I = 0, F = 0;
    uint64_t L = 0;  // leaves when built over explicit segments (from_sparse), else 0
    uint32_t R = 0;
    bool rank1 = true;
    DevBuf U, tree, tbuf, yv, Yp, err, scratch, segs;
    std::vector<double> y_host, Y_host;  // as given (validation / introspection)
    std::vector<uint64_t> segs_host;     // L + 1 leaf offsets (segmented trees)
    cudaStream_t stream = nullptr;
    std::mutex mu;
    uint64_t P() const { return uint64_t(R) * (R + 1) / 2; }
    const uint64_t* segs_d() const { return L ? segs.as<uint64_t>() : nullptr; }
    krpg::Topo topo() const {  // host-side topology (segment table in host memory)
        return L ? krpg::make_topo_segments(I, L, segs_host.data()) : krpg::make_topo(I, F);
    }
    void build() {
        const krpg::Topo t = topo();
        tree.ensure(sizeof(double) * t.L * P());
        uint64_t na, nb;
        krpg::tree_transient_doubles(I, R, &na, &nb, F, L);
        double* base = static_cast<double*>(tbuf.ensure(sizeof(double) * (na + nb) + 16));
        krpg::TreeBuildArgs a{};
        a.U = U.p;
        a.storage = KRPG_STORE_F64;
        a.I = I;
        a.R = R;
        a.F = F;
        a.segs = segs_d();
        a.segs_h = L ? segs_host.data() : nullptr;
        a.nleaves = L;
        a.compact = tree.as<double>();
        a.tbuf_a = base;
        a.tbuf_b = base + na;
        a.stream = stream;
        krpg::launch_tree_leaves(a);
        if (krpg::launch_tree_levels(a) < 0) throw CudaError("segment tree: level build failed");
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(stream));
    }
    ~krpg_segtree() {
        for (DevBuf* b : {&U, &tree, &tbuf, &yv, &Yp, &err, &scratch, &segs}) b->release();
        if (stream) cudaStreamDestroy(stream);
    }
};

// ---- CP-ARLS-LEV product sampler (sketch.cpp:86-149) ----
// Factors U[k] on the device (storage dtype), G[k] = their Grams on the host
// (R x R; only included factors are read). Outputs are device pointers.
namespace {
struct LevBufs {
    DevBuf *tab, *work, *g;
};
void product_lev_device(cudaStream_t s, LevBufs b, uint32_t N, uint32_t R, uint32_t storage,
                        const std::vector<const void*>& U, const std::vector<uint64_t>& I,
                        const std::vector<const double*>& G, int64_t excluded, uint64_t J, uint64_t seed,
                        uint64_t draw_offset, uint32_t* d_idx, double* d_prob, double* d_rows, double* d_margin) {
    std::vector<uint32_t> inc;
    for (uint32_t k = 0; k < N; ++k)
        if (excluded < 0 || uint32_t(excluded) != k) inc.push_back(k);
    require(!inc.empty(), "product_lev_sample: no factors left after exclusion");
    require(inc.size() <= krpg::LEV_MAX_FACTORS, "product_lev_sample: at most 16 included factors on device");
    const uint64_t P = uint64_t(R) * (R + 1) / 2, RR = uint64_t(R) * R;
    uint64_t tab = 0;
    size_t work = 0;
    for (uint32_t k : inc) {
        if (I[k] == 0) throw std::runtime_error("product_lev_sample: zero factor");
        tab += 2 * I[k];
        work = std::max(work, krpg::lev_scan_work_bytes(I[k]));
    }
    // host: G+ = pinv_psd(G_k) (dense_kernels.cpp:207), packed and dense
    const size_t gstride = P + RR;
    std::vector<double> gh(inc.size() * gstride);
    for (size_t q = 0; q < inc.size(); ++q) {
        const std::vector<double> gp = krpg::pinv_from_eigen(krpg::eigh_psd(G[inc[q]], R));
        const std::vector<double> pk = krpg::pack_upper(gp.data(), R);
        std::copy(pk.begin(), pk.end(), gh.begin() + q * gstride);
        std::copy(gp.begin(), gp.end(), gh.begin() + q * gstride + P);
    }
    double* dg = static_cast<double*>(b.g->ensure(8 * gh.size()));
    CK(cudaMemcpyAsync(dg, gh.data(), 8 * gh.size(), cudaMemcpyHostToDevice, s));
    double* dt = static_cast<double*>(b.tab->ensure(8 * tab));
    void* dw = b.work->ensure(work + 16);
    krpg::LevDrawArgs a;
    a.N = N;
    a.ninc = uint32_t(inc.size());
    a.R = R;
    a.storage = storage;
    a.J = J;
    a.seed = seed;
    a.draw_offset = draw_offset;
    uint64_t off = 0;
    for (size_t q = 0; q < inc.size(); ++q) {
        const uint32_t k = inc[q];
        double* p = dt + off;
        double* cum = p + I[k];
        off += 2 * I[k];
        krpg::launch_row_leverage(U[k], storage, I[k], R, dg + q * gstride, dg + q * gstride + P, p, s);
        if (krpg::launch_lev_scan(p, cum, I[k], dw, work + 16, s) < 0) throw CudaError("product_lev_sample: scan failed");
        a.inc[q] = k;
        a.p[q] = p;
        a.cum[q] = cum;
        a.U[q] = U[k];
        a.I[q] = I[k];
    }
    CK(cudaGetLastError());
    // totals (the reference's "zero factor" check, :113) before any draw
    std::vector<double> tot(inc.size());
    for (size_t q = 0; q < inc.size(); ++q)
        CK(cudaMemcpyAsync(&tot[q], a.cum[q] + a.I[q] - 1, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (double t : tot)
        if (!(t > 0.0)) throw std::runtime_error("product_lev_sample: zero factor");
    a.idx = d_idx;
    a.prob = d_prob;
    a.rows = d_rows;
    a.margin = d_margin;
    krpg::launch_lev_draws(a, s);
    CK(cudaGetLastError());
}
}  // namespace

extern "C" {

const char* krpg_last_error(void) { return g_err.c_str(); }

static void segtree_create_impl(const double* U, uint64_t I, uint32_t R, uint64_t F, const uint64_t* leaf_offsets,
                                uint64_t L, const double* Y, const double* y, int device, krpg_segtree_t* out) {
    {
        *out = nullptr;
        // validation and messages as segment_tree_sampler.cpp:26-45 / :47-65
        require(I >= 1 && R >= 1, "build_sampler: empty matrix");
        for (uint64_t e = 0; e < I * R; ++e) require(std::isfinite(U[e]), "build_sampler: non-finite entries");
        if (leaf_offsets) {  // explicit partition (init_tree's leaf_segments, :111-149)
            require(L >= 1, "build_sampler: no leaf segments");
            require(leaf_offsets[0] == 0 && leaf_offsets[L] == I, "build_sampler: leaf segments must cover [0, I)");
            for (uint64_t l = 0; l < L; ++l)
                require(leaf_offsets[l] < leaf_offsets[l + 1], "build_sampler: leaf segments must be non-empty and ascending");
        } else {
            require(F >= 1, "build_sampler: leaf capacity must be positive");
        }
        require(R <= 256, "krpg: rank above 256 is not supported on device");
        require((Y != nullptr) != (y != nullptr), "SegmentTreeSampler: give exactly one of Y (R x R) or y (R)");
        if (Y) {
            for (uint64_t e = 0; e < uint64_t(R) * R; ++e) require(std::isfinite(Y[e]), "build_sampler: non-finite Y");
            (void)krpg::eigh_psd(Y, R);  // rejects asymmetric or indefinite Y
        }
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, "krpg: no such CUDA device");
        auto t = std::make_unique<krpg_segtree>();
        t->device = device;
        t->I = I;
        t->R = R;
        t->F = leaf_offsets ? R : F;
        t->rank1 = y != nullptr;
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
        CK(cudaMemcpyAsync(t->U.ensure(8 * I * R), U, 8 * I * R, cudaMemcpyHostToDevice, t->stream));
        if (leaf_offsets) {
            t->L = L;
            t->segs_host.assign(leaf_offsets, leaf_offsets + L + 1);
            CK(cudaMemcpyAsync(t->segs.ensure(8 * (L + 1)), t->segs_host.data(), 8 * (L + 1),
                               cudaMemcpyHostToDevice, t->stream));
        }
        if (y) {
            t->y_host.assign(y, y + R);
            for (double v : t->y_host) require(std::isfinite(v), "build_sampler: non-finite y");
            CK(cudaMemcpyAsync(t->yv.ensure(8 * R), t->y_host.data(), 8 * R, cudaMemcpyHostToDevice, t->stream));
        } else {
            t->Y_host.assign(Y, Y + size_t(R) * R);
            for (double v : t->Y_host) require(std::isfinite(v), "build_sampler: non-finite Y");
            const std::vector<double> yp = krpg::pack_upper(Y, R);
            CK(cudaMemcpyAsync(t->Yp.ensure(8 * yp.size()), yp.data(), 8 * yp.size(), cudaMemcpyHostToDevice,
                               t->stream));
            CK(cudaStreamSynchronize(t->stream));
        }
        t->build();
        *out = t.release();
    }
}

int krpg_segtree_create(const double* U, uint64_t I, uint32_t R, uint64_t F, const double* Y, const double* y,
                        int device, krpg_segtree_t* out) {
    return guard([&] { segtree_create_impl(U, I, R, F, nullptr, 0, Y, y, device, out); });
}

int krpg_segtree_create_segments(const double* U, uint64_t I, uint32_t R, const uint64_t* leaf_offsets, uint64_t L,
                                 const double* Y, const double* y, int device, krpg_segtree_t* out) {
    return guard([&] {
        require(leaf_offsets != nullptr, "build_sampler: null leaf offsets");
        segtree_create_impl(U, I, R, 0, leaf_offsets, L, Y, y, device, out);
    });
}

int krpg_segtree_leaf_offsets(krpg_segtree_t t, uint64_t* offsets) {
    return guard([&] {
        require(t, "krpg: null tree");
        const krpg::Topo tp = t->topo();
        for (uint64_t l = 0; l <= tp.L; ++l) {
            uint64_t f = 0, e = 0;
            if (l < tp.L) {
                krpg::leaf_rows(tp, l, &f, &e);
                offsets[l] = f;
            } else {
                offsets[l] = t->I;
            }
        }
    });
}

int krpg_segtree_node_rows(krpg_segtree_t t, uint64_t v, uint64_t* first, uint64_t* last) {
    return guard([&] {
        require(t, "krpg: null tree");
        const krpg::Topo tp = t->topo();
        require(v < tp.n, "node_segment: node out of range");
        krpg::node_rows(tp, v, first, last);
    });
}

int krpg_segtree_clone(krpg_segtree_t t, krpg_segtree_t* out) {
    return guard([&] {
        *out = nullptr;
        require(t, "krpg: null tree");
        std::lock_guard<std::mutex> lk(t->mu);
        CK(cudaSetDevice(t->device));
        auto c = std::make_unique<krpg_segtree>();
        c->device = t->device;
        c->I = t->I;
        c->R = t->R;
        c->F = t->F;
        c->L = t->L;
        c->segs_host = t->segs_host;
        c->rank1 = t->rank1;
        c->y_host = t->y_host;
        c->Y_host = t->Y_host;
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        auto dup = [&](DevBuf& dst, const DevBuf& src) {
            if (!src.p) return;
            CK(cudaMemcpyAsync(dst.ensure(src.bytes), src.p, src.bytes, cudaMemcpyDeviceToDevice, t->stream));
        };
        dup(c->U, t->U);
        dup(c->tree, t->tree);
        dup(c->yv, t->yv);
        dup(c->Yp, t->Yp);
        dup(c->segs, t->segs);
        CK(cudaStreamSynchronize(t->stream));
        *out = c.release();
    });
}

int krpg_segtree_destroy(krpg_segtree_t t) {
    return guard([&] {
        if (!t) return;
        cudaSetDevice(t->device);
        delete t;
    });
}

int krpg_segtree_shape(krpg_segtree_t t, uint64_t* leaf_count, uint64_t* node_count) {
    return guard([&] {
        require(t, "krpg: null tree");
        const krpg::Topo tp = t->topo();
        *leaf_count = tp.L;
        *node_count = tp.n;
    });
}

int krpg_segtree_node_gram(krpg_segtree_t t, uint64_t node, double* out) {
    return guard([&] {
        require(t, "krpg: null tree");
        const krpg::Topo tp = t->topo();
        require(node < tp.n, "node_gram: node out of range");
        require(node == 0 || (node & 1), "node_gram: Gram of this node is not stored (compact layout)");
        std::lock_guard<std::mutex> lk(t->mu);
        CK(cudaSetDevice(t->device));
        const uint64_t slot = node == 0 ? 0 : (node + 1) / 2;
        std::vector<double> g(t->P());
        CK(cudaMemcpy(g.data(), t->tree.as<double>() + slot * t->P(), 8 * t->P(), cudaMemcpyDeviceToHost));
        krpg::unpack_upper(g.data(), t->R, out);
    });
}

static void segtree_sample_impl(krpg_segtree_t t, const double* H, uint64_t J, uint64_t seed, uint64_t stream0,
                                uint64_t counter, const uint64_t* keys, const uint64_t* counters, uint64_t* out,
                                double* margin);

int krpg_segtree_sample(krpg_segtree_t t, const double* H, uint64_t J, uint64_t seed, uint64_t stream0,
                        uint64_t counter, uint64_t* out, double* margin) {
    return guard([&] { segtree_sample_impl(t, H, J, seed, stream0, counter, nullptr, nullptr, out, margin); });
}

int krpg_segtree_sample_keyed(krpg_segtree_t t, const double* H, uint64_t J, const uint64_t* keys,
                              const uint64_t* counters, uint64_t* out, double* margin) {
    return guard([&] {
        require(keys && counters, "row_sample: null keys / counters");
        segtree_sample_impl(t, H, J, 0, 0, 0, keys, counters, out, margin);
    });
}

static void segtree_sample_impl(krpg_segtree_t t, const double* H, uint64_t J, uint64_t seed, uint64_t stream0,
                                uint64_t counter, const uint64_t* keys, const uint64_t* counters, uint64_t* out,
                                double* margin) {
    {
        require(t, "krpg: null tree");
        require(J >= 1, "row_sample: count must be positive");
        for (uint64_t e = 0; e < J * t->R; ++e) require(std::isfinite(H[e]), "row_sample: non-finite h");
        std::lock_guard<std::mutex> lk(t->mu);
        CK(cudaSetDevice(t->device));
        char* w = static_cast<char*>(t->scratch.ensure(8 * J * t->R + 8 * J * 4 + 256));
        double* dH = reinterpret_cast<double*>(w);
        uint64_t* dout = reinterpret_cast<uint64_t*>(w + 8 * J * t->R);
        double* dm = reinterpret_cast<double*>(w + 8 * J * t->R + 8 * J);
        uint64_t* dkeys = reinterpret_cast<uint64_t*>(w + 8 * J * t->R + 16 * J);
        uint64_t* dctr = dkeys + J;
        if (keys) {
            CK(cudaMemcpyAsync(dkeys, keys, 8 * J, cudaMemcpyHostToDevice, t->stream));
            CK(cudaMemcpyAsync(dctr, counters, 8 * J, cudaMemcpyHostToDevice, t->stream));
        }
        int* derr = static_cast<int*>(t->err.ensure(sizeof(int)));
        CK(cudaMemsetAsync(derr, 0, sizeof(int), t->stream));
        CK(cudaMemcpyAsync(dH, H, 8 * J * t->R, cudaMemcpyHostToDevice, t->stream));
        krpg::DrawArgs a{};
        a.R = t->R;
        a.N = 1;
        a.mode = t->rank1 ? 2 : 3;
        a.J = J;
        a.seed = seed;
        a.draw_offset = stream0;
        a.H = dH;
        a.margin = margin ? dm : nullptr;
        a.Y = t->rank1 ? nullptr : t->Yp.as<double>();
        a.yv = t->rank1 ? t->yv.as<double>() : nullptr;
        a.Z = t->tree.as<double>();
        a.U = t->U.p;
        a.storage = KRPG_STORE_F64;
        a.I = t->I;
        a.F = t->F;
        a.segs = t->segs_d();
        a.nleaves = t->L;
        a.counter = counter;
        a.keys = keys ? dkeys : nullptr;
        a.counters = keys ? dctr : nullptr;
        a.idx64 = dout;
        a.err = derr;
        a.stream = t->stream;
        krpg::launch_draws(a);
        CK(cudaGetLastError());
        int eh = 0;
        CK(cudaMemcpyAsync(out, dout, 8 * J, cudaMemcpyDeviceToHost, t->stream));
        if (margin) CK(cudaMemcpyAsync(margin, dm, 8 * J, cudaMemcpyDeviceToHost, t->stream));
        CK(cudaMemcpyAsync(&eh, derr, sizeof(int), cudaMemcpyDeviceToHost, t->stream));
        CK(cudaStreamSynchronize(t->stream));
        if (eh) throw std::runtime_error("row_sample: degenerate distribution (C <= 0)");
    }
}

int krpg_segtree_probabilities(krpg_segtree_t t, const double* h, double* out) {
    return guard([&] {
        require(t, "krpg: null tree");
        std::lock_guard<std::mutex> lk(t->mu);
        CK(cudaSetDevice(t->device));
        char* w = static_cast<char*>(t->scratch.ensure(8 * t->R + 8 * (t->I + 1) + 256));
        double* dh = reinterpret_cast<double*>(w);
        double* dout = dh + t->R;
        CK(cudaMemcpyAsync(dh, h, 8 * t->R, cudaMemcpyHostToDevice, t->stream));
        krpg::launch_segtree_masses(t->U.as<double>(), t->I, t->R, dh, t->rank1 ? t->yv.as<double>() : nullptr,
                                    t->rank1 ? nullptr : t->Yp.as<double>(), t->tree.as<double>(), dout, t->stream);
        std::vector<double> m(t->I + 1);
        CK(cudaMemcpyAsync(m.data(), dout, 8 * m.size(), cudaMemcpyDeviceToHost, t->stream));
        CK(cudaStreamSynchronize(t->stream));
        const double C = m[t->I];
        if (!std::isfinite(C) || C <= 0.0) throw std::runtime_error("row_sample: degenerate distribution (C <= 0)");
        for (uint64_t i = 0; i < t->I; ++i) out[i] = m[i] / C;
    });
}

int krpg_segtree_update_entry(krpg_segtree_t t, uint64_t r, uint32_t c, double value) {
    return guard([&] {
        require(t, "krpg: null tree");
        require(r < t->I && c < t->R, "update_entry: entry out of range");
        require(std::isfinite(value), "update_entry: non-finite value");
        std::lock_guard<std::mutex> lk(t->mu);
        CK(cudaSetDevice(t->device));
        const uint32_t R = t->R;
        std::vector<double> oldr(R), newr;
        CK(cudaMemcpy(oldr.data(), t->U.as<double>() + r * R, 8 * R, cudaMemcpyDeviceToHost));
        newr = oldr;
        newr[c] = value;
        char* w = static_cast<char*>(t->scratch.ensure(8 * 2 * R + 64));
        double* d_old = reinterpret_cast<double*>(w);
        double* d_new = d_old + R;
        uint64_t* d_row = reinterpret_cast<uint64_t*>(d_new + R);
        CK(cudaMemcpyAsync(d_old, oldr.data(), 8 * R, cudaMemcpyHostToDevice, t->stream));
        CK(cudaMemcpyAsync(d_new, newr.data(), 8 * R, cudaMemcpyHostToDevice, t->stream));
        CK(cudaMemcpyAsync(d_row, &r, 8, cudaMemcpyHostToDevice, t->stream));
        krpg::launch_row_deltas(t->tree.as<double>(), t->I, R, t->F, t->segs_d(), t->L, 1, d_row, d_old, d_new, t->stream);
        CK(cudaMemcpyAsync(t->U.as<double>() + r * R + c, &value, 8, cudaMemcpyHostToDevice, t->stream));
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(t->stream));
    });
}

int krpg_tensor_create(const uint64_t* dims, uint32_t N, const uint32_t* coords, const double* values, uint64_t nnz,
                       int device, krpg_tensor_t* out) {
    return guard([&] {
        *out = nullptr;
        require(N >= 1, "SparseTensorCoo: no dimensions");
        require(N <= 8, "krpg_tensor_create: at most 8 modes on device");
        for (uint32_t k = 0; k < N; ++k) require(dims[k] >= 1, "SparseTensorCoo: empty mode");
        for (uint64_t e = 0; e < nnz; ++e)
            for (uint32_t k = 0; k < N; ++k)
                require(coords[e * N + k] < dims[k], "SparseTensorCoo: coordinate out of range");
        unsigned __int128 prod = 1;
        for (uint32_t k = 0; k < N; ++k) prod *= dims[k];
        require(prod <= (unsigned __int128)(~uint64_t{0}), "krpg_tensor_create: tensor index space exceeds 2^64");
        require(nnz < (uint64_t{1} << 32), "krpg_tensor_create: more than 2^32 entries");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, "krpg: no such CUDA device");
        auto t = std::make_unique<krpg_tensor>();
        t->device = device;
        t->N = N;
        t->dims.assign(dims, dims + N);
        t->fib.resize(N);
        t->fib_built.assign(N, false);
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
        if (nnz) {
            DevBuf c_in, v_in;
            CK(cudaMemcpyAsync(c_in.ensure(4 * nnz * N), coords, 4 * nnz * N, cudaMemcpyHostToDevice, t->stream));
            CK(cudaMemcpyAsync(v_in.ensure(8 * nnz), values, 8 * nnz, cudaMemcpyHostToDevice, t->stream));
            uint32_t* co = nullptr;
            double* vo = nullptr;
            t->nnz = krpg::tensor_ingest(c_in.as<uint32_t>(), v_in.as<double>(), nnz, N, dims, &co, &vo, t->stream);
            t->coords.p = co;
            t->values.p = vo;
            c_in.release();
            v_in.release();
            std::vector<double> vh(t->nnz);
            CK(cudaMemcpy(vh.data(), vo, 8 * t->nnz, cudaMemcpyDeviceToHost));
            double sq = 0.0;
            for (double x : vh) sq += x * x;
            t->norm_sq = sq;
        }
        *out = t.release();
    });
}

int krpg_tensor_create_device(const uint64_t* dims, uint32_t N, const uint32_t* d_coords, const double* d_values,
                              uint64_t nnz, int device, krpg_tensor_t* out) {
    return guard([&] {
        *out = nullptr;
        require(N >= 1, "SparseTensorCoo: no dimensions");
        require(N <= 8, "krpg_tensor_create: at most 8 modes on device");
        for (uint32_t k = 0; k < N; ++k) require(dims[k] >= 1, "SparseTensorCoo: empty mode");
        unsigned __int128 prod = 1;
        for (uint32_t k = 0; k < N; ++k) prod *= dims[k];
        require(prod <= (unsigned __int128)(~uint64_t{0}), "krpg_tensor_create: tensor index space exceeds 2^64");
        require(nnz < (uint64_t{1} << 32), "krpg_tensor_create: more than 2^32 entries");
        require(nnz == 0 || (d_coords && d_values), "krpg_tensor_create_device: null input");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, "krpg: no such CUDA device");
        auto t = std::make_unique<krpg_tensor>();
        t->device = device;
        t->N = N;
        t->dims.assign(dims, dims + N);
        t->fib.resize(N);
        t->fib_built.assign(N, false);
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
        if (nnz) {
            // the caller's producer work is complete (legacy default stream semantics do
            // not apply to our non-blocking stream)
            CK(cudaDeviceSynchronize());
            require(krpg::coords_in_range(d_coords, nnz, N, dims, t->stream), "SparseTensorCoo: coordinate out of range");
            uint32_t* co = nullptr;
            double* vo = nullptr;
            t->nnz = krpg::tensor_ingest(d_coords, d_values, nnz, N, dims, &co, &vo, t->stream);
            t->coords.p = co;
            t->values.p = vo;
            t->norm_sq = krpg::sum_of_squares(vo, t->nnz, t->stream);
        }
        *out = t.release();
    });
}

int krpg_tensor_destroy(krpg_tensor_t t) {
    return guard([&] {
        if (!t) return;
        cudaSetDevice(t->device);
        delete t;
    });
}

int krpg_tensor_info(krpg_tensor_t t, uint64_t* nnz, double* norm_sq) {
    return guard([&] {
        require(t, "krpg: null tensor");
        if (nnz) *nnz = t->nnz;
        if (norm_sq) *norm_sq = t->norm_sq;
    });
}

int krpg_tensor_entries(krpg_tensor_t t, uint32_t* coords, double* values) {
    return guard([&] {
        require(t, "krpg: null tensor");
        CK(cudaSetDevice(t->device));
        if (coords && t->nnz) CK(cudaMemcpy(coords, t->coords.p, 4 * t->nnz * t->N, cudaMemcpyDeviceToHost));
        if (values && t->nnz) CK(cudaMemcpy(values, t->values.p, 8 * t->nnz, cudaMemcpyDeviceToHost));
    });
}

int krpg_sts_last_stats(krpg_t h, uint64_t* stats) {
    return guard([&] {
        require(h, "krpg: null handle");
        for (int i = 0; i < 3; ++i) stats[i] = h->sts_stats[i];
    });
}

int krpg_sts_solve(krpg_t h, krpg_tensor_t T, uint32_t j, uint64_t J, uint64_t seed, double* sigma) {
    return guard([&] {
        require(h && T, "krpg: null handle");
        require(j < h->N, "sts_solve: mode out of range");
        require(J >= 1, "KrpSample: sample count must be positive");
        std::lock_guard<std::mutex> lk(h->mu);
        std::lock_guard<std::mutex> lt(T->mu);
        h->set_device();
        h->flush_updates();
        h->sts_solve(*T, j, J, seed, sigma);
    });
}

int krpg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

static void validate_shapes(const uint64_t* I, uint32_t N, uint32_t R, uint32_t storage) {
    require(N >= 1, "KrpSampler: factor list is empty");
    require(R >= 1, "KrpSampler: empty factor");
    for (uint32_t k = 0; k < N; ++k) require(I[k] >= 1, "KrpSampler: empty factor");
    require(R <= 256, "krpg: rank above 256 is not supported on device");
    require(storage == KRPG_STORE_F64 || storage == KRPG_STORE_F32, "krpg: unknown storage type");
}

int krpg_create(const double* const* factors, const uint64_t* I, uint32_t N, uint32_t R, uint32_t storage,
                int device, krpg_t* out) {
    return guard([&] {
        *out = nullptr;
        validate_shapes(I, N, R, storage);
        for (uint32_t k = 0; k < N; ++k)
            for (uint64_t e = 0; e < I[k] * R; ++e)
                require(std::isfinite(factors[k][e]), "KrpSampler: non-finite factor entries");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, "krpg: no such CUDA device");
        auto* h = new krpg_sampler();
        try {
            h->device = device;
            h->N = N;
            h->R = R;
            h->storage = storage;
            h->P = uint64_t(R) * (R + 1) / 2;
            h->set_device();
            CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
            CK(cudaEventCreate(&h->ev0));
            CK(cudaEventCreate(&h->ev1));
            h->f.resize(N);
            h->pending.resize(N);
            for (uint32_t k = 0; k < N; ++k) {
                h->upload_factor(k, factors[k], I[k]);
                h->build_tree(k);
            }
            h->check_zero_krp();
        } catch (...) {
            krpg_destroy(h);
            throw;
        }
        *out = h;
    });
}

int krpg_create_device(const void* const* dev_factors, const uint64_t* I, uint32_t N, uint32_t R,
                       uint32_t storage, int device, krpg_t* out) {
    return guard([&] {
        *out = nullptr;
        validate_shapes(I, N, R, storage);
        auto* h = new krpg_sampler();
        try {
            h->device = device;
            h->N = N;
            h->R = R;
            h->storage = storage;
            h->P = uint64_t(R) * (R + 1) / 2;
            h->set_device();
            CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
            CK(cudaEventCreate(&h->ev0));
            CK(cudaEventCreate(&h->ev1));
            h->f.resize(N);
            h->pending.resize(N);
            for (uint32_t k = 0; k < N; ++k) {
                Factor& F = h->f[k];
                F.I = I[k];
                F.U.ensure(h->elt() * I[k] * R);
                CK(cudaMemcpyAsync(F.U.p, dev_factors[k], h->elt() * I[k] * R, cudaMemcpyDeviceToDevice, h->stream));
                h->build_tree(k);
            }
            for (uint32_t k = 0; k < N; ++k)
                for (double v : h->f[k].G) require(std::isfinite(v), "KrpSampler: non-finite factor entries");
            h->check_zero_krp();
        } catch (...) {
            krpg_destroy(h);
            throw;
        }
        *out = h;
    });
}

int krpg_destroy(krpg_t h) {
    if (!h) return KRPG_OK;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (Factor& F : h->f) {
        F.U.release();
        F.tree.release();
    }
    for (DevBuf* b : {&h->tbuf, &h->small, &h->Q, &h->err, &h->sH, &h->sIdx, &h->sProb, &h->sMargin, &h->rowbuf, &h->stswork,
                      &h->gstate, &h->zbuf, &h->levtab, &h->levwork, &h->levg, &h->gramwork})
        b->release();
    for (int i = 0; i < 2; ++i) {
        h->up[i].release();
        if (h->up_ev[i]) cudaEventDestroy(h->up_ev[i]);
    }
    h->errh.release();
    h->patchbuf.release();
    for (auto& kv : h->setup_cache) kv.second.etrees.release();
    for (cudaEvent_t e : h->out_ev)
        if (e) cudaEventDestroy(e);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    for (cudaStream_t x : h->sstreams) cudaStreamDestroy(x);
    for (cudaEvent_t x : h->sevents) cudaEventDestroy(x);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return KRPG_OK;
}

int krpg_info(krpg_t h, uint32_t* N, uint32_t* R, uint64_t* I) {
    return guard([&] {
        require(h, "krpg: null handle");
        if (N) *N = h->N;
        if (R) *R = h->R;
        if (I)
            for (uint32_t k = 0; k < h->N; ++k) I[k] = h->f[k].I;
    });
}

int krpg_factor_gram(krpg_t h, uint32_t j, double* out) {
    return guard([&] {
        require(h && j < h->N, "factor_gram: index out of range");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        std::memcpy(out, h->f[j].G.data(), sizeof(double) * h->R * h->R);
    });
}

int krpg_factor(krpg_t h, uint32_t j, double* out) {
    return guard([&] {
        require(h && j < h->N, "factor: index out of range");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        const uint64_t n = h->f[j].I * h->R;
        if (h->storage == KRPG_STORE_F32) {
            double* tmp = static_cast<double*>(h->rowbuf.ensure(8 * n));
            krpg::launch_convert_f32_to_f64(h->f[j].U.as<float>(), tmp, n, h->stream);
            CK(cudaMemcpyAsync(out, tmp, 8 * n, cudaMemcpyDeviceToHost, h->stream));
        } else {
            CK(cudaMemcpyAsync(out, h->f[j].U.p, 8 * n, cudaMemcpyDeviceToHost, h->stream));
        }
        CK(cudaStreamSynchronize(h->stream));
    });
}

int krpg_tree_shape(krpg_t h, uint32_t j, uint64_t* leaf_count, uint64_t* node_count) {
    return guard([&] {
        require(h && j < h->N, "tree: index out of range");
        const krpg::Topo t = krpg::make_topo(h->f[j].I, h->R);
        if (leaf_count) *leaf_count = t.L;
        if (node_count) *node_count = t.n;
    });
}

int krpg_node_gram(krpg_t h, uint32_t j, uint64_t node, double* out) {
    return guard([&] {
        require(h && j < h->N, "tree: index out of range");
        const krpg::Topo t = krpg::make_topo(h->f[j].I, h->R);
        require(node < t.n, "node_gram: node out of range");
        require(krpg::stored(node), "node_gram: partial Gram not stored at this node");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        std::vector<double> p(h->P);
        CK(cudaMemcpyAsync(p.data(), h->f[j].tree.as<double>() + krpg::slot_of(node) * h->P, 8 * h->P,
                           cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        krpg::unpack_upper(p.data(), h->R, out);
    });
}

int krpg_tree_grams(krpg_t h, uint32_t j, double* out) {
    return guard([&] {
        require(h && j < h->N, "tree: index out of range");
        const krpg::Topo t = krpg::make_topo(h->f[j].I, h->R);
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        CK(cudaMemcpyAsync(out, h->f[j].tree.p, 8 * t.L * h->P, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int krpg_sample_device(krpg_t h, int64_t excluded, uint64_t J, uint64_t seed, uint64_t draw_offset,
                       uint32_t mode, uint32_t* d_idx, double* d_prob, double* d_rows, double* d_margin) {
    return guard([&] {
        require(h, "krpg: null handle");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        h->sample_device(excluded, J, seed, draw_offset, mode, d_idx, d_prob, d_rows, d_margin);
    });
}

int krpg_sample(krpg_t h, int64_t excluded, uint64_t J, uint64_t seed, uint64_t draw_offset, uint32_t mode,
                uint32_t* idx, double* prob, double* rows, double* margin) {
    return guard([&] {
        require(h, "krpg: null handle");
        require(J >= 1, "KrpSample: sample count must be positive");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        uint32_t* di = idx ? static_cast<uint32_t*>(h->sIdx.ensure(4 * J * h->N)) : nullptr;
        double* dp = prob ? static_cast<double*>(h->sProb.ensure(8 * J)) : nullptr;
        double* dr = static_cast<double*>(h->sH.ensure(8 * J * h->R));
        double* dm = margin ? static_cast<double*>(h->sMargin.ensure(8 * J)) : nullptr;
        const bool trace = h->host_trace;
        const auto t0 = std::chrono::steady_clock::now();
        // page-locked destinations: the copies are pipelined with the last position's
        // compute inside sample_device; pageable ones are copied after it
        krpg_sampler::HostOut ho{idx, prob, rows, margin, false};
        const bool pipe = krpg_sampler::pinned(idx) && krpg_sampler::pinned(prob) &&
                          krpg_sampler::pinned(rows) && krpg_sampler::pinned(margin);
        h->sample_device(excluded, J, seed, draw_offset, mode, di, dp, dr, dm, pipe ? &ho : nullptr);
        const auto t1 = std::chrono::steady_clock::now();
        if (!ho.done) {
            if (idx) CK(cudaMemcpyAsync(idx, di, 4 * J * h->N, cudaMemcpyDeviceToHost, h->stream));
            if (prob) CK(cudaMemcpyAsync(prob, dp, 8 * J, cudaMemcpyDeviceToHost, h->stream));
            if (rows) CK(cudaMemcpyAsync(rows, dr, 8 * J * h->R, cudaMemcpyDeviceToHost, h->stream));
            if (margin) CK(cudaMemcpyAsync(margin, dm, 8 * J, cudaMemcpyDeviceToHost, h->stream));
        }
        h->sync_check();
        if (trace) {
            const auto t2 = std::chrono::steady_clock::now();
            std::fprintf(stderr, "krpg_sample host: setup+launch %.3f ms, wait %.3f ms\n",
                         std::chrono::duration<double, std::milli>(t1 - t0).count(),
                         std::chrono::duration<double, std::milli>(t2 - t1).count());
        }
    });
}

int krpg_product_lev_sample(krpg_t h, int64_t excluded, uint64_t J, uint64_t seed, uint64_t draw_offset,
                            uint32_t* idx, double* prob, double* rows, double* margin) {
    return guard([&] {
        require(h, "krpg: null handle");
        require(J >= 1, "product_lev_sample: J must be positive");
        if (excluded >= 0) require(uint64_t(excluded) < h->N, "product_lev_sample: excluded index out of range");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        h->sync_check();  // drain async calls before the synchronous path
        std::vector<const void*> U(h->N);
        std::vector<uint64_t> I(h->N);
        std::vector<const double*> G(h->N);
        for (uint32_t k = 0; k < h->N; ++k) {
            U[k] = h->f[k].U.p;
            I[k] = h->f[k].I;
            G[k] = h->f[k].G.data();
        }
        uint32_t* di = static_cast<uint32_t*>(h->sIdx.ensure(4 * J * h->N));
        double* dp = prob ? static_cast<double*>(h->sProb.ensure(8 * J)) : nullptr;
        double* dr = rows ? static_cast<double*>(h->sH.ensure(8 * J * h->R)) : nullptr;
        double* dm = margin ? static_cast<double*>(h->sMargin.ensure(8 * J)) : nullptr;
        cudaEvent_t t0 = h->pbegin();
        product_lev_device(h->stream, {&h->levtab, &h->levwork, &h->levg}, h->N, h->R, h->storage, U, I, G, excluded,
                           J, seed, draw_offset, di, dp, dr, dm);
        h->pend(KRPG_PROF_OTHER, t0, 0);
        if (idx) CK(cudaMemcpyAsync(idx, di, 4 * J * h->N, cudaMemcpyDeviceToHost, h->stream));
        if (prob) CK(cudaMemcpyAsync(prob, dp, 8 * J, cudaMemcpyDeviceToHost, h->stream));
        if (rows) CK(cudaMemcpyAsync(rows, dr, 8 * J * h->R, cudaMemcpyDeviceToHost, h->stream));
        if (margin) CK(cudaMemcpyAsync(margin, dm, 8 * J, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (h->prof_on) h->presolve();
    });
}

int krpg_product_lev_sample_factors(const double* const* factors, const uint64_t* I, uint32_t N, uint32_t R,
                                    int64_t excluded, uint64_t J, uint64_t seed, int device, uint32_t* idx,
                                    double* prob, double* rows, double* margin) {
    return guard([&] {
        // validation and messages as sketch.cpp:89-100
        require(N >= 1, "product_lev_sample: factor list is empty");
        require(J >= 1, "product_lev_sample: J must be positive");
        if (excluded >= 0) require(uint64_t(excluded) < N, "product_lev_sample: excluded index out of range");
        require(R >= 1 && R <= 256, "krpg: rank must be in [1, 256] on device");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, "krpg: no such CUDA device");
        CK(cudaSetDevice(device));
        cudaStream_t s = nullptr;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        std::vector<DevBuf> dU(N);
        DevBuf tab, work, g, gram, gwork, o_idx, o_prob, o_rows, o_m;
        auto cleanup = [&] {
            cudaStreamSynchronize(s);
            for (DevBuf& b : dU) b.release();
            for (DevBuf* b : {&tab, &work, &g, &gram, &gwork, &o_idx, &o_prob, &o_rows, &o_m}) b->release();
            cudaStreamDestroy(s);
        };
        try {
            std::vector<const void*> U(N, nullptr);
            std::vector<std::vector<double>> Gh(N);
            std::vector<const double*> G(N, nullptr);
            double* dgram = static_cast<double*>(gram.ensure(8 * size_t(R) * R));
            double* gw = static_cast<double*>(gwork.ensure(8 * krpg::full_gram_work_doubles(R)));
            for (uint32_t k = 0; k < N; ++k) {
                if (excluded >= 0 && uint32_t(excluded) == k) continue;
                if (I[k] == 0) throw std::runtime_error("product_lev_sample: zero factor");
                U[k] = dU[k].ensure(8 * I[k] * R);
                CK(cudaMemcpyAsync(dU[k].p, factors[k], 8 * I[k] * R, cudaMemcpyHostToDevice, s));
                // gram(U) (dense_kernels.cpp:19-42) on the device
                krpg::launch_full_gram(U[k], KRPG_STORE_F64, I[k], R, dgram, gw, s);
                Gh[k].resize(size_t(R) * R);
                CK(cudaMemcpyAsync(Gh[k].data(), dgram, 8 * size_t(R) * R, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                G[k] = Gh[k].data();
            }
            std::vector<uint64_t> Iv(I, I + N);
            uint32_t* di = static_cast<uint32_t*>(o_idx.ensure(4 * J * N));
            double* dp = static_cast<double*>(o_prob.ensure(8 * J));
            double* dr = static_cast<double*>(o_rows.ensure(8 * J * R));
            double* dm = margin ? static_cast<double*>(o_m.ensure(8 * J)) : nullptr;
            product_lev_device(s, {&tab, &work, &g}, N, R, KRPG_STORE_F64, U, Iv, G, excluded, J, seed, 0, di, dp, dr,
                               dm);
            if (idx) CK(cudaMemcpyAsync(idx, di, 4 * J * N, cudaMemcpyDeviceToHost, s));
            if (prob) CK(cudaMemcpyAsync(prob, dp, 8 * J, cudaMemcpyDeviceToHost, s));
            if (rows) CK(cudaMemcpyAsync(rows, dr, 8 * J * R, cudaMemcpyDeviceToHost, s));
            if (margin) CK(cudaMemcpyAsync(margin, dm, 8 * J, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

int krpg_leverage_scores(krpg_t h, uint32_t j, double* out) {
    return guard([&] {
        require(h && j < h->N, "leverage_scores: index out of range");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        h->sync_check();
        const uint32_t R = h->R;
        const uint64_t P = uint64_t(R) * (R + 1) / 2, I = h->f[j].I;
        const std::vector<double> gp = krpg::pinv_from_eigen(krpg::eigh_psd(h->f[j].G.data(), R));
        std::vector<double> gh = krpg::pack_upper(gp.data(), R);
        gh.insert(gh.end(), gp.begin(), gp.end());
        double* dg = static_cast<double*>(h->levg.ensure(8 * gh.size()));
        CK(cudaMemcpyAsync(dg, gh.data(), 8 * gh.size(), cudaMemcpyHostToDevice, h->stream));
        double* dp = static_cast<double*>(h->levtab.ensure(8 * I));
        krpg::launch_row_leverage(h->f[j].U.p, h->storage, I, R, dg, dg + P, dp, h->stream);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, dp, 8 * I, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int krpg_sync(krpg_t h) {
    return guard([&] {
        require(h, "krpg: null handle");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        h->sync_check();
    });
}

void* krpg_stream(krpg_t h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int krpg_conditional(krpg_t h, int64_t excluded, uint32_t k, const double* hist, double* probs,
                     double* mixture) {
    return guard([&] {
        require(h, "krpg: null handle");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        const uint32_t R = h->R;
        const size_t RR = size_t(R) * R;
        const std::vector<uint32_t> inc = h->included(excluded);
        size_t pos = inc.size();
        for (size_t p = 0; p < inc.size(); ++p)
            if (inc[p] == k) pos = p;
        require(pos < inc.size(), "conditional: factor k is not included");
        const std::vector<double> G = h->hadamard_of(inc);
        const std::vector<double> gp = krpg::pinv_from_eigen(krpg::eigh_psd(G.data(), R));
        std::vector<double> gk(RR, 1.0);
        krpg::hadamard_into(gk, gp.data());
        for (size_t q = pos + 1; q < inc.size(); ++q) krpg::hadamard_into(gk, h->f[inc[q]].G.data());
        const krpg::Eig eig = krpg::eigh_psd(gk.data(), R);
        std::vector<double> hc(RR, 1.0);
        krpg::hadamard_into(hc, h->f[k].G.data());
        krpg::hadamard_into(hc, gk.data());
        const double C = krpg::quadratic_form(hist, hc.data(), R, hist);
        if (!(C > 0.0)) throw std::runtime_error("conditional: zero normalizer");
        std::vector<double> HT(RR);
        for (uint32_t u = 0; u < R; ++u)
            for (uint32_t c = 0; c < R; ++c) HT[size_t(u) * R + c] = hist[c] * eig.vectors[size_t(c) * R + u];
        double* d = static_cast<double*>(h->small.ensure(sizeof(double) * (RR + 2 * R)));
        double* dHT = d;
        double* dN = d + RR;
        double* dW = dN + R;
        const uint64_t I = h->f[k].I;
        double* dP = static_cast<double*>(h->sProb.ensure(8 * I));
        CK(cudaMemcpyAsync(dHT, HT.data(), 8 * RR, cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemsetAsync(dN, 0, 8 * R, h->stream));
        krpg::launch_conditional_norms(h->f[k].U.p, h->storage, I, R, dHT, dN, h->stream);
        std::vector<double> norms(R), w(R, 0.0);
        CK(cudaMemcpyAsync(norms.data(), dN, 8 * R, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        for (uint32_t u = 0; u < R; ++u) {
            if (eig.values[u] == 0.0 || norms[u] == 0.0) continue;
            w[u] = eig.values[u] * norms[u] / C;
        }
        CK(cudaMemcpyAsync(dW, w.data(), 8 * R, cudaMemcpyHostToDevice, h->stream));
        krpg::launch_conditional_probs(h->f[k].U.p, h->storage, I, R, dHT, dW, dN, dP, h->stream);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(probs, dP, 8 * I, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        std::memcpy(mixture, w.data(), 8 * R);
    });
}

int krpg_update_factor(krpg_t h, uint32_t j, const double* U, uint64_t I) {
    return guard([&] {
        require(h && j < h->N, "update_factor: index out of range");
        require(I >= 1, "update_factor: invalid factor");
        for (uint64_t e = 0; e < I * h->R; ++e) require(std::isfinite(U[e]), "update_factor: invalid factor");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        h->upload_factor(j, U, I);
        h->build_tree(j);
    });
}

int krpg_update_factor_device(krpg_t h, uint32_t j, const void* dU, uint64_t I) {
    return guard([&] {
        require(h && j < h->N, "update_factor: index out of range");
        require(I >= 1 && dU, "update_factor: invalid factor");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        // validate before mutating (krp_sampler.cpp:198-205): the new factor and its tree
        // are built aside and swapped in only when the root Gram is finite (a non-finite
        // entry makes its row's diagonal, hence the root, non-finite)
        Factor nf;
        nf.I = I;
        nf.U.ensure(h->elt() * I * h->R);
        CK(cudaMemcpyAsync(nf.U.p, dU, h->elt() * I * h->R, cudaMemcpyDeviceToDevice, h->stream));
        std::swap(h->f[j], nf);
        try {
            h->build_tree(j);
            for (double x : h->f[j].G) require(std::isfinite(x), "update_factor: invalid factor");
        } catch (...) {
            std::swap(h->f[j], nf);
            CK(cudaStreamSynchronize(h->stream));
            nf.U.release();
            nf.tree.release();
            throw;
        }
        nf.U.release();
        nf.tree.release();
    });
}

int krpg_rebuild(krpg_t h, uint32_t j) {
    return guard([&] {
        require(h && j < h->N, "rebuild: index out of range");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        h->build_tree(j);
    });
}

int krpg_tree_device(krpg_t h, uint32_t j, double** d_tree, uint64_t* slots) {
    return guard([&] {
        require(h && j < h->N, "krpg_tree_device: index out of range");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        *d_tree = h->f[j].tree.as<double>();
        *slots = krpg::make_topo(h->f[j].I, h->R).L;
    });
}

int krpg_factor_device(krpg_t h, uint32_t j, void** d_U) {
    return guard([&] {
        require(h && j < h->N, "krpg_factor_device: index out of range");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        *d_U = h->f[j].U.p;
    });
}

int krpg_build_partition(krpg_t h, uint32_t j, uint32_t parts, uint32_t part, double* d_subroot) {
    return guard([&] {
        require(h && j < h->N, "krpg_build_partition: index out of range");
        require(d_subroot, "krpg_build_partition: null subroot buffer");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        h->build_partition(j, parts, part, d_subroot);
    });
}

int krpg_finish_partitions(krpg_t h, uint32_t j, uint32_t parts, const double* d_subroots) {
    return guard([&] {
        require(h && j < h->N, "krpg_finish_partitions: index out of range");
        require(d_subroots, "krpg_finish_partitions: null subroot buffer");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        h->finish_partitions(j, parts, d_subroots);
    });
}

int krpg_partition_rows(uint64_t I, uint32_t R, uint32_t parts, uint32_t part, uint64_t* first, uint64_t* last) {
    return guard([&] {
        require(I >= 1 && R >= 1, "krpg_partition_rows: empty factor");
        require(parts >= 1 && (parts & (parts - 1)) == 0 && part < parts, "krpg_partition_rows: bad partition");
        require(parts <= krpg::tree_positions(I, R), "krpg_partition_rows: more parts than tree positions");
        krpg::tree_partition_rows(I, R, parts, part, first, last);
    });
}

int krpg_update_entries(krpg_t h, uint32_t j, const uint64_t* r, const uint32_t* c, const double* v, uint64_t n) {
    return guard([&] {
        require(h && j < h->N, "update_factor_entry: index out of range");
        const uint32_t R = h->R;
        for (uint64_t e = 0; e < n; ++e) {
            require(r[e] < h->f[j].I && c[e] < R, "update_factor_entry: entry out of range");
            require(std::isfinite(v[e]), "update_factor_entry: non-finite value");
        }
        if (n == 0) return;
        std::lock_guard<std::mutex> lk(h->mu);
        // queued: applied as one device patch before the next call that reads this
        // handle's factors, trees or Grams (krpg_sampler::flush_updates)
        auto& q = h->pending[j];  // amortised growth: per-entry calls append one at a time
        for (uint64_t e = 0; e < n; ++e) q.push_back({r[e], c[e], v[e]});
    });
}

int krpg_validate(krpg_t h, double tol) {
    return guard([&] {
        require(h, "krpg: null handle");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        const uint32_t R = h->R;
        double* d = static_cast<double*>(h->small.ensure(8 * size_t(R) * R));
        std::vector<double> fresh(size_t(R) * R), root(h->P), G(size_t(R) * R);
        for (uint32_t j = 0; j < h->N; ++j) {
            krpg::launch_full_gram(h->f[j].U.p, h->storage, h->f[j].I, R, d, h->gram_work(), h->stream);
            CK(cudaMemcpyAsync(fresh.data(), d, 8 * size_t(R) * R, cudaMemcpyDeviceToHost, h->stream));
            CK(cudaMemcpyAsync(root.data(), h->f[j].tree.p, 8 * h->P, cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            krpg::unpack_upper(root.data(), R, G.data());
            for (uint32_t a = 0; a < R; ++a)
                for (uint32_t b = 0; b < R; ++b) {
                    const double scale = std::sqrt(std::abs(fresh[a * R + a] * fresh[b * R + b]));
                    const double lim = tol * std::max(scale, 1e-300);
                    if (std::abs(fresh[a * R + b] - G[a * R + b]) > lim)
                        throw std::runtime_error("KrpSampler::validate: tree root Gram drifted");
                    if (std::abs(fresh[a * R + b] - h->f[j].G[a * R + b]) > lim)
                        throw std::runtime_error("KrpSampler::validate: cached Gram drifted");
                }
        }
    });
}

int krpg_gather_sa_device(krpg_t h, uint64_t J, const double* d_prob, const double* d_rows, double* d_weights,
                          double* d_sa) {
    return guard([&] {
        require(h, "krpg: null handle");
        require(J >= 1, "make_sampling_weights: J must be positive");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        h->flush_updates();
        int* derr = static_cast<int*>(h->err.ensure(sizeof(int)));
        CK(cudaMemsetAsync(derr, 0, sizeof(int), h->stream));
        krpg::launch_gather_sa(d_prob, d_rows, J, h->R, d_weights, d_sa, derr, h->stream);
        CK(cudaGetLastError());
        int* eh = static_cast<int*>(h->errh.ensure(sizeof(int)));
        CK(cudaMemcpyAsync(eh, derr, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (*eh) throw std::invalid_argument("make_sampling_weights: sampled index has zero probability");
    });
}

int krpg_last_build_ms(krpg_t h, float* ms) {
    return guard([&] {
        require(h, "krpg: null handle");
        *ms = h->last_build_ms;
    });
}

int krpg_profile_enable(krpg_t h, int on) {
    return guard([&] {
        require(h, "krpg: null handle");
        std::lock_guard<std::mutex> lk(h->mu);
        h->prof_on = on != 0;
    });
}

int krpg_profile_read(krpg_t h, double* ms, uint64_t* launches, int reset) {
    return guard([&] {
        require(h, "krpg: null handle");
        std::lock_guard<std::mutex> lk(h->mu);
        h->set_device();
        CK(cudaStreamSynchronize(h->stream));  // resolve events of asynchronous calls
        h->presolve();
        for (int c = 0; c < KRPG_PROF_N; ++c) {
            if (ms) ms[c] = h->prof_ms[c];
            if (launches) launches[c] = h->prof_launches[c];
            if (reset) {
                h->prof_ms[c] = 0.0;
                h->prof_launches[c] = 0;
            }
        }
    });
}

int krpg_set_option(krpg_t h, int option, int64_t value) {
    return guard([&] {
        require(h, "krpg: null handle");
        std::lock_guard<std::mutex> lk(h->mu);
        if (option == KRPG_OPT_GROUPED_DESCENT)
            h->use_grouped = value != 0;
        else if (option == KRPG_OPT_PROFILE_DETAIL)
            h->prof_detail = value != 0;
        else if (option == KRPG_OPT_FUSED_DEEP)
            h->fused_deep = value != 0;
        else if (option == KRPG_OPT_SLICES) {
            require(value >= 1 && value <= 8, "krpg_set_option: slices must be in [1, 8]");
            h->nslices = uint32_t(value);
        } else if (option == KRPG_OPT_ASYNC) {
            if (!value && h->async_mode) h->sync_check();
            h->async_mode = value != 0;
        } else if (option == KRPG_OPT_HOST_TRACE)
            h->host_trace = value != 0;
        else if (option == KRPG_OPT_EVAL_REG)
            h->tune.eval_reg = value != 0;
        else if (option == KRPG_OPT_POS0_TABLES)
            h->tune.pos0_tables = value != 0;
        else if (option == KRPG_OPT_DEEP_THRESHOLD) {
            require(value >= 0 && value <= (int64_t(1) << 30), "krpg_set_option: deep threshold out of range");
            h->tune.deep_threshold = int(value);
        } else if (option == KRPG_OPT_DEEP_CHUNK) {
            require(value >= 0 && value <= 32, "krpg_set_option: deep chunk must be in [0, 32]");
            h->tune.deep_chunk = int(value);
        } else if (option == KRPG_OPT_EVAL_SPLIT) {
            require(value == 0 || value == 1 || value == 16, "krpg_set_option: eval split must be 0, 1 or 16");
            h->tune.eval_split = int(value);
        } else if (option == KRPG_OPT_DEEP_DMMA_MIN) {
            require(value >= 1 && value <= 64, "krpg_set_option: deep DMMA minimum must be in [1, 64]");
            h->tune.deep_dmma_min = int(value);
        } else if (option == KRPG_OPT_STS_DETERMINISTIC)
            h->tune.sts_deterministic = value != 0;
        else if (option == KRPG_OPT_OUT_SLICES) {
            require(value >= 1 && value <= 4, "krpg_set_option: output slices must be in [1, 4]");
            h->tune.out_slices = int(value);
        } else if (option == KRPG_OPT_EVAL_ML) {
            h->tune.eval_ml = value != 0;
        } else if (option == KRPG_OPT_LEAF_PAR) {
            require(value >= 0 && value <= 64, "krpg_set_option: leaf scan parallel bound must be in [0, 64]");
            h->tune.leaf_par = int(value);
        }
        else
            throw std::invalid_argument("krpg_set_option: unknown option");
    });
}

int krpg_topology_node_rows(uint64_t I, uint64_t F, uint64_t v, uint64_t* first, uint64_t* last,
                            uint64_t* leaf_count, uint64_t* node_count) {
    return guard([&] {
        require(I >= 1 && F >= 1, "topology: empty");
        const krpg::Topo t = krpg::make_topo(I, F);
        require(v < t.n, "node_segment: node out of range");
        krpg::node_rows(t, v, first, last);
        if (leaf_count) *leaf_count = t.L;
        if (node_count) *node_count = t.n;
    });
}

int krpg_is_checked_build(void) {
#ifdef KRPG_CHECKED
    return 1;
#else
    return 0;
#endif
}

int krpg_host_eigh(const double* G, uint32_t n, double* vectors, double* values) {
    return guard([&] {
        const krpg::Eig e = krpg::eigh_psd(G, n);
        std::memcpy(vectors, e.vectors.data(), sizeof(double) * n * n);
        std::memcpy(values, e.values.data(), sizeof(double) * n);
    });
}

}  // extern "C"
