// One grouped-descent level in isolation (config-2 shape: J = 65536 draws, R = 64, all draws
// in one node run as at the top of the tree), timed with events per launch:
//   usage: level_bench [J] [nruns]   (nruns: the draws are spread over that many node runs)
// The level kernel as the library launches it (default tuning);
// KRPG_FAKE_QF=1 skips the DMMA, =2 also the row / Gram loads (k_eval_reg only).
#define KRPG_LEVEL_BENCH 1
#include "../../paper_2301_12584_b200/csrc/descent_v2.cu"

#include <cstdio>
#include <random>
#include <vector>

using namespace krpg;
using namespace krpg::v2;

int main(int argc, char** argv) {
    const uint64_t J = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 65536;
    const uint32_t nruns = argc > 2 ? std::atoi(argv[2]) : 1;
    const uint32_t R = 64, P = R * (R + 1) / 2;
    const Topo tz = make_topo(1ull << 22, R);
    // level l such that 2^l >= nruns: draws at nodes 2^l - 1 + (d * nruns / J)
    uint32_t l = 0;
    while ((1u << l) < nruns) ++l;
    const uint32_t first = (1u << l) - 1;
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(-1, 1), U01(0, 1);
    std::vector<double> X(J * R), tree((size_t(tz.L)) * P), ud(J), invc(J), low(J, 0.0), mg(J, 1e300);
    const bool simple = std::getenv("LB_SIMPLE") != nullptr;  // low-entropy operands (power / clock probe)
    for (size_t i = 0; i < X.size(); ++i) X[i] = simple ? 1.0 + 0.125 * double(i % 7) : U(rng);
    for (size_t i = 0; i < tree.size(); ++i) tree[i] = simple ? 1e-3 * double(1 + i % 5) : U(rng) * 1e-3;
    for (uint64_t s = 0; s < tz.L; ++s)
        for (uint32_t a = 0; a < R; ++a) tree[s * P + pack_index(R, a, a)] = 10.0 + U01(rng);
    for (uint64_t d = 0; d < J; ++d) {
        ud[d] = U01(rng);
        invc[d] = 1.0 / (2 * 640.0);
    }
    std::vector<uint32_t> node(J), perm(J), nsort(J);
    for (uint64_t d = 0; d < J; ++d) {
        perm[d] = uint32_t(d);
        node[d] = first + uint32_t(d * nruns / J);
        nsort[d] = node[d];
    }
    // node ranges of the parents: GS/GE for level l nodes must be derivable; set GS/GE/cntL of parents
    const uint32_t nn = uint32_t(tz.n);
    std::vector<uint32_t> GS(nn, 0), GE(nn, 0), cntL(nn, 0);
    for (uint32_t r = 0; r < nruns; ++r) {
        const uint32_t v = first + r;
        const uint64_t s = uint64_t(r) * J / nruns, e = uint64_t(r + 1) * J / nruns;
        if (v == 0) continue;
        const uint32_t p = (v - 1) >> 1;
        if (v & 1) {
            GS[p] = uint32_t(s);
            cntL[p] = uint32_t(e - s);
        } else {
            GE[p] = uint32_t(e);
        }
    }
    auto up = [](const void* h, size_t bytes) {
        void* d;
        cudaMalloc(&d, bytes);
        cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
        return d;
    };
    EvalArgs a{};
    a.J = J;
    a.perm = static_cast<uint32_t*>(up(perm.data(), J * 4));
    a.nsort_in = static_cast<uint32_t*>(up(nsort.data(), J * 4));
    uint32_t* node_d = static_cast<uint32_t*>(up(node.data(), J * 4));
    a.node = node_d;
    cudaMalloc(&a.rank, J * 4);
    a.low = static_cast<double*>(up(low.data(), J * 8));
    a.invc = static_cast<double*>(up(invc.data(), J * 8));
    a.ud = static_cast<double*>(up(ud.data(), J * 8));
    a.margin = static_cast<double*>(up(mg.data(), J * 8));
    uint32_t* cntL_d = static_cast<uint32_t*>(up(cntL.data(), nn * 4));
    cudaMalloc(&a.cntR, size_t(nn) * 4);
    a.cntL = cntL_d;
    a.X = static_cast<double*>(up(X.data(), J * R * 8));
    a.tree = static_cast<double*>(up(tree.data(), tree.size() * 8));
    a.topo = tz;
    cudaMalloc(&a.err, 4);
    cudaMalloc(&a.perm_out, J * 4);
    cudaMalloc(&a.nsort_out, J * 4);
    a.GS = static_cast<uint32_t*>(up(GS.data(), nn * 4));
    a.GE = static_cast<uint32_t*>(up(GE.data(), nn * 4));
    const char* f = std::getenv("KRPG_FAKE_QF");
    a.fake = f ? std::atoi(f) : 0;
    const size_t ntr = (J / 8 + 64) * 16;
    cudaMalloc(&a.trace, ntr * 8);
    cudaMemset(a.trace, 0, ntr * 8);
    // counters of this level's nodes are reset before every launch (memset not timed)
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 1e30, sum = 0;
    const int K = 20;
    const char* mlv = std::getenv("LB_ML");
    const int ml = mlv ? std::atoi(mlv) : 0;
    uint32_t* gbar;
    cudaMalloc(&gbar, 128);
    if (const char* dbg = std::getenv("LB_ML_DBG")) {
        const int v = std::atoi(dbg);
        cudaMemcpyToSymbol(g_ml_dbg, &v, sizeof(int));
    }
    // the multi-level runs rewrite the order buffers: restore them before every launch
    uint32_t* perm0 = const_cast<uint32_t*>(a.perm);
    uint32_t* nsort0 = const_cast<uint32_t*>(a.nsort_in);
    for (int it = 0; it < K + 3; ++it) {
        cudaMemcpyAsync(node_d, node.data(), J * 4, cudaMemcpyHostToDevice, s);
        if (ml) {
            cudaMemcpyAsync(perm0, perm.data(), J * 4, cudaMemcpyHostToDevice, s);
            cudaMemcpyAsync(nsort0, nsort.data(), J * 4, cudaMemcpyHostToDevice, s);
            cudaMemcpyAsync(a.low, low.data(), J * 8, cudaMemcpyHostToDevice, s);
        }
        cudaMemsetAsync(a.cntR, 0, size_t(nn) * 4, s);
        cudaMemcpyAsync(cntL_d, cntL.data(), size_t(nn) * 4, cudaMemcpyHostToDevice, s);
        // level-l counters must start at zero (cntL of the parents is preset above)
        cudaMemsetAsync(cntL_d + first, 0, size_t(nruns) * 4, s);
        cudaEventRecord(e0, s);
        if (ml >= 2) {  // LB_ML=n: n consecutive levels in one cooperative launch (k_eval_reg_ml)
            cudaMemsetAsync(gbar, 0, 4, s);
            cudaEventRecord(e0, s);
            const bool ok = dispatch_eval_ml(R, a, uint32_t(ml), gbar, s, Tuning{});
            if (!ok) std::printf("cooperative launch refused: %s\n", cudaGetErrorString(cudaGetLastError()));
        } else if (ml == 1) {  // LB_ML=1 with LB_SEQ=n: n levels as n launches
            const char* sq = std::getenv("LB_SEQ");
            EvalArgs b = a;
            for (int q = 0; q < (sq ? std::atoi(sq) : 1); ++q) {
                dispatch_eval(R, EV_LEVEL, b, s, Tuning{});
                const uint32_t* t = b.perm_out;
                b.perm_out = const_cast<uint32_t*>(b.perm);
                b.perm = t;
                t = b.nsort_out;
                b.nsort_out = const_cast<uint32_t*>(b.nsort_in);
                b.nsort_in = t;
            }
        } else {
            dispatch_eval(R, EV_LEVEL, a, s, Tuning{});
        }
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 3) {
            best = std::min(best, double(ms));
            sum += ms;
        }
    }
    const cudaError_t err = cudaGetLastError();
    {
        std::vector<unsigned long long> tr(ntr);
        cudaMemcpy(tr.data(), a.trace, ntr * 8, cudaMemcpyDeviceToHost);
        unsigned long long t0min = ~0ull, t0max = 0, t5max = 0;
        double ph[5] = {0, 0, 0, 0, 0}, f6 = 0, f7 = 0, g8 = 0, g9 = 0, g10 = 0, g2 = 0, g11 = 0;
        int ng = 0;
        int n67 = 0;
        int nw = 0;
        for (size_t w = 0; w * 16 < ntr; ++w) {
            const unsigned long long* t = &tr[w * 16];
            if (!t[0] || !t[5]) continue;
            ++nw;
            t0min = std::min(t0min, t[0]);
            t0max = std::max(t0max, t[0]);
            t5max = std::max(t5max, t[5]);
            for (int k = 0; k < 5; ++k) ph[k] += double(t[k + 1] - t[k]);
            if (t[8] && t[9] && t[10] && t[11]) {
                g8 += double(t[8] - t[1]);
                g9 += double(t[9] - t[8]);
                g10 += double(t[10] - t[9]);
                g2 += double(t[2] - t[10]);
                g11 += double(t[11] - t[2]);
                ++ng;
            }
            if (t[6] && t[7]) {
                f6 += double(t[6] - t[2]);
                f7 += double(t[7] - t[6]);
                ++n67;
            }
        }
        if (nw)
            std::printf("  last launch: %d warps, span %.1f us, start skew %.1f us; per warp: positions %.2f, list %.2f, "
                        "sweep %.2f, claims %.2f, scatter %.2f us\n",
                        nw, (t5max - t0min) * 1e-3, (t0max - t0min) * 1e-3, ph[0] / nw * 1e-3, ph[1] / nw * 1e-3,
                        ph[2] / nw * 1e-3, ph[3] / nw * 1e-3, ph[4] / nw * 1e-3);
        if (ng) std::printf("  list phase: gram issue %.2f, block-0 rows %.2f, cp.async inputs %.2f, block list %.2f, "
                            "inputs wait %.2f us\n", g8 / ng * 1e-3, g9 / ng * 1e-3, g10 / ng * 1e-3, g2 / ng * 1e-3,
                            g11 / ng * 1e-3);
        if (n67) std::printf("  first block: gram + rows ready %.2f us after the list, its DMMA chain %.2f us\n", f6 / n67 * 1e-3, f7 / n67 * 1e-3);
    }
    std::vector<uint32_t> po(J);
    cudaMemcpy(po.data(), a.perm_out, J * 4, cudaMemcpyDeviceToHost);
    std::vector<char> seen(J, 0);
    uint64_t bad = 0;
    for (auto p : po) bad += (p >= J || seen[p]++) ? 1 : 0;
    std::printf("J %llu runs %u (level %u): best %.1f us  mean %.1f us  (DMMA floor at 37 TF/s: %.1f us)  perm %s  %s\n",
                (unsigned long long)J, nruns, l, best * 1e3, sum / K * 1e3, double(J) / 8 * 72 * 512 / 37e12 * 1e6,
                bad ? "BROKEN" : "ok", cudaGetErrorString(err));
}
