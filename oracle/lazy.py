"""TEST INFRASTRUCTURE ONLY -- the checker, never the product.

Lazy restatement of the reference's two-stage KRP sampler (krp_sampler.cpp:82-151
over segment_tree_sampler.cpp:258-293) for checking individual draws at full
problem size, where building the complete reference trees on the host would take
minutes: a node's partial Gram is formed only when a checked draw's walk needs it
(U[seg]^T U[seg], cached), the eigenvector stage uses the closed form of its leaf
masses (E-leaf u of the tree with rows sqrt(lam_u) V[:,u]^T and Y = G_k has mass
lam_u (h o v_u)^T G_k (h o v_u), segment_tree_sampler.cpp:225-239), and the uniforms
come from the pinned CounterRng restatement (counters 2p+1 / 2p+2, stream = draw).

Summation orders differ from the reference (BLAS Grams, numpy eigh), so draws
agree with it up to counted boundary draws (|cutoff - u| <= 1e-10), exactly the
bar the device is held to; tests/test_oracle.py pins this restatement against the
C oracle on enumerable problems.
"""
from __future__ import annotations

import numpy as np

from . import backend


class Topology:
    """init_tree (segment_tree_sampler.cpp:111-149): complete tree over L leaves."""

    def __init__(self, I: int, F: int):
        self.I, self.F = int(I), int(F)
        self.L = (self.I + self.F - 1) // self.F
        self.d = 0 if self.L <= 1 else (self.L - 1).bit_length()
        self.n = 2 * self.L - 1
        self.bottom = 2 * self.L - (1 << self.d)

    def is_leaf(self, v: int) -> bool:
        return 2 * v + 1 >= self.n

    def leaf_index(self, v: int) -> int:
        first_deep = (1 << self.d) - 1
        return v - first_deep if v >= first_deep else v - (self.L - 1) + self.bottom

    def rows(self, v: int) -> tuple[int, int]:
        a = v
        while not self.is_leaf(a):
            a = 2 * a + 1
        b = v
        while not self.is_leaf(b):
            b = 2 * b + 2
        la, lb = self.leaf_index(a), self.leaf_index(b)
        return la * self.F, min((lb + 1) * self.F, self.I)


def _eigh_desc(M):
    w, V = np.linalg.eigh(0.5 * (M + M.T))
    order = np.argsort(-w, kind="stable")
    w, V = w[order], V[:, order]
    lmax = max(w[0], 0.0)
    w = np.where((w < 0) & (w >= -1e-8 * lmax), 0.0, w)
    return w, V


class LazyKrp:
    def __init__(self, factors):
        self.U = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
        self.R = self.U[0].shape[1]
        self.topo = [Topology(u.shape[0], self.R) for u in self.U]
        self.cache = [dict() for _ in self.U]
        self.rng = backend("port")

    def node_gram(self, k: int, v: int) -> np.ndarray:
        g = self.cache[k].get(v)
        if g is None:
            f, l = self.topo[k].rows(v)
            X = self.U[k][f:l]
            g = X.T @ X
            self.cache[k][v] = g
        return g

    def sample(self, excluded, draws, seed):
        """Indices (len(draws) x N, excluded column 0xFFFFFFFF), probabilities,
        rows, margins (smallest |cutoff - u| over every comparison) of the given
        global draw ids."""
        N, R = len(self.U), self.R
        inc = [k for k in range(N) if k != excluded]
        grams = [self.node_gram(k, 0) for k in range(N)]
        G = np.ones((R, R))
        for k in inc:
            G = G * grams[k]
        lam, V = _eigh_desc(G)
        tau = R * np.finfo(float).eps * lam[0]
        keep = lam > tau
        rank = int(keep.sum())
        Gp = (V[:, keep] / lam[keep]) @ V[:, keep].T
        eig = []
        for p in range(len(inc)):
            Y = Gp.copy()
            for q in inc[p + 1:]:
                Y = Y * grams[q]
            eig.append(_eigh_desc(Y))
        out_i = np.full((len(draws), N), 0xFFFFFFFF, dtype=np.uint32)
        out_p = np.empty(len(draws))
        out_r = np.empty((len(draws), R))
        out_m = np.empty(len(draws))
        for t, d in enumerate(draws):
            u = self.rng.uniforms(seed, int(d), 2 * len(inc))
            h = np.ones(R)
            margin = np.inf
            for p, k in enumerate(inc):
                # eigenvector stage: leaf masses in closed form, walk over their prefix sums
                lam_p, Vp = eig[p]
                Zu = h[:, None] * Vp
                m = lam_p * np.einsum("au,ab,bu->u", Zu, grams[k], Zu)
                te = Topology(R, 1)
                uu, margin = self._walk(te, lambda v: m[slice(*te.rows(v))].sum(), u[2 * p], margin)
                ev = te.leaf_index(uu)
                z = h * Vp[:, ev]
                # factor stage: rank-1 M = z z^T on the factor tree
                tz = self.topo[k]
                node, margin, low, ic = self._walk_z(k, tz, z, u[2 * p + 1], margin)
                f, l = tz.rows(node)
                mass = (self.U[k][f:l] @ z) ** 2 * ic
                cum, pick, last_nz = low, -1, -1
                for i in range(l - f):
                    if mass[i] > 0:
                        last_nz = f + i
                    cum += mass[i]
                    margin = min(margin, abs(cum - u[2 * p + 1]))
                    if cum >= u[2 * p + 1]:
                        pick = f + i
                        break
                if pick < 0:
                    pick = last_nz if last_nz >= 0 else l - 1
                out_i[t, k] = pick
                h = h * self.U[k][pick]
            out_r[t] = h
            out_p[t] = float(h @ Gp @ h) / rank
            out_m[t] = margin
        return out_i, out_p, out_r, out_m

    @staticmethod
    def _walk(topo, mass_of, u, margin):
        C = mass_of(0)
        if not np.isfinite(C) or C <= 0:
            raise RuntimeError("row_sample: degenerate distribution (C <= 0)")
        ic, low, v = 1.0 / C, 0.0, 0
        while not topo.is_leaf(v):
            cutoff = low + ic * mass_of(2 * v + 1)
            margin = min(margin, abs(cutoff - u))
            if cutoff >= u:
                v = 2 * v + 1
            else:
                low, v = cutoff, 2 * v + 2
        return v, margin

    def _walk_z(self, k, topo, z, u, margin):
        qf = lambda v: float(z @ self.node_gram(k, v) @ z)  # noqa: E731
        C = qf(0)
        if not np.isfinite(C) or C <= 0:
            raise RuntimeError("row_sample: degenerate distribution (C <= 0)")
        ic, low, v = 1.0 / C, 0.0, 0
        while not topo.is_leaf(v):
            cutoff = low + ic * qf(2 * v + 1)
            margin = min(margin, abs(cutoff - u))
            if cutoff >= u:
                v = 2 * v + 1
            else:
                low, v = cutoff, 2 * v + 2
        return v, margin, low, ic
