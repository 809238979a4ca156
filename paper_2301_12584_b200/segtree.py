"""Device SegmentTreeSampler (the reference's secondary surface,
segment_tree_sampler.hpp:26-139): a standalone segment tree of partial Grams over
U (I x R) with leaf capacity F and a fixed PSD Y (rank-1 y y^T or general), built
and sampled with the same kernels as the KRP sampler (krpg_segtree_* in krpg.h)."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check

_dp = C.POINTER(C.c_double)


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


_u64p = C.POINTER(C.c_uint64)


def sparse_leaf_offsets(row_counts, R: int) -> np.ndarray:
    """Greedy row partition of from_sparse (segment_tree_sampler.cpp:88-101): a leaf
    closes before row i when adding its nonzeros would exceed R^2 and the leaf is
    non-empty. Returns the L + 1 leaf offsets."""
    cap = R * R
    offs, cur = [0], 0
    for i, rn in enumerate(np.asarray(row_counts, dtype=np.int64).tolist()):
        if cur + rn > cap and cur > 0:
            offs.append(i)
            cur = 0
        cur += rn
    offs.append(len(row_counts))
    return np.asarray(offs, dtype=np.uint64)


class SegmentTreeSampler:
    def __init__(self, U, F: Optional[int] = None, Y=None, y=None, device: int = 0, leaf_offsets=None):
        U = _c64(U)
        if U.ndim != 2:
            from ._lib import KrpgInvalidArgument
            raise KrpgInvalidArgument("SegmentTreeSampler: U must be a matrix")
        self.I, self.R = U.shape
        self.F = int(F) if F is not None else self.R
        self._U = U
        self._pattern = None  # sparse-built: set of stored (row, col)
        Yc = _c64(Y) if Y is not None else None
        yc = _c64(y) if y is not None else None
        self._h = C.c_void_p()
        Yp = Yc.ctypes.data_as(_dp) if Yc is not None else None
        yp = yc.ctypes.data_as(_dp) if yc is not None else None
        if leaf_offsets is None:
            check(_lib.lib().krpg_segtree_create(U.ctypes.data_as(_dp), self.I, self.R, self.F, Yp, yp, device,
                                                 C.byref(self._h)))
        else:
            offs = np.ascontiguousarray(leaf_offsets, dtype=np.uint64)
            check(_lib.lib().krpg_segtree_create_segments(U.ctypes.data_as(_dp), self.I, self.R,
                                                          offs.ctypes.data_as(_u64p), len(offs) - 1, Yp, yp,
                                                          device, C.byref(self._h)))

    @classmethod
    def from_sparse(cls, rows: int, cols: int, entry_rows, entry_cols, values, device: int = 0):
        """from_sparse (segment_tree_sampler.cpp:67-109): COO entries sorted row-major
        (strictly), Y = all-ones (y = 1), leaves by the R^2-nonzero greedy rule. The
        device stores the densified rows; draws are identical to the dense tree's."""
        from ._lib import KrpgInvalidArgument
        er = np.asarray(entry_rows, dtype=np.int64)
        ec = np.asarray(entry_cols, dtype=np.int64)
        ev = np.asarray(values, dtype=np.float64)
        if rows < 1 or cols < 1:
            raise KrpgInvalidArgument("build_sampler_sparse: empty matrix")
        if er.size == 0:
            raise KrpgInvalidArgument("build_sampler_sparse: matrix has no nonzeros")
        key = er * cols + ec
        if er.size > 1 and not np.all((er[1:] > er[:-1]) | ((er[1:] == er[:-1]) & (ec[1:] > ec[:-1]))):
            raise KrpgInvalidArgument("build_sampler_sparse: entries must be sorted row-major")
        if np.any(er < 0) or np.any(er >= rows) or np.any(ec < 0) or np.any(ec >= cols):
            raise KrpgInvalidArgument("build_sampler_sparse: entry out of range")
        if not np.all(np.isfinite(ev)):
            raise KrpgInvalidArgument("build_sampler_sparse: non-finite entry")
        U = np.zeros((rows, cols))
        U[er, ec] = ev
        offs = sparse_leaf_offsets(np.bincount(er, minlength=rows), cols)
        t = cls(U, None, y=np.ones(cols), device=device, leaf_offsets=offs)
        t._pattern = set(key.tolist())
        return t

    def sparse(self) -> bool:
        return self._pattern is not None

    def leaf_offsets(self) -> np.ndarray:
        out = np.empty(self.leaf_count() + 1, dtype=np.uint64)
        check(_lib.lib().krpg_segtree_leaf_offsets(self._h, out.ctypes.data_as(_u64p)))
        return out

    def leaf_segment(self, leaf: int):
        o = self.leaf_offsets()
        return int(o[leaf]), int(o[leaf + 1])

    def node_segment(self, node: int):
        f, l = C.c_uint64(), C.c_uint64()
        check(_lib.lib().krpg_segtree_node_rows(self._h, node, C.byref(f), C.byref(l)))
        return int(f.value), int(l.value)

    def rows(self) -> int:
        return self.I

    def cols(self) -> int:
        return self.R

    def shape(self):
        L, n = C.c_uint64(), C.c_uint64()
        check(_lib.lib().krpg_segtree_shape(self._h, C.byref(L), C.byref(n)))
        return int(L.value), int(n.value)

    def leaf_count(self) -> int:
        return self.shape()[0]

    def node_count(self) -> int:
        return self.shape()[1]

    def node_gram(self, node: int) -> np.ndarray:
        out = np.empty((self.R, self.R))
        check(_lib.lib().krpg_segtree_node_gram(self._h, node, out.ctypes.data_as(_dp)))
        return out

    def row_sample_batch(self, H, seed: int, stream0: int = 0, counter: int = 1, margin: bool = False):
        """Draw d uses history H[d] and CounterRng(seed, stream0 + d) at `counter`."""
        H = _c64(H).reshape(-1, self.R)
        J = H.shape[0]
        out = np.empty(J, dtype=np.uint64)
        mg = np.empty(J) if margin else None
        check(_lib.lib().krpg_segtree_sample(self._h, H.ctypes.data_as(_dp), J, seed, stream0, counter,
                                             out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                             mg.ctypes.data_as(_dp) if mg is not None else None))
        return (out, mg) if margin else out

    def row_sample(self, h, seed: int, stream: int, counter: int = 1) -> int:
        return int(self.row_sample_batch(np.asarray(h, dtype=np.float64)[None, :], seed, stream, counter)[0])

    def analytic_probabilities(self, h) -> np.ndarray:
        h = _c64(h)
        out = np.empty(self.I)
        check(_lib.lib().krpg_segtree_probabilities(self._h, h.ctypes.data_as(_dp), out.ctypes.data_as(_dp)))
        return out

    def update_entry(self, r: int, c: int, value: float) -> None:
        if self._pattern is not None and 0 <= r < self.I and 0 <= c < self.R and r * self.R + c not in self._pattern:
            from ._lib import KrpgInvalidArgument
            raise KrpgInvalidArgument("update_entry: entry outside the stored sparsity pattern")
        check(_lib.lib().krpg_segtree_update_entry(self._h, r, c, float(value)))
        self._U[r, c] = value

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.lib().krpg_segtree_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
