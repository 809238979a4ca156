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


class SegmentTreeSampler:
    def __init__(self, U, F: int, Y=None, y=None, device: int = 0):
        U = _c64(U)
        if U.ndim != 2:
            from ._lib import KrpgInvalidArgument
            raise KrpgInvalidArgument("SegmentTreeSampler: U must be a matrix")
        self.I, self.R = U.shape
        self.F = int(F)
        self._U = U
        Yc = _c64(Y) if Y is not None else None
        yc = _c64(y) if y is not None else None
        self._h = C.c_void_p()
        check(_lib.lib().krpg_segtree_create(
            U.ctypes.data_as(_dp), self.I, self.R, self.F,
            Yc.ctypes.data_as(_dp) if Yc is not None else None,
            yc.ctypes.data_as(_dp) if yc is not None else None, device, C.byref(self._h)))

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
