"""Device-resident sparse tensor for the STS-CP solve slice.

Mirrors the reference's SparseTensorCoo (tensor.hpp:18-70): ``from_entries``
validates coordinates, sums duplicates and sorts entries lexicographically --
here on the device (krpg_tensor_create). ``KrpSampler.sts_solve`` then runs one
STS-CP factor update (the StsCp branch of cp_als.cpp:279-313) against it.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import check


class SparseTensor:
    def __init__(self, dims: Sequence[int], coords, values, device: int = 0):
        self.dims = [int(d) for d in dims]
        N = len(self.dims)
        coords = np.ascontiguousarray(np.asarray(coords, dtype=np.uint32).reshape(-1, N))
        values = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
        if coords.shape[0] != values.shape[0]:
            from ._lib import KrpgInvalidArgument
            raise KrpgInvalidArgument("SparseTensorCoo: coords/values mismatch")
        self._h = C.c_void_p()
        dims_c = (C.c_uint64 * N)(*self.dims)
        check(_lib.lib().krpg_tensor_create(dims_c, N, coords.ctypes.data_as(C.POINTER(C.c_uint32)),
                                            values.ctypes.data_as(C.POINTER(C.c_double)), values.shape[0],
                                            device, C.byref(self._h)))

    @classmethod
    def from_entries(cls, dims, coords, values, device: int = 0) -> "SparseTensor":
        return cls(dims, coords, values, device)

    @classmethod
    def from_device(cls, dims, coords, values, device: int = 0) -> "SparseTensor":
        """From torch CUDA tensors (coords nnz x N int32/uint32, values nnz float64) without
        staging through host memory (krpg_tensor_create_device); inputs are only read."""
        import torch
        from ._lib import KrpgInvalidArgument
        from .sampler import _dev_tensor
        self = cls.__new__(cls)
        self.dims = [int(d) for d in dims]
        N = len(self.dims)
        nnz = int(values.shape[0])
        if coords.dim() != 2 or int(coords.shape[1]) != N or int(coords.shape[0]) != nnz:
            raise KrpgInvalidArgument("SparseTensorCoo: coords/values mismatch")
        pc = _dev_tensor(coords, "coords", coords.dtype if coords.dtype in (torch.int32,) else torch.int32, device)
        pv = _dev_tensor(values, "values", torch.float64, device)
        self._h = C.c_void_p()
        dims_c = (C.c_uint64 * N)(*self.dims)
        check(_lib.lib().krpg_tensor_create_device(dims_c, N, pc, pv, nnz, device, C.byref(self._h)))
        return self

    def ndim(self) -> int:
        return len(self.dims)

    def nnz(self) -> int:
        n = C.c_uint64()
        check(_lib.lib().krpg_tensor_info(self._h, C.byref(n), None))
        return int(n.value)

    def norm_squared(self) -> float:
        x = C.c_double()
        check(_lib.lib().krpg_tensor_info(self._h, None, C.byref(x)))
        return float(x.value)

    def entries(self):
        """(coords nnz x N, values nnz): deduplicated, lexicographically sorted."""
        n = self.nnz()
        c = np.empty((n, self.ndim()), dtype=np.uint32)
        v = np.empty(n)
        check(_lib.lib().krpg_tensor_entries(self._h, c.ctypes.data_as(C.POINTER(C.c_uint32)),
                                             v.ctypes.data_as(C.POINTER(C.c_double))))
        return c, v

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.lib().krpg_tensor_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
