"""Python mirror of the reference's C++ sampler API over the krpg C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/krplev/krp_sampler.hpp:17-101 so parity tests
read like the reference's own tests (test_krp_sampler.cpp). All work runs on
the GPU through libkrpg.so; there is no CPU execution path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (EXCLUDED, MODE_ONE_STAGE, MODE_TWO_STAGE, STORE_F32, STORE_F64, check,
                   KrpgError, KrpgInvalidArgument)

_dp = C.POINTER(C.c_double)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


_TORCH_DT = {np.dtype(np.uint32): "int32", np.dtype(np.float64): "float64"}


def _host_array(shape, dtype) -> np.ndarray:
    """Output buffer in page-locked host memory (torch's caching pinned
    allocator, so repeated calls reuse blocks) so device->host copies run at
    link speed; plain numpy memory when torch/CUDA is unavailable."""
    try:
        import torch
        if torch.cuda.is_available():
            t = torch.empty(shape, dtype=getattr(torch, _TORCH_DT[np.dtype(dtype)]), pin_memory=True)
            return t.numpy().view(dtype)
    except Exception:
        pass
    return np.empty(shape, dtype=dtype)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _dev_tensor(t, name: str, dtype, device: int, shape=None):
    """Validate a torch CUDA tensor handed to the C ABI as a raw pointer: dtype,
    contiguity, device and shape must match exactly, since the library reads and
    writes through data_ptr() with no further checks."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise KrpgInvalidArgument(f"{name}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise KrpgInvalidArgument(f"{name}: expected dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise KrpgInvalidArgument(f"{name}: tensor must be contiguous (row-major)")
    if t.device.index != device:
        raise KrpgInvalidArgument(f"{name}: tensor is on cuda:{t.device.index}, sampler on cuda:{device}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise KrpgInvalidArgument(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return C.c_void_p(t.data_ptr())


class RowOrder(enum.Enum):
    """krp_sampler.hpp:17-25."""
    Ascending = 0  # first factor varies slowest
    Reversed = 1   # first factor varies fastest (mode-j matricization order)


@dataclass
class SampleBatch:
    """krp_sampler.hpp:27-48: J draws with exact probabilities and KRP rows."""
    excluded: Optional[int]
    count: int
    factor_count: int
    dims: np.ndarray                 # per-factor rows, excluded slot = 0
    indices: np.ndarray              # J x N uint32, excluded column = kExcluded
    probabilities: np.ndarray        # J
    rows: np.ndarray                 # J x R
    margin: Optional[np.ndarray] = field(default=None)  # J (boundary accounting)

    kExcluded = EXCLUDED

    def index(self, draw: int, factor: int) -> int:
        return int(self.indices[draw, factor])

    def flat_indices(self, order: RowOrder = RowOrder.Ascending) -> np.ndarray:
        """Mixed-radix KRP row ids (krp_sampler.cpp:19-39)."""
        ks = [k for k in range(self.factor_count) if self.excluded is None or k != self.excluded]
        if order == RowOrder.Reversed:
            ks = ks[::-1]
        flat = np.zeros(self.count, dtype=np.uint64)
        for k in ks:
            flat = flat * np.uint64(self.dims[k]) + self.indices[:, k].astype(np.uint64)
        return flat

    def flat_index(self, draw: int, order: RowOrder = RowOrder.Ascending) -> int:
        ks = [k for k in range(self.factor_count) if self.excluded is None or k != self.excluded]
        if order == RowOrder.Reversed:
            ks = ks[::-1]
        flat = 0
        for k in ks:
            flat = flat * int(self.dims[k]) + int(self.indices[draw, k])
        return flat


@dataclass
class ConditionalDistribution:
    """krp_sampler.hpp:50-55."""
    probabilities: np.ndarray
    mixture_weights: np.ndarray


class KrpSampler:
    """Exact leverage-score sampler for the KRP U_1 o ... o U_N (krp_sampler.hpp:57-101).

    Holds one segment tree per factor in HBM (leaf capacity R, compact
    layout). ``sample`` reproduces the reference's two-stage draws bit-exactly
    (up to counted boundary draws); ``mode="one_stage"`` draws from the
    north-star's per-draw M = G+ o hh^T o G_{>k} directly.
    """

    def __init__(self, factors: Sequence[np.ndarray], storage: str = "f64", device: int = 0):
        L = _lib.lib()
        fs = [_f64(f) for f in factors]
        N = len(fs)
        if N == 0:
            raise KrpgInvalidArgument("KrpSampler: factor list is empty")
        for f in fs:
            if f.ndim != 2:
                raise KrpgInvalidArgument("KrpSampler: factors must be 2-D")
        R = fs[0].shape[1]
        if any(f.shape[1] != R for f in fs):
            raise KrpgInvalidArgument("KrpSampler: inconsistent column counts")
        I = (C.c_uint64 * N)(*[f.shape[0] for f in fs])
        ptrs = (_dp * N)(*[_ptr(f) for f in fs])
        h = C.c_void_p()
        st = STORE_F32 if storage == "f32" else STORE_F64
        check(L.krpg_create(ptrs, I, N, R, st, device, C.byref(h)))
        self._device = device
        self._h = h
        self._N, self._R = N, R
        self._dims = [f.shape[0] for f in fs]
        self._storage = st

    @classmethod
    def from_device(cls, factors, storage: str = "f64", device: int = 0) -> "KrpSampler":
        """Build from torch CUDA tensors (row-major, float64 for storage "f64",
        float32 for "f32", all on cuda:`device`). The library reads them on its own
        stream after the producer (torch's current stream) has finished."""
        import torch
        L = _lib.lib()
        N = len(factors)
        if N == 0:
            raise KrpgInvalidArgument("KrpSampler: factor list is empty")
        st = STORE_F32 if storage == "f32" else STORE_F64
        dt = torch.float32 if st == STORE_F32 else torch.float64
        if any(f.dim() != 2 for f in factors):
            raise KrpgInvalidArgument("KrpSampler: factors must be 2-D")
        R = int(factors[0].shape[1])
        if any(int(f.shape[1]) != R for f in factors):
            raise KrpgInvalidArgument("KrpSampler: inconsistent column counts")
        ptrs = (C.c_void_p * N)(*[_dev_tensor(f, f"factor {k}", dt, device) for k, f in enumerate(factors)])
        I = (C.c_uint64 * N)(*[int(f.shape[0]) for f in factors])
        torch.cuda.current_stream(device).synchronize()  # producer -> library (no handle/stream yet)
        h = C.c_void_p()
        check(L.krpg_create_device(ptrs, I, N, R, st, device, C.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        self._N, self._R = N, R
        self._dims = [int(f.shape[0]) for f in factors]
        self._storage = st
        self._device = device
        return self

    # ---- stream ordering between torch and the library's own stream ----
    def _lib_stream(self):
        import torch
        return torch.cuda.ExternalStream(self.stream(), device=torch.device("cuda", self._device))

    def _after_torch(self):
        """Library work issued next waits for what torch's current stream has queued."""
        import torch
        self._lib_stream().wait_stream(torch.cuda.current_stream(self._device))

    def _before_torch(self):
        """torch's current stream waits for the library's queued work (device outputs)."""
        import torch
        torch.cuda.current_stream(self._device).wait_stream(self._lib_stream())

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h:
            _lib.lib().krpg_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- accessors (krp_sampler.hpp:63-68) ----
    def factor_count(self) -> int:
        return self._N

    def rank(self) -> int:
        return self._R

    def factor(self, j: int) -> np.ndarray:
        if not 0 <= j < self._N:
            raise KrpgInvalidArgument("factor: index out of range")
        out = np.empty((self._dims[j], self._R))
        check(_lib.lib().krpg_factor(self._h, j, _ptr(out)))
        return out

    def factor_gram(self, j: int) -> np.ndarray:
        if not 0 <= j < self._N:
            raise KrpgInvalidArgument("factor_gram: index out of range")
        out = np.empty((self._R, self._R))
        check(_lib.lib().krpg_factor_gram(self._h, j, _ptr(out)))
        return out

    @property
    def handle(self):
        return self._h

    # ---- tree introspection (segment_tree_sampler.hpp:64-95) ----
    def tree_shape(self, j: int):
        lc, nc = C.c_uint64(), C.c_uint64()
        check(_lib.lib().krpg_tree_shape(self._h, j, C.byref(lc), C.byref(nc)))
        return int(lc.value), int(nc.value)

    def node_gram(self, j: int, node: int) -> np.ndarray:
        out = np.empty((self._R, self._R))
        check(_lib.lib().krpg_node_gram(self._h, j, node, _ptr(out)))
        return out

    def tree_grams(self, j: int) -> np.ndarray:
        L, _ = self.tree_shape(j)
        P = self._R * (self._R + 1) // 2
        out = np.empty((L, P))
        check(_lib.lib().krpg_tree_grams(self._h, j, _ptr(out)))
        return out

    # ---- sampling (krp_sampler.cpp:82-151) ----
    def sample(self, excluded: Optional[int], J: int, seed: int, *, mode: str = "two_stage",
               draw_offset: int = 0, margin: bool = False) -> SampleBatch:
        if J < 1:
            raise KrpgInvalidArgument("KrpSample: sample count must be positive")
        e = -1 if excluded is None else int(excluded)
        if e < -1:
            raise KrpgInvalidArgument("KrpSampler: excluded index out of range")
        N, R = self._N, self._R
        idx = _host_array((J, N), np.uint32)
        prob = _host_array((J,), np.float64)
        rows = _host_array((J, R), np.float64)
        mg = _host_array((J,), np.float64) if margin else None
        m = MODE_ONE_STAGE if mode == "one_stage" else MODE_TWO_STAGE
        check(_lib.lib().krpg_sample(self._h, e, J, seed, draw_offset, m,
                                     idx.ctypes.data_as(C.POINTER(C.c_uint32)), _ptr(prob), _ptr(rows),
                                     _ptr(mg) if mg is not None else None))
        dims = np.array([0 if (excluded is not None and k == excluded) else self._dims[k]
                         for k in range(N)], dtype=np.uint64)
        return SampleBatch(excluded, J, N, dims, idx, prob, rows, mg)

    def product_lev_sample(self, excluded: Optional[int], J: int, seed: int, *, draw_offset: int = 0,
                           margin: bool = False) -> SampleBatch:
        """CP-ARLS-LEV baseline (sketch.cpp:86-149) over the resident factors: each
        included mode drawn from its own normalised leverage scores."""
        if J < 1:
            raise KrpgInvalidArgument("product_lev_sample: J must be positive")
        e = -1 if excluded is None else int(excluded)
        if e < -1:
            raise KrpgInvalidArgument("product_lev_sample: excluded index out of range")
        N, R = self._N, self._R
        idx = _host_array((J, N), np.uint32)
        prob = _host_array((J,), np.float64)
        rows = _host_array((J, R), np.float64)
        mg = _host_array((J,), np.float64) if margin else None
        check(_lib.lib().krpg_product_lev_sample(self._h, e, J, seed, draw_offset,
                                                 idx.ctypes.data_as(C.POINTER(C.c_uint32)), _ptr(prob),
                                                 _ptr(rows), _ptr(mg) if mg is not None else None))
        dims = np.array([0 if (excluded is not None and k == excluded) else self._dims[k]
                         for k in range(N)], dtype=np.uint64)
        return SampleBatch(excluded, J, N, dims, idx, prob, rows, mg)

    def leverage_scores(self, j: int) -> np.ndarray:
        """u_i^T pinv(G_j) u_i for every row of factor j (unnormalised; sums to rank)."""
        out = np.empty(int(self._dims[j]))
        check(_lib.lib().krpg_leverage_scores(self._h, j, _ptr(out)))
        return out

    def sample_device(self, excluded: Optional[int], J: int, seed: int, idx=None, prob=None,
                      rows=None, margin=None, *, mode: str = "two_stage", draw_offset: int = 0) -> None:
        """Device-resident outputs (torch CUDA tensors or None)."""
        import torch
        e = -1 if excluded is None else int(excluded)
        m = MODE_ONE_STAGE if mode == "one_stage" else MODE_TWO_STAGE
        d = self._device

        def p(t, name, dtype, shape):
            return _dev_tensor(t, name, dtype, d, shape) if t is not None else None

        pi = p(idx, "idx", torch.int32, (J, self._N))
        pp = p(prob, "prob", torch.float64, (J,))
        pr = p(rows, "rows", torch.float64, (J, self._R))
        pm = p(margin, "margin", torch.float64, (J,))
        self._after_torch()
        check(_lib.lib().krpg_sample_device(self._h, e, J, seed, draw_offset, m, pi, pp, pr, pm))
        self._before_torch()

    def gather_sa_device(self, J: int, prob, rows, weights, sa) -> None:
        import torch
        d, R, f64 = self._device, self._R, torch.float64
        pp = _dev_tensor(prob, "prob", f64, d, (J,))
        pr = _dev_tensor(rows, "rows", f64, d, (J, R))
        pw = _dev_tensor(weights, "weights", f64, d, (J,)) if weights is not None else None
        ps = _dev_tensor(sa, "sa", f64, d, (J, R))
        self._after_torch()
        check(_lib.lib().krpg_gather_sa_device(self._h, J, pp, pr, pw, ps))
        self._before_torch()

    def update_factor_device(self, j: int, U) -> None:
        """New factor j from a torch CUDA tensor (storage dtype), full device rebuild."""
        import torch
        if not 0 <= j < self._N:
            raise KrpgInvalidArgument("update_factor: index out of range")
        dt = torch.float32 if self._storage == STORE_F32 else torch.float64
        if U.dim() != 2 or int(U.shape[1]) != self._R:
            raise KrpgInvalidArgument("update_factor: column count mismatch")
        pu = _dev_tensor(U, "U", dt, self._device)
        self._after_torch()
        check(_lib.lib().krpg_update_factor_device(self._h, j, pu, int(U.shape[0])))
        self._dims[j] = int(U.shape[0])

    def set_grouped_descent(self, on: bool) -> None:
        """Choose the level-synchronous grouped DMMA descent (default) or the per-draw kernel."""
        check(_lib.lib().krpg_set_option(self._h, _lib.OPT_GROUPED_DESCENT, 1 if on else 0))

    def set_fused_deep(self, on: bool) -> None:
        """Fused warp-local deep levels + leaf scan (default) or per-level global regrouping."""
        check(_lib.lib().krpg_set_option(self._h, _lib.OPT_FUSED_DEEP, 1 if on else 0))

    def set_slices(self, n: int) -> None:
        """Concurrent draw slices of the grouped descent (KRPG_OPT_SLICES, default 1)."""
        check(_lib.lib().krpg_set_option(self._h, _lib.OPT_SLICES, int(n)))

    def set_tuning(self, **opts) -> None:
        """Kernel-variant / tuning options of the grouped descent (include/krpg.h
        KRPG_OPT_EVAL_REG ...): eval_reg, pos0_tables, deep_threshold, deep_chunk,
        eval_split, deep_dmma_min, leaf_par."""
        for k, v in opts.items():
            if k not in _lib.TUNING:
                raise KrpgInvalidArgument(f"set_tuning: unknown option {k}")
            check(_lib.lib().krpg_set_option(self._h, _lib.TUNING[k], int(v)))

    def set_async(self, on: bool) -> None:
        """KRPG_OPT_ASYNC: sample_device returns once enqueued (no host sync), so
        the next call's host setup overlaps this call's kernels; errors surface
        at sync()."""
        check(_lib.lib().krpg_set_option(self._h, _lib.OPT_ASYNC, 1 if on else 0))

    def sync(self) -> None:
        """Wait for the handle's stream; raises an error left by an asynchronous call."""
        check(_lib.lib().krpg_sync(self._h))

    def rebuild(self, j: int) -> None:
        check(_lib.lib().krpg_rebuild(self._h, j))

    def sts_solve(self, T, j: int, J: int, seed: int) -> np.ndarray:
        """One STS-CP factor update of mode j against the sparse tensor T (cp_als.cpp:279-313,
        solver StsCp): factor j is replaced by the normalised solve and its tree rebuilt;
        returns the column norms sigma (normalize_columns, cp_als.cpp:39-52)."""
        sigma = np.empty(self._R)
        check(_lib.lib().krpg_sts_solve(self._h, T._h, j, J, seed, sigma.ctypes.data_as(C.POINTER(C.c_double))))
        return sigma

    def sts_last_stats(self) -> dict:
        st = (C.c_uint64 * 3)()
        check(_lib.lib().krpg_sts_last_stats(self._h, st))
        return {"draws_hitting_nonzero_fibers": int(st[0]), "distinct_fibers": int(st[1]),
                "entries_visited": int(st[2])}

    # ---- row-partitioned construction (multi-GPU, see sharding.build_partitioned) ----
    def tree_device(self, j: int):
        """Zero-copy torch view (L*P doubles) of factor j's compact tree in HBM."""
        import torch

        from .sharding import _DeviceArray
        ptr, slots = C.c_void_p(), C.c_uint64()
        check(_lib.lib().krpg_tree_device(self._h, j, C.byref(ptr), C.byref(slots)))
        P = self._R * (self._R + 1) // 2
        return torch.as_tensor(_DeviceArray(ptr.value, slots.value * P), device=f"cuda:{self._device}")

    def build_partition(self, j: int, parts: int, part: int, subroot) -> None:
        """Stored nodes of subtree `part` of `parts`; subtree root Gram -> `subroot` (P doubles, CUDA)."""
        import torch
        P = self._R * (self._R + 1) // 2
        ps = _dev_tensor(subroot, "subroot", torch.float64, self._device, (P,))
        self._after_torch()
        check(_lib.lib().krpg_build_partition(self._h, j, parts, part, ps))
        self._before_torch()

    def finish_partitions(self, j: int, parts: int, subroots) -> None:
        """Top levels from all subtree roots (parts x P doubles, CUDA, subtree order)."""
        import torch
        P = self._R * (self._R + 1) // 2
        ps = _dev_tensor(subroots, "subroots", torch.float64, self._device, (parts * P,))
        self._after_torch()
        check(_lib.lib().krpg_finish_partitions(self._h, j, parts, ps))
        self._before_torch()

    def profile_enable(self, on: bool = True, detail: bool = False) -> None:
        check(_lib.lib().krpg_profile_enable(self._h, 1 if on else 0))
        check(_lib.lib().krpg_set_option(self._h, _lib.OPT_PROFILE_DETAIL, 1 if detail else 0))

    def profile_read(self, reset: bool = True) -> dict:
        ms = np.zeros(16)
        n = np.zeros(16, dtype=np.uint64)
        check(_lib.lib().krpg_profile_read(self._h, _ptr(ms), n.ctypes.data_as(C.POINTER(C.c_uint64)),
                                           1 if reset else 0))
        return {name: {"ms": float(ms[i]), "launches": int(n[i])} for i, name in enumerate(_lib.PROF_NAMES)}

    def stream(self) -> int:
        return int(_lib.lib().krpg_stream(self._h) or 0)

    def last_build_ms(self) -> float:
        v = C.c_float()
        check(_lib.lib().krpg_last_build_ms(self._h, C.byref(v)))
        return float(v.value)

    # ---- conditional (krp_sampler.cpp:153-196) ----
    def conditional(self, excluded: Optional[int], k: int, h) -> ConditionalDistribution:
        h = _f64(h)
        if h.size != self._R:
            raise KrpgInvalidArgument("conditional: history vector has wrong length")
        if not 0 <= k < self._N:
            raise KrpgInvalidArgument("conditional: factor k is not included")
        e = -1 if excluded is None else int(excluded)
        probs = np.empty(self._dims[k])
        mix = np.empty(self._R)
        check(_lib.lib().krpg_conditional(self._h, e, k, _ptr(h), _ptr(probs), _ptr(mix)))
        return ConditionalDistribution(probs, mix)

    # ---- updates (krp_sampler.cpp:198-228) ----
    def update_factor(self, j: int, U) -> None:
        U = _f64(U)
        if not 0 <= j < self._N:
            raise KrpgInvalidArgument("update_factor: index out of range")
        if U.ndim != 2 or U.shape[1] != self._R:
            raise KrpgInvalidArgument("update_factor: column count mismatch")
        check(_lib.lib().krpg_update_factor(self._h, j, _ptr(U), U.shape[0]))
        self._dims[j] = U.shape[0]

    def update_factor_entry(self, j: int, r: int, c: int, value: float) -> None:
        self.update_factor_entries(j, [r], [c], [value])

    def update_factor_entries(self, j: int, r, c, v) -> None:
        r = np.ascontiguousarray(r, dtype=np.uint64)
        c = np.ascontiguousarray(c, dtype=np.uint32)
        v = _f64(v)
        if not (r.size == c.size == v.size):
            raise KrpgInvalidArgument("update_factor_entry: length mismatch")
        check(_lib.lib().krpg_update_entries(self._h, j, r.ctypes.data_as(C.POINTER(C.c_uint64)),
                                             c.ctypes.data_as(C.POINTER(C.c_uint32)), _ptr(v), v.size))

    def validate(self, tol: float = 1e-10) -> None:
        check(_lib.lib().krpg_validate(self._h, tol))


def product_lev_sample(factors: Sequence, excluded: Optional[int], J: int, seed: int, *, device: int = 0,
                       margin: bool = False) -> SampleBatch:
    """Free-function CP-ARLS-LEV sampler (sketch.cpp:86-149) over host factors: the
    factors are copied to the device, gram(U) is formed there, nothing persists."""
    if len(factors) == 0:
        raise KrpgInvalidArgument("product_lev_sample: factor list is empty")
    fs = [_f64(f) for f in factors]
    N, R = len(fs), fs[0].shape[1]
    e = -1 if excluded is None else int(excluded)
    for k, f in enumerate(fs):
        if k != e and f.shape[1] != R:
            raise KrpgInvalidArgument("product_lev_sample: inconsistent column counts")
    I = (C.c_uint64 * N)(*[f.shape[0] for f in fs])
    ptrs = (C.POINTER(C.c_double) * N)(*[_ptr(f) for f in fs])
    idx = np.empty((J, N), dtype=np.uint32)
    prob, rows = np.empty(J), np.empty((J, R))
    mg = np.empty(J) if margin else None
    check(_lib.lib().krpg_product_lev_sample_factors(ptrs, I, N, R, e, J, seed, device,
                                                     idx.ctypes.data_as(C.POINTER(C.c_uint32)), _ptr(prob),
                                                     _ptr(rows), _ptr(mg) if mg is not None else None))
    dims = np.array([0 if k == e else f.shape[0] for k, f in enumerate(fs)], dtype=np.uint64)
    return SampleBatch(excluded, J, N, dims, idx, prob, rows, mg)


def device_count() -> int:
    return int(_lib.lib().krpg_device_count())
