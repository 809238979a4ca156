"""TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.

ctypes front-ends for the two CPU oracles of the KRP leverage sampler:

* ``port``: ``oracle/build/libkrp_oracle.so`` — our plain-C restatement of the
  reference algorithm (oracle/krp_oracle.c), always buildable.
* ``ref``: ``oracle/_ref/libkrplev_ref.so`` — the unmodified reference
  (/root/reference/proj) compiled by oracle/Makefile; present wherever it was
  built (it travels to the GPU box as a prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "libkrp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkrplev_ref.so")
EXCLUDED = 0xFFFFFFFF

_u64 = C.c_uint64
_u32 = C.c_uint32
_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


def build(quiet: bool = True) -> None:
    """Compile the restatement (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


_lib_cache: dict[str, C.CDLL] = {}


def _load(path: str) -> C.CDLL:
    if path not in _lib_cache:
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        _lib_cache[path] = C.CDLL(path)
    return _lib_cache[path]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class _Backend:
    """Uniform view over the two libraries (prefix ko_ or kref_)."""

    def __init__(self, kind: str):
        self.kind = kind
        if kind == "port":
            if not os.path.exists(PORT_SO):
                build()
            self.lib = _load(PORT_SO)
            self.p = "ko_"
        elif kind == "ref":
            self.lib = _load(REF_SO)
            self.p = "kref_"
        else:
            raise ValueError(kind)
        getattr(self.lib, self.p + "last_error").restype = C.c_char_p

    def fn(self, name):
        return getattr(self.lib, self.p + name)

    def check(self, rc: int):
        if rc == 0:
            return
        msg = self.fn("last_error")().decode()
        if rc == 1:
            raise OracleInvalidArgument(msg)
        raise OracleError(msg)

    # ---- rng ----
    def uniforms(self, seed, stream, n):
        out = np.empty(n)
        self.fn("uniforms")(_u64(seed), _u64(stream), _u64(n), _dptr(out))
        return out

    def normals(self, seed, stream, n):
        out = np.empty(n)
        self.fn("normals")(_u64(seed), _u64(stream), _u64(n), _dptr(out))
        return out

    def derive_seed(self, seed, a, b=0):
        f = self.fn("derive_seed")
        f.restype = _u64
        return int(f(_u64(seed), _u64(a), _u64(b)))

    # ---- dense ----
    def eigh(self, G):
        G = _c64(G)
        n = G.shape[0]
        V = np.empty((n, n))
        lam = np.empty(n)
        self.check(self.fn("eigh")(_dptr(G), _u32(n), _dptr(V), _dptr(lam)))
        return V, lam

    def pinv(self, G):
        G = _c64(G)
        n = G.shape[0]
        out = np.empty((n, n))
        rank = _u64(0)
        self.check(self.fn("pinv")(_dptr(G), _u32(n), _dptr(out), C.byref(rank)))
        return out, int(rank.value)

    def leverage(self, factors):
        fs = [_c64(f) for f in factors]
        R = fs[0].shape[1]
        I = (_u64 * len(fs))(*[f.shape[0] for f in fs])
        ptrs = (_dp * len(fs))(*[_dptr(f) for f in fs])
        out = np.empty(int(np.prod([f.shape[0] for f in fs])))
        self.check(self.fn("leverage")(ptrs, I, _u32(len(fs)), _u32(R), _dptr(out)))
        return out

    def product_lev_sample(self, factors, excluded, J, seed):
        """CP-ARLS-LEV product_lev_sample (sketch.cpp:86-149): indices (J x N,
        excluded column 0xFFFFFFFF), probabilities, rows, margins (port only)."""
        fs = [_c64(f) for f in factors]
        N, R = len(fs), fs[0].shape[1]
        I = (_u64 * N)(*[f.shape[0] for f in fs])
        ptrs = (_dp * N)(*[_dptr(f) for f in fs])
        idx = np.empty((J, N), dtype=np.uint32)
        prob, rows, mg = np.empty(J), np.empty((J, R)), np.empty(J)
        e = -1 if excluded is None else int(excluded)
        self.check(self.fn("product_lev_sample")(ptrs, I, _u32(N), _u32(R), _i64(e), _u64(J), _u64(seed),
                                                  idx.ctypes.data_as(C.POINTER(_u32)), _dptr(prob), _dptr(rows),
                                                  _dptr(mg)))
        return idx, prob, rows, mg

    def sampling_weights(self, prob, J):
        prob = _c64(prob)
        w = np.empty_like(prob)
        self.check(self.fn("sampling_weights")(_dptr(prob), _u64(prob.size), _u64(J), _dptr(w)))
        return w


class OracleKrp:
    """KrpSampler through either CPU oracle (reference krp_sampler.hpp:61-101)."""

    def __init__(self, factors, backend: str = "port"):
        self.b = _Backend(backend)
        self.factors = [_c64(f).copy() for f in factors]
        self.N = len(self.factors)
        self.R = self.factors[0].shape[1] if self.N else 0
        I = (_u64 * max(self.N, 1))(*[f.shape[0] for f in self.factors])
        ptrs = (_dp * max(self.N, 1))(*[_dptr(f) for f in self.factors])
        h = _vp()
        create = self.b.fn("krp_create" if backend == "port" else "create")
        self.b.check(create(ptrs, I, _u32(self.N), _u32(self.R), C.byref(h)))
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.b.fn("krp_destroy" if self.b.kind == "port" else "destroy")(h)
            self.h = None

    def _name(self, port, ref):
        return self.b.fn(port if self.b.kind == "port" else ref)

    def factor_gram(self, j):
        out = np.empty((self.R, self.R))
        self.b.check(self._name("krp_factor_gram", "factor_gram")(self.h, _u32(j), _dptr(out)))
        return out

    def sample(self, excluded, J, seed, one_stage=False, want_margin=False, draw_offset=0):
        e = -1 if excluded is None else int(excluded)
        idx = np.empty((J, self.N), dtype=np.uint32)
        prob = np.empty(J)
        rows = np.empty((J, self.R))
        args = [self.h, _i64(e), _u64(J), _u64(seed), idx.ctypes.data_as(C.POINTER(_u32)),
                _dptr(prob), _dptr(rows)]
        margin = None
        if self.b.kind == "port":
            args.insert(4, _u64(draw_offset))
            margin = np.empty(J)
            args.append(_dptr(margin) if want_margin else None)
            f = self.b.fn("krp_sample_one_stage" if one_stage else "krp_sample")
        else:
            if draw_offset:
                raise ValueError("the reference has no draw offset")
            f = self.b.fn("sample_one_stage" if one_stage else "sample")
        self.b.check(f(*args))
        if want_margin:
            return idx, prob, rows, margin
        return idx, prob, rows

    def conditional(self, excluded, k, h):
        e = -1 if excluded is None else int(excluded)
        h = _c64(h)
        probs = np.empty(self.factors[k].shape[0])
        mix = np.empty(self.R)
        f = self._name("krp_conditional", "conditional")
        self.b.check(f(self.h, _i64(e), _u32(k), _dptr(h), _dptr(probs), _dptr(mix)))
        return probs, mix

    def update_factor(self, j, U):
        U = _c64(U)
        f = self._name("krp_update_factor", "update_factor")
        self.b.check(f(self.h, _u32(j), _dptr(U), _u64(U.shape[0])))
        self.factors[j] = U.copy()

    def update_entries(self, j, r, c, v):
        r = np.ascontiguousarray(r, dtype=np.uint64)
        c = np.ascontiguousarray(c, dtype=np.uint32)
        v = _c64(v)
        f = self._name("krp_update_entries", "update_entries")
        self.b.check(f(self.h, _u32(j), r.ctypes.data_as(C.POINTER(_u64)),
                       c.ctypes.data_as(C.POINTER(_u32)), _dptr(v), _u64(v.size)))
        for ri, ci, vi in zip(r, c, v):
            self.factors[j][ri, ci] = vi

    def node_gram(self, j, node):
        """Unpacked R x R Gram of a stored (root / left-child) node of factor j's tree."""
        R = self.R
        if self.b.kind == "ref":
            out = np.empty((R, R))
            self.b.check(self.b.fn("node_gram")(self.h, _u32(j), _u64(node), _dptr(out)))
            return out
        f = self.b.fn("krp_node_packed")
        f.restype = _dp
        p = f(self.h, _u32(j), _u64(node))
        packed = np.ctypeslib.as_array(p, shape=(R * (R + 1) // 2,)).copy()
        return unpack(packed, R)


def unpack(packed: np.ndarray, R: int) -> np.ndarray:
    """Packed upper triangle (row-major, segment_tree_sampler.hpp:111-115) -> R x R."""
    iu = np.triu_indices(R)
    G = np.zeros((R, R))
    G[iu] = packed
    G[(iu[1], iu[0])] = packed
    return G


class OracleTree:
    """SegmentTreeSampler through either oracle (segment_tree_sampler.hpp:26-95).
    Y=None -> rank-1 all-ones Y. The port stores every node (Full layout)."""

    def __init__(self, U, F, Y=None, backend="port", full=True):
        self.b = _Backend(backend)
        U = _c64(U)
        self.U = U.copy()
        self.R = U.shape[1]
        h = _vp()
        Yp = _dptr(_c64(Y)) if Y is not None else None
        self._Y = _c64(Y) if Y is not None else None
        if Y is not None:
            Yp = _dptr(self._Y)
        if backend == "port":
            self.b.check(self.b.fn("tree_create")(_dptr(self.U), _u64(U.shape[0]), _u32(self.R),
                                                  _u64(F), Yp, C.byref(h)))
        else:
            self.b.check(self.b.fn("tree_create")(_dptr(self.U), _u64(U.shape[0]), _u32(self.R),
                                                  _u64(F), Yp, C.c_int(1 if full else 0),
                                                  C.byref(h)))
        self.h = h
        for n in ("tree_node_count", "tree_leaf_count"):
            self.b.fn(n).restype = _u64

    @classmethod
    def from_sparse(cls, rows, cols, er, ec, ev, backend="port", full=True):
        """SegmentTreeSampler::from_sparse (segment_tree_sampler.cpp:67-109). The port
        restates the greedy R^2-nonzero leaf partition (:88-101) over the densified rows
        (ko_tree_create_segments); the reference backend calls from_sparse itself."""
        self = cls.__new__(cls)
        self.b = _Backend(backend)
        er = np.ascontiguousarray(er, dtype=np.uint32)
        ec = np.ascontiguousarray(ec, dtype=np.uint32)
        ev = _c64(ev)
        U = np.zeros((rows, cols))
        U[er.astype(np.int64), ec.astype(np.int64)] = ev
        self.U, self.R, self._Y = U, cols, None
        h = _vp()
        if backend == "ref":
            p32 = C.POINTER(C.c_uint32)
            self.b.check(self.b.fn("tree_create_sparse")(_u64(rows), _u64(cols), er.ctypes.data_as(p32),
                                                         ec.ctypes.data_as(p32), _dptr(ev), _u64(len(ev)),
                                                         C.c_int(1 if full else 0), C.byref(h)))
        else:
            counts = np.bincount(er.astype(np.int64), minlength=rows)
            offs, cur = [0], 0
            for i in range(rows):
                if cur + counts[i] > cols * cols and cur > 0:
                    offs.append(i)
                    cur = 0
                cur += int(counts[i])
            offs.append(rows)
            self.offsets = np.asarray(offs, dtype=np.uint64)
            self.b.check(self.b.fn("tree_create_segments")(_dptr(U), _u64(rows), _u32(cols),
                                                           self.offsets.ctypes.data_as(C.POINTER(_u64)),
                                                           _u64(len(offs) - 1), None, C.byref(h)))
        self.h = h
        for n in ("tree_node_count", "tree_leaf_count"):
            self.b.fn(n).restype = _u64
        return self

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.b.fn("tree_destroy")(h)
            self.h = None

    @property
    def node_count(self):
        return int(self.b.fn("tree_node_count")(self.h))

    @property
    def leaf_count(self):
        return int(self.b.fn("tree_leaf_count")(self.h))

    def node_gram(self, node):
        R = self.R
        if self.b.kind == "ref":
            out = np.empty((R, R))
            self.b.check(self.b.fn("tree_node_gram")(self.h, _u64(node), _dptr(out)))
            return out
        f = self.b.fn("tree_node_packed")
        f.restype = _dp
        p = f(self.h, _u64(node))
        return unpack(np.ctypeslib.as_array(p, shape=(R * (R + 1) // 2,)).copy(), R)

    def node_segment(self, node):
        a, b = _u64(0), _u64(0)
        if self.b.kind == "ref":
            self.b.check(self.b.fn("tree_node_segment")(self.h, _u64(node), C.byref(a), C.byref(b)))
        else:
            self.b.fn("tree_node_segment")(self.h, _u64(node), C.byref(a), C.byref(b))
        return int(a.value), int(b.value)

    def row_sample(self, h, seed, stream, n):
        h = _c64(h)
        out = np.empty(n, dtype=np.uint64)
        self.b.check(self.b.fn("tree_row_sample")(self.h, _dptr(h), _u64(seed), _u64(stream),
                                                   _u64(n), out.ctypes.data_as(C.POINTER(_u64))))
        return out

    def update_entry(self, r, c, v):
        self.b.check(self.b.fn("tree_update_entry")(self.h, _u64(r), _u64(c), C.c_double(v)))


def backend(kind: str = "port") -> _Backend:
    return _Backend(kind)


def random_matrix(rows, cols, seed, stream=0, kind="port"):
    """testsupport::random_matrix (tests/support.hpp:12-18): CounterRng normals."""
    return backend(kind).normals(seed, stream, rows * cols).reshape(rows, cols)
