"""CPU: the C-ABI library loads, exports every symbol include/krpg.h declares,
and its host-only logic (tree topology, R x R eigensolver) matches the oracle.
No compute call needs a GPU here; without one, device entry points must fail
loudly (no CPU fallback)."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2301_12584_b200 import _lib


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _lib.declared_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing


def test_python_signatures_cover_the_header():
    assert set(_lib.declared_symbols()) == set(_lib._SIGS)


def _node_rows(I, F, v):
    L = _lib.lib()
    f, l, lc, nc = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = L.krpg_topology_node_rows(C.c_uint64(I), C.c_uint64(F), C.c_uint64(v), C.byref(f), C.byref(l),
                                   C.byref(lc), C.byref(nc))
    _lib.check(rc)
    return (int(f.value), int(l.value)), int(lc.value), int(nc.value)


@pytest.mark.parametrize("I,F", [(1, 1), (2, 1), (3, 1), (5, 2), (64, 4), (29, 3), (33, 4), (100, 7),
                                 (4096, 16), (1000, 64), (257, 1), (5000, 64), (3, 8)])
def test_device_topology_matches_reference_init_tree(I, F):
    """krpg_device.cuh Topo/node_rows == SegmentTreeSampler::init_tree (segment_tree_sampler.cpp:111-149)."""
    t = oracle.OracleTree(np.ones((I, 2)), F, None, "port")
    for v in range(t.node_count):
        seg, lc, nc = _node_rows(I, F, v)
        assert lc == t.leaf_count and nc == t.node_count
        assert seg == t.node_segment(v), (I, F, v)


def test_topology_rejects_out_of_range():
    with pytest.raises(_lib.KrpgInvalidArgument):
        _node_rows(10, 2, 9)


def _host_eigh(G):
    L = _lib.lib()
    n = G.shape[0]
    G = np.ascontiguousarray(G, dtype=np.float64)
    V = np.empty((n, n))
    lam = np.empty(n)
    dp = C.POINTER(C.c_double)
    _lib.check(L.krpg_host_eigh(G.ctypes.data_as(dp), C.c_uint32(n), V.ctypes.data_as(dp), lam.ctypes.data_as(dp)))
    return V, lam


@pytest.mark.parametrize("n", [1, 2, 3, 7, 16, 64, 128])
def test_host_eigensolver_matches_reference_eigh(n):
    """host_linalg.cpp (Householder + QL) vs the reference Jacobi (dense_kernels.cpp:93-176):
    same eigenvalues to 1e-12 relative, same invariant subspaces, descending order."""
    B = oracle.random_matrix(2 * n, n, 31 + n)
    G = B.T @ B
    V, lam = _host_eigh(G)
    Vr, lr = oracle.backend("port").eigh(G)
    assert np.all(np.diff(lam) <= 0)
    assert np.max(np.abs(lam - lr)) <= 1e-12 * lr[0]
    assert np.max(np.abs(V.T @ V - np.eye(n))) < 1e-13
    # eigenvectors agree up to sign
    assert np.max(np.abs(np.abs(np.sum(V * Vr, axis=0)) - 1.0)) < 1e-9
    assert np.max(np.abs(V @ np.diag(lam) @ V.T - G)) < 1e-12 * lr[0]


def test_host_eigensolver_error_classes():
    with pytest.raises(_lib.KrpgInvalidArgument):
        _host_eigh(np.array([[1.0, 2.0], [0.0, 1.0]]))  # asymmetric
    with pytest.raises(_lib.KrpgInvalidArgument):
        _host_eigh(np.array([[1.0, 0.0], [0.0, -1.0]]))  # indefinite


def test_identity_eigenvectors_are_canonical():
    V, lam = _host_eigh(np.eye(4))
    assert np.array_equal(np.abs(V), np.eye(4)) and np.array_equal(lam, np.ones(4))


def test_device_entry_points_fail_loudly_without_gpu():
    if _lib.lib().krpg_device_count() > 0:
        pytest.skip("a GPU is present")
    from paper_2301_12584_b200 import KrpSampler, KrpgError
    with pytest.raises(KrpgError):
        KrpSampler([np.ones((4, 2)), np.ones((3, 2))])
