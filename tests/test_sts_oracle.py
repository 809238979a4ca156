"""CPU: the STS-CP restatement (oracle/sts_cp.py) pinned against the reference
itself (oracle/_ref: SparseTensorCoo::from_entries, sampled_rhs_rows, gram,
gram_cross, pinv_psd, matmul -- the StsCp branch of cp_als.cpp:279-313)."""
import ctypes as C

import numpy as np
import pytest

import oracle
from oracle import sts_cp
from parity_util import pareto_factors, sparse_tensor

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")

DIMS = (40, 30, 25)


def _ref():
    return oracle.backend("ref")


def test_from_entries_matches_reference():
    coords, values = sparse_tensor(DIMS, 3000, seed=1)
    b = _ref()
    n = C.c_uint64()
    dims = (C.c_uint64 * 3)(*DIMS)
    cp = coords.ctypes.data_as(C.POINTER(C.c_uint32))
    vp = values.ctypes.data_as(C.POINTER(C.c_double))
    b.check(b.fn("tensor_entries")(dims, C.c_uint32(3), cp, vp, C.c_uint64(len(values)), None, None, C.byref(n)))
    rc = np.empty((n.value, 3), dtype=np.uint32)
    rv = np.empty(n.value)
    b.check(b.fn("tensor_entries")(dims, C.c_uint32(3), cp, vp, C.c_uint64(len(values)),
                                   rc.ctypes.data_as(C.POINTER(C.c_uint32)), rv.ctypes.data_as(C.POINTER(C.c_double)),
                                   C.byref(n)))
    oc, ov = sts_cp.from_entries(DIMS, coords, values)
    assert np.array_equal(oc, rc)
    assert np.allclose(ov, rv, rtol=1e-15, atol=0)  # duplicate sums may associate differently
    assert len(ov) < len(values)  # the fixture does contain duplicates


@pytest.mark.parametrize("j", [0, 1, 2])
def test_sts_step_restatement_matches_reference(j):
    R, J, seed = 6, 2000, 17
    fs = pareto_factors([(d, R) for d in DIMS], seed=3)
    coords, values = sparse_tensor(DIMS, 3000, seed=2)
    oc, ov = sts_cp.from_entries(DIMS, coords, values)
    b = _ref()
    # reference end to end
    I = (C.c_uint64 * 3)(*DIMS)
    fptr = (C.POINTER(C.c_double) * 3)(*[f.ctypes.data_as(C.POINTER(C.c_double)) for f in fs])
    unew = np.empty((DIMS[j], R))
    sigma = np.empty(R)
    b.check(b.fn("sts_step")(fptr, I, C.c_uint32(3), C.c_uint32(R), oc.ctypes.data_as(C.POINTER(C.c_uint32)),
                             ov.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint64(len(ov)), C.c_uint32(j),
                             C.c_uint64(J), C.c_uint64(seed), unew.ctypes.data_as(C.POINTER(C.c_double)),
                             sigma.ctypes.data_as(C.POINTER(C.c_double))))
    # restatement on the reference's own batch
    idx, prob, rows = oracle.OracleKrp(fs, "ref").sample(j, J, seed)
    U, sg = sts_cp.sts_step(DIMS, oc, ov, j, idx, prob, rows, lambda G: b.pinv(G)[0])
    assert np.array_equal(sg, sigma)
    assert np.array_equal(U, unew)
