"""TEST INFRASTRUCTURE ONLY -- the checker, never the product.

numpy restatement of one STS-CP factor update (the StsCp branch of the
reference's CP-ALS loop, /root/reference/proj/src/cp_als.cpp:279-313), given the
sample batch the sampler drew (indices, probabilities, rows; the batch itself is
pinned by the sampler parity tests):

  from_entries        tensor.cpp:34-75    dedup (sum) + lexicographic sort
  fiber_index         tensor.cpp:104-129  entries grouped by mode-j column
  matricize_column    tensor.cpp:20-32    lowest mode fastest, mode j skipped
  sampled_rhs_rows    cp_als.cpp:122-145  dense J x I_j block (small cases only)
  sampling_weights    sketch.cpp:36-52    w = 1/sqrt(J q), q > 0 required
  gram / gram_cross   dense_kernels.cpp:19-56  sequential sums over rows
  matmul              dense_kernels.cpp:209-223  sequential over k
  normalize_columns   cp_als.cpp:39-52

Every sum runs in the reference's order with plain IEEE mul/add, so with the
reference's pinv (the oracle port's Jacobi eigh, pinned to the reference) the
result is bit-identical to the reference itself (tests/test_sts_oracle.py).
"""
from __future__ import annotations

import numpy as np


def from_entries(dims, coords, values):
    """SparseTensorCoo::from_entries: coordinates validated, duplicates summed in
    sorted order, entries sorted lexicographically (mode 0 slowest)."""
    dims = [int(d) for d in dims]
    N = len(dims)
    coords = np.asarray(coords, dtype=np.uint32).reshape(-1, N)
    values = np.asarray(values, dtype=np.float64)
    if np.any(coords >= np.asarray(dims, dtype=np.uint64)):
        raise ValueError("SparseTensorCoo: coordinate out of range")
    order = np.lexsort(coords.T[::-1])  # stable
    out_c, out_v = [], []
    for e in order:
        c = tuple(int(x) for x in coords[e])
        if out_c and out_c[-1] == c:
            out_v[-1] += values[e]
        else:
            out_c.append(c)
            out_v.append(float(values[e]))
    return np.asarray(out_c, dtype=np.uint32).reshape(-1, N), np.asarray(out_v)


def matricize_column(c, j, dims):
    u, stride = 0, 1
    for k, d in enumerate(dims):
        if k == j:
            continue
        u += int(c[k]) * stride
        stride *= int(d)
    return u


def fiber_index(dims, coords, j):
    """keys (distinct columns ascending), ptr, order (entry ids)."""
    col = np.array([matricize_column(c, j, dims) for c in coords], dtype=np.uint64)
    order = np.argsort(col, kind="stable")
    keys, ptr = [], []
    for p, e in enumerate(order):
        if not keys or keys[-1] != col[e]:
            keys.append(int(col[e]))
            ptr.append(p)
    ptr.append(len(order))
    return np.asarray(keys, dtype=np.uint64), np.asarray(ptr, dtype=np.int64), order


def sampled_rhs_rows(dims, coords, values, j, idx):
    """Dense J x I_j rows of the mode-j matricization picked by the batch (the
    batch's flat index in RowOrder::Reversed = the matricization column)."""
    keys, ptr, order = fiber_index(dims, coords, j)
    J = idx.shape[0]
    out = np.zeros((J, int(dims[j])))
    lookup = {int(k): g for g, k in enumerate(keys)}
    for d in range(J):
        u = matricize_column(idx[d], j, dims)
        g = lookup.get(u)
        if g is None:
            continue
        for p in range(ptr[g], ptr[g + 1]):
            e = order[p]
            out[d, coords[e][j]] = values[e]
    return out


def sampling_weights(prob, J):
    prob = np.asarray(prob, dtype=np.float64)
    if np.any(~(prob > 0.0)) or np.any(~np.isfinite(prob)):
        raise ValueError("make_sampling_weights: sampled index has zero probability")
    return 1.0 / np.sqrt(float(J) * prob)


def _gram_cross(A, B):
    C = np.zeros((A.shape[1], B.shape[1]))
    for i in range(A.shape[0]):  # sequential over rows, like the reference's loops
        C += np.outer(A[i], B[i])
    return C


def _matmul(A, B):
    C = np.zeros((A.shape[0], B.shape[1]))
    for k in range(A.shape[1]):
        a = A[:, k:k + 1]
        C += np.where(a != 0.0, a * B[k:k + 1, :], 0.0)
    return C


def normalize_columns(U):
    U = U.copy()
    nrm = np.zeros(U.shape[1])
    for i in range(U.shape[0]):
        nrm += U[i] * U[i]
    sigma = np.sqrt(nrm)
    for c in range(U.shape[1]):
        if sigma[c] > 0.0:
            U[:, c] /= sigma[c]
        else:
            U[c % U.shape[0], c] = 1.0
    return U, sigma


def sts_step(dims, coords, values, j, idx, prob, rows, pinv):
    """One StsCp factor update from a sample batch (idx J x N with the excluded
    column ignored, prob J, rows J x R). `pinv(G)` = the reference's pinv_psd."""
    J = idx.shape[0]
    w = sampling_weights(prob, J)
    sa = rows * w[:, None]
    sb = sampled_rhs_rows(dims, coords, values, j, idx) * w[:, None]
    gs = _gram_cross(sa, sa)
    U = _matmul(pinv(gs), _gram_cross(sa, sb)).T
    return normalize_columns(U)
