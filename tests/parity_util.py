"""Shared parity helpers: compare the device sampler with a CPU oracle.

Indices must be bit-exact except for *boundary draws*: draws whose uniform lies
within ``tol`` (1e-10, north_star) of a branch / leaf-scan threshold in either
implementation. Such draws are counted, and any mismatch outside that margin
is a failure.
"""
from __future__ import annotations

import numpy as np

BOUNDARY_TOL = 1e-10


def rel_err_matrix(A: np.ndarray, B: np.ndarray) -> float:
    """max |A-B| / sqrt(diag(A)_a diag(A)_b): Gram-scale relative error."""
    d = np.sqrt(np.abs(np.outer(np.diag(B), np.diag(B))))
    d = np.maximum(d, np.finfo(float).tiny)
    return float(np.max(np.abs(A - B) / d))


def compare_draws(gpu_idx, gpu_margin, ref_idx, ref_margin=None, tol=BOUNDARY_TOL):
    """Returns (n_mismatch, n_boundary_mismatch, n_unexplained)."""
    mism = np.any(gpu_idx != ref_idx, axis=1)
    n = int(mism.sum())
    m = gpu_margin[mism]
    if ref_margin is not None:
        m = np.minimum(m, ref_margin[mism])
    boundary = m <= tol
    return n, int(boundary.sum()), int((~boundary).sum())


def rel_err_vec(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


def rows_rel_err(a, b):
    """max over draws of |a-b|_inf / |b|_inf (rows are Hadamard products)."""
    a = np.asarray(a)
    b = np.asarray(b)
    scale = np.maximum(np.max(np.abs(b), axis=1, keepdims=True), 1e-300)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


def pareto_factors(shapes, seed, frac=1.0, alpha=1.5):
    """Config-1/2 inputs: N(0,1) entries, rows scaled by a Pareto(alpha) weight
    w = (1-u)^(-1/alpha); frac < 1 scales only that fraction of rows."""
    rng = np.random.default_rng(seed)
    out = []
    for (I, R) in shapes:
        U = rng.standard_normal((I, R))
        u = rng.random(I)
        w = (1.0 - rng.random(I)) ** (-1.0 / alpha)
        if frac < 1.0:
            w = np.where(u < frac, w, 1.0)
        out.append(U * w[:, None])
    return out


def config1_factors(shapes=((4096, 16),) * 3, seed=2301, kind="port"):
    """Config-1 inputs built only from the reference CounterRng (rng.hpp:13-48,
    support.hpp:12-18): entries N(0,1) from stream k, every row scaled by a
    Pareto(1.5) weight w = (1-u)^(-1/1.5) with u from stream 1000+k."""
    import oracle
    b = oracle.backend(kind)
    out = []
    for k, (I, R) in enumerate(shapes):
        U = b.normals(seed, k, I * R).reshape(I, R)
        u = b.uniforms(seed, 1000 + k, I)
        w = np.power(1.0 - u, -1.0 / 1.5)
        out.append(U * w[:, None])
    return out


def spiked_factors(shapes, seed, frac=0.01, scale=10.0, kind="port"):
    """testsupport::random_spiked_matrix (support.hpp:21-31): N(0,1) with about
    `frac` of entries scaled by `scale`, normal and uniform interleaved per entry."""
    import oracle
    b = oracle.backend(kind)
    out = []
    for k, (I, R) in enumerate(shapes):
        n = I * R
        # one normal() consumes two uniforms, then one uniform: 3 per entry
        u = b.uniforms(seed + k, 0, 3 * n).reshape(n, 3)
        z = np.sqrt(-2.0 * np.log(1.0 - u[:, 0])) * np.cos(6.283185307179586476925 * u[:, 1])
        z = np.where(u[:, 2] < frac, z * scale, z)
        out.append(z.reshape(I, R))
    return out


def digest(arrays) -> str:
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def sparse_tensor(dims, nnz, seed, s=1.1):
    """Synthetic COO in the config-5 style: per-mode Zipf(s)-skewed
    coordinates (so fibers repeat and duplicates occur), lognormal(0,1) values.
    Raw entries, duplicates not yet summed."""
    rng = np.random.default_rng(seed)
    coords = np.empty((nnz, len(dims)), dtype=np.uint32)
    for k, d in enumerate(dims):
        ranks = np.arange(1, d + 1, dtype=float)
        p = ranks ** (-s)
        p /= p.sum()
        perm = rng.permutation(d)  # popular indices scattered over the mode
        coords[:, k] = perm[rng.choice(d, size=nnz, p=p)]
    values = rng.lognormal(0.0, 1.0, size=nnz)
    return coords, values
