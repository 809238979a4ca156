import time, numpy as np, ctypes as C, sys
sys.path.insert(0, '/root/repo')
from paper_2301_12584_b200 import _lib
lib = _lib.lib()
for n in (64, 128, 256):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((4*n, n)); G = A.T @ A
    V = np.empty((n, n)); w = np.empty(n)
    p = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))
    lib.krpg_host_eigh(p(G), n, p(V), p(w))
    reps = 20 if n < 256 else 8
    t = time.perf_counter()
    for _ in range(reps): lib.krpg_host_eigh(p(G), n, p(V), p(w))
    dt = (time.perf_counter() - t) / reps
    print(n, f"host eigh {dt*1e3:.3f} ms", flush=True)
