import time, sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle
from parity_util import pareto_factors
t=time.time()
I=1<<22; R=64
rng=np.random.default_rng(5)
fs=[rng.standard_normal((I,R)) for _ in range(3)]
print('gen', time.time()-t, flush=True)
t=time.time()
o=oracle.OracleKrp(fs,'port')
print('oracle build', time.time()-t, flush=True)
t=time.time()
ri,rp,rr,rm=o.sample(None, 2048, 11, want_margin=True, draw_offset=1000000)
print('oracle sample 2048', time.time()-t, flush=True)
