import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins
from paper_1903_01855_b200.workloads import l2hmc
sf.init_runtime(sf.RuntimeOptions()); plugins.install()
B = 100000
s = l2hmc.L2HMCSampler(sf, B, "staged", seed=0)
for _ in range(3): s.step()
_native.sync(0)
xh = s.x.numpy()
T = {"make": 0, "upload": 0, "call": 0, "sync": 0, "d2h": 0}
n = 10
for _ in range(n):
    t0 = time.perf_counter(); x = sf.tensor_from_host(xh, (B, 2), sf.float32)
    t1 = time.perf_counter(); x._ptr()
    t2 = time.perf_counter(); xo, acc = s.transition(x)
    t3 = time.perf_counter(); _native.sync(0)
    t4 = time.perf_counter(); a = xo.numpy(); b = acc.numpy()
    t5 = time.perf_counter()
    for k, v in zip(T, (t1-t0, t2-t1, t3-t2, t4-t3, t5-t4)): T[k] += v
print({k: round(v / n * 1e3, 3) for k, v in T.items()}, "ms")
