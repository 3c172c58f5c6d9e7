"""Dev probe (GPU): where the end-to-end (host buffers in, host results out) time goes."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins
from paper_1903_01855_b200.workloads import l2hmc
sf.init_runtime(sf.RuntimeOptions()); plugins.install()
B = 100000
s = l2hmc.L2HMCSampler(sf, B, "staged", seed=0)
for _ in range(3): s.step()
_native.sync(0)
x_np = torch.from_numpy(s.x.numpy()).pin_memory().numpy()
T = {"make": 0, "call": 0, "d2h_x": 0, "d2h_acc": 0, "copyto": 0}
n = 20
def loop(n):
    for _ in range(n):
        t0 = time.perf_counter(); x = sf.tensor_from_host(x_np, (B, 2), sf.float32)
        t1 = time.perf_counter(); xo, acc = s.transition(x)
        t2 = time.perf_counter(); a = xo.numpy()
        t3 = time.perf_counter(); b = acc.numpy()
        t4 = time.perf_counter(); np.copyto(x_np, a)
        t5 = time.perf_counter()
        for k, v in zip(T, (t1-t0, t2-t1, t3-t2, t4-t3, t5-t4)): T[k] += v
loop(5)
for k in T: T[k] = 0
loop(n)
print({k: round(v / n * 1e3, 3) for k, v in T.items()}, "ms", "total", round(sum(T.values()) / n * 1e3, 3))
pr = cProfile.Profile(); pr.enable(); loop(n); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
