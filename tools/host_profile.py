"""Dev probe (GPU): host-side cost of one staged L2HMC transition call."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins
from paper_1903_01855_b200.workloads import l2hmc

sf.init_runtime(sf.RuntimeOptions()); plugins.install()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
s = l2hmc.L2HMCSampler(sf, B, "staged", seed=0)
for _ in range(3): s.step()
_native.sync(0)
n = 200
t = time.perf_counter()
for _ in range(n): s.step()
host = (time.perf_counter() - t) / n
_native.sync(0)
wall = (time.perf_counter() - t) / n
print(f"host {host*1e6:.1f} us/call, wall {wall*1e6:.1f} us/step")
pr = cProfile.Profile(); pr.enable()
for _ in range(n): s.step()
pr.disable(); _native.sync(0)
pstats.Stats(pr).sort_stats(sys.argv[2] if len(sys.argv) > 2 else "tottime").print_stats(30)
