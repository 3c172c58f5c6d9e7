"""Dev probe (GPU): real time spent in each layer of one staged L2HMC call."""
import sys, time, collections
sys.path.insert(0, ".")
import numpy as np
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins, executor, staging, ops, kernels
from paper_1903_01855_b200.workloads import l2hmc
sf.init_runtime(sf.RuntimeOptions()); plugins.install()
T = collections.defaultdict(int)
def wrap(obj, name, key):
    f = getattr(obj, name)
    def w(*a, **k):
        t = time.perf_counter_ns()
        try:
            return f(*a, **k)
        finally:
            T[key] += time.perf_counter_ns() - t
    setattr(obj, name, w)
B = 100000
s = l2hmc.L2HMCSampler(sf, B, "staged", seed=0)
for _ in range(3): s.step()
_native.sync(0)
wrap(_native.NativePlan, "run", "5 plan.run")
wrap(executor.Program, "_run_direct", "4 _run_direct")
wrap(executor, "_bind_inputs", "3b _bind_inputs")
wrap(executor, "execute_graph", "3 execute_graph")
wrap(ops, "_dispatch_eager", "2 _dispatch_eager")
wrap(staging, "call_concrete", "1b call_concrete")
wrap(staging.PolymorphicFunction, "__call__", "1 PolymorphicFunction.__call__")
x = s.x
n = 100
for _ in range(20): s.transition(x)
_native.sync(0); T.clear()
t0 = time.perf_counter_ns()
for _ in range(n): s.transition(x)
tt = time.perf_counter_ns() - t0
_native.sync(0)
print(f"total {tt/n/1e3:.1f} us/call (GPU runs behind)")
for k in sorted(T): print(f"  {k:34s} {T[k]/n/1e3:7.1f} us")
