"""Quick wall-clock probe of the main workloads (development aid)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins
from paper_1903_01855_b200.workloads.leapfrog import Leapfrog
from paper_1903_01855_b200.workloads.l2hmc import L2HMCSampler


def timeit(fn, n):
    fn(); fn()
    _native.sync(0)
    t = time.perf_counter()
    for _ in range(n):
        fn()
    _native.sync(0)
    return (time.perf_counter() - t) / n


sf.init_runtime(sf.RuntimeOptions())
for b in (200, 100000):
    for mode in ("eager", "staged"):
        wl = Leapfrog(b, mode)
        dt = timeit(wl.step, 20 if mode == "staged" else 3)
        print(f"leapfrog B={b} {mode}: {dt*1e6:.1f} us/traj, {b/dt:.3e} chains/s", flush=True)
plugins.install()
for b in (200,):
    for mode in ("staged", "eager"):
        t0 = time.perf_counter()
        wl = L2HMCSampler(sf, b, mode)
        wl.step()
        _native.sync(0)
        print(f"l2hmc first call {mode}: {time.perf_counter()-t0:.2f}s", flush=True)
        dt = timeit(wl.step, 5)
        print(f"l2hmc B={b} {mode}: {dt*1e3:.2f} ms/transition, {b/dt:.3e} samples/s", flush=True)
        if mode == "staged":
            prog = list(wl.transition.cached_functions()[0].graph._plan.values())[0]
            print("  segments", len(prog.segments), "launches", prog.n_launches)
