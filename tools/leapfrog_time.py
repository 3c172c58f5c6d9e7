"""Staged / eager time per trajectory of the reference-pinned leapfrog
workload (bench.py extra "leapfrog") at the given batch sizes.

    python tools/leapfrog_time.py 200 100000
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, plugins  # noqa: E402
from paper_1903_01855_b200.workloads.leapfrog import Leapfrog  # noqa: E402

out = {}
for b in [int(x) for x in sys.argv[1:]] or [200]:
    sf.init_runtime(sf.RuntimeOptions(seed=0))
    plugins.install()
    lf = Leapfrog(b, "staged")
    dt = bench._time_steps(lf.step, 200, _native, warm=5)
    import time
    t = time.perf_counter()
    for _ in range(200):
        lf.step()
    _native.sync(0)
    out[b] = {"us_per_trajectory": dt * 1e6,
              "no_gc_freeze_us": (time.perf_counter() - t) / 200 * 1e6}
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("SF_")}, **out}))
