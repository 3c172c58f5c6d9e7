"""L2HMC training step time (workloads/l2hmc.py L2HMCTrain), staged and
eager, wall clock per step incl. host cost.

    python tools/l2hmc_train_time.py 200 10000
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, plugins  # noqa: E402
from paper_1903_01855_b200.workloads import l2hmc  # noqa: E402

out = {}
for b in [int(x) for x in sys.argv[1:]] or [200]:
    row = {}
    for mode, n in (("staged", 20), ("eager", 2)):
        if mode == "eager" and b > 1000:
            continue
        sf.init_runtime(sf.RuntimeOptions(seed=1))
        plugins.install()
        tr = l2hmc.L2HMCTrain(sf, b, mode, seed=0)
        t = time.perf_counter()
        tr.step()
        _native.sync(0)
        first = time.perf_counter() - t
        tr.step()
        _native.sync(0)
        t = time.perf_counter()
        for _ in range(n):
            tr.step()
        _native.sync(0)
        dt = (time.perf_counter() - t) / n
        row[mode] = {"ms_per_step": dt * 1e3, "samples_per_sec": b / dt, "first_step_s": first}
    out[b] = row
print(json.dumps(out))
