"""Staged L2HMC transition time (CUDA events, warm) over chain counts —
for A/B runs of row-kernel code-generation options (SF_ROW_* env vars).

    python tools/l2hmc_sweep.py 200 10000 100000
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, plugins  # noqa: E402
from paper_1903_01855_b200.workloads import l2hmc  # noqa: E402

out = {}
for b in [int(x) for x in sys.argv[1:]] or [200, 100000]:
    sf.init_runtime(sf.RuntimeOptions(seed=1))
    plugins.install()
    s = l2hmc.L2HMCSampler(sf, b, "staged", seed=0)
    for _ in range(3):
        s.step()
    _native.sync(0)
    import time
    n = 50
    t = time.perf_counter()
    for _ in range(n):
        s.step()
    _native.sync(0)
    out[b] = (time.perf_counter() - t) / n * 1e6
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("SF_")},
                  "us_per_transition": out}))
