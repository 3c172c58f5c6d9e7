"""Where the L2HMC headline e2e step (bench.py e2e: host state in, host
state + acceptance out, through the public API) spends its time.

    python tools/e2e_breakdown.py [chains]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, plugins  # noqa: E402
from paper_1903_01855_b200.workloads import l2hmc  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
sf.init_runtime(sf.RuntimeOptions(seed=1))
plugins.install()
s = l2hmc.L2HMCSampler(sf, B, "staged", seed=0)
for _ in range(5):
    s.step()
_native.sync(0)
x_host = s.x.raw()
n = 200


def timed(fn):
    for _ in range(5):
        fn()
    _native.sync(0)
    t = time.perf_counter()
    for _ in range(n):
        fn()
    _native.sync(0)
    return (time.perf_counter() - t) / n * 1e6


out = {}
out["h2d_only_us"] = timed(lambda: sf.tensor_from_host(x_host, (B, 2), sf.float32)._ptr())
xd = sf.tensor_from_host(x_host, (B, 2), sf.float32)
out["transition_device_in_out_us"] = timed(lambda: s.transition(xd))
xo, acc = s.transition(xd)
_native.sync(0)


def reads():
    a, b = s.transition(xd)
    a.raw(), b.raw()


out["transition_plus_d2h_us"] = timed(reads)


def e2e():
    global x_host
    x = sf.tensor_from_host(x_host, (B, 2), sf.float32)
    a, b = s.transition(x)
    x_host = a.raw()
    b.raw()


out["e2e_us"] = timed(e2e)
print(json.dumps(out))
_ = np
