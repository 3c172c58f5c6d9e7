"""C2 microbenchmark staged / eager timing (wall clock per chain incl. host
cost; device time of the staged chain with CUDA events).

    python tools/c2_time.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402  (events only)

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, plugins  # noqa: E402
from paper_1903_01855_b200.workloads import microbench  # noqa: E402

sf.init_runtime(sf.RuntimeOptions())
plugins.install()
out = {}
for mode, n in (("staged", 200), ("eager", 50)):
    ch = microbench.Chain(mode)
    for _ in range(3):
        ch.step()
    _native.sync(0)
    t = time.perf_counter()
    for _ in range(n):
        ch.step()
    _native.sync(0)
    out[mode + "_us_per_op"] = (time.perf_counter() - t) / n * 1e6 / 300
    if mode == "staged":
        stream = torch.cuda.ExternalStream(_native.stream_of(0))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            ch.step()
        e1.record(stream)
        e1.synchronize()
        out["staged_device_us_per_chain"] = e0.elapsed_time(e1) * 1e3 / n
print(json.dumps(out))
