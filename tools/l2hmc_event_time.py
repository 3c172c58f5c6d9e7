"""Device time per staged L2HMC transition (CUDA events around N back-to-back
steps on the backend stream) vs the wall clock per step: separates kernel
latency from host cost at small chain counts.

    python tools/l2hmc_event_time.py 200 10000
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402  (events only)

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, plugins  # noqa: E402
from paper_1903_01855_b200.workloads import l2hmc  # noqa: E402

out = {}
stream = torch.cuda.ExternalStream(_native.stream_of(0))
for b in [int(x) for x in sys.argv[1:]] or [200]:
    sf.init_runtime(sf.RuntimeOptions(seed=1))
    plugins.install()
    s = l2hmc.L2HMCSampler(sf, b, "staged", seed=0)
    for _ in range(5):
        s.step()
    _native.sync(0)
    n = 50
    if os.environ.get("FLUSH") == "1":
        # as bench.py times the headline: 256 MiB written between steps
        buf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
        ts = []
        for _ in range(n):
            with torch.cuda.stream(stream):
                buf.fill_(1.0)
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
            s.step()
            a1.record(stream)
            ts.append((a0, a1))
        _native.sync(0)
        out[f"{b}_flushed"] = {"device_us": sum(a.elapsed_time(c) for a, c in ts) * 1e3 / n}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t = time.perf_counter()
    for _ in range(n):
        s.step()
    e1.record(stream)
    host = (time.perf_counter() - t) / n * 1e6
    e1.synchronize()
    out[b] = {"device_us": e0.elapsed_time(e1) * 1e3 / n, "host_enqueue_us": host}
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("SF_")}, **out}))
