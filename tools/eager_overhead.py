"""Host cost per eager op: native front-end + launch queue vs one launch per
op vs the Python dispatcher (prints one JSON line).

    python tools/eager_overhead.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _fastpath, _native, plugins  # noqa: E402
from paper_1903_01855_b200.workloads import microbench  # noqa: E402
from paper_1903_01855_b200.workloads.leapfrog import Leapfrog  # noqa: E402


def mode(name):
    _fastpath.set_enabled(name != "python")
    _native.queue_config(0, 64 if name == "queue" else 0)


def timeit(fn, reps):
    fn()
    _native.sync(0)
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    _native.sync(0)
    return (time.perf_counter() - t) / reps


def main():
    sf.init_runtime(sf.RuntimeOptions())
    plugins.install()
    out = {}
    x = sf.constant(np.ones((1, 16), np.float32))
    for m in ("queue", "direct", "python"):
        mode(m)
        r = {}
        rt = sf.get_runtime()
        f0 = _fastpath.pending(rt)
        q0 = _native.queue_stats(0)
        r["add_us"] = timeit(lambda: sf.add(x, x), 20000) * 1e6
        r["fast_dispatches"] = _fastpath.pending(rt) - f0
        r["queue_pushed_flushes"] = [a - b for a, b in zip(_native.queue_stats(0), q0)]
        r["dispatch_add_us"] = timeit(lambda: _fastpath.ext.dispatch("add", [x, x]), 20000) * 1e6
        r["noop_us"] = timeit(lambda: None, 20000) * 1e6
        r["mul_scalar_us"] = timeit(lambda: x * 0.5, 20000) * 1e6
        ch = microbench.Chain("eager", seed=0)
        r["c2_us_per_op"] = timeit(lambda: ch.step().numpy(), 50) * 1e6 / 300
        lf = Leapfrog(200, "eager", seed=0)
        r["leapfrog200_us_per_dispatch"] = timeit(lf.run_iteration, 20) * 1e6 / 260
        out[m] = r
    mode("queue")
    print(json.dumps({"eager_overhead": out}))


if __name__ == "__main__":
    main()
