"""Dev probe (GPU): per-step event times of the bench loop, with/without L2 flush + clock sampler."""
import sys, time
sys.path.insert(0, ".")
import torch
import bench
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins
from paper_1903_01855_b200.workloads import l2hmc

sf.init_runtime(sf.RuntimeOptions()); plugins.install()
s = l2hmc.L2HMCSampler(sf, 100000, "staged", seed=0)
for _ in range(3): s.step()
_native.sync(0)
stream = torch.cuda.ExternalStream(_native.stream_of(0))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for flush_on in (True, False):
    for clocks in (True, False):
        times = []
        cm = bench.Clocks(0) if clocks else None
        if cm: cm.__enter__()
        for _ in range(20):
            with torch.cuda.stream(stream):
                if flush_on: flush.fill_(1.0)
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            s.step()
            e1.record(stream)
            times.append((e0, e1))
        _native.sync(0); torch.cuda.synchronize()
        if cm: cm.__exit__(None, None, None)
        ms = [a.elapsed_time(b) for a, b in times]
        print(f"flush={flush_on} clocks={clocks}: " + " ".join(f"{m:.3f}" for m in ms))
