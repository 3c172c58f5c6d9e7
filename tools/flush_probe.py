"""Dev probe (GPU): cost of a cold L2 on the staged L2HMC step, by chain count and flush kind."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins
from paper_1903_01855_b200.workloads import l2hmc

sf.init_runtime(sf.RuntimeOptions()); plugins.install()
stream = torch.cuda.ExternalStream(_native.stream_of(0))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for B in (1000, 100000):
    s = l2hmc.L2HMCSampler(sf, B, "staged", seed=0)
    for _ in range(3): s.step()
    _native.sync(0)
    for kind in ("none", "write", "read"):
        times = []
        for _ in range(15):
            with torch.cuda.stream(stream):
                if kind == "write": flush.fill_(1.0)
                elif kind == "read": flush.sum()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            s.step()
            e1.record(stream)
            times.append((e0, e1))
        _native.sync(0); torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in times[3:])
        print(f"B={B} flush={kind}: median {ms[len(ms)//2]:.3f} ms")
