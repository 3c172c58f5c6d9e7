"""One staged ResNet-50 b32 training step after warm-up, bracketed by
cudaProfilerStart/Stop — the command for ncu launch lists of the C4 step
(`ncu --profile-from-start off ...`).

    python tools/resnet_step.py [batch]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402  (profiler range only)

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, nn  # noqa: E402
from paper_1903_01855_b200.workloads import resnet  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sf.init_runtime(sf.RuntimeOptions())
nn.install()
tr = resnet.ResNetTrain(sf, batch=batch, mode="staged", seed=0)
for _ in range(4):
    tr.step()
_native.sync(0)
t = time.perf_counter()
torch.cuda.profiler.start()
tr.step()
_native.sync(0)
torch.cuda.profiler.stop()
print("step ms", (time.perf_counter() - t) * 1e3)
