"""Staged ResNet-50 C4 step time only (bench.py's resnet_extra staged leg):
a short command for iterating on the ResNet kernels.

    python tools/c4_time.py [steps] [staged|eager]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, nn  # noqa: E402
from paper_1903_01855_b200.workloads import resnet  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
mode = sys.argv[2] if len(sys.argv) > 2 else "staged"
sf.init_runtime(sf.RuntimeOptions())
nn.install()
tr = resnet.ResNetTrain(sf, batch=32, mode=mode, image=224, seed=0)
dt = bench._time_steps(tr.step, n, _native, warm=3)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("SF_")},
                  "mode": mode, "c4_ms": dt * 1e3, "img_per_sec": 32 / dt}))
_ = np
