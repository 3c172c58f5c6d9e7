"""Time one float32 convolution forward: implicit GEMM (sf_conv2d_tc) vs
im2col + GEMM, at ResNet-50 b32 layer shapes.

    python tools/conv_time.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402  (events only)

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, nn  # noqa: E402

sf.init_runtime(sf.RuntimeOptions())
nn.install()
stream = torch.cuda.ExternalStream(_native.stream_of(0))
out = {}
for (n, h, c, co, k, s, p) in [(32, 56, 64, 64, 3, 1, 1), (32, 28, 128, 128, 3, 1, 1),
                               (32, 14, 256, 256, 3, 1, 1), (32, 7, 512, 512, 3, 1, 1),
                               (32, 56, 256, 512, 1, 2, 0)]:
    rng = np.random.default_rng(0)
    x = sf.constant(rng.standard_normal((n, h, h, c)).astype(np.float32))
    w = sf.constant(rng.standard_normal((k, k, c, co)).astype(np.float32))
    row = {}
    for mode in (True, False):
        nn.IMPLICIT_CONV = mode
        for _ in range(3):
            nn.conv2d(x, w, s, p)
        _native.sync(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(20):
            nn.conv2d(x, w, s, p)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        ho = (h + 2 * p - k) // s + 1
        flops = 2 * n * ho * ho * co * k * k * c
        row["implicit" if mode else "explicit"] = {"us": ms * 1e3, "useful_tflops": flops / ms / 1e9}
    out[f"{n}x{h}x{h}x{c} k{k} s{s} -> {co}"] = row
print(json.dumps(out, indent=1))
