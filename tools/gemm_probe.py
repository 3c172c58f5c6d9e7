"""Dev probe (GPU): tcgen05 3xTF32 GEMM time, lo precomputed vs derived in shared memory."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native
sf.init_runtime(sf.RuntimeOptions())
stream = torch.cuda.ExternalStream(_native.stream_of(0))
shapes = [(100352, 64, 576), (100352, 256, 64), (25088, 128, 1152), (6272, 256, 2304),
          (1568, 512, 4608), (100352, 64, 64), (4096, 4096, 4096)]
for m, n, k in shapes:
    a = sf.constant(np.random.default_rng(0).standard_normal((m, k)).astype(np.float32))
    b = sf.constant(np.random.default_rng(1).standard_normal((n, k)).astype(np.float32))
    ah, al = _native.split_tf32(0, m, k, a._ptr())
    bh, bl = _native.split_tf32(0, n, k, b._ptr())
    res = []
    for lo in (True, False):
        f = (lambda: _native.gemm_tf32x3(0, m, n, k, ah.ptr, al.ptr, bh.ptr, bl.ptr)) if lo else \
            (lambda: _native.gemm_tf32x3(0, m, n, k, ah.ptr, 0, bh.ptr, 0))
        for _ in range(3): f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(20): f()
        e1.record(stream); _native.sync(0)
        ms = e0.elapsed_time(e1) / 20
        res.append((ms, 2 * m * n * k / ms / 1e9))
    print(f"{m}x{n}x{k}: lo-in-HBM {res[0][0]*1e3:7.1f} us {res[0][1]:6.1f} TF | lo-in-smem {res[1][0]*1e3:7.1f} us {res[1][1]:6.1f} TF")
