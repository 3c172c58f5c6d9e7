"""Dev probe (GPU): does tcgen05 kind::tf32 ignore the low 13 mantissa bits of
fp32 operands (i.e. is the raw fp32 tile usable as the TF32 'hi' part)?"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native
sf.init_runtime(sf.RuntimeOptions())
rng = np.random.default_rng(0)
for (m, n, k) in [(256, 64, 64), (1024, 128, 576), (300, 200, 100)]:
    a = sf.constant(rng.standard_normal((m, k)).astype(np.float32))
    b = sf.constant(rng.standard_normal((n, k)).astype(np.float32))
    ahi, alo = _native.split_tf32(0, m, k, a._ptr())
    bhi, blo = _native.split_tf32(0, n, k, b._ptr())
    ref = _native.gemm_tf32x3(0, m, n, k, ahi.ptr, alo.ptr, bhi.ptr, blo.ptr)
    raw = _native.gemm_tf32x3(0, m, n, k, a._ptr(), alo.ptr, b._ptr(), blo.ptr)
    r1 = _native.download(ref, np.float32, (m, n)); r2 = _native.download(raw, np.float32, (m, n))
    print((m, n, k), "bitwise equal:", r1.tobytes() == r2.tobytes(), "max diff", float(np.abs(r1 - r2).max()))
