"""Dev probe (GPU): MN-major tcgen05 GEMM operands vs numpy."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native
sf.init_runtime(sf.RuntimeOptions())
rng = np.random.default_rng(0)
for (m, n, k) in [(128, 64, 32), (128, 128, 32), (256, 128, 64)]:
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((n, k)).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64).T
    for a_mn, b_mn in [(False, False), (False, True), (True, False), (True, True)]:
        As = np.ascontiguousarray(a.T if a_mn else a); Bs = np.ascontiguousarray(b.T if b_mn else b)
        ta, tb = sf.constant(As), sf.constant(Bs)
        ah, al = _native.split_tf32(0, *As.shape, ta._ptr())
        bh, bl = _native.split_tf32(0, *Bs.shape, tb._ptr())
        c = _native.gemm_tf32x3_ex(0, m, n, k, a_mn, b_mn, k, k, ah.ptr, al.ptr, bh.ptr, bl.ptr)
        got = _native.download(c, np.float32, (m, n))
        err = np.abs(got - want).max()
        # which transpose of the truth does it match?
        print((m, n, k), a_mn, b_mn, "maxabs", float(np.abs(got).max()), "err", float(err),
              "nonzero frac", float((got != 0).mean()))
