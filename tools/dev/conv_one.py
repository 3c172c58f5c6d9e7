import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, nn
sf.init_runtime(sf.RuntimeOptions()); nn.install()
n, h, c, co, k, s, p = [int(v) for v in sys.argv[1:8]]
rng = np.random.default_rng(0)
x = sf.constant(rng.standard_normal((n, h, h, c)).astype(np.float32))
w = sf.constant(rng.standard_normal((k, k, c, co)).astype(np.float32))
nn.IMPLICIT_CONV = os.environ.get("IMPL", "1") == "1"
for _ in range(5):
    nn.conv2d(x, w, s, p)
_native.sync(0)
