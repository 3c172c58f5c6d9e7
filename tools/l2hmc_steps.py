"""Run N staged L2HMC transitions (bench.py's headline program) — a short
command for ncu captures of the row kernel.

    python tools/l2hmc_steps.py [chains] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, plugins  # noqa: E402
from paper_1903_01855_b200.workloads import l2hmc  # noqa: E402

chains = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
sf.init_runtime(sf.RuntimeOptions(seed=1234))
plugins.install()
s = l2hmc.L2HMCSampler(sf, chains, "staged", seed=0)
for _ in range(steps):
    s.step()
_native.sync(0)
print("ok", float(s.accept.numpy().mean()))
