"""C2 microbenchmark (100 x tanh(x @ W_i + b_i)) eager and staged, a few
chains each after warm-up: the command profiled for the launch-overhead
evidence (ncu launch list: kernels per chain and their device time)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native, plugins  # noqa: E402
from paper_1903_01855_b200.workloads import microbench  # noqa: E402


def main():
    sf.init_runtime(sf.RuntimeOptions())
    plugins.install()
    for mode in ("eager", "staged"):
        ch = microbench.Chain(mode)
        for _ in range(3):
            ch.step().numpy()
        _native.sync(0)
        l0 = _native.launch_count(0)
        for _ in range(2):
            ch.step().numpy()
        print(mode, "kernel launches per chain:", (_native.launch_count(0) - l0) / 2)


if __name__ == "__main__":
    main()
