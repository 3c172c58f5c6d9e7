"""SCK1 checkpoint fixtures written by the REFERENCE (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ckpt_golden.py

Builds tests/ckpt_graph.py's object graph with the reference package and
saves it with stageflow.checkpoint.save (reference checkpoint.py), with and
without variables.  tests/test_checkpoint.py checks that this package
writes the same bytes and restores from them.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

import stageflow as ref  # noqa: E402
from ckpt_graph import build  # noqa: E402

ref.init_runtime(ref.RuntimeOptions())
for name, with_vars in (("ckpt_ref.sck1", True), ("ckpt_ref_novars.sck1", False)):
    data = ref.save(build(ref, with_vars)).to_bytes()
    with open(os.path.join(HERE, name), "wb") as f:
        f.write(data)
    print(name, len(data), "bytes")
