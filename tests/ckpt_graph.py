"""The object graph the SCK1 checkpoint fixtures are built from.  Written
against the public API only, so the same function builds it with the
reference (tests/golden/make_ckpt_golden.py) and with this package."""
import numpy as np


def build(sf, with_variables=True, scale=1.0):
    class Model(sf.Trackable):
        pass

    root = Model()
    root.dense = Model()
    if with_variables:
        root.dense.kernel = sf.Variable(
            sf.constant((np.arange(12, dtype=np.float32) * scale).reshape(3, 4)))
        root.dense.bias = sf.Variable(sf.constant(np.array([0.5, -1.0, 2.0, 3.5]) * scale))
        root.step = sf.Variable(sf.constant(np.int32(7 * scale)))
        root.flag = sf.Variable(sf.constant(bool(scale == 1.0)))
    root.table = (np.arange(6, dtype=np.int64) * int(scale)).reshape(2, 3)
    it = sf.SequenceIterator([10, 20, 30, 40])
    if scale == 1.0:
        next(it)
        next(it)
    root.data = it
    root.dense.parent = root  # a cycle: restore must stay finite
    return root
