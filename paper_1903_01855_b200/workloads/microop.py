"""The reference's microop_loop workload (stageflow/bench.py:186-206): a
chain of 1000 scalar adds, x <- x + 1.0 on a float32 0-d tensor — pure
dispatch overhead.

Eager: 1000 dispatches per iteration, each one launch of the add kernel
with the 1.0 as a launch immediate.  Staged: one call; the traced graph
(1000 constants + 1000 adds) lowers to a single uniform kernel in which one
thread carries x through the 1000 adds in registers.
"""
from __future__ import annotations

import numpy as np

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import ops

N_OPS = 1000


def chain(x):
    for _ in range(N_OPS):
        x = ops.add(x, 1.0)
    return x


class MicroOpLoop:
    gate_tol = 1e-5

    def __init__(self, mode: str, seed: int = 0):
        del seed  # the workload has no random state (reference :189-191)
        self.x = sf.tensor_from_host(np.zeros(1, dtype=np.float32), (), sf.float32)
        self.mode = mode
        self.chain = sf.stage(chain) if mode == "staged" else chain
        self.staged_functions = [self.chain] if mode == "staged" else []

    def step(self):
        self.x = self.chain(self.x)
        return self.x

    def run_iteration(self) -> float:
        self.step()
        return float(self.x)

    def cache_size(self) -> int:
        return sum(pf.cache_size for pf in self.staged_functions)
