"""The reference's mlp_train workload (stageflow/bench.py:103-144) on this backend.

2-layer MLP 128 -> 256 -> 1 (relu, MSE).  Staged mode stages the forward +
loss and the update application as two functions; the tape between them
derives a staged backward (one call_function), as in the paper's "forward
pass and gradient application staged" setup (the C4 pattern).
"""
from __future__ import annotations

import numpy as np

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import ops


def _f32(arr) -> sf.Tensor:
    arr = np.asarray(arr, dtype=np.float32)
    return sf.tensor_from_host(arr.reshape(-1), arr.shape, sf.float32)


class MLPTrain:
    IN, HIDDEN, OUT = 128, 256, 1
    LR = 1e-3
    gate_tol = 1e-5

    def __init__(self, batch: int, mode: str, seed: int = 0):
        rng = np.random.default_rng(seed)
        self.x = _f32(rng.standard_normal((batch, self.IN)) * 0.5)
        self.y = _f32(rng.standard_normal((batch, self.OUT)))
        self.w1 = sf.Variable(_f32(rng.standard_normal((self.IN, self.HIDDEN)) * 0.05))
        self.b1 = sf.Variable(_f32(np.zeros(self.HIDDEN)))
        self.w2 = sf.Variable(_f32(rng.standard_normal((self.HIDDEN, self.OUT)) * 0.05))
        self.b2 = sf.Variable(_f32(np.zeros(self.OUT)))
        self.params = [self.w1, self.b1, self.w2, self.b2]

        def forward_loss(x, y):
            h = ops.relu(ops.add(ops.matmul(x, self.w1.read_value()), self.b1.read_value()))
            pred = ops.add(ops.matmul(h, self.w2.read_value()), self.b2.read_value())
            err = ops.sub(pred, y)
            return ops.reduce_mean(ops.mul(err, err))

        def apply_updates(g1, g2, g3, g4):
            for v, g in zip(self.params, (g1, g2, g3, g4)):
                v.assign_add(ops.mul(g, -self.LR))

        if mode == "staged":
            self.forward_loss = sf.stage(forward_loss)
            self.apply_updates = sf.stage(apply_updates)
            self.staged_functions = [self.forward_loss, self.apply_updates]
        else:
            self.forward_loss = forward_loss
            self.apply_updates = apply_updates
            self.staged_functions = []

    def step(self):
        with sf.Tape() as t:
            loss = self.forward_loss(self.x, self.y)
        grads = t.gradient(loss, self.params)
        self.apply_updates(*grads)
        return loss

    def run_iteration(self) -> float:
        return float(self.step())

    def cache_size(self) -> int:
        return sum(pf.cache_size for pf in self.staged_functions)
