"""The reference's leapfrog workload on this backend
(reference: stageflow/bench.py:147-183, the C1/C3 stand-in).

q, p ~ N(0, 1) of shape (B, 2) from ``default_rng(seed)``; 10 steps of
step 0.1 of a symplectic integrator on U(q) = sum(q^2)/2 whose force is a
tape gradient.  Staged mode stages the whole trajectory: the traced graph
(50 constants + 120 elementwise ops after folding) lowers to ONE fused
kernel that reads q, p once and writes them once (32 B per chain).
"""
from __future__ import annotations

import numpy as np

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import ops

STEP = 0.1
N_STEPS = 10


def _f32(arr) -> sf.Tensor:
    arr = np.asarray(arr, dtype=np.float32)
    return sf.tensor_from_host(arr.reshape(-1), arr.shape, sf.float32)


def force(q):
    with sf.Tape() as t:
        t.watch(q)
        u = ops.mul(ops.reduce_sum(ops.mul(q, q)), 0.5)
    return t.gradient(u, q)


def trajectory(q, p):
    half = STEP / 2.0
    for _ in range(N_STEPS):
        p = ops.sub(p, ops.mul(force(q), half))
        q = ops.add(q, ops.mul(p, STEP))
        p = ops.sub(p, ops.mul(force(q), half))
    return q, p


class Leapfrog:
    gate_tol = 1e-6

    def __init__(self, batch: int, mode: str, seed: int = 0):
        rng = np.random.default_rng(seed)
        self.batch = batch
        self.q = _f32(rng.standard_normal((batch, 2)))
        self.p = _f32(rng.standard_normal((batch, 2)))
        self.mode = mode
        self.trajectory = sf.stage(trajectory) if mode == "staged" else trajectory
        self.staged_functions = [self.trajectory] if mode == "staged" else []

    def step(self):
        """One trajectory, device-resident (no host fetch)."""
        self.q, self.p = self.trajectory(self.q, self.p)
        return self.q, self.p

    def run_iteration(self):
        """One trajectory plus the host fetch of q and p (reference :181-183)."""
        self.step()
        return np.concatenate([self.q.numpy().ravel(), self.p.numpy().ravel()])

    def cache_size(self) -> int:
        return sum(pf.cache_size for pf in self.staged_functions)
