"""NumPy restatements of the benchmark workloads (oracle; test-only).

Each follows the op order of the reference program it restates, in the
same dtype, so with NumPy underneath it reproduces the reference's own
results bit-for-bit (pinned by tests/test_oracle.py against the golden
vectors generated from the reference).
"""
from __future__ import annotations

import numpy as np

F32 = np.float32


# ---------------------------------------------------------------------------
# leapfrog — stageflow/bench.py:147-183
# ---------------------------------------------------------------------------

def _leapfrog_force(q):
    # Tape gradient of U = 0.5 * sum(q*q): the mul rule contributes
    # up*q twice (gradients.py:125-132) with up = broadcast(0.5), accumulated
    # by add (tape.py:200-211).
    half = F32(0.5) * F32(1.0)
    g = np.full(q.shape, half, dtype=F32)
    return np.add(g * q, g * q)


def leapfrog_init(batch, seed=0):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((batch, 2)).astype(F32)
    p = rng.standard_normal((batch, 2)).astype(F32)
    return q, p


def leapfrog_trajectory(q, p, n_steps=10, step=0.1):
    half = F32(step / 2.0)
    eps = F32(step)
    for _ in range(n_steps):
        p = p - _leapfrog_force(q) * half
        q = q + p * eps
        p = p - _leapfrog_force(q) * half
    return q, p


def leapfrog(batch, seed=0, trajectories=1):
    """Concatenated (q, p) after `trajectories` trajectories (run_iteration output)."""
    q, p = leapfrog_init(batch, seed)
    for _ in range(trajectories):
        q, p = leapfrog_trajectory(q, p)
    return np.concatenate([q.ravel(), p.ravel()])


# ---------------------------------------------------------------------------
# mlp_train — stageflow/bench.py:103-144
# ---------------------------------------------------------------------------

class MLPTrain:
    IN, HIDDEN, OUT = 128, 256, 1
    LR = 1e-3

    def __init__(self, batch, seed=0):
        rng = np.random.default_rng(seed)
        self.x = (rng.standard_normal((batch, self.IN)) * 0.5).astype(F32)
        self.y = rng.standard_normal((batch, self.OUT)).astype(F32)
        self.w1 = (rng.standard_normal((self.IN, self.HIDDEN)) * 0.05).astype(F32)
        self.b1 = np.zeros(self.HIDDEN, dtype=F32)
        self.w2 = (rng.standard_normal((self.HIDDEN, self.OUT)) * 0.05).astype(F32)
        self.b2 = np.zeros(self.OUT, dtype=F32)

    def step(self):
        x, y = self.x, self.y
        pre = np.matmul(x, self.w1) + self.b1
        h = np.maximum(pre, 0).astype(F32)
        pred = np.matmul(h, self.w2) + self.b2
        err = pred - y
        loss = np.mean(err * err)
        count = err.size
        g = np.full(err.shape, F32(1.0) * F32(1.0 / count), dtype=F32)
        g_err = np.add(g * err, g * err)
        g_b2 = np.sum(g_err, axis=0).astype(F32)
        g_h = np.matmul(g_err, np.ascontiguousarray(self.w2.T))
        g_w2 = np.matmul(np.ascontiguousarray(h.T), g_err)
        g_pre = g_h * (pre > 0).astype(F32)
        g_b1 = np.sum(g_pre, axis=0).astype(F32)
        g_w1 = np.matmul(np.ascontiguousarray(x.T), g_pre)
        lr = F32(-self.LR)
        self.w1 = self.w1 + g_w1 * lr
        self.b1 = self.b1 + g_b1 * lr
        self.w2 = self.w2 + g_w2 * lr
        self.b2 = self.b2 + g_b2 * lr
        return float(loss)


def mlp_losses(batch, iterations, seed=0):
    m = MLPTrain(batch, seed)
    return np.array([m.step() for _ in range(iterations)], dtype=np.float64)


# ---------------------------------------------------------------------------
# C2 microbenchmark — builder-defined
# ---------------------------------------------------------------------------

C2_LAYERS, C2_WIDTH = 100, 16


def c2_params(seed=0, layers=C2_LAYERS, width=C2_WIDTH):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((1, width)).astype(F32)
    ws, bs = [], []
    for _ in range(layers):
        ws.append((rng.standard_normal((width, width)) * 0.3).astype(F32))
        bs.append((rng.standard_normal((1, width)) * 0.1).astype(F32))
    return x, ws, bs


def c2_chain(x, ws, bs):
    for w, b in zip(ws, bs):
        x = np.tanh(np.matmul(x, w) + b)
    return x


def c2_chain_grad(x, ws, bs):
    """d sum(chain(x)) / dx via the tanh rule up*(1 - y*y)."""
    ys = []
    h = x
    for w, b in zip(ws, bs):
        h = np.tanh(np.matmul(h, w) + b)
        ys.append(h)
    g = np.ones_like(h)
    for w, y in zip(reversed(ws), reversed(ys)):
        g = g * (F32(1.0) - y * y)
        g = np.matmul(g, np.ascontiguousarray(w.T))
    return g
