"""C2 small-op microbenchmark: a chain of 100 x tanh(matmul(x, W_i) + b_i).

Builder-defined: x (1,16), W_i (16,16) ~ 0.3 N(0,1),
b_i (1,16) ~ 0.1 N(0,1), drawn from ``default_rng(seed)`` in the order x,
then (W_i, b_i) per layer; all float32, closed over (captured) by the
staged function.  ``tanh`` is the plugin op (plugins.py).  300 primitive
ops per chain; the metric is primitive ops per second.
"""
from __future__ import annotations

import numpy as np

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import plugins

LAYERS, WIDTH = 100, 16


def params(seed=0, layers=LAYERS, width=WIDTH):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((1, width)).astype(np.float32)
    ws, bs = [], []
    for _ in range(layers):
        ws.append((rng.standard_normal((width, width)) * 0.3).astype(np.float32))
        bs.append((rng.standard_normal((1, width)) * 0.1).astype(np.float32))
    return x, ws, bs


class Chain:
    def __init__(self, mode: str, seed: int = 0):
        plugins.install()
        x, ws, bs = params(seed)
        self.x = sf.constant(x)
        self.ws = [sf.constant(w) for w in ws]
        self.bs = [sf.constant(b) for b in bs]

        def chain(v):
            for w, b in zip(self.ws, self.bs):
                v = sf.dispatch("tanh", [sf.add(sf.matmul(v, w), b)])[0]
            return v

        self.fn = sf.stage(chain) if mode == "staged" else chain
        self.out = None

    def step(self):
        self.out = self.fn(self.x)
        return self.out
