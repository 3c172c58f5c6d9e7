"""ResNet-50 v1.5 training step (BASELINE configs C4 / C5), NHWC, float32.

Written against an API module ``sf`` (this backend, or the reference with
the numpy plugin ops of oracle/ref_plugins.py) so the same program is both
the workload and, on the reference, its oracle.  Mirrors the reference's
mlp_train staging pattern (stageflow/bench.py:103-144): the forward pass +
loss is one staged function, the tape derives its (staged) backward, and
the SGD update ``v += -lr * g`` over all 161 variables is a second staged
function.  Batch norm uses batch statistics and is composed from built-in
primitives (reduce_mean / sub / mul / add) plus the ``rsqrt`` plugin op.
"""
from __future__ import annotations

import math

import numpy as np

LAYERS = (3, 4, 6, 3)
WIDTHS = (64, 128, 256, 512)
EXPANSION = 4
BN_EPS = 1e-5


def _f32(sf, arr, dtype=None):
    dtype = dtype or sf.float32
    arr = np.asarray(arr, dtype=dtype.np_dtype)
    return sf.tensor_from_host(arr.reshape(-1), arr.shape, dtype)


class ResNet50:
    def __init__(self, sf, num_classes: int = 1000, seed: int = 0, width_div: int = 1,
                 dtype=None):
        self.sf = sf
        rng = np.random.default_rng(seed)
        self.params = []

        def var(arr):
            v = sf.Variable(_f32(sf, arr, dtype))
            self.params.append(v)
            return v

        def conv(kh, cin, cout):
            std = math.sqrt(2.0 / (kh * kh * cout))  # He (fan_out), as torchvision
            return var(rng.standard_normal((kh, kh, cin, cout)) * std)

        def bn(c):
            return var(np.ones(c)), var(np.zeros(c))

        w = [max(1, x // width_div) for x in WIDTHS]
        stem = max(1, 64 // width_div)
        self.stem = (conv(7, 3, stem), bn(stem))
        self.blocks = []
        cin = stem
        for stage, (n_blocks, width) in enumerate(zip(LAYERS, w)):
            for b in range(n_blocks):
                stride = 2 if (b == 0 and stage > 0) else 1
                cout = width * EXPANSION
                blk = {
                    "c1": (conv(1, cin, width), bn(width)),
                    "c2": (conv(3, width, width), bn(width)),
                    "c3": (conv(1, width, cout), bn(cout)),
                    "stride": stride,
                    "down": (conv(1, cin, cout), bn(cout)) if (stride != 1 or cin != cout) else None,
                }
                self.blocks.append(blk)
                cin = cout
        bound = 1.0 / math.sqrt(cin)
        self.fc_w = var(rng.uniform(-bound, bound, (cin, num_classes)))
        self.fc_b = var(rng.uniform(-bound, bound, (num_classes,)))

    # -- layers -----------------------------------------------------------------
    def _bn(self, x, gamma_beta, relu):
        sf = self.sf
        gamma, beta = gamma_beta
        mean = sf.reduce_mean(x, axes=(0, 1, 2))
        xc = sf.sub(x, mean)
        var = sf.reduce_mean(sf.mul(xc, xc), axes=(0, 1, 2))
        inv = sf.dispatch("rsqrt", [sf.add(var, BN_EPS)])[0]
        y = sf.add(sf.mul(sf.mul(xc, inv), gamma.read_value()), beta.read_value())
        return sf.relu(y) if relu else y

    def _conv(self, x, w, stride, pad):
        return self.sf.dispatch("conv2d", [x, w.read_value()], {"stride": stride, "pad": pad})[0]

    def forward(self, x):
        sf = self.sf
        w, g = self.stem
        h = self._bn(self._conv(x, w, 2, 3), g, relu=True)
        h = sf.dispatch("max_pool", [h], {"ksize": 3, "stride": 2, "pad": 1})[0]
        for blk in self.blocks:
            s = blk["stride"]
            (w1, g1), (w2, g2), (w3, g3) = blk["c1"], blk["c2"], blk["c3"]
            o = self._bn(self._conv(h, w1, 1, 0), g1, relu=True)
            o = self._bn(self._conv(o, w2, s, 1), g2, relu=True)
            o = self._bn(self._conv(o, w3, 1, 0), g3, relu=False)
            if blk["down"] is not None:
                wd, gd = blk["down"]
                h = self._bn(self._conv(h, wd, s, 0), gd, relu=False)
            h = sf.relu(sf.add(o, h))
        pooled = sf.reduce_mean(h, axes=(1, 2))
        return sf.add(sf.matmul(pooled, self.fc_w.read_value()), self.fc_b.read_value())


class ResNetTrain:
    """One SGD training step per ``step()``; staged or eager."""

    LR = 1e-3

    def __init__(self, sf, batch: int, mode: str = "staged", image: int = 224, seed: int = 0,
                 width_div: int = 1, num_classes: int = 1000, dtype=None):
        self.sf = sf
        self.model = ResNet50(sf, num_classes=num_classes, seed=seed, width_div=width_div,
                              dtype=dtype)
        rng = np.random.default_rng(seed + 1)
        self.x = _f32(sf, rng.standard_normal((batch, image, image, 3)), dtype)
        labels = rng.integers(0, num_classes, size=(batch,))
        self.labels = sf.tensor_from_host(labels, (batch,), sf.int32)
        params = self.model.params

        def forward_loss(x, labels):
            logits = self.model.forward(x)
            return sf.reduce_mean(sf.dispatch("softmax_xent", [logits, labels])[0])

        def apply_updates(*grads):
            for v, gr in zip(params, grads):
                v.assign_add(sf.mul(gr, -self.LR))

        if mode == "staged":
            self.forward_loss = sf.stage(forward_loss, name="resnet50_forward_loss")
            self.apply_updates = sf.stage(apply_updates, name="resnet50_apply_updates")
            self.staged_functions = [self.forward_loss, self.apply_updates]
        else:
            self.forward_loss = forward_loss
            self.apply_updates = apply_updates
            self.staged_functions = []

    def step(self, x=None, labels=None):
        sf = self.sf
        with sf.Tape() as t:
            loss = self.forward_loss(self.x if x is None else x,
                                     self.labels if labels is None else labels)
        grads = t.gradient(loss, self.model.params)
        self.apply_updates(*grads)
        return loss

    def run_iteration(self) -> float:
        return float(self.step())
