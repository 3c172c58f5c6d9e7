"""NumPy restatement of the reference's primitive kernels (oracle; test-only).

Each entry cites the reference kernel it restates
(paths relative to /root/reference/pkg/src).
"""
from __future__ import annotations

import numpy as np


def add(a, b):  # stageflow/kernels.py:116-130 (np.add)
    return np.add(a, b)


def sub(a, b):  # :116-130 (np.subtract)
    return np.subtract(a, b)


def mul(a, b):  # :116-130 (np.multiply)
    return np.multiply(a, b)


def div(a, b):  # :156-158 (errstate-guarded np.divide)
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.divide(a, b)


def neg(x):  # :144-153
    return np.negative(x)


def exp(x):  # :161-163
    with np.errstate(over="ignore"):
        return np.exp(x)


def log(x):  # :166-168
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.log(x)


def softplus(x):  # :171-173 — logaddexp(0, x)
    return np.logaddexp(0.0, x).astype(x.dtype)


def relu(x):  # :176-177 — np.maximum(x, 0)
    return np.maximum(x, 0).astype(x.dtype)


def step_positive(x):  # :180-181
    return np.greater(x, 0).astype(x.dtype)


def greater(a, b):  # :222-232
    return np.greater(a, b)


def matmul(a, b):  # :184-208 — OpenBLAS sgemm/dgemm via np.matmul
    return np.matmul(a, b)


def transpose(x):  # :211-219
    return np.ascontiguousarray(x.T)


def reduce_sum(x, axes=None, keepdims=False):  # :323-364 (pairwise np.sum)
    out = np.sum(x, axis=None if axes is None else tuple(axes), keepdims=keepdims)
    return np.asarray(out).astype(x.dtype)


def reduce_mean(x, axes=None, keepdims=False):  # :323-364 (np.mean)
    out = np.mean(x, axis=None if axes is None else tuple(axes), keepdims=keepdims)
    return np.asarray(out).astype(x.dtype)


def tanh(x):  # builder plugin (np.tanh); no reference kernel exists
    return np.tanh(x)


KERNELS = dict(add=add, sub=sub, mul=mul, div=div, neg=neg, exp=exp, log=log, softplus=softplus,
               relu=relu, step_positive=step_positive, greater=greater, matmul=matmul,
               transpose=transpose, reduce_sum=reduce_sum, reduce_mean=reduce_mean, tanh=tanh)
