"""NumPy kernels for the NN plugin ops (oracle; test-only).

conv2d / conv2d_grad_input / conv2d_grad_filter / max_pool / max_pool_grad /
softmax_xent / softmax_xent_grad in NHWC, matching the semantics of
paper_1903_01855_b200/nn.py.  Cross-checked against torch CPU fp32 in
tests/test_oracle_nn.py; registered into the reference runtime by
oracle/ref_plugins.register_nn.
"""
from __future__ import annotations

import numpy as np


def out_hw(h, w, k, s, p):
    return (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1


def im2col(x, kh, kw, s, p):
    n, h, w, c = x.shape
    ho, wo = out_hw(h, w, kh, s, p)
    xp = np.pad(x, ((0, 0), (p, p), (p, p), (0, 0)))
    cols = np.empty((n, ho, wo, kh, kw, c), dtype=x.dtype)
    for i in range(kh):
        for j in range(kw):
            cols[:, :, :, i, j, :] = xp[:, i:i + s * ho:s, j:j + s * wo:s, :]
    return cols.reshape(n * ho * wo, kh * kw * c)


def col2im(dcols, shape, kh, kw, s, p):
    n, h, w, c = shape
    ho, wo = out_hw(h, w, kh, s, p)
    d = dcols.reshape(n, ho, wo, kh, kw, c)
    dxp = np.zeros((n, h + 2 * p, w + 2 * p, c), dtype=dcols.dtype)
    for i in range(kh):
        for j in range(kw):
            dxp[:, i:i + s * ho:s, j:j + s * wo:s, :] += d[:, :, :, i, j, :]
    return dxp[:, p:p + h, p:p + w, :]


def conv2d(x, w, stride, pad):
    kh, kw, ci, co = w.shape
    n, h, wd, c = x.shape
    ho, wo = out_hw(h, wd, kh, stride, pad)
    cols = im2col(x, kh, kw, stride, pad)
    return (cols @ w.reshape(kh * kw * ci, co)).reshape(n, ho, wo, co)


def conv2d_grad_input(dy, w, stride, pad, input_shape):
    kh, kw, ci, co = w.shape
    n, ho, wo, _ = dy.shape
    dcols = dy.reshape(n * ho * wo, co) @ w.reshape(kh * kw * ci, co).T
    return col2im(dcols, input_shape, kh, kw, stride, pad)


def conv2d_grad_filter(x, dy, stride, pad, filter_shape):
    kh, kw, ci, co = filter_shape
    cols = im2col(x, kh, kw, stride, pad)
    return (cols.T @ dy.reshape(-1, co)).reshape(filter_shape)


def max_pool(x, k, s, p):
    n, h, w, c = x.shape
    ho, wo = out_hw(h, w, k, s, p)
    xp = np.pad(x, ((0, 0), (p, p), (p, p), (0, 0)), constant_values=-np.inf)
    out = np.full((n, ho, wo, c), -np.inf, dtype=x.dtype)
    for i in range(k):
        for j in range(k):
            out = np.maximum(out, xp[:, i:i + s * ho:s, j:j + s * wo:s, :])
    return out.astype(x.dtype)


def max_pool_grad(x, dy, k, s, p):
    """Route each window's gradient to its first maximum (window order kh, kw)."""
    n, h, w, c = x.shape
    ho, wo = out_hw(h, w, k, s, p)
    xp = np.pad(x, ((0, 0), (p, p), (p, p), (0, 0)), constant_values=-np.inf)
    best = np.full((n, ho, wo, c), -np.inf, dtype=x.dtype)
    arg = np.full((n, ho, wo, c), -1, dtype=np.int64)
    for i in range(k):
        for j in range(k):
            v = xp[:, i:i + s * ho:s, j:j + s * wo:s, :]
            take = v > best
            best = np.where(take, v, best)
            arg = np.where(take, i * k + j, arg)
    dxp = np.zeros((n, h + 2 * p, w + 2 * p, c), dtype=dy.dtype)
    for i in range(k):
        for j in range(k):
            dxp[:, i:i + s * ho:s, j:j + s * wo:s, :] += np.where(arg == i * k + j, dy, 0)
    return dxp[:, p:p + h, p:p + w, :]


def softmax_xent(logits, labels):
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    s = e.sum(axis=1)
    return (np.log(s) + m[:, 0] - logits[np.arange(len(labels)), labels]).astype(logits.dtype)


def softmax_xent_grad(logits, labels, g):
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    p = e / e.sum(axis=1, keepdims=True)
    p[np.arange(len(labels)), labels] -= 1
    return (p * g[:, None]).astype(logits.dtype)
