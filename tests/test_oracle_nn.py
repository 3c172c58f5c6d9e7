"""Pin the numpy NN oracle (oracle/nn_np.py) against torch CPU fp32 — an
independent implementation — since the reference has no conv/pool/xent."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import nn_np

GEOMS = [  # (N, H, W, Cin, Cout, K, stride, pad)
    (2, 9, 9, 3, 4, 7, 2, 3), (2, 8, 8, 5, 6, 3, 1, 1), (1, 9, 7, 4, 3, 3, 2, 1),
    (2, 6, 6, 8, 16, 1, 2, 0), (3, 5, 5, 4, 4, 1, 1, 0),
]


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).double().requires_grad_(True)


@pytest.mark.parametrize("g", GEOMS)
def test_conv_fwd_and_grads_vs_torch(g):
    n, h, w, ci, co, k, s, p = g
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n, h, w, ci))
    wt = rng.standard_normal((k, k, ci, co))
    y = nn_np.conv2d(x, wt, s, p)
    tx, tw = _t(x), _t(wt)
    ty = F.conv2d(tx.permute(0, 3, 1, 2), tw.permute(3, 2, 0, 1), stride=s, padding=p)
    np.testing.assert_allclose(y, ty.permute(0, 2, 3, 1).detach().numpy(), rtol=1e-10, atol=1e-10)
    dy = rng.standard_normal(y.shape)
    ty.permute(0, 2, 3, 1).backward(torch.from_numpy(dy))
    np.testing.assert_allclose(nn_np.conv2d_grad_input(dy, wt, s, p, x.shape), tx.grad.numpy(),
                               rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(nn_np.conv2d_grad_filter(x, dy, s, p, wt.shape), tw.grad.numpy(),
                               rtol=1e-10, atol=1e-10)


def test_max_pool_vs_torch():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 9, 9, 3))
    y = nn_np.max_pool(x, 3, 2, 1)
    tx = _t(x)
    ty = F.max_pool2d(tx.permute(0, 3, 1, 2), 3, 2, 1)
    np.testing.assert_allclose(y, ty.permute(0, 2, 3, 1).detach().numpy())
    dy = rng.standard_normal(y.shape)
    ty.permute(0, 2, 3, 1).backward(torch.from_numpy(dy))
    np.testing.assert_allclose(nn_np.max_pool_grad(x, dy, 3, 2, 1), tx.grad.numpy(), atol=1e-12)


def test_softmax_xent_vs_torch():
    rng = np.random.default_rng(2)
    logits = rng.standard_normal((5, 7))
    labels = rng.integers(0, 7, size=5)
    got = nn_np.softmax_xent(logits, labels)
    tl = _t(logits)
    want = F.cross_entropy(tl, torch.from_numpy(labels), reduction="none")
    np.testing.assert_allclose(got, want.detach().numpy(), rtol=1e-12)
    g = rng.uniform(0.5, 1.5, size=5)
    want.backward(torch.from_numpy(g))
    np.testing.assert_allclose(nn_np.softmax_xent_grad(logits, labels, g), tl.grad.numpy(),
                               rtol=1e-10, atol=1e-12)
