"""GPU parity of the ResNet-50 plugin ops and training step (configs C4/C5).

Ops are checked against the numpy oracle (itself pinned to torch CPU, see
test_oracle_nn.py); the training step against golden losses produced by the
reference runtime with numpy plugin ops (tests/golden/make_golden.py).
"""
import os

import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import nn
from paper_1903_01855_b200.workloads import resnet
from oracle import nn_np

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
GEOMS = [(2, 9, 9, 3, 4, 7, 2, 3), (2, 8, 8, 5, 6, 3, 1, 1), (1, 9, 7, 4, 3, 3, 2, 1),
         (2, 6, 6, 8, 16, 1, 2, 0), (3, 5, 5, 4, 4, 1, 1, 0), (2, 16, 16, 64, 64, 3, 1, 1)]


@pytest.fixture(autouse=True)
def _nn():
    nn.install()


@pytest.mark.parametrize("g", GEOMS)
def test_conv_vs_oracle(g):
    n, h, w, ci, co, k, s, p = g
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n, h, w, ci)).astype(np.float32)
    wt = rng.standard_normal((k, k, ci, co)).astype(np.float32)
    tx, tw = sf.constant(x), sf.constant(wt)
    y = nn.conv2d(tx, tw, s, p)
    want = nn_np.conv2d(x.astype(np.float64), wt.astype(np.float64), s, p)
    # sums of K = k*k*ci unit-scale products: fp32-class absolute error ~ 1e-5 * sqrt(K)
    atol = 1e-4 * np.sqrt(k * k * ci)
    np.testing.assert_allclose(y.numpy(), want, rtol=1e-4, atol=atol)
    dy = rng.standard_normal(want.shape).astype(np.float32)
    with sf.Tape() as t:
        t.watch(tx)
        t.watch(tw)
        yy = nn.conv2d(tx, tw, s, p)
        loss = sf.reduce_sum(sf.mul(yy, sf.constant(dy)))
    gx, gw = t.gradient(loss, [tx, tw])
    np.testing.assert_allclose(gx.numpy(), nn_np.conv2d_grad_input(
        dy.astype(np.float64), wt.astype(np.float64), s, p, x.shape), rtol=1e-4, atol=1e-4)
    np.testing.assert_allclose(gw.numpy(), nn_np.conv2d_grad_filter(
        x.astype(np.float64), dy.astype(np.float64), s, p, wt.shape), rtol=1e-4, atol=1e-3)


def test_conv_weight_grad_split_k():
    # N*H*W >= 16384 takes the split-K GEMM path
    rng = np.random.default_rng(3)
    x = rng.standard_normal((4, 64, 64, 8)).astype(np.float32)
    dy = rng.standard_normal((4, 64, 64, 16)).astype(np.float32)
    gw = sf.dispatch("conv2d_grad_filter", [sf.constant(x), sf.constant(dy)],
                     {"stride": 1, "pad": 1, "filter_shape": (3, 3, 8, 16)})[0].numpy()
    want = nn_np.conv2d_grad_filter(x.astype(np.float64), dy.astype(np.float64), 1, 1,
                                    (3, 3, 8, 16))
    np.testing.assert_allclose(gw, want, rtol=1e-4, atol=2e-3)


@pytest.mark.parametrize("shape,k,s,p", [((2, 9, 9, 8), 3, 2, 1), ((2, 10, 7, 64), 3, 1, 1),
                                         ((1, 12, 12, 4), 2, 2, 0), ((3, 8, 8, 12), 3, 2, 0)])
def test_maxpool_grad_vectorised_vs_oracle(shape, k, s, p):
    """The 4-channel gather (C % 4 == 0) visits exactly the windows holding
    each pixel; ties and overlapping windows (the argmax of several windows)
    accumulate like the oracle."""
    rng = np.random.default_rng(3)
    x = rng.integers(-3, 3, size=shape).astype(np.float32)  # many ties
    tx = sf.constant(x)
    with sf.Tape() as t:
        t.watch(tx)
        y = nn.max_pool(tx, k, s, p)
        dy = rng.standard_normal(y.shape).astype(np.float32)
        loss = sf.reduce_sum(sf.mul(y, sf.constant(dy)))
    np.testing.assert_array_equal(y.numpy(), nn_np.max_pool(x, k, s, p))
    np.testing.assert_allclose(t.gradient(loss, tx).numpy(), nn_np.max_pool_grad(x, dy, k, s, p),
                               rtol=1e-6, atol=1e-6)


def test_maxpool_vectorised_nan_first_wins():
    """NaNs in the 4-channel forward kernel: a window holding a NaN yields
    NaN (np.maximum's propagation, the oracle); lanes without NaNs are exact."""
    rng = np.random.default_rng(5)
    x = rng.integers(-3, 3, size=(2, 9, 9, 8)).astype(np.float32)
    x[rng.random(x.shape) < 0.1] = np.nan
    y = nn.max_pool(sf.constant(x), 3, 2, 1)
    np.testing.assert_array_equal(y.numpy(), nn_np.max_pool(x, 3, 2, 1))


def test_maxpool_and_xent_vs_oracle():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 9, 9, 3)).astype(np.float32)
    tx = sf.constant(x)
    with sf.Tape() as t:
        t.watch(tx)
        y = nn.max_pool(tx, 3, 2, 1)
        dy = rng.standard_normal(y.shape).astype(np.float32)
        loss = sf.reduce_sum(sf.mul(y, sf.constant(dy)))
    np.testing.assert_array_equal(y.numpy(), nn_np.max_pool(x, 3, 2, 1))
    np.testing.assert_allclose(t.gradient(loss, tx).numpy(), nn_np.max_pool_grad(x, dy, 3, 2, 1),
                               rtol=1e-6, atol=1e-6)
    logits = rng.standard_normal((6, 1000)).astype(np.float32)
    labels = rng.integers(0, 1000, size=6)
    tl = sf.constant(logits)
    tlab = sf.tensor_from_host(labels, (6,), sf.int32)
    with sf.Tape() as t:
        t.watch(tl)
        l = nn.softmax_xent(tl, tlab)
        loss = sf.reduce_mean(l)
    np.testing.assert_allclose(l.numpy(), nn_np.softmax_xent(logits.astype(np.float64), labels),
                               rtol=1e-5)
    np.testing.assert_allclose(t.gradient(loss, tl).numpy(), nn_np.softmax_xent_grad(
        logits.astype(np.float64), labels, np.full(6, 1 / 6)), rtol=1e-4, atol=1e-7)


def test_resnet50_training_f64_matches_reference():
    """Three staged SGD steps in float64: the deep BN stack (batch statistics
    over as few as 16 values per channel at this size) amplifies round-off,
    so the step-to-step trajectory is compared where round-off is 1e-16."""
    tr = resnet.ResNetTrain(sf, batch=4, mode="staged", image=64, seed=0, dtype=sf.float64)
    losses = [tr.run_iteration() for _ in range(3)]
    np.testing.assert_allclose(losses, GOLD["resnet_f64_losses"], rtol=1e-9)
    assert [tr.forward_loss.trace_count, tr.apply_updates.trace_count] == \
        list(GOLD["resnet_trace_counts"])


@pytest.mark.parametrize("mode", ["eager", "staged"])
def test_resnet50_f32_first_step_matches_reference(mode):
    tr = resnet.ResNetTrain(sf, batch=4, mode=mode, image=64, seed=0)
    loss = tr.run_iteration()
    np.testing.assert_allclose(loss, GOLD[f"resnet_{mode}_losses"][0], rtol=1e-5)


def test_resnet50_eager_equals_staged_bitwise():
    e = resnet.ResNetTrain(sf, batch=2, mode="eager", image=32, seed=0)
    s = resnet.ResNetTrain(sf, batch=2, mode="staged", image=32, seed=0)
    for _ in range(2):
        assert np.float32(e.run_iteration()).tobytes() == np.float32(s.run_iteration()).tobytes()
    assert e.model.fc_w.numpy().tobytes() == s.model.fc_w.numpy().tobytes()


@pytest.mark.parametrize("mode,dtype,tag,tol", [
    ("eager", "float64", "grad64", 1e-9), ("staged", "float64", "grad64", 1e-9),
    ("staged", "float32", "grad0", 1e-4)])
def test_resnet50_initial_gradients_match_reference(mode, dtype, tag, tol):
    dt = getattr(sf, dtype)
    tr = resnet.ResNetTrain(sf, batch=4, mode=mode, image=64, seed=0, dtype=dt)
    with sf.Tape() as t:
        loss = tr.forward_loss(tr.x, tr.labels)
    grads = t.gradient(loss, tr.model.params)
    assert abs(float(loss) - float(GOLD[f"resnet_{tag}_loss"][0])) < tol * 10
    # f32: parameters near the output are well conditioned and must meet 1e-4;
    # f64: every sampled parameter, down to the stem, must meet 1e-9
    # (the reference's own f32 gradients differ from its f64 ones by ~3% on the
    # deep parameters: f32 parity is asserted where f32 itself is meaningful)
    for i in ((0, 1, 2, 3, 10, 100, 159, 160) if dtype == "float64" else (160,)):
        want = GOLD[f"resnet_{tag}_{i}"]
        scale = max(1e-30, float(np.abs(want).max()))
        err = float(np.abs(grads[i].numpy().ravel()[:want.size] - want).max()) / scale
        assert err < tol, (i, err)
