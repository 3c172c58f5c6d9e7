"""ResNet-50 at the benchmarked configuration C4 (batch 32, 224x224x3,
seed 0) against the REFERENCE run at the same configuration
(tests/golden/make_golden_r2.py: stageflow + numpy plugin ops, eager tape,
float32 and float64).

What the reference's own numbers say about the bar: its float32 gradients
differ from its float64 ones by up to ~9% element-wise on the deep
convolution/BN parameters (batch-norm backward subtracts nearly equal batch
means: a ~1e6 round-off amplification), and by 5e-8 on the classifier bias.
So:

* float64 on the GPU must match the reference's float64 to 1e-8 on every
  one of the 161 gradients (norms and sums) and on the sampled slices — the
  algorithm is the same, the amplified round-off is ~1e-10;
* float32 on the GPU (the benchmarked staged step, 3xTF32 GEMMs) must be,
  over the 161 gradients, no less accurate than the reference's own float32
  (median, maximum, and count within 1e-4 of float64), each gradient within
  max(5e-4, 4 x the reference's float32 error), and the classifier within
  rtol 1e-4 element-wise (bounds recorded in DESIGN.md §3);
* eager and staged float32 steps on the GPU are bit-identical at C4.
"""
import os

import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import nn
from paper_1903_01855_b200.workloads import resnet

pytestmark = pytest.mark.gpu
GOLD2 = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_r2.npz"))
PARAMS = [int(i) for i in GOLD2["resnet_c4_params"]]


@pytest.fixture(autouse=True)
def _nn():
    nn.install()


def _grads(mode, dtype):
    tr = resnet.ResNetTrain(sf, batch=32, mode=mode, image=224, seed=0, dtype=dtype)
    with sf.Tape() as t:
        loss = tr.forward_loss(tr.x, tr.labels)
    grads = t.gradient(loss, tr.model.params)
    return float(loss), [g.numpy() for g in grads]


def _norms_sums(grads):
    a = [g.astype(np.float64).ravel() for g in grads]
    return np.array([np.sqrt(np.square(x).sum()) for x in a]), np.array([x.sum() for x in a])


def _slice_err(got, want):
    got = got.ravel()[:want.size].astype(np.float64)
    return float(np.abs(got - want).max() / max(1e-300, np.abs(want).max()))


def test_c4_float64_gradients_match_reference():
    loss, grads = _grads("staged", sf.float64)
    assert len(grads) == 161
    np.testing.assert_allclose(loss, GOLD2["resnet_c4_f64_loss"][0], rtol=1e-12)
    norms, sums = _norms_sums(grads)
    want_n, want_s = GOLD2["resnet_c4_f64_grad_norms"], GOLD2["resnet_c4_f64_grad_sums"]
    np.testing.assert_allclose(norms, want_n, rtol=1e-8)
    # sums cancel: compare them on the scale of the norm
    assert np.all(np.abs(sums - want_s) <= 1e-8 * want_n * np.sqrt([g.size for g in grads]))
    for i in PARAMS:
        assert _slice_err(grads[i], GOLD2[f"resnet_c4_f64_grad_{i}"]) < 1e-8, i


@pytest.mark.parametrize("mode", ["staged", "eager"])
def test_c4_float32_gradients_within_reference_bound(mode):
    loss, grads = _grads(mode, sf.float32)
    ref64 = GOLD2["resnet_c4_f64_loss"][0]
    np.testing.assert_allclose(loss, ref64, rtol=1e-5)
    norms, _ = _norms_sums(grads)
    n64, n32 = GOLD2["resnet_c4_f64_grad_norms"], GOLD2["resnet_c4_f32_grad_norms"]
    ref_err = np.abs(n32 - n64) / n64
    err = np.abs(norms - n64) / n64
    # (1) as a distribution over the 161 gradients, ours is no less accurate
    # than the reference's own float32 (measured: median 3.9e-4 vs 1.2e-3,
    # max 7.9e-3 vs 2.0e-2; profiles/r02_c4_grad_errors.json)
    assert np.median(err) <= np.median(ref_err)
    assert err.max() <= ref_err.max()
    assert (err < 1e-4).sum() >= (ref_err < 1e-4).sum()
    # (2) per gradient: within 4x the reference's own float32 error, with a
    # 5e-4 floor (a gradient whose reference f32 error happens to be tiny is
    # not better conditioned: layer-4 BN betas are column sums of a
    # cancelling dy, ref 3.5e-5, ours 2.6e-4)
    bound = np.maximum(5e-4, 4 * ref_err)
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, [(int(i), float(err[i]), float(bound[i])) for i in bad]
    for i in PARAMS:
        want = GOLD2[f"resnet_c4_f64_grad_{i}"]
        ref_e = _slice_err(GOLD2[f"resnet_c4_f32_grad_{i}"], want)
        e = _slice_err(grads[i], want)
        assert e < max(5e-4, 4 * ref_e), (i, e, ref_e)
    # the classifier (no BN behind it) meets rtol 1e-4 element-wise
    for i in (159, 160):
        want = GOLD2[f"resnet_c4_f64_grad_{i}"]
        np.testing.assert_allclose(grads[i].ravel()[:want.size], want, rtol=1e-4,
                                   atol=1e-4 * np.abs(want).max())


def test_c4_eager_equals_staged_bitwise():
    le, ge = _grads("eager", sf.float32)
    ls, gs = _grads("staged", sf.float32)
    assert np.float32(le).tobytes() == np.float32(ls).tobytes()
    for a, b in zip(ge, gs):
        assert a.tobytes() == b.tobytes()
