"""The data-parallel step on one GPU (world-size-1 NCCL communicator):
the C-ABI all-reduce, the gradient all-reduce folded into the staged
backward's plan, and proof that the update consumes the reduced gradients
(a scaled collective) — SURVEY.md §8(e), config C5."""
import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import comm as sfcomm
from paper_1903_01855_b200 import dist as sfdist
from paper_1903_01855_b200 import nn
from paper_1903_01855_b200.workloads import resnet

pytestmark = pytest.mark.gpu

SMALL = dict(image=32, width_div=16)


@pytest.fixture
def comm():
    c = sfcomm.Communicator(1, 0, 0)
    yield c
    c.close()


def test_allreduce_c_abi_world1(comm):
    x = sf.constant(np.arange(1000, dtype=np.float32).reshape(10, 100) / 7)
    (s,) = comm.allreduce([x])
    assert s.numpy().tobytes() == x.numpy().tobytes() and s is not x
    (d,) = comm.allreduce([x], scale=2.0)
    np.testing.assert_array_equal(d.numpy(), x.numpy() * np.float32(2))
    y = sf.constant(np.ones((3,), np.float64))
    (e,) = comm.allreduce([y], scale=0.5)
    np.testing.assert_array_equal(e.numpy(), np.full(3, 0.5))


def _local_params(lr_scale=1.0):
    sf.init_runtime(sf.RuntimeOptions())
    nn.install()
    tr = resnet.ResNetTrain(sf, batch=4, mode="staged", seed=0, **SMALL)
    tr.LR = resnet.ResNetTrain.LR * lr_scale
    rng = np.random.default_rng(1000)  # the DP rank-0 data
    x = sf.tensor_from_host(rng.standard_normal((4, 32, 32, 3)).astype(np.float32),
                            (4, 32, 32, 3), sf.float32)
    labels = sf.tensor_from_host(rng.integers(0, 1000, size=(4,)), (4,), sf.int32)
    for _ in range(2):
        tr.step(x, labels)
    return [p.read_value().numpy() for p in tr.model.params]


def _dp_params(grad_scale=1.0, bucket_bytes=sfcomm.BUCKET_BYTES):
    sf.init_runtime(sf.RuntimeOptions())
    nn.install()
    com = sfcomm.Communicator(1, 0, 0)
    dp = sfdist.ResNetDataParallel(sf, 4, com, seed=0, grad_scale=grad_scale,
                                   bucket_bytes=bucket_bytes, **SMALL)
    for _ in range(2):
        dp.step()
    out = [p.read_value().numpy() for p in dp.train.model.params]
    return out, dp, com


def test_dp_step_world1_equals_local_step():
    want = _local_params()
    got, _, com = _dp_params()
    com.close()
    for a, b in zip(got, want):
        assert a.tobytes() == b.tobytes()


def test_scaled_collective_feeds_the_update():
    """The all-reduce sums 2 x grad (NCCL premul sum); the update then equals
    a local step with twice the learning rate, bit for bit — the reduced
    buffers are what the update reads."""
    want = _local_params(lr_scale=2.0)
    got, _, com = _dp_params(grad_scale=2.0)
    com.close()
    for a, b in zip(got, want):
        assert a.tobytes() == b.tobytes()
    plain = _local_params()
    assert any(a.tobytes() != b.tobytes() for a, b in zip(got, plain))


def test_allreduce_steps_sit_inside_the_backward_plan():
    _, dp, com = _dp_params(bucket_bytes=64 << 10)
    plans = dp.backward_plans()
    assert plans
    kinds = [k for p in plans for k, _, _ in p.step_stats()]
    ar = [i for i, k in enumerate(kinds) if k == 12]
    assert len(ar) >= 3  # several buckets
    # the first bucket goes out while backward kernels are still to come
    assert ar[0] < max(i for i, k in enumerate(kinds) if k != 12)
    com.close()
