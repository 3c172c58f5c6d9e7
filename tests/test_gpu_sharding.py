"""Chain sharding below the trace cache (paper_1903_01855_b200/sharding.py,
SURVEY.md §8(e)): contiguous shards of the batch, traced once at the full
batch, equal the unsharded run bit for bit (the reference's own property:
3 leapfrog trajectories at B=200 split into 2 or 8 shards are identical)."""
import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins
from paper_1903_01855_b200.sharding import NotShardable, shard
from paper_1903_01855_b200.workloads import l2hmc
from paper_1903_01855_b200.workloads.leapfrog import Leapfrog

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_leapfrog_shards_equal_unsharded(shards):
    ref = Leapfrog(200, "staged", seed=0)
    want = [ref.run_iteration() for _ in range(3)]
    wl = Leapfrog(200, "staged", seed=0)
    f = shard(wl.trajectory, shards=shards)
    q, p = wl.q, wl.p
    for t in range(3):
        q, p = f(q, p)
        got = np.concatenate([q.numpy().ravel(), p.numpy().ravel()])
        assert got.tobytes() == want[t].tobytes()
    assert wl.trajectory.cache_size == 1  # traced once, at the full batch


def test_l2hmc_draws_as_inputs_shards_equal_unsharded():
    plugins.install()
    ref = l2hmc.L2HMCSampler(sf, 300, "staged", seed=0, draws="inputs", draw_seed=5)
    s = l2hmc.L2HMCSampler(sf, 300, "staged", seed=0, draws="inputs", draw_seed=5)
    f = shard(s.transition, shards=2)
    x = s.x
    for _ in range(2):
        draws = ref.host_draws()
        ref.step(draws)
        ts = [sf.tensor_from_host(d.reshape(-1), d.shape, sf.float32) for d in draws]
        x, acc = f(x, *ts)
        assert x.numpy().tobytes() == ref.x.numpy().tobytes()
        assert acc.numpy().tobytes() == ref.accept.numpy().tobytes()
    assert s.transition.cache_size == 1


def test_cross_chain_graph_is_not_shardable():
    f = sf.stage(lambda x: sf.mul(x, sf.reduce_sum(x)))
    x = sf.constant(np.ones((8, 2), np.float32))
    with pytest.raises(NotShardable):
        shard(f, shards=2)(x)


@pytest.mark.skipif(_native.device_count() < 2, reason="needs two GPUs")
def test_leapfrog_shards_on_two_gpus():
    sf.init_runtime(sf.RuntimeOptions(gpus=2))
    ref = Leapfrog(200, "staged", seed=0)
    want = ref.run_iteration()
    wl = Leapfrog(200, "staged", seed=0)
    devs = [d.name for d in sf.get_runtime().devices]
    q, p = shard(wl.trajectory, devices=devs)(wl.q, wl.p)
    assert np.concatenate([q.numpy().ravel(), p.numpy().ravel()]).tobytes() == want.tobytes()


two_gpus = pytest.mark.skipif(_native.device_count() < 2, reason="needs two GPUs")


@two_gpus
def test_add_across_gpus_counts_two_copies():
    """reference tests/test_devices.py:40-49 with GPU:0 / GPU:1 for CPU:0 /
    ACCEL:0: two tensors on GPU:0 added under a GPU:1 scope -> 2 copies."""
    rt = sf.init_runtime(sf.RuntimeOptions(gpus=2))
    g1 = rt.devices[1].name
    a, b = sf.constant(1.0), sf.constant(2.0)
    before = rt.stats.snapshot()["transparent_copies"]
    with sf.device_scope(g1):
        c = sf.add(a, b)
    assert float(c) == 3.0 and c.device == g1
    assert rt.stats.snapshot()["transparent_copies"] - before == 2


@two_gpus
def test_value_device_independence_across_gpus():
    """reference tests/test_devices.py:134-139: same bytes on either device."""
    rt = sf.init_runtime(sf.RuntimeOptions(gpus=2))
    x = sf.constant(np.linspace(-1, 1, 8).astype(np.float32))
    on0 = sf.softplus(x)
    with sf.device_scope(rt.devices[1].name):
        on1 = sf.softplus(x)
    assert on0.numpy().tobytes() == on1.numpy().tobytes()


@two_gpus
def test_executor_copies_counted_in_graphs_across_gpus():
    """reference tests/test_devices.py:141-153: a mul pinned to GPU:1 in a
    graph run on GPU:0 -> x copied over, the product copied back: 2 copies."""
    from paper_1903_01855_b200.devices import DeviceName
    from paper_1903_01855_b200.graph import GraphBuilder

    rt = sf.init_runtime(sf.RuntimeOptions(gpus=2))
    b = GraphBuilder()
    x = b.add_placeholder("x", sf.float32, ())
    (m,) = b.add_node("mul", [x, x], {}, rt.devices[1].name, [(sf.float32, ())])
    (y,) = b.add_node("add", [m, x], {}, None, [(sf.float32, ())])
    gf = b.finalize("mixed", [y], ["y"])
    before = rt.stats.snapshot()["transparent_copies"]
    out = sf.execute(gf, [sf.constant(3.0)])
    assert float(out[0]) == 12.0
    assert rt.stats.snapshot()["transparent_copies"] - before == 2
