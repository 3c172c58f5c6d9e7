"""The native eager front-end (csrc/sf_eager.cpp) and the launch queue
(csrc/sf_queue.cu) against the reference-semantics Python dispatcher.

Three executions of the same eager program must agree bit-for-bit, with the
same RuntimeStats and the same tape gradients:
  * native fast path + launch queue (the default),
  * native fast path, queue disabled (one kernel per op),
  * Python dispatcher (``ops._dispatch_py`` — the reference's
    stageflow/ops.py:294-362 logic) with the queue disabled.
The queue must also keep stream order against everything that is not queued
(reductions, large ops, host reads, staged calls).
"""
import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _fastpath, _native
from paper_1903_01855_b200 import ops as sfops
from paper_1903_01855_b200 import plugins

pytestmark = pytest.mark.gpu

MODES = ("queue", "direct", "python")


class _Mode:
    def __init__(self, mode):
        self.mode = mode

    def __enter__(self):
        self.was = _fastpath.set_enabled(self.mode != "python")
        _native.queue_config(0, 0 if self.mode != "queue" else 64)
        return self

    def __exit__(self, *exc):
        _native.queue_flush(0)
        _native.queue_config(0, 64)
        _fastpath.set_enabled(self.was)


def _random_program(seed, n_ops=40, shape=(7, 5)):
    """A random eager program over elementwise ops, matmuls, transposes,
    reshapes, broadcasts, reductions and scalar operands (the op mix of the
    reference's randomized eager==staged test, tests/test_ops.py:163-171)."""
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(0.5, 1.5, size=shape).astype(np.float32)
    w0 = rng.uniform(-0.5, 0.5, size=(shape[1], shape[1])).astype(np.float32)
    plan = [(rng.integers(0, 12), float(rng.uniform(0.5, 2.0)), int(rng.integers(0, 1 << 30)))
            for _ in range(n_ops)]

    def run():
        x = sf.constant(x0)
        w = sf.constant(w0)
        vals = [x]
        for kind, c, pick in plan:
            a = vals[pick % len(vals)]
            b = vals[(pick >> 8) % len(vals)]
            if kind == 0:
                y = sf.add(a, b)
            elif kind == 1:
                y = a * c
            elif kind == 2:
                y = c - a
            elif kind == 3:
                y = sf.div(a, sf.add(sf.relu(b), 1.0))
            elif kind == 4:
                y = sf.matmul(a, w)
            elif kind == 5:
                y = sf.transpose(sf.transpose(a))
            elif kind == 6:
                y = sf.reshape(sf.reshape(a, (shape[1], shape[0])), shape)
            elif kind == 7:
                y = sf.broadcast_to(sf.reduce_sum(a, axes=(0,), keepdims=True), shape)
            elif kind == 8:
                y = plugins.tanh(a)
            elif kind == 9:
                y = sf.softplus(sf.neg(a))
            elif kind == 10:
                y = sf.exp(sf.mul(a, 0.1))
            else:
                y = sf.sub(a, sf.reduce_mean(b))
            vals.append(y)
        return [v.numpy() for v in vals[-6:]]

    return run


@pytest.mark.parametrize("seed", range(8))
def test_random_programs_bitwise_across_paths(seed):
    plugins.install()
    run = _random_program(seed)
    outs = {}
    for mode in MODES:
        with _Mode(mode):
            outs[mode] = run()
    for mode in MODES[1:]:
        for got, want in zip(outs[mode], outs["queue"]):
            assert got.tobytes() == want.tobytes(), mode


def test_stats_match_python_dispatcher():
    plugins.install()
    run = _random_program(3, n_ops=30)
    snaps = {}
    for mode in ("queue", "python"):
        rt = sf.init_runtime(sf.RuntimeOptions())
        plugins.install()
        with _Mode(mode):
            run()
        snaps[mode] = rt.stats.snapshot()
    assert snaps["queue"] == snaps["python"]
    assert snaps["queue"]["eager_dispatches"] > 30


def test_fast_path_counts_fold_into_stats():
    rt = sf.get_runtime()
    x = sf.constant(np.ones((3, 3), np.float32))
    before = rt.stats.eager_dispatches
    for _ in range(5):
        x = x + 1.0
    assert rt.stats.eager_dispatches - before == 5
    assert rt.stats.eager_op_counts["add"] >= 5
    rt.stats.reset()
    assert rt.stats.eager_dispatches == 0
    x = x * 2.0
    assert rt.stats.snapshot()["eager_op_counts"] == {"mul": 1}


def _tape_program():
    rng = np.random.default_rng(0)
    q0 = rng.standard_normal((200, 2)).astype(np.float32)
    w0 = rng.standard_normal((2, 2)).astype(np.float32)

    def run():
        q = sf.constant(q0)
        w = sf.constant(w0)
        with sf.Tape(persistent=True) as tape:
            tape.watch(q)
            tape.watch(w)
            h = plugins.tanh(sf.matmul(q, w))
            u = sf.reduce_sum(sf.mul(sf.mul(h, h), 0.5)) + sf.reduce_sum(sf.softplus(q))
        gq, gw = tape.gradient(u, [q, w])
        return gq.numpy(), gw.numpy()

    return run


def test_tape_gradients_bitwise_across_paths():
    plugins.install()
    run = _tape_program()
    got = {}
    for mode in MODES:
        with _Mode(mode):
            got[mode] = run()
    for mode in MODES[1:]:
        for a, b in zip(got[mode], got["queue"]):
            assert a.tobytes() == b.tobytes(), mode


def test_leapfrog_eager_matches_reference_golden_via_queue():
    from paper_1903_01855_b200.workloads.leapfrog import Leapfrog
    from oracle import workloads_np

    eager = Leapfrog(200, "eager", seed=0)
    staged = Leapfrog(200, "staged", seed=0)
    e = eager.run_iteration()
    s = staged.run_iteration()
    assert e.tobytes() == s.tobytes()
    np.testing.assert_allclose(e, workloads_np.leapfrog(200, seed=0, trajectories=1),
                               rtol=1e-4, atol=1e-6)


def test_queue_batches_launches():
    _native.queue_flush(0)
    pushed0, flushes0 = _native.queue_stats(0)
    launches0 = _native.launch_count(0)
    x = sf.constant(np.arange(16, dtype=np.float32).reshape(1, 16))
    for _ in range(100):
        x = x * 1.0001 + 0.5
    out = x.numpy()
    pushed, flushes = _native.queue_stats(0)
    assert pushed - pushed0 >= 200
    assert flushes - flushes0 <= 5  # 64 ops per launch
    assert _native.launch_count(0) - launches0 <= 6
    want = np.arange(16, dtype=np.float32).reshape(1, 16)
    for _ in range(100):
        want = (want * np.float32(1.0001)).astype(np.float32) + np.float32(0.5)
    assert out.tobytes() == want.astype(np.float32).tobytes()


def test_queue_order_against_unqueued_work():
    """Queued ops interleaved with direct launches (a large op), reductions,
    staged calls and host reads see each other's results in program order."""
    big = sf.constant(np.ones((300, 100), np.float32))   # 30000 > queue limit
    small = sf.constant(np.full((4, 4), 2.0, np.float32))

    @sf.stage
    def staged(a):
        return a * 3.0

    s = small
    for _ in range(3):
        s = s + 1.0                       # queued
        b = big + 1.0                     # direct launch (too big to queue)
        r = sf.reduce_sum(s)              # reduction (flushes the queue)
        s = staged(s)                     # staged call (flushes)
        s = s - sf.reshape(r, (1, 1))     # queued, reads r
    got = s.numpy()
    want = np.full((4, 4), 2.0, np.float32)
    for _ in range(3):
        want = want + np.float32(1.0)
        r = np.float32(want.sum(dtype=np.float32))
        want = want * np.float32(3.0)
        want = want - r
    np.testing.assert_array_equal(got, want)
    assert float(sf.reduce_sum(b)) == 60000.0


def test_queue_survives_freed_inputs():
    """Tensors dropped while their readers are still queued: the allocator
    only hands their blocks to later (ordered) writers."""
    vals = []
    x = sf.constant(np.full((8, 8), 1.0, np.float32))
    for i in range(60):
        y = sf.add(x, float(i))
        x = sf.mul(y, 1.0)     # y dropped next iteration while queued
        vals.append(float(i))
    got = x.numpy()
    want = np.full((8, 8), 1.0, np.float32)
    for v in vals:
        want = want + np.float32(v)
    np.testing.assert_array_equal(got, want)


def test_int32_and_bool_through_queue():
    a = sf.constant(np.array([[2 ** 31 - 1, -5, 7]], np.int32))
    b = sf.constant(np.array([[2, 3, -7]], np.int32))
    np.testing.assert_array_equal(sf.mul(a, b).numpy(),
                                  (a.numpy().astype(np.int64) * b.numpy()).astype(np.int32))
    g = sf.greater(a, b)
    assert g.dtype is sf.boolean
    np.testing.assert_array_equal(g.numpy(), a.numpy() > b.numpy())
    np.testing.assert_array_equal(sf.broadcast_to(g, (2, 3)).numpy(),
                                  np.broadcast_to(a.numpy() > b.numpy(), (2, 3)))
    np.testing.assert_array_equal((a + 3).numpy(), a.numpy() + np.int32(3))


def test_scalar_coercion_matches_reference():
    """Python scalars are taken 'like' the tensor (reference _as_operand,
    ops.py:370-383): f32 rounding of a double, reflected operators."""
    x = sf.constant(np.array([1.0, 2.0, 3.0], np.float32))
    c = 0.1
    np.testing.assert_array_equal((x * c).numpy(), x.numpy() * np.float32(c))
    np.testing.assert_array_equal((c - x).numpy(), np.float32(c) - x.numpy())
    np.testing.assert_array_equal((2 / x).numpy(), np.float32(2) / x.numpy())
    np.testing.assert_array_equal((-x).numpy(), -x.numpy())
    np.testing.assert_array_equal((x > 1.5).numpy(), x.numpy() > 1.5)
    np.testing.assert_array_equal((0.5 < x).numpy(), x.numpy() > 0.5)  # reflected __gt__
    with pytest.raises(TypeError):
        _ = x < 1.0
    assert (x == x) is True and (x != x) is False
    d = sf.constant(np.array([1.0, 2.0], np.float64))
    np.testing.assert_array_equal((d * 0.1).numpy(), d.numpy() * 0.1)


def test_errors_identical_on_fast_path():
    from paper_1903_01855_b200.errors import KernelError

    f = sf.constant(np.ones(3, np.float32))
    i = sf.constant(np.ones(3, np.int32))
    for fn in (lambda: sf.add(f, i), lambda: sf.div(i, i), lambda: sf.exp(i),
               lambda: sf.add(sf.constant(np.ones((2, 3), np.float32)),
                              sf.constant(np.ones((4,), np.float32))),
               lambda: sf.matmul(f, f), lambda: sf.reshape(f, (2, 2))):
        msgs = []
        for mode in ("queue", "python"):
            with _Mode(mode):
                with pytest.raises(KernelError) as e:
                    fn()
                msgs.append(str(e.value))
        assert msgs[0] == msgs[1]


def test_identity_is_fresh_handle_and_reshape_is_view():
    x = sf.constant(np.arange(6, dtype=np.float32))
    y = sfops.identity(x)
    assert y is not x and y.numpy().tobytes() == x.numpy().tobytes()
    z = sf.reshape(x, (2, 3))
    assert z.shape == (2, 3)
    np.testing.assert_array_equal(z.numpy(), np.arange(6, dtype=np.float32).reshape(2, 3))


# -- the native staged-call path (StagedFast, csrc/sf_eager.cpp) ----------------


def _staged_program():
    rng = np.random.default_rng(5)
    w = sf.constant(rng.standard_normal((4, 4)).astype(np.float32))
    b = sf.constant(rng.standard_normal((1, 4)).astype(np.float32))

    def body(x, y):
        h = plugins.tanh(sf.add(sf.matmul(x, w), b))
        return sf.mul(h, y), sf.reduce_sum(h)

    return body


def test_staged_fast_path_bitwise_and_counters():
    plugins.install()
    rng = np.random.default_rng(0)
    xs = [sf.constant(rng.standard_normal((64, 4)).astype(np.float32)) for _ in range(4)]
    y = sf.constant(np.full((64, 4), 0.5, np.float32))
    results, snaps = {}, {}
    for mode in ("queue", "python"):
        rt = sf.init_runtime(sf.RuntimeOptions())
        plugins.install()
        with _Mode(mode):
            f = sf.stage(_staged_program())
            outs = [f(x, y) for x in xs]
            results[mode] = [(a.numpy(), s.numpy()) for a, s in outs]
            snaps[mode] = (rt.stats.snapshot(), f.cache_size)
            if mode == "queue":
                assert f._fast is not None  # armed after the first call
    for (a0, s0), (a1, s1) in zip(results["queue"], results["python"]):
        assert a0.tobytes() == a1.tobytes() and s0.tobytes() == s1.tobytes()
    assert snaps["queue"] == snaps["python"]
    assert snaps["queue"][0]["eager_op_counts"]["call_function"] == 4
    assert snaps["queue"][0]["traces"] == 1


def test_staged_fast_path_misses_fall_back():
    plugins.install()
    rt = sf.get_runtime()
    f = sf.stage(_staged_program())
    y = sf.constant(np.ones((8, 4), np.float32))
    a = f(sf.constant(np.ones((8, 4), np.float32)), y)
    launches = rt.stats.graph_launches
    b = f(sf.constant(np.ones((8, 4), np.float32)), y)          # fast path
    assert rt.stats.graph_launches == launches + 1
    assert a[0].numpy().tobytes() == b[0].numpy().tobytes()
    c = f(sf.constant(np.ones((16, 4), np.float32)),               # new shape: retrace
          sf.constant(np.ones((16, 4), np.float32)))
    assert c[0].shape == (16, 4) and f.cache_size == 2
    with sf.Tape() as t:                                           # a tape: reference path
        x = sf.constant(np.ones((8, 4), np.float32))
        t.watch(x)
        out, s = f(x, y)
    g = t.gradient(s, x)
    assert g.shape == (8, 4)
    sf.init_runtime(sf.RuntimeOptions())                           # a new runtime: miss
    plugins.install()
    d = f(sf.constant(np.ones((8, 4), np.float32)), sf.constant(np.ones((8, 4), np.float32)))
    assert d[0].numpy().tobytes() == a[0].numpy().tobytes()


def test_l2hmc_staged_fast_path_matches_reference_path():
    from paper_1903_01855_b200.workloads import l2hmc

    outs = {}
    for mode in ("queue", "python"):
        sf.init_runtime(sf.RuntimeOptions(seed=3))
        plugins.install()
        with _Mode(mode):
            s = l2hmc.L2HMCSampler(sf, 200, "staged", seed=0)
            outs[mode] = np.stack([s.run_iteration() for _ in range(4)])
    assert outs["queue"].tobytes() == outs["python"].tobytes()
