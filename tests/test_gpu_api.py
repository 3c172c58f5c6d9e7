"""API-level parity on the GPU: tapes, staging, graph functions, variables,
host callbacks.  Restates the reference's behavioural tests
(tests/test_tape.py, test_staging.py, test_graph.py, test_state.py,
test_escape.py) against this backend, plus traced-graph structure parity
against SGF1 bytes produced by the reference itself."""
import gc
import os
import threading
import time

import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200.errors import (CallbackError, ConsumedTape, DeadVariable, InputMismatch,
                                          MissingFunction, NonScalarTarget, NotSerializable,
                                          ShapeMismatch, SignatureMismatch, SignatureViolation,
                                          StagingError, UnwatchedSource, VariableCreationError)
from paper_1903_01855_b200.graph import GraphBuilder, constant_fold, optimize, prune
from paper_1903_01855_b200.serial import deserialize, serialize

from helpers import (FD_OPS, build_mlp, central_diff, fd_case, fd_loss, max_rel_err,
                     random_graph, tape_grads)

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


# ---------------------------------------------------------------- tapes
def test_read_only_pinned_result_uploads_asynchronously():
    """A result array from Tensor.raw() fed back (the e2e sampler loop):
    pooled page-locked memory behind a read-only memoryview, uploaded by an
    asynchronous DMA, doubles as the tensor's host copy; the pool block is
    reused only by later copies on the same stream, so churning downloads
    cannot corrupt the upload.  An array the caller froze itself (numpy() +
    writeable=False) is copied: the caller could unfreeze it."""
    from paper_1903_01855_b200 import _native

    n = 300000
    base = np.arange(n, dtype=np.float32)
    h = sf.constant(base).raw()
    assert _native.frozen_pinned(h)
    with pytest.raises(ValueError):
        h.flags.writeable = True
    t = sf.tensor_from_host(h, (n,), sf.float32)
    assert np.shares_memory(t.raw(), h)  # aliased (async DMA), not copied
    y = sf.add(t, sf.constant(np.float32(1.0)))
    del h
    for _ in range(5):
        z = y.numpy()
    np.testing.assert_array_equal(z, base + np.float32(1.0))
    # a caller-frozen array is not trusted: synchronous private copy
    u = sf.constant(base).numpy()
    u.flags.writeable = False
    assert not _native.frozen_pinned(u)
    t3 = sf.tensor_from_host(u, (n,), sf.float32)
    assert not np.shares_memory(t3.raw(), u)
    u.flags.writeable = True
    u[:] = -1
    np.testing.assert_array_equal(t3.numpy(), base)
    # writable or user-owned arrays keep the synchronous copy
    w = base.copy()
    t2 = sf.tensor_from_host(w, (n,), sf.float32)
    w[:] = -1
    np.testing.assert_array_equal(t2.numpy(), base)


def test_staged_variable_updates_fold_into_groups_bitwise():
    """v.assign_add(g * -lr) for several same-shape variables: the staged
    program stores v + increment from the group that computes the increment
    (in place); values match eager bit for bit, and a read after the update
    inside the same function sees the new value."""
    rng = np.random.default_rng(8)
    shapes = [(64, 32), (64, 32), (128,)]
    init = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    grads = [sf.constant(rng.standard_normal(s).astype(np.float32)) for s in shapes]

    def run(staged):
        vs = [sf.Variable(sf.constant(a)) for a in init]

        def update(*gs):
            for v, g in zip(vs, gs):
                v.assign_add(sf.mul(g, -0.125))
            return sf.reduce_sum(sf.mul(vs[0].read_value(), 2.0))

        f = sf.stage(update) if staged else update
        outs = [f(*grads).numpy() for _ in range(3)]
        return [v.read_value().numpy() for v in vs], outs

    (ve, oe), (vs_, os_) = run(False), run(True)
    for a, b in zip(ve, vs_):
        assert a.tobytes() == b.tobytes()
    for a, b in zip(oe, os_):
        assert a.tobytes() == b.tobytes()


def test_staged_backward_computes_only_gradients_that_can_be_read():
    """A tape over a staged call asks its backward only for gradients that
    can reach a requested source: the input images' gradient is pruned and
    conv2d_grads narrows to the filter gradient; results are unchanged."""
    from paper_1903_01855_b200 import nn
    from paper_1903_01855_b200.backprop import get_forward_backward

    nn.install()
    rng = np.random.default_rng(4)
    x = sf.constant(rng.standard_normal((2, 9, 9, 8)).astype(np.float32))
    w = sf.Variable(sf.constant(rng.standard_normal((3, 3, 8, 4)).astype(np.float32)))

    def loss(x):
        return sf.reduce_sum(nn.conv2d(x, w.read_value(), stride=1, pad=1))

    staged = sf.stage(loss)
    grads = []
    for f in (loss, staged):
        with sf.Tape() as t:
            val = f(x)
        grads.append(t.gradient(val, [w])[0].numpy())
    np.testing.assert_allclose(grads[1], grads[0], rtol=1e-5, atol=1e-4)
    cf = staged.cached_functions()[0]
    bwd = get_forward_backward(cf.graph)[1]
    sel = list(getattr(bwd, "_selected", {}).values())
    assert sel, "the backward was not restricted to the readable gradients"
    ops_used = {n.op for n in sel[0].graph.nodes}
    assert "conv2d_grad_filter" in ops_used and "conv2d_grads" not in ops_used


def test_reading_one_output_reads_small_siblings_in_the_same_round_trip():
    rng = np.random.default_rng(2)
    xa = rng.standard_normal((50000, 2)).astype(np.float32)

    @sf.stage
    def f(x):
        return sf.mul(x, 2.0), sf.reduce_sum(sf.exp(x), axes=(1,))

    x = sf.constant(xa)
    for _ in range(2):  # second call: the traced program is warm
        a, b = f(x)
    ha = a.numpy()
    assert b._pend is not None          # enqueued with a's read
    hb = b.numpy()
    assert b._pend is None
    np.testing.assert_array_equal(ha, xa * np.float32(2.0))
    np.testing.assert_allclose(hb, np.exp(xa.astype(np.float64)).sum(1), rtol=1e-6)
    a2, b2 = f(x)
    assert b2.raw().tobytes() == hb.tobytes() and not b2.raw().flags.writeable


def test_listing_square_and_nested():
    x = sf.constant(3.0)
    with sf.Tape() as t1:
        with sf.Tape() as t2:
            t1.watch(x)
            t2.watch(x)
            y = x * x
        dy = t2.gradient(y, x)
    assert float(dy) == 6.0 and float(t1.gradient(dy, x)) == 2.0


def test_variable_auto_watch():
    x = sf.Variable(3.0)
    with sf.Tape() as t1:
        with sf.Tape() as t2:
            y = x * x
        dy = t2.gradient(y, x)
    assert float(dy) == 6.0 and float(t1.gradient(dy, x)) == 2.0


def test_tape_errors_and_zeros():
    x, z = sf.constant([1.0, 2.0]), sf.constant(5.0)
    with sf.Tape() as t:
        t.watch(x)
        t.watch(z)
        y = sf.reduce_sum(x)
    g = t.gradient(y, z)
    assert g.shape == () and float(g) == 0.0
    with pytest.raises(ConsumedTape):
        t.gradient(y, x)
    with sf.Tape() as t:
        t.watch(x)
        y = sf.mul(x, x)
    with pytest.raises(NonScalarTarget):
        t.gradient(y, x)
    with sf.Tape() as t:
        y = sf.mul(z, z)
    with pytest.raises(UnwatchedSource):
        t.gradient(y, z)


def test_persistent_and_relu_kink():
    x = sf.constant(2.0)
    with sf.Tape(persistent=True) as t:
        t.watch(x)
        y = x * x
        z = y * x
    assert float(t.gradient(y, x)) == 4.0 and float(t.gradient(z, x)) == 12.0
    x = sf.constant(0.0)
    with sf.Tape() as t:
        t.watch(x)
        y = sf.relu(x)
    assert float(t.gradient(y, x)) == 0.0


def test_dropout_gradient_is_mask():
    x = sf.constant(np.full(64, 2.0, dtype=np.float32))
    with sf.Tape() as t:
        t.watch(x)
        out, mask = sf.dispatch("dropout", [x], {"rate": 0.5})
        y = sf.reduce_sum(out)
    np.testing.assert_array_equal(t.gradient(y, x).numpy(), mask.numpy())


@pytest.mark.parametrize("op_name", sorted(FD_OPS))
def test_fd_float64(op_name):
    spec = FD_OPS[op_name]
    rng = np.random.default_rng(11)
    worst = 0.0
    for _ in range(3):
        arrays, weights = fd_case(op_name, spec, rng, sf.float64)
        grads = tape_grads(op_name, spec, arrays, weights)
        loss = fd_loss(op_name, spec, weights)
        for i in range(len(arrays)):
            worst = max(worst, max_rel_err(grads[i], central_diff(loss, arrays, i, 1e-3), 1e-6))
    assert worst < 1e-6, f"{op_name}: {worst}"


@pytest.mark.parametrize("op_name", ["mul", "matmul", "softplus", "relu"])
def test_fd_float32(op_name):
    spec = FD_OPS[op_name]
    rng = np.random.default_rng(5)
    for _ in range(3):
        arrays, weights = fd_case(op_name, spec, rng, sf.float32)
        grads = tape_grads(op_name, spec, arrays, weights)
        loss = fd_loss(op_name, spec, weights)
        for i in range(len(arrays)):
            assert max_rel_err(grads[i], central_diff(loss, arrays, i, 1e-3), 1e-3) < 1e-3


@pytest.mark.parametrize("x0", [-2.0, 0.0, 2.0])
def test_cubic_second_derivative_exact(x0):
    x = sf.tensor_from_host([x0], (), sf.float64)

    def c(v):
        return sf.tensor_from_host([v], (), sf.float64)

    with sf.Tape() as outer:
        outer.watch(x)
        with sf.Tape() as inner:
            inner.watch(x)
            y = sf.sub(sf.add(sf.sub(sf.mul(c(2.0), sf.mul(x, sf.mul(x, x))),
                                     sf.mul(c(3.0), sf.mul(x, x))), sf.mul(c(4.0), x)), c(1.0))
        dy = inner.gradient(y, x)
    assert float(dy) == 6.0 * x0 ** 2 - 6.0 * x0 + 4.0
    assert float(outer.gradient(dy, x)) == 12.0 * x0 - 6.0


def test_staged_gradients_match_eager_mlp():
    rng = np.random.default_rng(0)
    params, forward = build_mlp(rng)
    x = sf.constant(rng.standard_normal((4, 16)).astype(np.float32))

    def loss_fn(v):
        out = forward(v)
        return sf.reduce_mean(sf.mul(out, out))

    order = [params[k] for k in ("w1", "b1", "w2", "b2")]
    with sf.Tape() as t:
        loss = loss_fn(x)
    eager = [g.numpy() for g in t.gradient(loss, order)]
    staged = sf.stage(loss_fn)
    with sf.Tape() as t2:
        loss_s = staged(x)
    got = [g.numpy() for g in t2.gradient(loss_s, order)]
    assert abs(float(loss) - float(loss_s)) < 1e-6
    for ge, gs in zip(eager, got):
        np.testing.assert_allclose(gs, ge, rtol=1e-6, atol=1e-6)


def test_staged_backward_is_one_call():
    pf = sf.stage(lambda v: sf.reduce_sum(sf.mul(v, v)))
    x = sf.constant(np.ones(8, dtype=np.float32))
    with sf.Tape() as t:
        t.watch(x)
        y = pf(x)
    before = dict(sf.get_runtime().stats.snapshot()["eager_op_counts"])
    g = t.gradient(y, x)
    after = sf.get_runtime().stats.snapshot()["eager_op_counts"]
    delta = {k: after.get(k, 0) - before.get(k, 0) for k in set(after) | set(before)}
    assert {k: v for k, v in delta.items() if v} == {"call_function": 1}
    np.testing.assert_array_equal(g.numpy(), 2.0 * np.ones(8, dtype=np.float32))


# ---------------------------------------------------------------- staging
def test_trace_cache_hits_and_misses():
    pf = sf.stage(lambda x: sf.reduce_sum(x))
    a = sf.constant(np.zeros((3, 5), dtype=np.float32))
    pf(a)
    pf(sf.constant(np.ones((3, 5), dtype=np.float32)))
    assert pf.cache_size == 1 and pf.trace_count == 1
    pf(sf.constant(np.ones((4, 5), dtype=np.float32)))
    assert pf.cache_size == 2 and pf.trace_count == 2


def test_listing5_dropout_specialisation():
    def lossy(w, x, training=True):
        out = sf.matmul(w, x)
        return sf.dropout(out, 0.2) if training else out

    pf = sf.stage(lossy)
    w, x = sf.random_normal((3, 5)), sf.random_normal((5, 1))
    pf(w, x, training=True)
    pf(w, x, training=False)
    assert pf.cache_size == 2
    assert sorted("dropout" in cf.graph.op_counts() for cf in pf.cached_functions()) == [False, True]


def test_host_rng_freezes():
    def f():
        return sf.add(sf.eye(5), sf.constant(np.random.default_rng().standard_normal((5, 5))
                                             .astype(np.float32)))

    staged = sf.stage(f)
    first = staged().numpy()
    for _ in range(3):
        np.testing.assert_array_equal(staged().numpy(), first)


def test_concurrent_same_key_traces_once():
    pf = sf.stage(lambda x: sf.mul(x, x))
    x = sf.constant(2.0)
    errors = []

    def call():
        try:
            assert float(pf(x)) == 4.0
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ts = [threading.Thread(target=call) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors and pf.cache_size == 1 and pf.trace_count == 1


def test_pinned_wildcard_signature():
    pf = sf.stage(lambda x: sf.reduce_sum(x, axes=(1,)), signature=[(sf.float32, (None, 5))])
    a = pf(sf.constant(np.ones((2, 5), dtype=np.float32)))
    b = pf(sf.constant(np.ones((7, 5), dtype=np.float32)))
    assert a.shape == (2,) and b.shape == (7,) and pf.cache_size == 1 and pf.trace_count == 1
    np.testing.assert_array_equal(b.numpy(), np.full(7, 5.0, np.float32))
    with pytest.raises(SignatureMismatch):
        pf(sf.constant(np.ones((2, 5), dtype=np.float64)))


def test_capture_and_mutation_semantics():
    outside = sf.constant([1.0, 2.0])
    f = sf.stage(lambda x: sf.add(sf.add(x, outside), outside))
    x = sf.constant([0.5, 0.5])
    np.testing.assert_array_equal(f(x).numpy(), [2.5, 4.5])
    assert len(f.get_concrete(f.trace_key_for(x)).graph.inputs) == 2
    v = sf.Variable(0.0)

    @sf.stage
    def mutate():
        v.assign_add(1.0)
        return v.read_value()

    mutate()
    assert float(v.read_value()) == 1.0
    v.assign_add(1.0)
    assert float(v.read_value()) == 2.0
    mutate()
    assert float(v.read_value()) == 3.0


def test_dead_variable():
    v = sf.Variable(1.0)

    @sf.stage
    def read():
        return sf.add(v.read_value(), 1.0)

    assert float(read()) == 2.0
    del v
    gc.collect()
    with pytest.raises(DeadVariable):
        read()


def test_state_creation_contract():
    state = {"v": None}

    def f(x):
        if state["v"] is None:
            state["v"] = sf.Variable(10.0)
        return sf.add(x, state["v"].read_value())

    pf = sf.stage(f)
    assert float(pf(sf.constant(1.0))) == 11.0 and pf.trace_count == 2
    assert float(pf(sf.constant(2.0))) == 12.0 and pf.trace_count == 2

    def g(x):
        return sf.add(x, sf.Variable(1.0).read_value())

    with pytest.raises(VariableCreationError):
        sf.stage(g)(sf.constant(1.0))


def test_nested_call_and_loops():
    inner = sf.stage(lambda a: sf.relu(a), name="inner_relu")

    @sf.stage
    def outer(a, b):
        return inner(sf.matmul(a, b))

    e = sf.eye(3)
    d = sf.constant(np.diag([-1.0, 1.0, 2.0]).astype(np.float32))
    np.testing.assert_array_equal(outer(e, d).numpy(),
                                  np.diag([0.0, 1.0, 2.0]).astype(np.float32))
    graph = outer.get_concrete(outer.trace_key_for(e, d)).graph
    calls = [n for n in graph.nodes if n.op == "call_function"]
    assert len(calls) == 1 and "relu" in graph.library[calls[0].attrs["function"]].op_counts()

    @sf.stage
    def unrolled(x):
        for _ in range(11):
            x = sf.add(x, x)
        return x

    assert float(unrolled(sf.constant(1.0))) == 2048.0


def test_cond_and_while():
    def run(x):
        return sf.cond(sf.greater(x, 0.0), lambda v: sf.mul(v, 2.0), lambda v: sf.neg(v), [x])

    assert float(run(sf.constant(3.0))) == 6.0 and float(run(sf.constant(-3.0))) == 3.0
    staged = sf.stage(run)
    assert float(staged(sf.constant(3.0))) == 6.0 and float(staged(sf.constant(-3.0))) == 3.0

    def sum_to(n):
        _, acc = sf.while_loop(lambda i, acc: sf.greater(i, 0),
                               lambda i, acc: (sf.sub(i, 1), sf.add(acc, i)),
                               [n, sf.constant(0, dtype=sf.int32)])
        return acc

    n = sf.constant(6, dtype=sf.int32)
    assert int(sum_to(n).item()) == 21 and int(sf.stage(sum_to)(n).item()) == 21


def test_device_while_loop_matches_host_loop():
    """while_loop on the device (CUDA graph WHILE node, executor.device_while):
    the first call of a signature loops on the host, later calls replay the
    recorded graph; both must give the host loop's bits, for any trip count."""
    from paper_1903_01855_b200 import executor

    rng = np.random.default_rng(5)
    W = sf.constant(rng.standard_normal((8, 8)).astype(np.float32) * 0.3)

    def iterate(x, n):
        def body(i, v):
            return sf.sub(i, 1), sf.add(sf.matmul(v, W), sf.mul(v, 0.5))

        _, out = sf.while_loop(lambda i, v: sf.greater(i, 0), body, [n, x])
        return out

    staged = sf.stage(iterate)
    x = sf.constant(rng.standard_normal((64, 8)).astype(np.float32))
    cases = [0, 1, 7, 40, 3]
    executor.DEVICE_WHILE = False
    try:
        want = [staged(x, sf.constant(k, dtype=sf.int32)).numpy() for k in cases]
    finally:
        executor.DEVICE_WHILE = True
    got = [staged(x, sf.constant(k, dtype=sf.int32)).numpy() for k in cases * 2]
    for g, w in zip(got, want * 2):
        assert g.tobytes() == w.tobytes()
    progs = [v for gf in _while_bodies(staged) for v in gf.__dict__.get("_device_while",
                                                                       {}).values()]
    assert any(isinstance(p, executor._WhileProgram) for p in progs)
    # int32 accumulation as in the reference's own test (stageflow tests: 21)
    def sum_to(n):
        _, acc = sf.while_loop(lambda i, acc: sf.greater(i, 0),
                               lambda i, acc: (sf.sub(i, 1), sf.add(acc, i)),
                               [n, sf.constant(0, dtype=sf.int32)])
        return acc

    s = sf.stage(sum_to)
    assert [int(s(sf.constant(k, dtype=sf.int32)).item()) for k in (6, 6, 100, 0)] == \
        [21, 21, 5050, 0]


def _while_bodies(pf):
    out = []
    for cf in pf.cached_functions():
        for gf in cf.graph.library.values():
            out.append(gf)
    return out


# ---------------------------------------------------------------- graph functions
def test_constant_fold_and_execute():
    b = GraphBuilder()
    x = b.add_placeholder("x", sf.float32, (2, 2))
    (c1,) = b.add_node("constant", [], {"value": sf.constant([[1.0, 1.0], [1.0, 1.0]])}, None,
                       [(sf.float32, (2, 2))])
    (c2,) = b.add_node("constant", [], {"value": sf.constant([[2.0, 2.0], [2.0, 2.0]])}, None,
                       [(sf.float32, (2, 2))])
    (s,) = b.add_node("add", [c1, c2], {}, None, [(sf.float32, (2, 2))])
    (y,) = b.add_node("matmul", [s, x], {}, None, [(sf.float32, (2, 2))])
    gf = b.finalize("f", [y], ["y"])
    folded = optimize(gf)
    assert folded.op_counts() == {"constant": 1, "matmul": 1}
    xv = sf.constant(np.eye(2, dtype=np.float32))
    np.testing.assert_array_equal(sf.execute(folded, [xv])[0].numpy(), sf.execute(gf, [xv])[0].numpy())


def test_long_chain_and_errors():
    b = GraphBuilder()
    x = b.add_placeholder("x", sf.float64, ())
    ref = x
    for _ in range(1000):
        (ref,) = b.add_node("add", [ref, ref], {}, None, [(sf.float64, ())])
    gf = b.finalize("chain", [ref], ["y"])
    assert float(sf.execute(gf, [sf.tensor_from_host([1.0], (), sf.float64)])[0]) == 2.0 ** 1000
    b = GraphBuilder()
    x = b.add_placeholder("x", sf.float32, ())
    (y,) = b.add_node("call_function", [x], {"function": "ghost"}, None, [(sf.float32, ())])
    with pytest.raises(MissingFunction):
        sf.execute(b.finalize("caller", [y], ["y"]), [sf.constant(1.0)])
    b = GraphBuilder()
    x = b.add_placeholder("x", sf.float32, (2,))
    (y,) = b.add_node("mul", [x, x], {}, None, [(sf.float32, (2,))])
    with pytest.raises(InputMismatch):
        sf.execute(b.finalize("sq", [y], ["y"]), [sf.constant([1.0, 2.0, 3.0])])


def test_optimizer_soundness_random_graphs():
    for seed in range(40):
        gf, inputs, _ = random_graph(seed, max_nodes=25)
        base = sf.execute(gf, inputs)[0].numpy()
        opt = prune(constant_fold(gf))
        assert sf.execute(opt, inputs)[0].numpy().tobytes() == base.tobytes(), seed
        assert len(opt.nodes) <= len(gf.nodes)
    for seed in range(10):
        clean, _, _ = random_graph(seed, max_nodes=20, with_dead=0)
        dirty, _, _ = random_graph(seed, max_nodes=20, with_dead=5)
        assert len(optimize(dirty).nodes) == len(optimize(clean).nodes)


def test_stateful_graph_round_trip():
    v = sf.Variable(0.0)

    @sf.stage
    def bump():
        v.assign_add(1.0)
        return v.read_value()

    bump()
    gf = bump.get_concrete(bump.trace_key_for()).graph
    restored = deserialize(serialize(gf))
    assert float(sf.execute(restored, [], captured=[v])[0]) == 2.0


# ---------------------------------------------------------------- structure parity vs the reference
def test_leapfrog_graph_bytes_match_reference():
    from paper_1903_01855_b200.workloads.leapfrog import Leapfrog

    for b in (10, 200):
        wl = Leapfrog(b, "staged")
        wl.step()
        pf = wl.staged_functions[0]
        gf = pf.cached_functions()[0].graph
        assert serialize(gf) == GOLD[f"leapfrog_graph_{b}"].tobytes()
        assert pf.trace_count == int(GOLD[f"leapfrog_trace_count_{b}"][0])


def test_mlp_graph_bytes_match_reference():
    from paper_1903_01855_b200.workloads.mlp import MLPTrain

    wl = MLPTrain(32, "staged")
    losses = [wl.run_iteration() for _ in range(10)]
    np.testing.assert_allclose(losses, GOLD["mlp_staged_32_losses"], rtol=1e-4)
    gf = wl.forward_loss.cached_functions()[0].graph
    assert serialize(gf) == GOLD["mlp_fwd_graph_32"].tobytes()
    assert serialize(gf._fwd_bwd[1].graph) == GOLD["mlp_bwd_graph_32"].tobytes()
    counts = GOLD["mlp_staged_32_counts"]
    assert [wl.forward_loss.trace_count, wl.apply_updates.trace_count,
            sf.get_runtime().stats.snapshot()["derived_traces"]] == list(counts)


def test_c2_chain_matches_reference():
    from paper_1903_01855_b200.workloads import microbench

    for mode in ("eager", "staged"):
        mb = microbench.Chain(mode)
        out = mb.step().numpy()
        np.testing.assert_allclose(out, GOLD[f"c2_{mode}"], rtol=1e-4, atol=1e-6)
    mb = microbench.Chain("staged")
    mb.step()
    gf = mb.fn.cached_functions()[0].graph
    assert serialize(gf) == GOLD["c2_graph"].tobytes()
    e, s = microbench.Chain("eager").step(), microbench.Chain("staged").step()
    assert e.numpy().tobytes() == s.numpy().tobytes()


# ---------------------------------------------------------------- variables / host callbacks
def test_variable_semantics():
    v = sf.Variable([1.0, 1.0])
    snap = v.read_value()
    v.assign_add([1.0, 1.0])
    np.testing.assert_array_equal(snap.numpy(), [1.0, 1.0])
    np.testing.assert_array_equal(v.numpy(), [2.0, 2.0])
    with pytest.raises(ShapeMismatch):
        v.assign([1.0, 2.0, 3.0])
    a, b = sf.Variable(sf.constant([1.0, 2.0])), sf.Variable(sf.constant([1.0, 2.0]))
    a.assign([9.0, 9.0])
    np.testing.assert_array_equal(b.numpy(), [1.0, 2.0])


def test_host_calls():
    cb = sf.register_callback(lambda x: sf.mul(x, x), [(sf.float32, ())])
    x = sf.constant(3.0)
    with sf.Tape() as t:
        t.watch(x)
        (y,) = sf.host_call(cb, [x])
    assert float(y) == 9.0 and float(t.gradient(y, x)) == 6.0

    def f(v):
        (y,) = sf.host_call(cb, [v])
        return sf.mul(y, 2.0)

    staged = sf.stage(f)
    with sf.Tape() as t2:
        t2.watch(x)
        ys = staged(x)
    assert float(ys) == 18.0 and float(t2.gradient(ys, x)) == 12.0
    bad = sf.register_callback(lambda v: sf.constant([1.0, 2.0]), [(sf.float32, ())])
    with pytest.raises(SignatureViolation):
        sf.host_call(bad, [x])
    boom = sf.register_callback(lambda v: 1 / 0, [(sf.float32, ())])
    with pytest.raises(CallbackError):
        sf.host_call(boom, [x])
    with pytest.raises(NotSerializable):
        serialize(staged.cached_functions()[0].graph)


def test_escape_trace():
    seen = {}

    @sf.stage
    def f(x):
        with sf.escape_trace():
            c = sf.add(sf.constant(2.0), sf.constant(3.0))
            seen["concrete"] = not c.is_symbolic
        return sf.add(x, c)

    assert float(f(sf.constant(1.0))) == 6.0 and seen["concrete"]
    assert f.cached_functions()[0].graph.op_counts()["add"] == 1


def test_device_cond_matches_host_cond():
    """cond on the device (CUDA graph IF/ELSE node, executor.device_cond): both
    branches, repeated calls, captured tensors; bits equal to the host read."""
    from paper_1903_01855_b200 import executor

    rng = np.random.default_rng(9)
    W = sf.constant(rng.standard_normal((8, 8)).astype(np.float32))

    def f(x, flag):
        return sf.cond(flag, lambda v: sf.matmul(v, W), lambda v: sf.mul(sf.neg(v), 2.0), [x])

    staged = sf.stage(f)
    x = sf.constant(rng.standard_normal((16, 8)).astype(np.float32))
    flags = [True, False, True, False, False, True]
    want = [staged(x, sf.constant(b)).numpy() for b in flags]
    executor.DEVICE_COND = True
    try:
        got = [staged(x, sf.constant(b)).numpy() for b in flags * 2]
    finally:
        executor.DEVICE_COND = False
    for g, w in zip(got, want * 2):
        assert g.tobytes() == w.tobytes()
    progs = [p for gf in _while_bodies(staged) for p in gf.__dict__.get("_device_cond",
                                                                      {}).values()]
    assert any(isinstance(p, executor._CondProgram) for p in progs)


def test_program_graph_replay_semantics():
    """Whole-program CUDA-graph replay (executor._ProgramGraph): replays give
    the direct run's bits; fresh input data is copied in; variables are read
    live; an output still held by the caller is never overwritten (the next
    call runs directly instead)."""
    from paper_1903_01855_b200 import executor

    rng = np.random.default_rng(2)
    Ws = [sf.Variable(sf.constant(rng.standard_normal((64, 64)).astype(np.float32) * 0.2))
          for _ in range(12)]

    def f(x):
        h = x
        for W in Ws:
            h = sf.relu(sf.matmul(h, W.read_value()))
        return h, sf.reduce_sum(h)

    def direct(x):
        executor.GRAPH_REPLAY = False
        try:
            return [t.numpy() for t in sf.stage(f)(x)]
        finally:
            executor.GRAPH_REPLAY = True

    staged = sf.stage(f)
    xs = [sf.constant(rng.standard_normal((64, 64)).astype(np.float32)) for _ in range(4)]
    got = [[t.numpy() for t in staged(x)] for x in xs]           # 2nd call records the graph
    prog = next(iter(staged.cached_functions()[0].graph._plan.values()))
    assert isinstance(prog.__dict__.get("_replay"), executor._ProgramGraph)
    for x, g in zip(xs, got):
        for a, b in zip(g, direct(x)):
            assert a.tobytes() == b.tobytes()
    held = staged(xs[0])                       # keep these outputs alive ...
    snapshot = [t.numpy().copy() for t in held]
    other = staged(xs[1])                      # ... so this call must not reuse them
    assert all(t.numpy().tobytes() == s.tobytes() for t, s in zip(held, snapshot))
    assert other[0].numpy().tobytes() == direct(xs[1])[0].tobytes()
    del held, other
    Ws[3].assign(sf.constant(np.eye(64, dtype=np.float32)))   # variables are read live
    after = [t.numpy() for t in staged(xs[2])]
    for a, b in zip(after, direct(xs[2])):
        assert a.tobytes() == b.tobytes()
