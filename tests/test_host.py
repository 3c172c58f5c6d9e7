"""CPU-only tests: the C-ABI library, and the host-side logic of the front
end (no kernel launches).  Mirrors the host-level cases of the reference's
tests (test_tensor.py, test_devices.py, test_staging.py trace keys,
test_graph.py builder/prune/serialization, test_tape.py lifecycle)."""
import ctypes
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native
from paper_1903_01855_b200.errors import (BroadcastIncompatible, ConsumedTape, CorruptGraph,
                                          FormatVersionMismatch, InactiveTape, LengthMismatch,
                                          MissingConcreteFunction, NarrowingOverflow,
                                          NonNestedEnd, SignatureMismatch, StagingError,
                                          UnencodableArgument, UnknownDevice)
from paper_1903_01855_b200.graph import GraphBuilder, prune
from paper_1903_01855_b200.serial import deserialize, serialize
from paper_1903_01855_b200.staging import infer_trace_key

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- the C-ABI
def _header_symbols():
    text = open(os.path.join(ROOT, "include", "sfb200.h")).read()
    return sorted(set(re.findall(r"\b(sf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in _header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_header_symbols()) <= set(_native.EXPORTED_SYMBOLS) | {"sf_elementwise"}


def test_library_loads_without_gpu_and_fails_loudly():
    lib = _native.load_library()
    assert lib.sf_version() >= 100
    if _native.device_count() == 0:
        n = ctypes.c_int(0)
        assert lib.sf_init(ctypes.byref(n)) == 6  # SF_ERR_NO_DEVICE
        with pytest.raises(sf.errors.DeviceUnavailable):
            sf.add(sf.constant(1.0), sf.constant(2.0))


def test_jit_compiles_generated_kernel_without_gpu():
    src = ('#include "sf_ops.cuh"\nextern "C" __global__ void k_test(float* p) '
           "{ p[threadIdx.x] = sf::softplus(p[threadIdx.x]); }")
    assert _native.jit_compile("k_test", src) != 0


def test_jit_disk_cache_across_processes(tmp_path):
    """The NVRTC cubin cache (sf_jit.cpp) persists across processes and
    ignores a corrupted entry."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1903_01855_b200 import _native\n"
            "src = '#include \"sf_ops.cuh\"\\nextern \"C\" __global__ void k_cache(float* p) "
            "{ p[threadIdx.x] = sf::exp_(p[threadIdx.x]); }'\n"
            "assert _native.jit_compile('k_cache', src) != 0\n") % ROOT
    env = dict(os.environ, SF_JIT_CACHE=str(tmp_path))
    subprocess.run([sys.executable, "-c", code], env=env, check=True)
    files = sorted(tmp_path.glob("*.cubin"))
    assert len(files) == 1 and files[0].stat().st_size > 100
    before = files[0].stat().st_mtime_ns
    subprocess.run([sys.executable, "-c", code], env=env, check=True)  # served from disk
    assert files[0].stat().st_mtime_ns == before
    files[0].write_bytes(b"garbage")                                   # corrupted: recompiled
    subprocess.run([sys.executable, "-c", code], env=env, check=True)
    assert files[0].stat().st_size > 100


# ---------------------------------------------------------------- tensors / dtypes
def test_tensor_from_host_checks():
    t = sf.tensor_from_host([2.0, -2.0], (2, 1), sf.float32)
    assert t.shape == (2, 1)
    np.testing.assert_array_equal(t.numpy(), [[2.0], [-2.0]])
    with pytest.raises(LengthMismatch):
        sf.tensor_from_host([1.0, 2.0, 3.0], (2,), sf.float32)
    with pytest.raises(NarrowingOverflow):
        sf.tensor_from_host([2 ** 31], (1,), sf.int32)
    with pytest.raises(NarrowingOverflow):
        sf.tensor_from_host([1.5], (1,), sf.int32)
    src = np.ones(3, dtype=np.float32)
    t = sf.tensor_from_host(src, (3,), sf.float32)
    src[0] = 9.0
    assert t.numpy()[0] == 1.0
    with pytest.raises(ValueError):
        sf.constant([1.0, 2.0]).raw()[0] = 5.0


@pytest.mark.parametrize("dtype", [sf.float32, sf.float64, sf.int32, sf.boolean])
def test_to_host_round_trip(dtype):
    data = {sf.boolean: [True, False, True, True], sf.int32: [1, -5, 7, 0]}.get(
        dtype, [1.25, -0.5, 3.0, 0.125])
    back, shape, dt = sf.to_host(sf.tensor_from_host(data, (2, 2), dtype))
    assert back == data and shape == (2, 2) and dt is dtype


def test_constant_default_dtypes():
    assert sf.constant(1.0).dtype is sf.float32
    assert sf.constant(1).dtype is sf.int32
    assert sf.constant(True).dtype is sf.boolean
    assert sf.constant(np.zeros(2)).dtype is sf.float64


@settings(max_examples=40, deadline=None)
@given(st.lists(st.sampled_from([1, 2, 3, 5]), max_size=3),
       st.lists(st.sampled_from([1, 2, 3, 5]), max_size=3))
def test_broadcast_commutative(a, b):
    a, b = tuple(a), tuple(b)
    try:
        left = sf.broadcast_shapes(a, b)
    except BroadcastIncompatible:
        with pytest.raises(BroadcastIncompatible):
            sf.broadcast_shapes(b, a)
        return
    assert left == sf.broadcast_shapes(b, a) == tuple(np.broadcast_shapes(a, b))


def test_broadcast_wildcards():
    assert sf.broadcast_shapes((None, 3), (4, 3)) == (4, 3)
    assert sf.broadcast_shapes((None, 3), (1, 3)) == (None, 3)


# ---------------------------------------------------------------- devices
def test_device_names():
    n = sf.DeviceName.parse("/job:training/task:2/device:GPU:0")
    assert (n.job, n.task, n.kind, n.index) == ("training", 2, "GPU", 0)
    assert sf.DeviceName.parse(n.render()) == n
    with pytest.raises(ValueError):
        sf.DeviceName.parse("cpu:0")
    assert [d.render() for d in sf.list_devices()][0] == "/job:local/task:0/device:GPU:0"
    with pytest.raises(UnknownDevice):
        with sf.device_scope("/job:local/task:0/device:GPU:77"):
            pass


# ---------------------------------------------------------------- trace keys / staging (no launches)
def test_trace_keys():
    assert infer_trace_key([sf.constant(1.0), True]) != infer_trace_key([sf.constant(1.0), False])
    assert infer_trace_key([sf.constant([1.0, 2.0])]) == infer_trace_key([sf.constant([9.0, -9.0])])
    with pytest.raises(UnencodableArgument):
        infer_trace_key([object()])
    v = sf.Variable([1.0, 2.0])
    enc = infer_trace_key([v]).encoding
    assert enc[0][0] == ("variable", "float32", (2,), id(v)) and enc[1] is None


def test_trace_without_folding_records_structure():
    pf = sf.stage(lambda a, b: sf.matmul(a, b))
    a = sf.constant(np.eye(2, dtype=np.float32))
    assert pf.cache_size == 0
    with pytest.raises(MissingConcreteFunction):
        pf.get_concrete(sf.TraceKey(("x",)))
    key = pf.trace_key_for(a, a)
    bound = pf._bind((a, a), {})
    pf._cache[key] = pf._trace_to_concrete(bound)
    graph = pf.get_concrete(key).graph
    assert [n.op for n in graph.nodes] == ["matmul"] and pf.trace_count == 1


def test_pinned_signature_checks():
    pf = sf.stage(lambda x: x, signature=[(sf.float32, (None, 5))])
    with pytest.raises(SignatureMismatch):
        pf.trace_key_for(sf.constant(np.ones((2, 4), dtype=np.float32)))
    with pytest.raises(SignatureMismatch):
        pf.trace_key_for(3.0)


def test_staging_errors_at_trace_time():
    pf = sf.stage(lambda x: "nope")
    with pytest.raises(StagingError):
        pf._trace_to_concrete(pf._bind((sf.constant(1.0),), {}))


# ---------------------------------------------------------------- graph IR
def _square(extra_dead=False):
    b = GraphBuilder()
    x = b.add_placeholder("x", sf.float32, (2,))
    (y,) = b.add_node("mul", [x, x], {}, None, [(sf.float32, (2,))])
    if extra_dead:
        b.add_node("exp", [x], {}, None, [(sf.float32, (2,))])
    return b.finalize("square", [y], ["y"])


def test_prune_and_idempotence():
    gf = _square(extra_dead=True)
    p = prune(gf)
    assert len(gf.nodes) - len(p.nodes) == 1 and "exp" not in p.op_counts()
    assert p.structurally_equal(prune(p))


def test_prune_keeps_stateful():
    b = GraphBuilder()
    x = b.add_placeholder("x", sf.float32, (2,))
    s = b.add_placeholder("state", sf.float32, (2,), is_variable_ref=True)
    (y,) = b.add_node("mul", [x, x], {}, None, [(sf.float32, (2,))])
    b.add_node("assign_variable", [s, y], {}, None, [])
    b.add_node("exp", [x], {}, None, [(sf.float32, (2,))])
    pr = prune(b.finalize("writer", [y], ["y"]))
    assert "assign_variable" in pr.op_counts() and "exp" not in pr.op_counts()


def test_corrupt_graph_rejected():
    from paper_1903_01855_b200.graph import GraphFunction, Node, Placeholder

    with pytest.raises(CorruptGraph):
        GraphFunction("bad", [Placeholder("x", sf.float32, ())],
                      [Node("neg", ((5, 0),), {}, None, ((sf.float32, ()),))], [("y", (1, 0))])


def test_serialization_round_trip_and_errors():
    gf = _square()
    blob = serialize(gf)
    assert blob[:4] == b"SGF1"
    assert gf.structurally_equal(deserialize(blob))
    bad = bytearray(blob)
    bad[4] = 99
    with pytest.raises(FormatVersionMismatch):
        deserialize(bytes(bad))
    with pytest.raises(CorruptGraph):
        deserialize(b"XXXX" + blob[4:])
    with pytest.raises(CorruptGraph):
        deserialize(blob[: len(blob) // 2])


def test_deserialize_plugin_ops_through_the_registry():
    """the reference's deserialize infers node specs from a
    global table and cannot load plugin ops (stageflow/serial.py:397); here
    inference goes through the live registry, so a registered plugin op
    round-trips."""
    from paper_1903_01855_b200 import plugins

    plugins.install()
    b = GraphBuilder()
    x = b.add_placeholder("x", sf.float32, (4,))
    (y,) = b.add_node("tanh", [x], {}, None, [(sf.float32, (4,))])
    (z,) = b.add_node("select", [b.add_node("greater", [y, x], {}, None,
                                            [(sf.boolean, (4,))])[0], y, x], {}, None,
                      [(sf.float32, (4,))])
    gf = b.finalize("plug", [z], ["z"])
    blob = serialize(gf)
    back = deserialize(blob)
    assert serialize(back) == blob and [n.op for n in back.nodes] == ["tanh", "greater", "select"]


# ---------------------------------------------------------------- tapes (lifecycle only)
def test_tape_lifecycle():
    t1, t2 = sf.Tape(), sf.Tape()
    t1.begin()
    t2.begin()
    with pytest.raises(NonNestedEnd):
        t1.end()
    t2.end()
    t1.end()
    t = sf.Tape()
    t.begin()
    t.end()
    with pytest.raises(InactiveTape):
        t.watch(sf.constant(1.0))


def test_sequence_iterator_and_trackable():
    it = sf.SequenceIterator("abcd")
    assert next(it) == "a" and next(it) == "b" and it.position == 2
    assert list(it) == ["c", "d"]

    class Box(sf.Trackable):
        pass

    b = Box()
    b.v = sf.Variable(1.0)
    b.blob = np.arange(3)
    b.other = "x"
    assert set(b.tracked_children()) == {"v", "blob"}
    del b.v
    assert set(b.tracked_children()) == {"blob"}
