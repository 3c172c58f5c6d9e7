"""GPU parity of the eager primitives and of eager vs staged execution.

Mirrors the reference's tests/test_ops.py (golden values :69-77, repeat
bit-identity :100-104, dropout mask :106-111, eager==staged :118-171) and
adds elementwise/reduction/matmul parity against NumPy (the reference's
arithmetic) with the tolerances of the north-star contract.
"""
import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import ops as sfops
from paper_1903_01855_b200.errors import ArityMismatch, AttrMismatch, KernelError, UnknownOp

from helpers import random_pure_function

pytestmark = pytest.mark.gpu

RTOL_F32 = 1e-6   # transcendental ulp differences (CUDA libm vs numpy SIMD)
RTOL_F64 = 1e-13


def _np(op, *xs):
    with np.errstate(all="ignore"):
        return {
            "add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide,
            "greater": np.greater, "neg": np.negative, "exp": np.exp, "log": np.log,
            "softplus": lambda x: np.logaddexp(0.0, x), "relu": lambda x: np.maximum(x, 0),
            "step_positive": lambda x: np.greater(x, 0).astype(x.dtype),
        }[op](*xs)


def test_listing_golden_values():
    a = sf.constant([[1.0, 0.0]])
    x = sf.constant([[2.0], [-2.0]])
    np.testing.assert_array_equal(sfops.dispatch("matmul", [a, x])[0].numpy(), [[2.0]])
    assert float(sf.add(sf.constant(1.0), sf.constant(2.0))) == 3.0


def test_dispatch_errors():
    with pytest.raises(ArityMismatch):
        sfops.dispatch("add", [sf.constant(1.0)])
    with pytest.raises(AttrMismatch):
        sfops.dispatch("reshape", [sf.constant(1.0)], {"bogus": 1})
    with pytest.raises(UnknownOp):
        sfops.dispatch("no_such_op", [])
    with pytest.raises(KernelError):
        sf.add(sf.constant(1.0), sf.tensor_from_host([2.0], (), sf.float64))
    t = sf.constant([True, False])
    with pytest.raises(KernelError):
        sf.add(t, t)


@pytest.mark.parametrize("dtype", [sf.float32, sf.float64])
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "greater"])
@pytest.mark.parametrize("shapes", [((3, 4), (3, 4)), ((3, 4), ()), ((5, 1, 4), (3, 1)),
                                    ((), (7,)), ((1000, 2), (1000, 2)), ((4097,), ())])
def test_binary_vs_numpy(op, dtype, shapes):
    rng = np.random.default_rng(1)
    a = rng.uniform(0.5, 2.0, size=shapes[0]).astype(dtype.np_dtype)
    b = rng.uniform(0.5, 2.0, size=shapes[1]).astype(dtype.np_dtype)
    got = sfops.dispatch(op, [sf.constant(a), sf.constant(b)])[0].numpy()
    want = _np(op, a, b)
    assert got.dtype == want.dtype and got.shape == want.shape
    # IEEE +,-,*,/ and comparisons are bit-exact with numpy
    assert got.tobytes() == np.asarray(want).tobytes()


@pytest.mark.parametrize("dtype", [sf.float32, sf.float64])
@pytest.mark.parametrize("op", ["neg", "exp", "log", "softplus", "relu", "step_positive"])
def test_unary_vs_numpy(op, dtype):
    rng = np.random.default_rng(2)
    x = rng.uniform(-3.0, 3.0, size=(33, 17)).astype(dtype.np_dtype)
    if op == "log":
        x = np.abs(x) + 0.1
    got = sf.dispatch(op, [sf.constant(x)])[0].numpy()
    want = _np(op, x)
    rtol = RTOL_F32 if dtype is sf.float32 else RTOL_F64
    np.testing.assert_allclose(got, want, rtol=rtol, atol=0)


def test_unary_edge_values():
    x = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -100.0, 100.0, 1e-45], dtype=np.float32)
    for op in ("relu", "softplus", "exp", "step_positive", "neg"):
        got = sf.dispatch(op, [sf.constant(x)])[0].numpy()
        want = _np(op, x)
        np.testing.assert_allclose(got, want, rtol=1e-6, equal_nan=True, err_msg=op)
        if op == "relu":
            assert not np.any(np.signbit(got[:2]))
    # softplus keeps denormals: softplus(-100) = 3.78e-44 in f32
    sp = sf.softplus(sf.constant(np.float32(-100.0))).numpy()
    assert 3.7e-44 < float(sp) < 3.9e-44


def test_int32_wraps():
    a = sf.tensor_from_host([2 ** 31 - 1], (1,), sf.int32)
    two = sf.tensor_from_host([2], (1,), sf.int32)
    assert sf.mul(a, two).numpy()[0] == -2
    assert sf.add(a, sf.tensor_from_host([1], (1,), sf.int32)).numpy()[0] == -(2 ** 31)
    arr = np.arange(-50, 2950, dtype=np.int32) * np.int32(1 << 20)
    big = sf.tensor_from_host(arr, arr.shape, sf.int32)
    # numpy accumulates in int64 and the reference's _wrap casts back (mod 2^32)
    assert sf.reduce_sum(big).item() == int(np.sum(arr).astype(np.int32))


@pytest.mark.parametrize("xs,ys", [((3136, 64), (64,)), ((3136, 64), (3136, 1)), ((50, 256), (1, 256)),
                                   ((7, 2048), (7, 2048)), ((12, 4, 8), (4, 1)), ((6, 12), (12,))])
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div"])
def test_row_column_broadcast_bitwise(xs, ys, op):
    """2-D broadcasts (the vectorised NHWC-vs-channel path and its fallbacks)
    are bit-exact with numpy's float32 arithmetic, in both operand orders."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal(xs).astype(np.float32)
    y = (rng.standard_normal(ys).astype(np.float32) + np.float32(3.0))
    f = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide}[op]
    got = sf.dispatch(op, [sf.constant(x), sf.constant(y)])[0].numpy()
    assert got.tobytes() == f(x, y).tobytes()
    got = sf.dispatch(op, [sf.constant(y), sf.constant(x + np.float32(4.0))])[0].numpy()
    assert got.tobytes() == f(y, x + np.float32(4.0)).tobytes()


@pytest.mark.parametrize("shape", [(100, 64), (20000, 3 * 64), (50000, 8), (33, 33), (1568, 2048),
                                   (3000, 256), (1025, 4), (40, 132), (301 * 1024 + 77, 64),
                                   (600 * 1024, 128)])
def test_column_reduction_matches_row_reduction_bitwise(shape):
    """The coalesced column kernels (scalar, and 16-byte at every block width)
    and the warp kernel implement one order (CRO)."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal(shape, dtype=np.float32)
    x[:, 1] = -0.0  # an all-(-0.0) column sums to -0.0 (folds start from the first element)
    cols = sf.reduce_sum(sf.constant(x), axes=(0,)).numpy()
    rows = sf.reduce_sum(sf.constant(np.ascontiguousarray(x.T)), axes=(1,)).numpy()
    assert cols.tobytes() == rows.tobytes()
    assert cols[1] == 0.0 and np.signbit(cols[1])


def test_int32_mean_truncates_eagerly():
    t = sf.tensor_from_host([7, 0, 0], (3,), sf.int32)
    assert sf.reduce_mean(t).item() == 2


@pytest.mark.parametrize("shape,axes,keepdims", [
    ((2, 3), None, False), ((2, 3), (1,), False), ((2, 3), (0,), True), ((4, 5, 6), (0, 2), False),
    ((100000, 2), None, False), ((3, 20000), (1,), True), ((64,), (-1,), False), ((), None, False),
    ((7, 1, 9), (1,), False), ((40, 3), (0,), False)])
@pytest.mark.parametrize("op", ["reduce_sum", "reduce_mean"])
def test_reductions_vs_numpy(op, shape, axes, keepdims):
    rng = np.random.default_rng(3)
    x = rng.standard_normal(shape).astype(np.float32)
    got = sf.dispatch(op, [sf.constant(x)], {"axes": axes, "keepdims": keepdims})[0].numpy()
    fn = np.sum if op == "reduce_sum" else np.mean
    want = fn(x.astype(np.float64), axis=axes, keepdims=keepdims)
    assert got.shape == np.shape(want)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5 * np.sqrt(max(1, x.size)))


@pytest.mark.parametrize("m,k,n", [(1, 16, 16), (4, 16, 32), (200, 2, 10), (256, 128, 256),
                                   (97, 33, 65), (3, 0, 4)])
@pytest.mark.parametrize("dtype", [sf.float32, sf.float64])
def test_matmul_vs_numpy(m, k, n, dtype):
    rng = np.random.default_rng(4)
    a = rng.standard_normal((m, k)).astype(dtype.np_dtype)
    b = rng.standard_normal((k, n)).astype(dtype.np_dtype)
    got = sf.matmul(sf.constant(a), sf.constant(b)).numpy()
    want = a.astype(np.float64) @ b.astype(np.float64)
    tol = 1e-5 if dtype is sf.float32 else 1e-12
    np.testing.assert_allclose(got, want, rtol=tol, atol=tol * max(1, k))


def test_transpose_reshape_broadcast():
    x = np.arange(12, dtype=np.float32).reshape(3, 4)
    t = sf.constant(x)
    np.testing.assert_array_equal(sf.dispatch("transpose", [t])[0].numpy(), x.T)
    np.testing.assert_array_equal(sf.reshape(t, (4, 3)).numpy(), x.reshape(4, 3))
    np.testing.assert_array_equal(sf.broadcast_to(sf.constant([[1.0, 2.0]]), (3, 2)).numpy(),
                                  np.broadcast_to(np.array([[1.0, 2.0]], np.float32), (3, 2)))
    with pytest.raises(KernelError):
        sf.broadcast_to(sf.constant([1.0, 2.0]), (3,))


def test_repeat_dispatch_bit_identical():
    a = sf.constant(np.linspace(-1, 1, 12).reshape(3, 4).astype(np.float32))
    assert sf.softplus(a).numpy().tobytes() == sf.softplus(a).numpy().tobytes()


def test_dropout_mask_semantics():
    x = sf.constant(np.ones((100,), dtype=np.float32))
    out, mask = sfops.dispatch("dropout", [x], {"rate": 0.5})
    m = mask.numpy()
    assert set(np.unique(m)).issubset({0.0, 2.0})
    np.testing.assert_array_equal(out.numpy(), m)


def test_operators_on_tensors():
    x = sf.constant([1.0, 2.0])
    np.testing.assert_allclose(((x + 1.0) * 2.0 - x / x).numpy(), [3.0, 5.0])


def test_single_op_eager_equals_staged():
    cases = [("add", 2, None), ("sub", 2, None), ("mul", 2, None), ("div", 2, None),
             ("neg", 1, None), ("exp", 1, None), ("softplus", 1, None), ("relu", 1, None),
             ("identity", 1, None), ("reduce_sum", 1, {"axes": None, "keepdims": False})]
    rng = np.random.default_rng(7)
    for op, arity, attrs in cases:
        args = [sf.constant(rng.uniform(0.5, 1.5, size=(2, 3)).astype(np.float32))
                for _ in range(arity)]
        eager = sfops.dispatch(op, args, attrs)[0].numpy()
        staged = sf.stage(lambda *xs: sfops.dispatch(op, list(xs), attrs)[0])(*args).numpy()
        assert eager.tobytes() == staged.tobytes(), op


@pytest.mark.parametrize("shape,bshape,cshape", [
    ((16, 8, 64), (64,), (16, 8, 1)), ((256, 12), (1, 12), (256, 1)), ((4, 6, 6, 32), (32,), ()),
    ((2, 512), (2, 512), (512,)), ((1023, 3), (3,), (1023, 1))])
def test_fused_broadcast_groups_eager_equals_staged(shape, bshape, cshape):
    """Fused elementwise groups (16-byte vector codegen when the innermost
    extent allows it, scalar otherwise) are bit-exact with eager dispatch,
    for row-, column- and scalar-broadcast operands and several outputs."""
    rng = np.random.default_rng(11)
    x = sf.constant(rng.standard_normal(shape).astype(np.float32))
    b = sf.constant(rng.standard_normal(bshape).astype(np.float32))
    c = sf.constant((rng.uniform(1.0, 2.0, cshape)).astype(np.float32))

    def f(x, b, c):
        y = sf.relu(x * b + c)
        z = sf.exp(y / c) - x
        return y, z * b

    eager = f(x, b, c)
    staged = sf.stage(f)(x, b, c)
    for e, s in zip(eager, staged):
        assert e.shape == s.shape and e.raw().tobytes() == s.raw().tobytes()


@pytest.mark.parametrize("shape", [(2, 7, 7, 64), (32, 14, 14, 16), (4, 28, 28, 128), (3, 11, 13, 8),
                                   (40, 1000)])
def test_reduction_fusion_eager_equals_staged(shape):
    """Normalisation-style graphs: column reductions folded into the group
    that computes their input (one or several chunks, sum and mean, several
    reductions per group, values also stored for later use) are bit-exact
    with eager dispatch, which materialises every value and reduces it."""
    from paper_1903_01855_b200 import lowering

    rng = np.random.default_rng(13)
    x = sf.constant(rng.standard_normal(shape).astype(np.float32))
    g = sf.constant(rng.uniform(0.5, 1.5, shape[-1:]).astype(np.float32))
    axes = tuple(range(len(shape) - 1))

    def f(x, g):
        mean = sf.reduce_mean(x, axes=axes)
        xc = sf.sub(x, mean)
        var = sf.reduce_mean(sf.mul(xc, xc), axes=axes)
        y = sf.mul(sf.mul(xc, g), var)
        s1 = sf.reduce_sum(sf.mul(y, x), axes=axes)
        s2 = sf.reduce_sum(sf.relu(y), axes=axes, keepdims=True)
        return y, var, s1, s2

    eager = f(x, g)
    assert lowering.RED_FUSE
    staged = sf.stage(f)(x, g)
    for e, s in zip(eager, staged):
        assert e.shape == s.shape and e.raw().tobytes() == s.raw().tobytes()


@pytest.mark.parametrize("seed", range(50))
def test_random_programs_eager_equals_staged(seed):
    fn, inputs = random_pure_function(seed)
    eager = fn(*inputs)
    staged = sf.stage(fn)(*inputs)
    assert eager.dtype is staged.dtype and eager.shape == staged.shape
    assert eager.raw().tobytes() == staged.raw().tobytes(), seed


def test_zero_bias_elision_is_bitwise_with_signed_zeros():
    """A staged relu(t + (x + 0-bias)) with +-0 / NaN / inf inputs: the add
    the staged compiler drops (lowering.elide_zero_adds) changes no bit of
    the relu output against the eager path, which performs it."""
    vals = np.array([0.0, -0.0, 1.0, -1.0, np.nan, np.inf, -np.inf, 1e-45, -1e-45, 3.0],
                    np.float32)
    x = np.stack([vals, vals[::-1], -vals, np.roll(vals, 3)]).astype(np.float32)
    t = np.stack([-vals, vals, np.roll(vals, 5), vals[::-1]]).astype(np.float32)
    bias = sf.constant(np.zeros(10, np.float32))

    def f(a, b):
        return sf.relu(sf.add(b, sf.add(a, bias)))

    tx, tt = sf.constant(x), sf.constant(t)
    eager = f(tx, tt).numpy()
    staged = sf.stage(f)(tx, tt).numpy()
    np.testing.assert_array_equal(eager.view(np.uint32), staged.view(np.uint32))
