"""Ready-made plugin ops, registered through the reference's own plugin API.

The reference has no tanh, uniform draws, min/max, select or casts (SURVEY.md
§0 "Gaps"); the L2HMC sampler and the C2 microbenchmark need them.  They
are defined here exactly as a user would define them — ``OpDef`` +
``register_op`` (reference: stageflow/ops.py:45-59, :155-157) — with GPU
kernels, inference rules, gradient rules written in dispatched ops, and a
``lowering`` hint so the staged compiler fuses them into generated kernels.

``install()`` registers the set into the live runtime (idempotent; call it
after ``init_runtime``).
"""
from __future__ import annotations

from typing import List

from . import _fastpath, _native, dtypes
from .dtypes import DType
from .errors import KernelError
from .kernels import _bcast, launch_ew, ordinal_of
from .ops import DTYPE, FLOAT, SHAPE, OpDef, _schema, dispatch, get_runtime
from .tensor import Tensor, tensor_from_host


def _float_unary(name):
    def kernel(attrs, inputs, env):
        (x,) = inputs
        if not x.dtype.is_float:
            raise KernelError(f"{name} requires a float tensor, got {x.dtype.value}")
        return [launch_ew(name, x.dtype, x.dtype, (x,), env.device)]

    def infer(attrs, in_specs, env=None):
        dt, shape = in_specs[0]
        if not dt.is_float:
            raise KernelError(f"{name} requires a float tensor, got {dt.value}")
        return [(dt, shape)]

    _fastpath.mark_fast(kernel, _fastpath.K_EW1, _native.OP[name], _fastpath.F_FLOATS_ONLY)
    return kernel, infer


def _same_binary(name, out_bool=False):
    def kernel(attrs, inputs, env):
        a, b = inputs
        if a.dtype is not b.dtype:
            raise KernelError(f"{name}: mixed dtypes {a.dtype.value} and {b.dtype.value}")
        if a.dtype is DType.boolean:
            raise KernelError(f"{name} is not defined for boolean tensors")
        out_dt = DType.boolean if out_bool else a.dtype
        return [launch_ew(name, a.dtype, out_dt, (a, b), env.device)]

    def infer(attrs, in_specs, env=None):
        (da, sa), (db, sb) = in_specs
        if da is not db:
            raise KernelError(f"{name}: mixed dtypes {da.value} and {db.value}")
        if da is DType.boolean:
            raise KernelError(f"{name} is not defined for boolean tensors")
        return [(DType.boolean if out_bool else da, _bcast(sa, sb))]

    _fastpath.mark_fast(kernel, _fastpath.K_EW2, _native.OP[name],
                        _fastpath.F_OUT_BOOL if out_bool else 0)
    return kernel, infer


def _one(dt: DType) -> Tensor:
    return tensor_from_host([1.0], (), dt)


# -- gradient rules (dispatched ops only) ---------------------------------------


def _grad_tanh(ctx):
    from .ops import mul, sub

    y = ctx.output(0)
    return [mul(ctx.out_grad(), sub(_one(y.dtype), mul(y, y)))]


def _grad_sigmoid(ctx):
    from .ops import mul, sub

    y = ctx.output(0)
    return [mul(ctx.out_grad(), mul(y, sub(_one(y.dtype), y)))]


def _grad_square(ctx):
    from .ops import add, mul

    x = ctx.input(0)
    return [mul(ctx.out_grad(), add(x, x))]


def _grad_sqrt(ctx):
    from .ops import add, div

    y = ctx.output(0)
    return [div(ctx.out_grad(), add(y, y))]


def _grad_rsqrt(ctx):
    # d/dx x^-1/2 = -1/2 * y^3
    from .ops import mul

    y = ctx.output(0)
    half = tensor_from_host([-0.5], (), y.dtype)
    return [mul(ctx.out_grad(), mul(half, mul(y, mul(y, y))))]


def _mask(cond_op, x, y, dt):
    return dispatch("cast", [dispatch(cond_op, [x, y])[0]], {"dtype": dt})[0]


def _grad_minmax(is_max: bool):
    # max: a gets up where a >= b, b where a < b; min: a where b >= a, b where a > b
    def rule(ctx):
        from .gradients import _unbroadcast
        from .ops import mul

        up = ctx.out_grad()
        a, b = ctx.input(0), ctx.input(1)
        dt = ctx.in_spec(0)[0]
        if is_max:
            ma, mb = _mask("greater_equal", a, b, dt), _mask("less", a, b, dt)
        else:
            ma, mb = _mask("greater_equal", b, a, dt), _mask("greater", a, b, dt)
        return [_unbroadcast(mul(up, ma), ctx.in_spec(0)[1]),
                _unbroadcast(mul(up, mb), ctx.in_spec(1)[1])]

    return rule


def _grad_select(ctx):
    from .gradients import _unbroadcast, zeros_for

    up = ctx.out_grad()
    c = ctx.input(0)
    zero = zeros_for((up.dtype, ()))
    ga = dispatch("select", [c, up, zero])[0]
    gb = dispatch("select", [c, zero, up])[0]
    return [None, _unbroadcast(ga, ctx.in_spec(1)[1]), _unbroadcast(gb, ctx.in_spec(2)[1])]


# -- select / cast / random_uniform ---------------------------------------------------


def _select_kernel(attrs, inputs, env):
    c, a, b = inputs
    if c.dtype is not DType.boolean:
        raise KernelError("select: condition must be boolean")
    if a.dtype is not b.dtype:
        raise KernelError("select: branches must share a dtype")
    return [launch_ew("select", a.dtype, a.dtype, (c, a, b), env.device)]


def _select_infer(attrs, in_specs, env=None):
    (dc, sc), (da, sa), (db, sb) = in_specs
    if dc is not DType.boolean:
        raise KernelError("select: condition must be boolean")
    if da is not db:
        raise KernelError("select: branches must share a dtype")
    return [(da, _bcast(_bcast(sc, sa), sb))]


def _cast_kernel(attrs, inputs, env):
    (x,) = inputs
    dt: DType = attrs["dtype"]
    if x.dtype is dt:
        from .kernels import relabel

        return [relabel(x, env.device)]
    n = x.size
    buf = _native.cast(ordinal_of(env.device), x.dtype.tag, dt.tag, n, x._ptr() if n else 0,
                       n * dt.width)
    return [Tensor._adopt(dt, x.shape, env.device, buf)]


def _cast_infer(attrs, in_specs, env=None):
    return [(attrs["dtype"], in_specs[0][1])]


def _isfinite_kernel(attrs, inputs, env):
    (x,) = inputs
    return [launch_ew("isfinite", x.dtype, DType.boolean, (x,), env.device)]


def _isfinite_infer(attrs, in_specs, env=None):
    return [(DType.boolean, in_specs[0][1])]


def _random_uniform_infer(attrs, in_specs, env=None):
    dt = attrs["dtype"]
    if not dt.is_float:
        raise KernelError("random_uniform produces float tensors")
    return [(dt, tuple(attrs["shape"]))]


def _plugin_defs() -> List[OpDef]:
    from .kernels import _random_uniform_kernel

    defs = []
    for name, grad in (("tanh", _grad_tanh), ("sigmoid", _grad_sigmoid),
                       ("square", _grad_square), ("sqrt", _grad_sqrt),
                       ("rsqrt", _grad_rsqrt)):
        k, inf = _float_unary(name)
        defs.append(OpDef(name, 1, {}, 1, False, k, inf, grad, (), ("ew", name)))
    for name, grad in (("maximum", _grad_minmax(True)), ("minimum", _grad_minmax(False))):
        k, inf = _same_binary(name)
        defs.append(OpDef(name, 2, {}, 1, False, k, inf, grad, (), ("ew", name)))
    for name in ("less", "equal", "greater_equal"):
        k, inf = _same_binary(name, out_bool=True)
        defs.append(OpDef(name, 2, {}, 1, False, k, inf, None, (), ("ew", name)))
    defs.append(OpDef("select", 3, {}, 1, False, _select_kernel, _select_infer, _grad_select, (),
                      ("ew", "select")))
    defs.append(OpDef("cast", 1, _schema(dtype=DTYPE), 1, False, _cast_kernel, _cast_infer, None,
                      (), ("cast",)))
    defs.append(OpDef("is_finite", 1, {}, 1, False, _isfinite_kernel, _isfinite_infer, None, (),
                      ("ew", "isfinite")))
    defs.append(OpDef("random_uniform", 0, _schema(shape=SHAPE, dtype=DTYPE), 1, True,
                      _random_uniform_kernel, _random_uniform_infer, None, (), ("rng", 1)))
    return defs


def install() -> None:
    """Register every plugin op not yet known to the live runtime."""
    from .ops import register_op

    reg = get_runtime().registry
    for d in _plugin_defs():
        try:
            reg.get(d.name)
        except Exception:
            register_op(d)


# thin wrappers ------------------------------------------------------------------


def _w1(op):
    def fn(x):
        from .ops import _as_operand

        return dispatch(op, [_as_operand(x)])[0]

    fn.__name__ = op
    return _fastpath.wrap(op, 1, fn)


def _w2(op):
    def fn(a, b):
        from .ops import _as_operand

        a = _as_operand(a, like=b if isinstance(b, Tensor) else None)
        b = _as_operand(b, like=a)
        return dispatch(op, [a, b])[0]

    fn.__name__ = op
    return _fastpath.wrap(op, 2, fn)


tanh = _w1("tanh")
sigmoid = _w1("sigmoid")
square = _w1("square")
sqrt = _w1("sqrt")
rsqrt = _w1("rsqrt")
is_finite = _w1("is_finite")
maximum = _w2("maximum")
minimum = _w2("minimum")
less = _w2("less")
equal = _w2("equal")
greater_equal = _w2("greater_equal")


def select(cond, a, b) -> Tensor:
    from .ops import _as_operand

    a = _as_operand(a, like=b if isinstance(b, Tensor) else None)
    b = _as_operand(b, like=a)
    return dispatch("select", [cond, a, b])[0]


def cast(x, dtype: DType) -> Tensor:
    return dispatch("cast", [x], {"dtype": dtype})[0]


def random_uniform(shape, dtype: DType = dtypes.float32) -> Tensor:
    return dispatch("random_uniform", [], {"shape": tuple(shape), "dtype": dtype})[0]
