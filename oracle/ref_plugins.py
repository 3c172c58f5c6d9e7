"""NumPy plugin ops for the REFERENCE runtime (oracle; test-only).

The builder-defined workloads (C2 tanh chain, L2HMC) need ops the
reference lacks.  To run those same user programs on the reference — the
oracle for them — this module registers numpy-kernel OpDefs into a live
reference runtime through its own ``register_op`` (stageflow/ops.py:155).
Names, attrs, inference and gradient rules match
paper_1903_01855_b200/plugins.py op for op, so traced graphs match too.
"""
from __future__ import annotations

import numpy as np


def register_all(ref, OpDef, register_op) -> None:
    K = ref.kernels
    from stageflow.errors import KernelError  # the reference's own taxonomy
    from stageflow.gradients import _unbroadcast, zeros_for
    from stageflow.ops import DTYPE, SHAPE, _schema, dispatch, mul, sub, add, div
    from stageflow.runtime import get_runtime
    from stageflow.tensor import tensor_from_host

    def one(dt):
        return tensor_from_host([1.0], (), dt)

    def f_unary(fn):
        def kernel(attrs, inputs, env):
            (x,) = inputs
            if not x.dtype.is_float:
                raise KernelError("requires a float tensor")
            with np.errstate(all="ignore"):
                return [K._wrap(fn(x.raw()), x.dtype, env)]

        def infer(attrs, in_specs, env=None):
            return [in_specs[0]]

        return kernel, infer

    def f_binary(fn, out_bool=False):
        def kernel(attrs, inputs, env):
            a, b = inputs
            if a.dtype is not b.dtype:
                raise KernelError("mixed dtypes")
            out = fn(a.raw(), b.raw())
            dt = ref.boolean if out_bool else a.dtype
            return [K._wrap(out, dt, env)]

        def infer(attrs, in_specs, env=None):
            (da, sa), (db, sb) = in_specs
            return [(ref.boolean if out_bool else da, K._broadcast("op", sa, sb))]

        return kernel, infer

    def g_tanh(ctx):
        y = ctx.output(0)
        return [mul(ctx.out_grad(), sub(one(y.dtype), mul(y, y)))]

    def g_sigmoid(ctx):
        y = ctx.output(0)
        return [mul(ctx.out_grad(), mul(y, sub(one(y.dtype), y)))]

    def g_square(ctx):
        x = ctx.input(0)
        return [mul(ctx.out_grad(), add(x, x))]

    def g_sqrt(ctx):
        y = ctx.output(0)
        return [div(ctx.out_grad(), add(y, y))]

    def g_rsqrt(ctx):
        y = ctx.output(0)
        half = tensor_from_host([-0.5], (), y.dtype)
        return [mul(ctx.out_grad(), mul(half, mul(y, mul(y, y))))]

    def mask(op, x, y, dt):
        return dispatch("cast", [dispatch(op, [x, y])[0]], {"dtype": dt})[0]

    def g_minmax(is_max):
        def rule(ctx):
            up = ctx.out_grad()
            a, b = ctx.input(0), ctx.input(1)
            dt = ctx.in_spec(0)[0]
            if is_max:
                ma, mb = mask("greater_equal", a, b, dt), mask("less", a, b, dt)
            else:
                ma, mb = mask("greater_equal", b, a, dt), mask("greater", a, b, dt)
            return [_unbroadcast(mul(up, ma), ctx.in_spec(0)[1]),
                    _unbroadcast(mul(up, mb), ctx.in_spec(1)[1])]

        return rule

    def g_select(ctx):
        up = ctx.out_grad()
        c = ctx.input(0)
        zero = zeros_for((up.dtype, ()))
        ga = dispatch("select", [c, up, zero])[0]
        gb = dispatch("select", [c, zero, up])[0]
        return [None, _unbroadcast(ga, ctx.in_spec(1)[1]), _unbroadcast(gb, ctx.in_spec(2)[1])]

    def sigmoid_np(x):
        one_ = x.dtype.type(1.0)
        return one_ / (one_ + np.exp(-x))

    unary = {"tanh": (np.tanh, g_tanh), "sigmoid": (sigmoid_np, g_sigmoid),
             "square": (lambda x: x * x, g_square), "sqrt": (np.sqrt, g_sqrt),
             "rsqrt": (lambda x: x.dtype.type(1.0) / np.sqrt(x), g_rsqrt)}
    for name, (fn, grad) in unary.items():
        k, inf = f_unary(fn)
        register_op(OpDef(name, 1, {}, 1, False, k, inf, grad, ()))
    for name, fn, grad in (("maximum", np.maximum, g_minmax(True)),
                           ("minimum", np.minimum, g_minmax(False))):
        k, inf = f_binary(fn)
        register_op(OpDef(name, 2, {}, 1, False, k, inf, grad, ()))
    for name, fn in (("less", np.less), ("equal", np.equal), ("greater_equal", np.greater_equal)):
        k, inf = f_binary(fn, out_bool=True)
        register_op(OpDef(name, 2, {}, 1, False, k, inf, None, ()))

    def select_kernel(attrs, inputs, env):
        c, a, b = inputs
        return [K._wrap(np.where(c.raw(), a.raw(), b.raw()), a.dtype, env)]

    def select_infer(attrs, in_specs, env=None):
        (_, sc), (da, sa), (_, sb) = in_specs
        return [(da, K._broadcast("select", K._broadcast("select", sc, sa), sb))]

    register_op(OpDef("select", 3, {}, 1, False, select_kernel, select_infer, g_select, ()))

    def cast_kernel(attrs, inputs, env):
        (x,) = inputs
        return [K._wrap(x.raw().astype(attrs["dtype"].np_dtype), attrs["dtype"], env)]

    register_op(OpDef("cast", 1, _schema(dtype=DTYPE), 1, False, cast_kernel,
                      lambda attrs, s, env=None: [(attrs["dtype"], s[0][1])], None, ()))

    def isfinite_kernel(attrs, inputs, env):
        return [K._wrap(np.isfinite(inputs[0].raw()), ref.boolean, env)]

    register_op(OpDef("is_finite", 1, {}, 1, False, isfinite_kernel,
                      lambda attrs, s, env=None: [(ref.boolean, s[0][1])], None, ()))

    def uniform_kernel(attrs, inputs, env):
        shape, dt = tuple(attrs["shape"]), attrs["dtype"]
        arr = get_runtime().draw(lambda rng: rng.random(shape))
        return [K._wrap(arr, dt, env)]

    register_op(OpDef("random_uniform", 0, _schema(shape=SHAPE, dtype=DTYPE), 1, True,
                      uniform_kernel,
                      lambda attrs, s, env=None: [(attrs["dtype"], tuple(attrs["shape"]))],
                      None, ()))
    register_nn(ref, OpDef, register_op)


def register_nn(ref, OpDef, register_op) -> None:
    """conv2d / max_pool / softmax_xent (and their gradient ops) as numpy
    plugins, same names/attrs/rules as paper_1903_01855_b200/nn.py."""
    from stageflow.ops import INT, SHAPE, _schema, dispatch

    from oracle import nn_np

    K = ref.kernels

    def wrap(arr, like, env):
        return K._wrap(np.ascontiguousarray(arr), like.dtype, env)

    def conv_k(attrs, ins, env):
        x, w = ins
        return [wrap(nn_np.conv2d(x.raw(), w.raw(), attrs["stride"], attrs["pad"]), x, env)]

    def conv_i(attrs, in_specs, env=None):
        (dx, (n, h, w, c)), (_, (kh, kw, ci, co)) = in_specs
        ho, wo = nn_np.out_hw(h, w, kh, attrs["stride"], attrs["pad"])
        return [(dx, (n, ho, wo, co))]

    def conv_g(ctx):
        x, w = ctx.input(0), ctx.input(1)
        up = ctx.out_grad()
        a = {"stride": ctx.attrs["stride"], "pad": ctx.attrs["pad"]}
        gx = dispatch("conv2d_grad_input", [up, w], dict(a, input_shape=tuple(ctx.in_spec(0)[1])))[0]
        gw = dispatch("conv2d_grad_filter", [x, up],
                      dict(a, filter_shape=tuple(ctx.in_spec(1)[1])))[0]
        return [gx, gw]

    def gi_k(attrs, ins, env):
        dy, w = ins
        return [wrap(nn_np.conv2d_grad_input(dy.raw(), w.raw(), attrs["stride"], attrs["pad"],
                                             tuple(attrs["input_shape"])), dy, env)]

    def gf_k(attrs, ins, env):
        x, dy = ins
        return [wrap(nn_np.conv2d_grad_filter(x.raw(), dy.raw(), attrs["stride"], attrs["pad"],
                                              tuple(attrs["filter_shape"])), x, env)]

    def pool_k(attrs, ins, env):
        (x,) = ins
        return [wrap(nn_np.max_pool(x.raw(), attrs["ksize"], attrs["stride"], attrs["pad"]), x, env)]

    def pool_i(attrs, in_specs, env=None):
        dt, (n, h, w, c) = in_specs[0]
        ho, wo = nn_np.out_hw(h, w, attrs["ksize"], attrs["stride"], attrs["pad"])
        return [(dt, (n, ho, wo, c))]

    def pool_g(ctx):
        a = {k: ctx.attrs[k] for k in ("ksize", "stride", "pad")}
        return [dispatch("max_pool_grad", [ctx.input(0), ctx.out_grad()], a)[0]]

    def pool_gk(attrs, ins, env):
        x, dy = ins
        return [wrap(nn_np.max_pool_grad(x.raw(), dy.raw(), attrs["ksize"], attrs["stride"],
                                         attrs["pad"]), x, env)]

    def xent_k(attrs, ins, env):
        lg, lab = ins
        return [wrap(nn_np.softmax_xent(lg.raw(), lab.raw()), lg, env)]

    def xent_g(ctx):
        return [dispatch("softmax_xent_grad", [ctx.input(0), ctx.input(1), ctx.out_grad()])[0],
                None]

    def xent_gk(attrs, ins, env):
        lg, lab, g = ins
        return [wrap(nn_np.softmax_xent_grad(lg.raw(), lab.raw(), g.raw()), lg, env)]

    same = lambda attrs, s, env=None: [s[0]]  # noqa: E731
    conv_attrs = _schema(stride=INT, pad=INT)
    pool_attrs = _schema(ksize=INT, stride=INT, pad=INT)
    register_op(OpDef("conv2d", 2, conv_attrs, 1, False, conv_k, conv_i, conv_g, ()))
    register_op(OpDef("conv2d_grad_input", 2, _schema(stride=INT, pad=INT, input_shape=SHAPE), 1,
                      False, gi_k, lambda attrs, s, env=None: [(s[0][0], tuple(attrs["input_shape"]))],
                      None, ()))
    register_op(OpDef("conv2d_grad_filter", 2, _schema(stride=INT, pad=INT, filter_shape=SHAPE),
                      1, False, gf_k,
                      lambda attrs, s, env=None: [(s[0][0], tuple(attrs["filter_shape"]))], None, ()))
    register_op(OpDef("max_pool", 1, pool_attrs, 1, False, pool_k, pool_i, pool_g, ()))
    register_op(OpDef("max_pool_grad", 2, pool_attrs, 1, False, pool_gk, same, None, ()))
    register_op(OpDef("softmax_xent", 2, {}, 1, False, xent_k,
                      lambda attrs, s, env=None: [(s[0][0], (s[0][1][0],))], xent_g, ()))
    register_op(OpDef("softmax_xent_grad", 3, {}, 1, False, xent_gk, same, None, ()))
