"""Host logic of the elementwise / reduction fusion passes
(paper_1903_01855_b200/lowering.py): group hoisting, vector-width selection,
reduction fusion, and the generated sources (compiled with NVRTC, which
needs no GPU).  Bit-exactness of the generated kernels is checked on the GPU
(tests/test_gpu_ops.py)."""
from paper_1903_01855_b200 import _native, lowering
from paper_1903_01855_b200.dtypes import DType
from paper_1903_01855_b200.lowering import FusedGroup, LOp, LV


class _Prog:
    def __init__(self):
        self.n = 0
        self.ops = []

    def lv(self, shape, kind="op", dtype=DType.float32):
        self.n += 1
        return LV(self.n, dtype, shape, kind)

    def op(self, kind, name, ins, shape, attrs=None, dtype=DType.float32):
        o = self.lv(shape, dtype=dtype)
        self.ops.append(LOp(kind, name, list(ins), [o], attrs or {}))
        o.producer = self.ops[-1]
        return o


S = (8, 14, 14, 64)


def _bn_like():
    """x - mean(x); var = mean(xc^2); y = xc * var (per-channel operands)."""
    P = _Prog()
    x = P.lv(S, "input")
    mean = P.op("reduce", "reduce_mean", [x], (64,), {"axes": (0, 1, 2)})
    xc = P.op("ew", "sub", [x, mean], S)
    sq = P.op("ew", "mul", [xc, xc], S)
    var = P.op("reduce", "reduce_mean", [sq], (64,), {"axes": (0, 1, 2)})
    y = P.op("ew", "mul", [xc, var], S)
    s = P.op("reduce", "reduce_sum", [y], (64,), {"axes": (0, 1, 2)})
    return P, (x, mean, xc, sq, var, y, s)


def test_hoisting_joins_latest_group_only_when_operands_exist():
    P, (x, mean, xc, sq, var, y, s) = _bn_like()
    units = lowering.fuse(P.ops, True)
    groups = [u for u in units if isinstance(u, FusedGroup)]
    # y needs var, produced after the (sub, mul) group: it starts a new group
    assert [[op.name for op in g.ops] for g in groups] == [["sub", "mul"], ["mul"]]
    # an op whose operands all exist earlier joins the earlier group
    P2 = _Prog()
    a = P2.lv(S, "input")
    b = P2.lv(S, "input")
    t1 = P2.op("ew", "add", [a, b], S)
    r = P2.op("reduce", "reduce_sum", [t1], (64,), {"axes": (0, 1, 2)})
    t2 = P2.op("ew", "mul", [a, a], S)  # independent of r: hoisted into t1's group
    units = lowering.fuse(P2.ops, True)
    assert len([u for u in units if isinstance(u, FusedGroup)]) == 1
    assert [op.name for op in units[0].ops] == ["add", "mul"]


def test_reduction_fusion_attaches_column_reductions():
    P, (x, mean, xc, sq, var, y, s) = _bn_like()
    units = lowering.fuse_reductions(lowering.fuse(P.ops, True))
    groups = [u for u in units if isinstance(u, FusedGroup)]
    # mean(x) reads an input: stays a reduction launch; var and s are folded
    assert [op.outs[0] for op in groups[0].reduces] == [var]
    assert [op.outs[0] for op in groups[1].reduces] == [s]
    assert sum(1 for u in units if isinstance(u, LOp) and u.kind == "reduce") == 1


def test_reduction_fusion_skips_non_column_and_small_cases():
    P = _Prog()
    x = P.lv((40, 6), "input")           # innermost 6: not a multiple of 4
    t = P.op("ew", "mul", [x, x], (40, 6))
    P.op("reduce", "reduce_sum", [t], (6,), {"axes": (0,)})
    y = P.lv((20, 64), "input")          # 20 rows: short reduction order
    u = P.op("ew", "mul", [y, y], (20, 64))
    P.op("reduce", "reduce_sum", [u], (64,), {"axes": (0,)})
    z = P.lv((64, 64), "input")          # reduce over the innermost axis
    v = P.op("ew", "mul", [z, z], (64, 64))
    P.op("reduce", "reduce_sum", [v], (64,), {"axes": (1,)})
    units = lowering.fuse_reductions(lowering.fuse(P.ops, True))
    assert all(not u.reduces for u in units if isinstance(u, FusedGroup))


def test_vector_width_rules():
    P = _Prog()
    x = P.lv(S, "input")
    ch = P.lv((64,), "input")
    col = P.lv((8, 14, 14, 1), "input")
    g = FusedGroup(S)
    g.ops.append(LOp("ew", "mul", [x, ch], [P.lv(S)]))
    g.ops.append(LOp("ew", "add", [g.ops[0].outs[0], col], [P.lv(S)]))
    ext, _ = lowering._group_ext(g)
    assert lowering._vector_width(g, ext, []) == 4
    g2 = FusedGroup((8, 14, 14, 6))
    x6 = P.lv((8, 14, 14, 6), "input")
    g2.ops.append(LOp("ew", "mul", [x6, x6], [P.lv((8, 14, 14, 6))]))
    ext2, _ = lowering._group_ext(g2)
    assert lowering._vector_width(g2, ext2, []) == 1
    g3 = FusedGroup(S)  # boolean output: scalar path
    g3.ops.append(LOp("ew", "greater", [x, ch], [P.lv(S, dtype=DType.boolean)]))
    ext3, _ = lowering._group_ext(g3)
    assert lowering._vector_width(g3, ext3, []) == 1


def test_fused_sources_compile():
    P, (x, mean, xc, sq, var, y, s) = _bn_like()
    units = lowering.fuse_reductions(lowering.fuse(P.ops, True))
    groups = [u for u in units if isinstance(u, FusedGroup)]
    # group 0: xc is needed later (by y), sq only by the folded reduction
    name, src, ext, outs, reds, grid, block, n_chunks, c = lowering.generate_reduce_group(
        groups[0], {id(xc)}, 148)
    assert outs == [xc] and [op.outs[0] for op in reds] == [var] and c == 64
    assert n_chunks == 2 and "atomicAdd(&a.counters" in src and "cp.async" not in src
    _native.jit_compile(name, src)
    name, src, *_ = lowering.generate_reduce_group(groups[1], set(), 148)
    _native.jit_compile(name, src)
    g = FusedGroup(S)
    g.ops.append(LOp("ew", "mul", [x, mean], [P.lv(S)]))
    name, src, ext, outs = lowering.generate_group(g, {id(g.ops[0].outs[0])})
    assert g.vec == 4 and "float4" in src
    _native.jit_compile(name, src)


def test_variable_update_folds_into_increment_group_unless_touched():
    P = _Prog()
    g = P.lv((32, 8), "input")
    v = P.lv((32, 8), "var")
    w = P.lv((32, 8), "var")
    inc = P.op("ew", "mul", [g, g], (32, 8))
    P.ops.append(LOp("var_add", "var_add", [v, inc], []))
    P.ops.append(LOp("var_read", "var_read", [w], [P.lv((32, 8))]))  # touches w only
    inc2 = P.op("ew", "mul", [g, inc], (32, 8))
    P.ops.append(LOp("var_add", "var_add", [w, inc2], []))  # w read after inc2's group: kept
    units = lowering.fuse(P.ops, True)
    groups = [u for u in units if isinstance(u, FusedGroup)]
    assert list(groups[0].inplace.values()) == [v]
    assert [op.name for op in groups[0].ops] == ["mul", "add", "mul"]
    # w's update: w was read after the group ran, so it stays a separate op
    assert any(isinstance(u, LOp) and u.kind == "var_add" for u in units)


def test_zero_bias_add_elided_only_before_relu():
    """x + (+0) is dropped when its value reaches only relu through add/sub
    (sign-of-zero differences vanish there); a -0 bias, a kept value, or a
    multiply on the way keeps the add."""
    import numpy as np

    def net(bias_vals, tail="relu", keep_sum=False):
        P = _Prog()
        x = P.lv((4, 10), "input")
        t = P.lv((4, 10), "input")
        b = P.lv((10,), "input")
        b.vals = np.asarray(bias_vals, np.float32)
        z = P.op("ew", "add", [x, b], (4, 10))
        s = P.op("ew", "add", [t, z], (4, 10))
        y = P.op("ew", tail, [s, s] if tail == "mul" else [s], (4, 10))
        keep = {id(y)} | ({id(s)} if keep_sum else set())
        return P, x, z, lowering.elide_zero_adds(P.ops, frozenset(keep))

    P, x, z, ops = net(np.zeros(10))
    assert [op.name for op in ops] == ["add", "relu"] and z.root() is x
    for kwargs in ({"bias_vals": -np.zeros(10)}, {"bias_vals": np.r_[np.zeros(9), 1.0]},
                   {"bias_vals": np.zeros(10), "tail": "mul"},
                   {"bias_vals": np.zeros(10), "keep_sum": True}):
        P, x, z, ops = net(**kwargs)
        assert len(ops) == 3 and z.root() is z, kwargs
