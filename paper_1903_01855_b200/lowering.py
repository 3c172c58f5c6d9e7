"""Lowering of graph functions to native programs (the staged executor's compiler).

Replaces the reference's per-node interpreter (stageflow/executor.py:58-269).
A GraphFunction is compiled once per (device, concrete input signature):

1. *Flatten*: nodes become lowered ops over lowered values (``LV``).
   ``call_function`` callees are inlined; ``reshape``/``identity`` become
   aliases (no data movement); ``constant`` becomes a plan-owned buffer or,
   when it is one element or a splat, an immediate literal.
2. *Fuse*: maximal runs of elementwise/broadcast ops over one iteration
   shape become a single generated CUDA kernel (registers only, one load per
   external input element, one store per value needed outside the group),
   compiled for sm_100a by NVRTC against the same ``sf_ops.cuh`` the eager
   kernels use — hence bit-identical results.
3. *Segment*: ops the native executor cannot run (host callbacks, cond /
   while predicates, plugin ops without a lowering, host-RNG parity draws)
   split the program; everything between them is one native plan executed
   by a single ``sf_plan_run`` call (csrc/sf_plan.cpp), with temporaries
   allocated at their defining step and freed after their last use.
"""
from __future__ import annotations

import hashlib
import os
import re
import struct
from typing import Any, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native, dtypes
from .dtypes import DType
from .errors import KernelError, MissingFunction, StageflowError
from .tensor import Tensor

# ---------------------------------------------------------------------------
# lowered values and ops
# ---------------------------------------------------------------------------


class LV:
    """A lowered value.  kinds: input, var, const, op, alias."""

    __slots__ = ("id", "dtype", "shape", "kind", "index", "tensor", "base", "imm", "producer",
                 "vals")

    def __init__(self, id_, dtype: DType, shape, kind: str):
        self.id = id_
        self.dtype = dtype
        self.shape = tuple(shape)
        self.kind = kind
        self.index = -1       # input ordinal
        self.tensor = None    # const value
        self.base = None      # alias target
        self.imm = None       # scalar literal if the value is a known splat
        self.producer = None  # LOp
        # host values of an immutable captured tensor the program is
        # specialised on (row kernels read its elements as literals)
        self.vals = None

    @property
    def numel(self) -> int:
        return dtypes.element_count(self.shape)

    @property
    def nbytes(self) -> int:
        return self.numel * self.dtype.width

    def root(self) -> "LV":
        v = self
        while v.kind == "alias":
            v = v.base
        return v


class LOp:
    __slots__ = ("kind", "name", "ins", "outs", "attrs", "node_idx", "op_def")

    def __init__(self, kind, name, ins, outs, attrs=None, node_idx=-1, op_def=None):
        self.kind = kind      # ew | matmul | reduce | transpose | eye | rng | dropout |
        self.name = name      # var_read | var_assign | var_add | py
        self.ins = ins
        self.outs = outs
        self.attrs = attrs or {}
        self.node_idx = node_idx
        self.op_def = op_def


# elementwise ops the fuser understands: name -> (arity, result dtype rule)
_EW_BUILTIN = {
    "add": 2, "sub": 2, "mul": 2, "div": 2, "neg": 1, "exp": 1, "log": 1, "softplus": 1,
    "relu": 1, "step_positive": 1, "greater": 2,
}


class Lowerer:
    def __init__(self, device_ordinal: int, rng_mode: str):
        self.dev = device_ordinal
        self.rng_mode = rng_mode
        self.values: List[LV] = []
        self.ops: List[LOp] = []
        self.inputs: List[LV] = []
        # fold nodes computed only from specialised captures and constants at
        # compile time (Program sets it together with capture specialisation)
        self.fold_captures = False
        self.fold_max_numel = 1024

    def new(self, dtype, shape, kind) -> LV:
        v = LV(len(self.values), dtype, shape, kind)
        self.values.append(v)
        return v

    # -- graph flattening -------------------------------------------------------
    def lower_graph(self, gf, in_vals: Sequence[LV], libraries) -> List[LV]:
        from .ops import get_op_def

        libs = (gf.library,) + tuple(libraries)
        n_in = len(gf.inputs)
        env: Dict[Tuple[int, int], LV] = {}
        for i, v in enumerate(in_vals):
            env[(i, 0)] = v
        for j, node in enumerate(gf.nodes):
            ins = [env[r] for r in node.inputs]
            op_def = get_op_def(node.op)
            outs = self._fold(node, ins, op_def, gf.library) if self.fold_captures else None
            if outs is None:
                outs = self.lower_node(node, j, ins, libs, op_def)
            for k, o in enumerate(outs):
                env[(n_in + j, k)] = o
        return [env[ref] for _, ref in gf.outputs]

    @staticmethod
    def _value_of(lv: LV):
        """The immutable tensor behind a lowered value, if it has one (a
        specialised capture or a constant; reshaped views included)."""
        r = lv.root()
        t = r.tensor
        if t is None or r.kind not in ("const", "input"):
            return None
        if tuple(lv.shape) == tuple(t.shape):
            return t
        host = t._host.reshape(lv.shape) if t._host is not None else None
        return Tensor._adopt(t.dtype, tuple(lv.shape), t.device, t._buf, host)

    def _fold(self, node, ins, op_def, library):
        """Constant-fold a node computed only from specialised captures and
        constants, with the backend's own kernels (the reference's
        constant_fold does the same for graph constants,
        stageflow/graph.py:306-431; captured tensors are immutable, and a
        program is compiled per capture identity): the sampler's chain-
        independent values (weight transforms, time embeddings) become
        literals of the row kernel and the per-call uniform kernel goes
        away.  Returns the output values, or None when the node stays."""
        if (op_def.stateful or node.op in ("constant", "call_function", "cond", "while_loop",
                                           "host_call") or not ins
                or any(dtypes.element_count(shape) > self.fold_max_numel
                       for _, shape in node.out_specs if None not in tuple(shape))):
            return None
        vals = [self._value_of(x) for x in ins]
        if any(v is None for v in vals):
            return None
        from . import executor

        try:
            res = executor.run_node_for_folding(node, vals, library)
        except StageflowError:
            return None
        outs = []
        for t in res:
            v = self.new(t.dtype, t.shape, "const")
            v.tensor = t
            v.imm = _splat_value(t)
            if t.dtype.is_float and 0 < t.size <= self.fold_max_numel:
                v.vals = t.raw().reshape(-1)
            outs.append(v)
        return outs

    def _out(self, node, k=0) -> LV:
        dt, shape = node.out_specs[k]
        return self.new(dt, shape, "op")

    def emit(self, kind, name, ins, outs, node_idx, attrs=None, op_def=None) -> List[LV]:
        op = LOp(kind, name, ins, outs, attrs, node_idx, op_def)
        for o in outs:
            o.producer = op
        self.ops.append(op)
        return outs

    def lower_node(self, node, j, ins: List[LV], libs, op_def) -> List[LV]:
        op = node.op
        if op == "constant":
            t: Tensor = node.attrs["value"]
            v = self.new(t.dtype, t.shape, "const")
            v.tensor = t
            v.imm = _splat_value(t)
            return [v]
        if op in ("reshape", "identity"):
            dt, shape = node.out_specs[0]
            v = self.new(dt, _concrete(shape, ins[0].shape if op == "identity" else None), "alias")
            v.base = ins[0]
            v.imm = ins[0].imm if ins[0].kind in ("const", "alias") else None
            if v.imm is None and ins[0].root().kind == "const":
                v.imm = ins[0].root().imm
            return [v]
        if op in _EW_BUILTIN:
            return self.emit("ew", op, ins, [self._shaped_out(node, ins)], j)
        if op == "broadcast_to":
            return self.emit("ew", "identity", ins, [self._shaped_out(node, ins)], j)
        if op == "matmul":
            a, b = ins
            out = self.new(a.dtype, (a.shape[0], b.shape[1]), "op")
            return self.emit("matmul", op, ins, [out], j, {"ta": 0, "tb": 0})
        if op == "transpose":
            x = ins[0]
            out = self.new(x.dtype, tuple(reversed(x.shape)), "op")
            return self.emit("transpose", op, ins, [out], j)
        if op in ("reduce_sum", "reduce_mean"):
            from .kernels import normalize_axes, reduced_shape

            x = ins[0]
            if x.dtype is DType.boolean or (op == "reduce_mean" and x.dtype is DType.int32):
                return self._py(node, j, ins, op_def)
            axes = normalize_axes(op, len(x.shape), node.attrs.get("axes"))
            shape = reduced_shape(op, x.shape, node.attrs.get("axes"),
                                  node.attrs.get("keepdims", False))
            out = self.new(x.dtype, shape, "op")
            return self.emit("reduce", op, ins, [out], j, {"axes": axes})
        if op == "eye":
            dt = node.attrs["dtype"]
            n = node.attrs["size"]
            return self.emit("eye", op, [], [self.new(dt, (n, n), "op")], j)
        if op == "random_normal" and self.rng_mode == "device":
            dt = node.attrs["dtype"]
            return self.emit("rng", op, [], [self.new(dt, tuple(node.attrs["shape"]), "op")], j,
                             {"kind": 0})
        if op == "dropout" and self.rng_mode == "device":
            x = ins[0]
            outs = [self.new(x.dtype, x.shape, "op"), self.new(x.dtype, x.shape, "op")]
            return self.emit("dropout", op, ins, outs, j, {"rate": node.attrs["rate"]})
        if op == "read_variable":
            v = ins[0]
            return self.emit("var_read", op, ins, [self.new(v.dtype, v.shape, "op")], j)
        if op == "assign_variable":
            return self.emit("var_assign", op, ins, [], j)
        if op == "assign_add_variable":
            return self.emit("var_add", op, ins, [], j)
        if op == "call_function":
            callee = _resolve(node.attrs["function"], libs)
            outs = self.lower_graph(callee, ins, libs)
            return outs
        low = getattr(op_def, "lowering", None)
        if low is not None:
            kind = low[0]
            if kind == "ew":
                return self.emit("ew", low[1], ins, [self._shaped_out(node, ins)], j)
            if kind == "cast":
                return self.emit("ew", "cast_" + node.out_specs[0][0].value, ins,
                                 [self._shaped_out(node, ins)], j)
            if kind == "rng" and self.rng_mode == "device":
                dt = node.attrs["dtype"]
                return self.emit("rng", op, [], [self.new(dt, tuple(node.attrs["shape"]), "op")],
                                 j, {"kind": low[1]})
        return self._py(node, j, ins, op_def)

    def _shaped_out(self, node, ins) -> LV:
        dt, shape = node.out_specs[0]
        if None in tuple(shape):
            shape = ins[0].shape
            for x in ins[1:]:
                shape = dtypes.broadcast_shapes(shape, x.shape)
        return self.new(dt, shape, "op")

    def _py(self, node, j, ins, op_def) -> List[LV]:
        outs = [self.new(dt, shape, "op") for dt, shape in node.out_specs]
        return self.emit("py", node.op, ins, outs, j, dict(node.attrs), op_def)


def _concrete(shape, fallback):
    if None in tuple(shape):
        if fallback is None:
            raise KernelError("lowering needs concrete shapes")
        return fallback
    return shape


def _resolve(name_or_fn, libs):
    from .graph import GraphFunction

    if isinstance(name_or_fn, GraphFunction):
        return name_or_fn
    for lib in libs:
        f = lib.get(name_or_fn)
        if f is not None:
            return f
    raise MissingFunction(f"no graph function named {name_or_fn!r} in scope")


def _splat_value(t: Tensor):
    """The single value of a constant whose elements are all equal (or None)."""
    if t.size == 0:
        return None
    if t.size == 1:
        h = t._host if t._host is not None else t.raw()
        return h.reshape(-1)[0].item()
    if t.size > (1 << 22):
        return None
    h = t.raw().reshape(-1)
    first = h[0]
    if t.dtype.is_float:
        # bitwise comparison (distinguishes -0.0 and NaN payloads)
        view = h.view(np.uint32 if t.dtype is DType.float32 else np.uint64)
        if np.all(view == view[0]):
            return first.item()
        return None
    return first.item() if np.all(h == first) else None


# ---------------------------------------------------------------------------
# fusion of elementwise runs
# ---------------------------------------------------------------------------


class FusedGroup:
    __slots__ = ("ops", "shape", "outs_needed", "ext_inputs", "vec", "reduces", "inplace")

    def __init__(self, shape):
        self.ops: List[LOp] = []
        self.shape = shape
        self.outs_needed: List[LV] = []
        self.ext_inputs: List[LV] = []
        self.vec = 1  # elements per thread of the generated kernel
        self.reduces: List[LOp] = []  # column reductions folded in (fuse_reductions)
        self.inplace: Dict[int, LV] = {}  # id(out) -> variable it is stored into (var_add)


_PURE_KINDS = frozenset(("ew", "matmul", "reduce", "transpose", "eye"))


def _is_pos_zero(v: LV) -> bool:
    """v is a float constant (splat literal or specialised capture) whose
    every element is +0.0."""
    r = v.root()
    if not r.dtype.is_float:
        return False
    if r.kind == "const" and r.imm is not None:
        return float(r.imm) == 0.0 and not np.signbit(r.imm)
    if r.vals is not None:
        a = np.asarray(r.vals)
        return a.size > 0 and not a.any() and not np.signbit(a).any()
    return False


def elide_zero_adds(ops: List[LOp], keep) -> List[LOp]:
    """x + (+0) -> x where the sum only reaches relu through add/sub chains.

    x + (+0) equals x except that -0 becomes +0.  Two values that differ only
    in the sign of a zero still differ only that way after adding or
    subtracting any third value, and relu maps both zeros to +0 (NaNs pass
    unchanged), so every relu output is bit-identical with the add removed.
    A network layer with zero-initialised biases (the L2HMC nets) thereby
    drops one vector add per layer.  Values the program returns (keep) and
    any other consumer keep the add."""
    users: Dict[int, List[LOp]] = {}
    for op in ops:
        for x in op.ins:
            users.setdefault(id(x.root()), []).append(op)
    memo: Dict[int, bool] = {}

    def insensitive(v: LV, depth: int = 0) -> bool:
        r = v.root()
        if id(r) in memo:
            return memo[id(r)]
        ok = id(r) not in keep and depth < 16 and bool(users.get(id(r)))
        if ok:
            for u in users[id(r)]:
                if u.kind != "ew" or len(u.outs) != 1:
                    ok = False
                elif u.name == "relu":
                    continue
                elif u.name in ("add", "sub") and u.outs[0].shape == v.shape:
                    if not insensitive(u.outs[0], depth + 1):
                        ok = False
                else:
                    ok = False
                if not ok:
                    break
        memo[id(r)] = ok
        return ok

    out: List[LOp] = []
    for op in ops:
        if (op.kind == "ew" and op.name == "add" and len(op.ins) == 2 and len(op.outs) == 1
                and op.outs[0].dtype.is_float):
            o = op.outs[0]
            for a, b in ((op.ins[0], op.ins[1]), (op.ins[1], op.ins[0])):
                if (_is_pos_zero(b) and tuple(a.shape) == tuple(o.shape)
                        and a.dtype is o.dtype and insensitive(o)):
                    o.kind = "alias"
                    o.base = a
                    o.producer = None
                    break
            else:
                out.append(op)
            continue
        out.append(op)
    return out


def cse(ops: List[LOp]) -> List[LOp]:
    """Common-subexpression elimination over deterministic ops.

    A traced sampler recomputes the same chain-independent values (weight
    transposes, time encodings) once per unrolled step; each repeat becomes
    an alias of the first result, so it is computed, stored and staged once
    per call.  Results are unchanged bit for bit (same op, same operands)."""
    table: Dict[tuple, LV] = {}
    out: List[LOp] = []
    for op in ops:
        if op.kind in _PURE_KINDS and len(op.outs) == 1:
            ins = []
            for x in op.ins:
                r = x.root()
                if r.kind == "const" and r.imm is not None:
                    ins.append(("imm", repr(r.imm), r.dtype.value, tuple(x.shape)))
                else:
                    ins.append((id(r), tuple(x.shape)))
            o = op.outs[0]
            key = (op.kind, op.name, repr(sorted(op.attrs.items())), tuple(ins),
                   o.dtype.value, tuple(o.shape))
            prev = table.get(key)
            if prev is not None:
                o.kind = "alias"
                o.base = prev
                o.producer = None
                continue
            table[key] = o
        out.append(op)
    return out


def fuse(ops: List[LOp], fuse_enabled: bool) -> List[Any]:
    """Group elementwise ops sharing one output shape into fused kernels.

    An elementwise op joins the latest group of its shape when every operand
    is available where that group runs (produced before the group, or inside
    it); it is then computed at the group's position, which is safe because
    lowered values are immutable and its consumers all come later.  So the
    per-channel arithmetic of a normalisation layer, interleaved with the
    reductions that feed it, still becomes one launch per shape instead of
    one per op."""
    units: List[Any] = []
    produced_at: Dict[int, int] = {}
    latest: Dict[tuple, int] = {}  # shape -> index of the latest group of that shape
    var_touch: Dict[int, int] = {}  # id(variable) -> unit index of its last access
    barrier = -1                    # unit index of the last Python-executed op

    def record(unit_ops, u):
        for o_op in unit_ops:
            for o in getattr(o_op, "outs", ()):
                produced_at[id(o)] = u

    for op in ops:
        if isinstance(op, tuple):  # (RowProgram, planner) from rowfuse.plan_rows
            units.append(op)
            record(op[0].ops, len(units) - 1)
            continue
        if op.kind == "var_add" and fuse_enabled and FUSE_UPDATES:
            # v += x with x computed by an earlier group of v's shape: the
            # group stores v + x into v itself (one launch instead of two);
            # legal when nothing touched v since that group ran
            v, x = op.ins
            g = produced_at.get(id(x.root()), -1)
            grp = units[g] if g >= 0 else None
            if (isinstance(grp, FusedGroup) and x.root() is x and v.root() is v
                    and tuple(grp.shape) == tuple(v.shape) == tuple(x.shape)
                    and v.dtype is x.dtype and v.dtype in _VEC4
                    and var_touch.get(id(v), -1) < g and barrier < g):
                o = LV(-1, v.dtype, v.shape, "op")
                upd = LOp("ew", "add", [v, x], [o])
                o.producer = upd
                grp.ops.append(upd)
                grp.inplace[id(o)] = v
                var_touch[id(v)] = g
                continue
        if op.kind == "ew" and fuse_enabled:
            shape = tuple(op.outs[0].shape)
            g = latest.get(shape)
            if g is not None and all(produced_at.get(id(x.root()), -1) <= g for x in op.ins):
                units[g].ops.append(op)
                record([op], g)
                continue
            grp = FusedGroup(op.outs[0].shape)
            grp.ops.append(op)
            units.append(grp)
            latest[shape] = len(units) - 1
            record([op], len(units) - 1)
            continue
        units.append(op)
        record([op], len(units) - 1)
        if op.kind in ("var_read", "var_assign", "var_add") and op.ins:
            var_touch[id(op.ins[0].root())] = len(units) - 1
        elif op.kind == "py":
            barrier = len(units) - 1
    return units


FUSE_UPDATES = True  # var_add folded into the group computing its increment


# ---------------------------------------------------------------------------
# code generation
# ---------------------------------------------------------------------------

_CTYPE = {DType.float32: "float", DType.float64: "double", DType.int32: "int",
          DType.boolean: "bool"}

_UNARY_FN = {
    "neg": "sf::neg", "exp": "sf::exp_", "log": "sf::log_", "softplus": "sf::softplus",
    "relu": "sf::relu", "step_positive": "sf::step_pos", "tanh": "sf::tanh_",
    "sqrt": "sf::sqrt_", "rsqrt": "sf::rsqrt_", "sigmoid": "sf::sigmoid", "abs": "sf::abs_",
    "square": "sf::square", "reciprocal": "sf::recip", "cos": "sf::cos_", "sin": "sf::sin_",
}
_BINARY_FN = {"add": "sf::add", "sub": "sf::sub", "mul": "sf::mul", "div": "sf::div",
              "maximum": "sf::maximum", "minimum": "sf::minimum"}
_COMPARE = {"greater": ">", "less": "<", "equal": "==", "greater_equal": ">="}


def ew_expr(nm: str, args: List[str], ct: str) -> str:
    """C expression of one elementwise op (same functions as the eager kernels)."""
    if nm == "identity":
        return args[0]
    if nm in _UNARY_FN:
        return f"{_UNARY_FN[nm]}({args[0]})"
    if nm in _BINARY_FN:
        return f"{_BINARY_FN[nm]}({args[0]}, {args[1]})"
    if nm in _COMPARE:
        return f"({args[0]} {_COMPARE[nm]} {args[1]})"
    if nm == "isfinite":
        return f"sf::isfinite_({args[0]})"
    if nm == "logical_not":
        return f"(!{args[0]})"
    if nm == "select":
        return f"({args[0]} ? {args[1]} : {args[2]})"
    if nm.startswith("cast_"):
        return f"({ct})({args[0]})"
    raise KernelError(f"fusion: no code for elementwise op {nm!r}")


def alias_unwritten_reads(ops: List["LOp"], keep) -> List["LOp"]:
    """read_variable of a variable no op of the program writes returns the
    same value wherever it sits in the program's stateful chain: the read
    becomes an alias of the variable's buffer instead of a snapshot copy, so
    network weights stay uniform operands of the row programs (a trainable
    L2HMC's 2,560 weight reads otherwise cut its transition into ~1,000
    kernels).  A read whose value leaves the program (``keep``: outputs,
    e.g. values saved for the backward) keeps its snapshot: the caller may
    hold it across a later assignment) as a copy — an elementwise identity,
    which the row planner treats as one more uniform op (the value is the
    same at any point of the program)."""
    written = {id(op.ins[0].root()) for op in ops
               if op.kind in ("var_assign", "var_add") and op.ins}
    out = []
    for op in ops:
        if op.kind == "var_read" and op.ins and id(op.ins[0].root()) not in written:
            if id(op.outs[0]) in keep:
                op.kind, op.name = "ew", "identity"
            else:
                o = op.outs[0]
                o.kind = "alias"
                o.base = op.ins[0]
                o.producer = None
                continue
        out.append(op)
    return out


def c_literal(value, dtype: DType) -> str:
    if dtype is DType.float32:
        bits = struct.unpack("<I", struct.pack("<f", float(value)))[0]
        return f"__int_as_float(0x{bits:08x})"
    if dtype is DType.float64:
        bits = struct.unpack("<Q", struct.pack("<d", float(value)))[0]
        return f"__longlong_as_double(0x{bits:016x}ll)"
    if dtype is DType.int32:
        v = int(value)
        return f"(int){v}" if v != -(2 ** 31) else "(int)(-2147483647 - 1)"
    return "true" if value else "false"


def _strides_for(src_shape, out_shape):
    nd = len(out_shape)
    cs, acc = [], 1
    for d in reversed(src_shape):
        cs.append(acc)
        acc *= d
    cs = cs[::-1]
    pad = nd - len(src_shape)
    return [0] * pad + [0 if src_shape[i] == 1 else cs[i] for i in range(len(src_shape))]


def _index_expr(src_shape, out_shape, idx: str) -> str:
    """C expression for the flat offset of the broadcast source at flat index idx."""
    if tuple(src_shape) == tuple(out_shape):
        return idx
    if dtypes.element_count(src_shape) == 1:
        return "0"
    strides = _strides_for(src_shape, out_shape)
    terms = []
    inner = 1
    for d in range(len(out_shape) - 1, -1, -1):
        ext = out_shape[d]
        st = strides[d]
        if st and ext != 1:
            coord = f"({idx} / {inner})" if inner != 1 else idx
            if d != 0:
                coord = f"({coord} % {ext})"
            terms.append(f"{coord} * {st}" if st != 1 else coord)
        inner *= ext
    return " + ".join(terms) if terms else "0"


_VEC4 = {DType.float32: "float4", DType.int32: "int4"}


def _vector_width(group: FusedGroup, ext, outs) -> int:
    """4 when every thread can own 4 consecutive elements of one innermost
    row: 4-byte dtypes only, innermost extent % 4 == 0, and each external
    operand either full-shape, row-broadcast (innermost stride 1: one 16-byte
    load) or column-broadcast (innermost stride 0: one scalar load)."""
    shape = tuple(group.shape)
    if not shape or shape[-1] % 4 or dtypes.element_count(shape) < 1024:
        return 1
    for op in group.ops:
        if any(o.dtype not in _VEC4 for o in op.outs):
            return 1
    for x, r in ext:
        xs = tuple(x.shape)
        if r.dtype not in _VEC4:
            return 1
        if xs == shape or dtypes.element_count(xs) == 1:
            continue
        if len(xs) > len(shape) or any(a not in (1, b) for a, b in zip(xs[::-1], shape[::-1])):
            return 1  # not a plain broadcast (e.g. a reshaped view): scalar path
    return 4


def _x4_parts(group: FusedGroup, ext, names, outs, reds=()):
    """Pieces of a 4-elements-per-thread group body over flat index i (t = i/4):
    (operand loads, vector declarations, per-lane body, vector stores).  Each
    value in ``reds`` (in-group LVs) is also exposed as float4 red{k}_v."""
    shape = tuple(group.shape)
    lines = []
    for k, (x, r) in enumerate(ext):
        ct, vt = _CTYPE[r.dtype], _VEC4[r.dtype]
        xs = tuple(x.shape)
        if xs == shape:
            lines.append(f"    const {vt} in{k}_v = ((const {vt}*)a.p[{k}])[t];")
        elif dtypes.element_count(xs) == 1:
            lines.append(f"    const {ct} in{k}_s = ((const {ct}*)a.p[{k}])[0];")
            lines.append(f"    const {vt} in{k}_v = {{in{k}_s, in{k}_s, in{k}_s, in{k}_s}};")
        else:
            off = _index_expr(xs, shape, "i")
            inner_bcast = len(xs) == 0 or xs[-1] == 1
            if inner_bcast:
                lines.append(f"    const {ct} in{k}_s = ((const {ct}*)a.p[{k}])[{off}];")
                lines.append(f"    const {vt} in{k}_v = {{in{k}_s, in{k}_s, in{k}_s, in{k}_s}};")
            else:
                lines.append(f"    const {vt} in{k}_v = *(const {vt}*)((const {ct}*)a.p[{k}] + ({off}));")
    body = []
    for k, (x, r) in enumerate(ext):
        body.append(f"      const {_CTYPE[r.dtype]} in{k} = ((const {_CTYPE[r.dtype]}*)&in{k}_v)[e];")

    def ref(x: LV) -> str:
        r = x.root()
        nm = names.get((id(r), x.shape)) or names.get((id(r), r.shape))
        if nm is not None:
            return nm
        if r.kind == "const" and r.imm is not None:
            return c_literal(r.imm, r.dtype)
        raise KernelError("fusion: unresolved operand")

    for t, op in enumerate(group.ops):
        o = op.outs[0]
        ct = _CTYPE[o.dtype]
        body.append(f"      const {ct} v{t} = {ew_expr(op.name, [ref(x) for x in op.ins], ct)};")
        names[(id(o), o.shape)] = f"v{t}"
    for k, o in enumerate(outs):
        body.append(f"      ((({_CTYPE[o.dtype]}*)&out{k}_v))[e] = {names[(id(o), o.shape)]};")
    for k, x in enumerate(reds):
        body.append(f"      ((float*)&red{k}_v)[e] = {names[(id(x), x.shape)]};")
    decl = [f"    {_VEC4[o.dtype]} out{k}_v;" for k, o in enumerate(outs)]
    decl += [f"    float4 red{k}_v;" for k in range(len(reds))]
    stores = [f"    (({_VEC4[o.dtype]}*)a.p[{len(ext) + k}])[t] = out{k}_v;"
              for k, o in enumerate(outs)]
    return lines, decl, body, stores


def _generate_group_x4(group: FusedGroup, ext, names, outs, idx_t):
    """Fused elementwise kernel with 16-byte loads/stores (see _vector_width)."""
    lines, decl, body, stores = _x4_parts(group, ext, names, outs)
    n_ptr = len(ext) + len(outs)
    src_core = (f"struct Params {{ void* p[{max(1, n_ptr)}]; long long n; }};\n"
                f"extern \"C\" __global__ void __launch_bounds__(256) KNAME(const __grid_constant__ "
                f"Params a) {{\n"
                f"  const {idx_t} stride = ({idx_t})gridDim.x * blockDim.x;\n"
                f"  const {idx_t} n4 = ({idx_t})(a.n >> 2);\n"
                f"  for ({idx_t} t = ({idx_t})blockIdx.x * blockDim.x + threadIdx.x; t < n4;"
                f" t += stride) {{\n"
                f"    const {idx_t} i = t << 2;\n"
                + "\n".join(lines + decl) + "\n"
                f"#pragma unroll\n    for (int e = 0; e < 4; ++e) {{\n"
                + "\n".join(body) + "\n    }\n"
                + "\n".join(stores) + "\n  }\n}\n")
    digest = hashlib.sha1(src_core.encode()).hexdigest()[:16]
    name = f"sf_fused4_{digest}"
    source = '#include "sf_ops.cuh"\n' + src_core.replace("KNAME", name)
    return name, source, [r for _, r in ext], outs


def _group_ext(group: FusedGroup):
    """External inputs of a group: [(view as consumed, storage root)] and the
    name table; an alias (reshape) is loaded with its own shape over the
    root's buffer."""
    produced = {id(o) for op in group.ops for o in op.outs}
    ext: List[Tuple[LV, LV]] = []
    names: Dict[Tuple[int, tuple], str] = {}
    for op in group.ops:
        for x in op.ins:
            r = x.root()
            if id(r) in produced:
                continue
            if r.kind == "const" and r.imm is not None:
                continue
            key = (id(r), x.shape)
            if key not in names:
                names[key] = f"in{len(ext)}"
                ext.append((x, r))
    return ext, names


# ---------------------------------------------------------------------------
# reduction fusion: column reductions folded into their producing group
# ---------------------------------------------------------------------------

RED_FUSE = True          # fold column reductions into the group computing their input
_RED_MAX_PER_GROUP = 8


def _column_geometry(x: LV):
    """(R, C) when reducing x over all but its innermost axis is the float32
    16-byte column kernel's case (reduce_cols_f32x4 in sf_reduce.cu), else None."""
    shape = tuple(x.shape)
    if x.dtype is not DType.float32 or len(shape) < 2 or None in shape:
        return None
    c = shape[-1]
    r = dtypes.element_count(shape) // c if c else 0
    if c % 4 or c < 8 or r <= 32 or c // 4 > 65536 or (r + 1023) // 1024 >= 65536:
        return None
    return r, c


def fuse_reductions(units: List[Any]) -> List[Any]:
    """Attach each column reduction (reduce_sum/mean over all but the last
    axis) whose input is computed by an earlier fused group to that group:
    the group's kernel then folds the value in registers instead of writing it
    to HBM for a separate reduction launch.  The reduction moves to the
    group's position, which is safe because its only input is computed there
    and its consumers all come later.  The fold follows the eager kernel's
    canonical order exactly, so results are unchanged bit for bit."""
    if not RED_FUSE:
        return units
    out: List[Any] = []
    where: Dict[int, int] = {}
    for unit in units:
        if isinstance(unit, FusedGroup):
            for op in unit.ops:
                where[id(op.outs[0])] = len(out)
            out.append(unit)
            continue
        if (isinstance(unit, LOp) and unit.kind == "reduce"
                and unit.name in ("reduce_sum", "reduce_mean")):
            x = unit.ins[0]
            g = where.get(id(x))
            nd = len(x.shape)
            if (g is not None and _column_geometry(x) is not None
                    and tuple(sorted(unit.attrs.get("axes") or ())) == tuple(range(nd - 1))):
                grp = out[g]
                ext, _ = _group_ext(grp)
                outs_all = [op.outs[0] for op in grp.ops]
                if (tuple(grp.shape) == tuple(x.shape) and len(grp.reduces) < _RED_MAX_PER_GROUP
                        and _vector_width(grp, ext, outs_all) == 4):
                    grp.reduces.append(unit)
                    continue
        out.append(unit)
    return out


RED_UNROLL = int(os.environ.get("SF_RED_UNROLL", "4"))


def _unroll_rename(line: str, u: int) -> str:
    """An operand-load line of _x4_parts for unrolled row u (its index
    variables i/t and its in*_s / in*_v names suffixed with u)."""
    line = re.sub(r"\b(in\d+_[sv])\b", rf"\g<1>{u}", line)
    line = re.sub(r"\bi\b", f"i{u}", line)
    return re.sub(r"\bt\b", f"t{u}", line)


def generate_reduce_group(group: FusedGroup, needed_after: set, sm_count: int):
    """CUDA source of a fused group that also folds column reductions of its
    values (see fuse_reductions).  Thread (tx, l) of a block owns 4 adjacent
    columns and partial lane l of one 1024-row chunk — rows l, l+32, ... —
    computing the group's values there (storing the ones needed elsewhere) and
    folding each reduced value left to right; the 32 lane partials of a column
    are combined with the xor butterfly; with several chunks the last block of
    a column group folds the chunk partials (arrival counter) and applies the
    mean.  This is reduce_cols_f32x4 + reduce_partials' order exactly.

    Returns (name, source, ext roots, stored outs, reduce ops, grid, block,
    n_chunks, C)."""
    shape = tuple(group.shape)
    r_rows, c = _column_geometry(group.reduces[0].ins[0])
    ext, names = _group_ext(group)
    outs = [op.outs[0] for op in group.ops if id(op.outs[0]) in needed_after]
    reds = group.reduces
    k_red = len(reds)
    chunk = min(1024, r_rows)
    n_chunks = (r_rows + chunk - 1) // chunk
    target = 4 * sm_count
    xt = 32 if (c // 128) * n_chunks >= target else 16 if (c // 64) * n_chunks >= target else 8
    while xt > 8 and k_red * 32 * (xt * 4 + 1) * 4 > 40000:
        xt //= 2
    gx = (c // 4 + xt - 1) // xt
    lines, decl, body, stores = _x4_parts(group, ext, names, outs, [op.ins[0] for op in reds])
    base_red = len(ext) + len(outs)
    base_part = base_red + k_red
    n_ptr = base_part + (k_red if n_chunks > 1 else 0)
    fold = []
    for k in range(k_red):
        fold.append(f"      if (first) acc{k} = red{k}_v;\n      else {{ acc{k}.x += red{k}_v.x; "
                    f"acc{k}.y += red{k}_v.y; acc{k}.z += red{k}_v.z; acc{k}.w += red{k}_v.w; }}")
    countf = c_literal(float(r_rows), DType.float32)

    def final(k, val):
        o = f"((float*)a.p[{base_red + k}])[col]"
        mean = reds[k].name == "reduce_mean"
        return f"{o} = {val} / {countf};" if mean else f"{o} = {val};"

    src = [f"struct Params {{ void* p[{n_ptr}]; unsigned* counters; }};",
           f"extern \"C\" __global__ void __launch_bounds__({xt * 32}) KNAME("
           f"const __grid_constant__ Params a) {{",
           f"  __shared__ float acc_s[{k_red}][32][{xt * 4 + 1}];",
           f"  const int tx = threadIdx.x % {xt}, tl = threadIdx.x / {xt};",
           f"  const int bx = blockIdx.x % {gx};",
           f"  const long long j = blockIdx.x / {gx};",
           f"  const long long c0 = ((long long)bx * {xt} + tx) * 4;",
           f"  const long long g0 = j * {chunk};",
           f"  const long long len = {r_rows}LL - g0 < {chunk} ? {r_rows}LL - g0 : {chunk};"]
    src += [f"  float4 acc{k} = make_float4(0.f, 0.f, 0.f, 0.f);" for k in range(k_red)]
    # RED_UNROLL rows of a lane per iteration: all their operand loads are
    # issued first, then the rows are computed and folded in row order (the
    # CRO is unchanged; a 1024-row chunk is 32 dependent load rounds without
    # this, which left the late layers' reductions latency-bound)
    U = RED_UNROLL
    src += [f"  if (c0 < {c} && tl < len) {{",
            "    bool first = true;",
            f"    for (long long row = g0 + tl; row < g0 + len; row += {32 * U}) {{"]
    loaded = []
    for u in range(U):
        src += [f"    const long long row{u} = min(row + {32 * u}LL, g0 + len - 1);",
                f"    const long long i{u} = row{u} * {c} + c0;",
                f"    const long long t{u} = i{u} >> 2;"]
        for ln in lines:
            m = re.match(r"\s*const (\S+) (in\d+_[sv]) =", ln)
            if m and u == 0:
                loaded.append((m.group(1), m.group(2)))
            src.append(_unroll_rename(ln, u))
    for u in range(U):
        guard = "" if u == 0 else f"if (row + {32 * u} < g0 + len) "
        src += [f"    {guard}{{", f"    const long long i = i{u}, t = t{u};"]
        src += [f"    const {ty} {nm} = {nm}{u};" for ty, nm in loaded]
        src += decl
        src += ["#pragma unroll", "    for (int e = 0; e < 4; ++e) {"] + body + ["    }"]
        src += stores + fold + ["      first = false;", "    }"]
    src += ["    }", "  }"]
    for k in range(k_red):
        src += [f"  acc_s[{k}][tl][tx * 4 + 0] = acc{k}.x; acc_s[{k}][tl][tx * 4 + 1] = acc{k}.y;",
                f"  acc_s[{k}][tl][tx * 4 + 2] = acc{k}.z; acc_s[{k}][tl][tx * 4 + 3] = acc{k}.w;"]
    butterfly = ["#pragma unroll",
                 "      for (int off = 16; off >= 1; off >>= 1) {",
                 "        const float ov = __shfl_xor_sync(0xffffffffu, v, off);",
                 "        const bool op = __shfl_xor_sync(0xffffffffu, present, off);",
                 "        if (present && op) v = v + ov;",
                 "        else if (op) v = ov;",
                 "        present = present || op;",
                 "      }"]
    src += ["  __syncthreads();",
            "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;",
            f"  for (int k = 0; k < {k_red}; ++k) {{",
            "#pragma unroll",
            "    for (int q = 0; q < 4; ++q) {",
            "      const int cl = warp * 4 + q;",
            f"      const long long col = (long long)bx * {xt * 4} + cl;",
            "      float v = acc_s[k][lane][cl];",
            "      bool present = lane < len;"] + butterfly
    if n_chunks == 1:
        src += [f"      if (lane == 0 && col < {c}) {{",
                "        switch (k) {"]
        src += [f"          case {k}: {final(k, 'v')} break;" for k in range(k_red)]
        src += ["        }", "      }", "    }", "  }", "}"]
    else:
        src += [f"      if (lane == 0 && col < {c}) "
                f"((float*)a.p[{base_part} + k])[col * {n_chunks} + j] = v;",
                "    }", "  }",
                "  __shared__ bool last;",
                "  __threadfence();",
                "  __syncthreads();",
                "  if (threadIdx.x == 0) {",
                "    const unsigned prev = atomicAdd(&a.counters[bx], 1u);",
                f"    last = prev == {n_chunks - 1}u;",
                "    if (last) a.counters[bx] = 0;",
                "  }",
                "  __syncthreads();",
                "  if (!last) return;",
                "  __threadfence();",
                f"  for (int k = 0; k < {k_red}; ++k) {{",
                "    for (int q = 0; q < 4; ++q) {",
                f"      const long long col = (long long)bx * {xt * 4} + warp * 4 + q;",
                f"      if (col >= {c}) continue;",
                f"      const float* pc = (const float*)a.p[{base_part} + k] + col * {n_chunks};",
                "      float v = 0.f;",
                "      bool present = false;",
                f"      for (int qq = lane; qq < {n_chunks}; qq += 32) {{",
                "        const float w = __ldcg(pc + qq);",
                "        v = present ? v + w : w;",
                "        present = true;",
                "      }"] + butterfly
        src += ["      if (lane == 0) {", "        switch (k) {"]
        src += [f"          case {k}: {final(k, 'v')} break;" for k in range(k_red)]
        src += ["        }", "      }", "    }", "  }", "}"]
    src_core = "\n".join(src) + "\n"
    digest = hashlib.sha1(src_core.encode()).hexdigest()[:16]
    name = f"sf_fusedred_{digest}"
    source = '#include "sf_ops.cuh"\n' + src_core.replace("KNAME", name)
    return (name, source, [r for _, r in ext], outs, list(reds), gx * n_chunks, xt * 32,
            n_chunks, c)


def generate_group(group: FusedGroup, needed_after: set) -> Tuple[str, str, List[LV], List[LV]]:
    """CUDA source for a fused group. Returns (name, source, in_values, out_values)."""
    shape = group.shape
    n = dtypes.element_count(shape)
    ext, names = _group_ext(group)
    outs = [op.outs[0] for op in group.ops if id(op.outs[0]) in needed_after]
    idx_t = "long long" if n >= (1 << 31) else "int"
    vec = _vector_width(group, ext, outs)
    group.vec = vec
    if vec == 4:
        return _generate_group_x4(group, ext, names, outs, idx_t)
    lines = []
    for k, (x, r) in enumerate(ext):
        ct = _CTYPE[r.dtype]
        lines.append(f"    const {ct} in{k} = ((const {ct}*)a.p[{k}])"
                     f"[{_index_expr(x.shape, shape, 'i')}];")

    def ref(x: LV) -> str:
        r = x.root()
        nm = names.get((id(r), x.shape)) or names.get((id(r), r.shape))
        if nm is not None:
            return nm
        if r.kind == "const" and r.imm is not None:
            return c_literal(r.imm, r.dtype)
        raise KernelError("fusion: unresolved operand")

    for t, op in enumerate(group.ops):
        o = op.outs[0]
        ct = _CTYPE[o.dtype]
        # operands of a broadcasting op that have a different (smaller) shape
        # were loaded through broadcast indexing already (ext inputs), and
        # in-group values always have the group shape.
        expr = ew_expr(op.name, [ref(x) for x in op.ins], ct)
        lines.append(f"    const {ct} v{t} = {expr};")
        names[(id(o), o.shape)] = f"v{t}"
    for k, o in enumerate(outs):
        ct = _CTYPE[o.dtype]
        lines.append(f"    (({ct}*)a.p[{len(ext) + k}])[i] = {names[(id(o), o.shape)]};")
    body = "\n".join(lines)
    n_ptr = len(ext) + len(outs)
    src_core = (f"struct Params {{ void* p[{max(1, n_ptr)}]; long long n; }};\n"
                f"extern \"C\" __global__ void __launch_bounds__(256) KNAME(const __grid_constant__ "
                f"Params a) {{\n"
                f"  const {idx_t} stride = ({idx_t})gridDim.x * blockDim.x;\n"
                f"  for ({idx_t} i = ({idx_t})blockIdx.x * blockDim.x + threadIdx.x; i < ({idx_t})a.n;"
                f" i += stride) {{\n{body}\n  }}\n}}\n")
    digest = hashlib.sha1(src_core.encode()).hexdigest()[:16]
    name = f"sf_fused_{digest}"
    source = '#include "sf_ops.cuh"\n' + src_core.replace("KNAME", name)
    return name, source, [r for _, r in ext], outs


# ---------------------------------------------------------------------------
# plan serialisation (format documented in csrc/sf_plan.cpp)
# ---------------------------------------------------------------------------

SLOT_INPUT, SLOT_CONST, SLOT_TEMP, SLOT_OUTPUT = 0, 1, 2, 3


class PlanWriter:
    def __init__(self):
        self.slots: List[list] = []   # [kind, dtype_tag, index, nbytes, const_ptr, def, last]
        self.steps: List[Tuple[int, bytes]] = []
        self.n_inputs = 0
        self.n_outputs = 0

    def slot(self, kind, dtype: DType, nbytes: int, index=-1, const_ptr=0) -> int:
        self.slots.append([kind, dtype.tag, index, nbytes, const_ptr, -1, -1])
        return len(self.slots) - 1

    def step(self, kind: int, payload: bytes, defs=(), uses=()) -> int:
        s = len(self.steps)
        self.steps.append((kind, payload))
        for d in defs:
            if self.slots[d][5] < 0:
                self.slots[d][5] = s
        for u in list(uses) + list(defs):
            self.slots[u][6] = max(self.slots[u][6], s)
        return s

    def serialize(self) -> bytes:
        parts = [struct.pack("<IIiiii", 0x4C504653, 1, len(self.slots), self.n_inputs,
                             self.n_outputs, len(self.steps))]
        for kind, tag, index, nbytes, cptr, d, last in self.slots:
            parts.append(struct.pack("<BBHiQQii", kind, tag, 0, index, max(1, nbytes), cptr, d,
                                     last))
        for kind, payload in self.steps:
            parts.append(struct.pack("<II", kind, len(payload)))
            parts.append(payload)
        return b"".join(parts)


def pack_ew_step(op: int, dtype: DType, out_shape, in_slots, in_shapes, imms, out_slot) -> bytes:
    nd = len(out_shape)
    if nd > _native.MAX_DIMS:
        raise KernelError("rank exceeds backend limit")
    shp = list(out_shape) + [1] * (_native.MAX_DIMS - nd)
    slots = list(in_slots) + [-1] * (3 - len(in_slots))
    ims = list(imms) + [0.0] * (3 - len(imms))
    strides = []
    for j in range(3):
        if j < len(in_shapes) and in_shapes[j] is not None:
            st = in_shapes[j] if isinstance(in_shapes[j], list) else _strides_for(in_shapes[j],
                                                                                  out_shape)
        else:
            st = [0] * nd
        strides.extend(list(st) + [0] * (_native.MAX_DIMS - nd))
    return struct.pack("<iiii3ii3d8q24q", op, dtype.tag, nd, len(in_slots), *slots, out_slot, *ims,
                       *shp, *strides)
