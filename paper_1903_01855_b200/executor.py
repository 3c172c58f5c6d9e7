"""Execution of graph functions (reference: stageflow/executor.py).

``execute_graph`` validates the bound inputs exactly like the reference
(:153-193), then runs the graph's *native program*: the lowered, fused form
built by lowering.py once per (device, input signature) and cached on
``gf._plan``.  A program is a sequence of segments — native plans (one
``sf_plan_run`` each) and the few nodes that must run through Python
(host callbacks, tensor-dependent control flow, plugin ops without a
lowering, host-RNG parity draws).

Graphs that pin nodes to other devices on a multi-GPU runtime run through
``_interpret`` instead: per-node launches with the reference's transparent
copy accounting (:231-261), so copy counters stay identical.
"""
from __future__ import annotations

import struct
import threading
import weakref
from contextlib import contextmanager
from typing import Dict, List, Optional, Sequence, Tuple

from . import _native, dtypes
from .dtypes import DType
from .errors import (CallbackError, DeadVariable, InputMismatch, KernelError, MissingFunction,
                     NotSerializable, SignatureViolation, StageflowError)
from .graph import GraphFunction, Node
from .kernels import KernelEnv, ordinal_of, relabel
from .lowering import (FusedGroup, LOp, Lowerer, LV, PlanWriter, SLOT_CONST, SLOT_INPUT,
                       alias_unwritten_reads, elide_zero_adds,
                       SLOT_OUTPUT, SLOT_TEMP, cse, fuse, fuse_reductions, generate_group,
                       generate_reduce_group, pack_ew_step)
from .runtime import current_context, get_runtime
from .tensor import Tensor

_PASSTHROUGH = (CallbackError, SignatureViolation, DeadVariable, MissingFunction, InputMismatch,
                NotSerializable)


def _known(shape) -> bool:
    return None not in tuple(shape)


def _bind_inputs(gf: GraphFunction, values: Sequence) -> None:
    """Check every value against its placeholder (reference: executor.py
    _bind_inputs).  Tensors are immutable and a Variable's dtype and shape
    never change, so an object that passed for a placeholder passes forever:
    the captured weights a staged sampler feeds every call are checked on the
    first call only (weak references: nothing is kept alive, and a dead
    variable is still reported)."""
    from .state import Variable

    if len(values) != len(gf.inputs):
        raise InputMismatch(f"{gf.name} takes {len(gf.inputs)} inputs (including captures), "
                            f"got {len(values)}")
    ok = gf.__dict__.setdefault("_bound_ok", [None] * len(gf.inputs))
    for i, (ph, v) in enumerate(zip(gf.inputs, values)):
        w = ok[i]
        if w is not None and w() is v:
            continue
        _bind_one(gf, ph, v, Variable)
        ok[i] = weakref.ref(v)


def _bind_one(gf, ph, v, Variable) -> None:
    if ph.is_variable_ref or isinstance(v, Variable):
        if not isinstance(v, Variable):
            raise InputMismatch(f"{gf.name}: input {ph.name!r} expects a variable")
        if v.dtype is not ph.dtype or (_known(ph.shape) and v.shape != ph.shape):
            raise InputMismatch(
                f"{gf.name}: variable bound to {ph.name!r} is {v.dtype.value}{list(v.shape)}, "
                f"expected {ph.dtype.value}{list(ph.shape)}")
        return
    if not isinstance(v, Tensor):
        raise InputMismatch(f"{gf.name}: input {ph.name!r} expects a tensor, got "
                            f"{type(v).__name__}")
    if v._symbolic is not None:
        raise InputMismatch(f"{gf.name}: symbolic tensor passed for {ph.name!r}")
    if v.dtype is not ph.dtype or len(v.shape) != len(ph.shape) or any(
            w is not None and h != w for h, w in zip(v.shape, ph.shape)):
        raise InputMismatch(
            f"{gf.name}: input {ph.name!r} is {v.dtype.value}{list(v.shape)}, expected "
            f"{ph.dtype.value}{list(ph.shape)}")


# ---------------------------------------------------------------------------
# native programs
# ---------------------------------------------------------------------------

_SM_COUNT: Dict[int, int] = {}


def _sm_count(dev: int) -> int:
    n = _SM_COUNT.get(dev)
    if n is None:
        import ctypes

        c = ctypes.c_int(0)
        L = _native.require_device()
        L.sf_device_info(dev, ctypes.byref(c), None, None, None)
        n = _SM_COUNT[dev] = max(1, c.value)
    return n


def _unit_ops(unit):
    if isinstance(unit, FusedGroup):
        return unit.ops + unit.reduces if unit.reduces else unit.ops
    if isinstance(unit, tuple):  # (RowProgram, planner)
        return unit[0].ops
    return [unit]


class _NativeSegment:
    __slots__ = ("plan", "in_roots", "out_roots", "n_launches")


class _PySegment:
    __slots__ = ("op",)


class Program:
    """A graph function lowered for one device and input signature."""

    def __init__(self, gf: GraphFunction, inputs: Sequence, device, libraries, rng_mode: str,
                 fuse_enabled: bool, collective=None):
        self.gf = gf
        # data-parallel gradient exchange (comm.py): (GradientCollective,
        # output indices to sum over ranks) or None; the indices not reduced
        # inside a plan are reduced after the run (post_reduce)
        self.collective = collective
        self.post_reduce: List[int] = []
        self.device = device
        self.dev = ordinal_of(device)
        self.keep: List = []  # constant tensors whose buffers plans point at
        lw = Lowerer(self.dev, rng_mode)
        lw.fold_captures = fuse_enabled and BAKE
        self.in_vals: List[LV] = []
        # inputs the program is specialised on (index -> weakref of the tensor)
        self.baked: Dict[int, "weakref.ref"] = {}
        for i, (ph, v) in enumerate(zip(gf.inputs, inputs)):
            lv = lw.new(v.dtype, v.shape, "var" if ph.is_variable_ref else "input")
            lv.index = i
            if fuse_enabled and bakeable(ph, v):
                lv.vals = v.raw().reshape(-1)
                lv.tensor = v  # (compile-time folding of nodes computed from it)
                self.baked[i] = weakref.ref(v)
            self.in_vals.append(lv)
        self.out_vals = lw.lower_graph(gf, self.in_vals, libraries)
        from . import rowfuse
        from .rowfuse import plan_rows

        rowfuse.SM_COUNT = _sm_count(self.dev)
        keep = frozenset(id(v.root()) for v in self.out_vals)
        ops = alias_unwritten_reads(lw.ops, keep) if fuse_enabled else lw.ops
        ops = cse(ops) if fuse_enabled else ops
        if fuse_enabled and ELIDE_ZERO_ADDS:
            ops = elide_zero_adds(ops, keep)
        self.has_rng = any(op.kind in ("rng", "dropout") for op in ops)
        keep = frozenset(id(v.root()) for v in self.out_vals)
        units = fuse(plan_rows(ops, keep) if fuse_enabled else ops, fuse_enabled)
        if fuse_enabled:
            units = fuse_reductions(units)
        self.segments = self._segment(units)
        self.n_launches = sum(s.n_launches for s in self.segments
                              if isinstance(s, _NativeSegment))
        if self.collective is not None:
            self.post_reduce = [i for i in self.collective[1]
                                if id(self.out_vals[i].root()) not in self._coll_done]

    # -- construction -------------------------------------------------------------
    def _segment(self, units) -> list:
        # last unit index at which each root is used (graph outputs count as "after all")
        last_use: Dict[int, int] = {}
        end = len(units)
        for u, unit in enumerate(units):
            for op in _unit_ops(unit):
                for x in op.ins:
                    last_use[id(x.root())] = max(last_use.get(id(x.root()), -1), u)
        self._read_by = dict(last_use)  # last unit reading each root (outputs aside)
        for v in self.out_vals:
            last_use[id(v.root())] = end
        # collective outputs: root id -> index into out_vals (first occurrence)
        self._coll_roots: Dict[int, int] = {}
        if self.collective is not None:
            for i in self.collective[1]:
                self._coll_roots.setdefault(id(self.out_vals[i].root()), i)
        self._coll_done: set = set()
        produced_in: Dict[int, int] = {}
        for u, unit in enumerate(units):
            for op in _unit_ops(unit):
                for o in op.outs:
                    produced_in[id(o)] = u
        self._precompile_rows(units, last_use)

        segs: list = []
        run: list = []
        run_start = 0

        def flush(upto: int):
            if run:
                segs.append(self._build_native(run, run_start, upto, last_use, produced_in))

        for u, unit in enumerate(units):
            if isinstance(unit, LOp) and unit.kind == "py":
                flush(u)
                run = []
                s = _PySegment()
                s.op = unit
                segs.append(s)
                run_start = u + 1
            else:
                if not run:
                    run_start = u
                run.append(unit)
        flush(len(units))
        return segs

    @staticmethod
    def _precompile_rows(units, last_use) -> None:
        """Generate every row-program chunk and compile them on parallel threads."""
        import os
        from concurrent.futures import ThreadPoolExecutor

        from .rowfuse import generate_rowprog

        jobs = []
        for u, unit in enumerate(units):
            if isinstance(unit, tuple):
                needed = {id(o) for op in unit[0].ops for o in op.outs
                          if last_use.get(id(o), -1) > u}
                name, src = generate_rowprog(unit[0], unit[1], needed)[:2]
                jobs.append((name, src))
        if len(jobs) > 1:
            with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as pool:
                list(pool.map(lambda j: _native.jit_compile(*j), jobs))

    def _build_native(self, units, start, stop, last_use, produced_in) -> _NativeSegment:
        pw = PlanWriter()
        slot_of: Dict[int, int] = {}
        in_roots: List[LV] = []
        out_roots: List[LV] = []
        seg_range = range(start, stop)

        def needed_outside(root: LV) -> bool:
            return last_use.get(id(root), -1) >= stop

        def slot_for_use(x: LV) -> int:
            r = x.root()
            s = slot_of.get(id(r))
            if s is not None:
                return s
            if r.kind == "const":
                t = r.tensor
                self.keep.append(t)
                s = pw.slot(SLOT_CONST, r.dtype, r.nbytes, const_ptr=t._ptr() if r.numel else 0)
            else:
                # defined outside this segment: an input of the plan
                s = pw.slot(SLOT_INPUT, r.dtype, r.nbytes, index=len(in_roots))
                in_roots.append(r)
            slot_of[id(r)] = s
            return s

        def slot_for_def(o: LV) -> int:
            s = slot_of.get(id(o))
            if s is None:
                if needed_outside(o):
                    s = pw.slot(SLOT_OUTPUT, o.dtype, o.nbytes, index=len(out_roots))
                    out_roots.append(o)
                else:
                    s = pw.slot(SLOT_TEMP, o.dtype, o.nbytes)
                slot_of[id(o)] = s
            return s

        n_launch = 0
        coll = self.collective
        pending: List[Tuple[int, int]] = []  # (slot, nbytes) awaiting their bucket
        pending_bytes = 0
        reduced_here: set = set()

        def flush_bucket():
            nonlocal pending, pending_bytes, n_launch
            if not pending:
                return
            spec = coll[0]
            slots = [sl for sl, _ in pending]
            dtype = pw.slots[slots[0]][1]
            payload = struct.pack("<Qiid", spec.comm.handle, dtype, len(slots), float(spec.scale))
            payload += struct.pack("<%di" % len(slots), *slots)
            pw.step(12, payload, uses=slots)
            n_launch += 1
            pending, pending_bytes = [], 0

        def collect(u: int):
            """Gradient outputs defined by now and read by nothing later join
            the current bucket (in the order the backward produced them)."""
            nonlocal pending_bytes
            for rid, i in self._coll_roots.items():
                if rid in reduced_here or rid in self._coll_done:
                    continue
                sl = slot_of.get(rid)
                if sl is None or pw.slots[sl][0] != SLOT_OUTPUT or pw.slots[sl][5] < 0:
                    continue
                if self._read_by.get(rid, -1) > u:
                    continue
                if pending and pw.slots[pending[0][0]][1] != pw.slots[sl][1]:
                    flush_bucket()  # one dtype per grouped call
                reduced_here.add(rid)
                nb = pw.slots[sl][3]
                pending.append((sl, nb))
                pending_bytes += nb
                if pending_bytes >= coll[0].bucket_bytes:
                    flush_bucket()

        for u_off, unit in enumerate(units):
            u = start + u_off
            if isinstance(unit, tuple):
                needed = {id(o) for op in unit[0].ops for o in op.outs
                          if last_use.get(id(o), -1) > u}
                n_launch += self._emit_rows(pw, unit, needed, slot_for_use, slot_for_def)
            elif isinstance(unit, FusedGroup):
                needed = set(unit.inplace)  # variable updates are always stored
                for op in unit.ops:
                    o = op.outs[0]
                    if last_use.get(id(o), -1) > u:
                        needed.add(id(o))
                inplace = unit.inplace

                def group_def(o, _inplace=inplace):
                    # an in-place variable update writes the variable's buffer
                    v = _inplace.get(id(o))
                    return slot_for_use(v) if v is not None else slot_for_def(o)

                n_launch += self._emit_group(pw, unit, needed, slot_for_use,
                                             group_def if inplace else slot_for_def)
            else:
                n_launch += self._emit_op(pw, unit, slot_for_use, slot_for_def)
            if coll is not None and self._coll_roots:
                collect(u)
        if coll is not None:
            flush_bucket()
            self._coll_done |= reduced_here
        pw.n_inputs = len(in_roots)
        pw.n_outputs = len(out_roots)
        seg = _NativeSegment()
        seg.plan = _native.NativePlan(self.dev, pw.serialize(), len(in_roots), len(out_roots))
        seg.in_roots = in_roots
        seg.out_roots = out_roots
        seg.n_launches = n_launch
        return seg

    def _emit_reduce_group(self, pw, group: FusedGroup, needed, use, define) -> int:
        name, src, ext, outs, reds, grid, block, n_chunks, c = generate_reduce_group(
            group, needed, _sm_count(self.dev))
        kernel = _native.jit_compile(name, src)
        in_slots = [use(r) for r in ext]
        out_slots = [define(o) for o in outs]
        red_slots = [define(op.outs[0]) for op in reds]
        # chunk partials: scratch that lives for this launch only
        part_slots = ([pw.slot(SLOT_TEMP, DType.float32, 4 * c * n_chunks) for _ in reds]
                      if n_chunks > 1 else [])
        ptrs = in_slots + out_slots + red_slots + part_slots
        payload = struct.pack("<QIIII", kernel, grid, block, 0, len(ptrs))
        payload += struct.pack("<%di" % len(ptrs), *ptrs)
        payload += struct.pack("<IQ", 8, _native.reduce_counters(self.dev))
        pw.step(1, payload, defs=out_slots + red_slots + part_slots, uses=in_slots)
        return 1

    def _emit_group(self, pw, group: FusedGroup, needed, use, define) -> int:
        if group.reduces:
            return self._emit_reduce_group(pw, group, needed, use, define)
        if len(group.ops) == 1 and (dtypes.element_count(group.shape) < SINGLE_OP_JIT_NUMEL
                                    or group.ops[0].name.startswith("cast_")):
            # small single ops: the precompiled eager kernel (no JIT);
            # large ones get a generated kernel with compile-time shapes and
            # 16-byte accesses (measured 2.5 -> 4+ TB/s on NHWC x channel)
            return self._emit_single_ew(pw, group.ops[0], use, define)
        name, src, ext, outs = generate_group(group, needed)
        if not outs:
            return 0
        kernel = _native.jit_compile(name, src)
        in_slots = [use(r) for r in ext]
        out_slots = [define(o) for o in outs]
        n = dtypes.element_count(group.shape)
        grid = max(1, min((n // group.vec + 255) // 256, _sm_count(self.dev) * 16))
        ptrs = in_slots + out_slots
        payload = struct.pack("<QIIII", kernel, grid, 256, 0, len(ptrs))
        payload += struct.pack("<%di" % len(ptrs), *ptrs)
        payload += struct.pack("<Iq", 8, n)
        pw.step(1, payload, defs=out_slots, uses=in_slots)
        return 1

    def _emit_rows(self, pw, unit, needed, use, define) -> int:
        from .rowfuse import generate_rowprog

        rp, planner = unit
        name, src, ext, outs, rng_counts, _n_ptr = generate_rowprog(rp, planner, needed)
        if not outs:
            return 0
        kernel = _native.jit_compile(name, src)
        in_slots = [use(r) for r in ext]
        out_slots = [define(o) for o in outs]
        rows = rp.batch
        per_cta = rp.rows_per_cta  # 128 x replicas, or 64 for a team-split kernel
        grid = 1 if rp.uniform_only else max(1, (rows + per_cta - 1) // per_cta)
        ptrs = in_slots + out_slots
        n_rng = max(1, len(rng_counts))
        scalars = struct.pack("<qQ", rows, 0) + b"\0" * (8 * n_rng)
        block = rp.block  # one chain per thread; uniform kernels: one warp per op of a level
        payload = struct.pack("<QIIII", kernel, grid, block, rp.dyn_smem, len(ptrs))
        payload += struct.pack("<%di" % len(ptrs), *ptrs)
        payload += struct.pack("<I", len(scalars)) + scalars
        patches = [(0, 8, 0)] + [(1, 16 + 8 * i, c) for i, c in enumerate(rng_counts)]
        payload += struct.pack("<I", len(patches))
        for kind, off, count in patches:
            payload += struct.pack("<IIQ", kind, off, count)
        if rp.cpool:
            # uniform operands gathered into the kernel's __constant__ pool
            pool_bytes, entries = rp.cpool
            payload += struct.pack("<II", pool_bytes, len(entries))
            for k, off, n, width, N, Np in entries:
                payload += struct.pack("<iIIIII", in_slots[k], off, n, width, N, Np)
        pw.step(1, payload, defs=out_slots, uses=in_slots)
        return 1 + (-(-len(rp.cpool[1]) // 960) if rp.cpool else 0)

    def _emit_single_ew(self, pw, op: LOp, use, define) -> int:
        o = op.outs[0]
        in_slots, in_shapes, imms = [], [], []
        for x in op.ins:
            r = x.root()
            if r.kind == "const" and r.imm is not None:
                in_slots.append(-1)
                imms.append(float(r.imm))
                in_shapes.append(None)
            else:
                in_slots.append(use(x))
                imms.append(0.0)
                in_shapes.append(x.shape)
        name = op.name
        if name.startswith("cast_"):
            # casts lower to the cast kernel
            src = op.ins[0]
            if in_slots[0] < 0:
                raise KernelError("cast of an immediate should have been folded")
            out = define(o)
            pw.step(11, struct.pack("<iiiiq", src.dtype.tag, o.dtype.tag, in_slots[0], out, o.numel),
                    defs=[out], uses=[in_slots[0]])
            return 1
        opcode = _native.OP[name]
        in_dtype = op.ins[0].dtype if name != "select" else op.ins[1].dtype
        out = define(o)
        pw.step(8, pack_ew_step(opcode, in_dtype, o.shape, in_slots, in_shapes, imms, out),
                defs=[out], uses=[s for s in in_slots if s >= 0])
        return 1

    def _emit_op(self, pw, op: LOp, use, define) -> int:
        k = op.kind
        if k == "matmul":
            a, b = op.ins
            o = op.outs[0]
            sa, sb = use(a), use(b)
            so = define(o)
            m, n = o.shape
            kk = a.shape[0] if op.attrs["ta"] else a.shape[1]
            pw.step(2, struct.pack("<iiiiiiqqq", o.dtype.tag, op.attrs["ta"], op.attrs["tb"], sa, sb,
                                   so, m, n, kk), defs=[so], uses=[sa, sb])
            return 1
        if k == "reduce":
            x = op.ins[0]
            o = op.outs[0]
            sx = use(x)
            so = define(o)
            mask = 0
            for ax in op.attrs["axes"]:
                mask |= 1 << ax
            shape = list(x.shape) + [1] * (8 - len(x.shape))
            pw.step(3, struct.pack("<iiiIii8q", 1 if op.name == "reduce_mean" else 0, x.dtype.tag,
                                   len(x.shape), mask, sx, so, *shape), defs=[so], uses=[sx])
            return 1
        if k == "transpose":
            x = op.ins[0]
            o = op.outs[0]
            sx = use(x)
            so = define(o)
            if len(x.shape) == 2:
                pw.step(4, struct.pack("<iiiiqq", x.dtype.tag, sx, so, 0, x.shape[0], x.shape[1]),
                        defs=[so], uses=[sx])
            else:
                from .kernels import _contiguous_strides

                strides = list(reversed(_contiguous_strides(x.shape)))
                pw.step(8, pack_ew_step(_native.OP["identity"], x.dtype, o.shape, [sx], [strides],
                                        [0.0], so), defs=[so], uses=[sx])
            return 1
        if k == "eye":
            o = op.outs[0]
            so = define(o)
            pw.step(6, struct.pack("<iiq", o.dtype.tag, so, o.shape[0]), defs=[so])
            return 1
        if k == "rng":
            o = op.outs[0]
            so = define(o)
            pw.step(9, struct.pack("<iiiiq", op.attrs["kind"], o.dtype.tag, so, 0, o.numel),
                    defs=[so])
            return 1
        if k == "dropout":
            x = op.ins[0]
            sx = use(x)
            so, sm = define(op.outs[0]), define(op.outs[1])
            pw.step(10, struct.pack("<iiiiqd", x.dtype.tag, sx, so, sm, x.numel, op.attrs["rate"]),
                    defs=[so, sm], uses=[sx])
            return 1
        if k == "var_read":
            v = op.ins[0]
            sv = use(v)
            so = define(op.outs[0])
            pw.step(7, struct.pack("<iiq", sv, so, v.nbytes), defs=[so], uses=[sv])
            return 0
        if k == "var_assign":
            v, x = op.ins
            sv = use(v)
            if x.root().kind == "const" and x.root().imm is not None and v.numel > 0:
                pw.step(5, struct.pack("<iiqd", v.dtype.tag, sv, v.numel, float(x.root().imm)),
                        uses=[sv])
                return 1
            sx = use(x)
            pw.step(7, struct.pack("<iiq", sx, sv, v.nbytes), uses=[sx, sv])
            return 0
        if k == "var_add":
            v, x = op.ins
            sv = use(v)
            r = x.root()
            if r.kind == "const" and r.imm is not None:
                slots, shapes, imms = [sv, -1], [v.shape, None], [0.0, float(r.imm)]
            else:
                slots, shapes, imms = [sv, use(x)], [v.shape, x.shape], [0.0, 0.0]
            pw.step(8, pack_ew_step(_native.OP["add"], v.dtype, v.shape, slots, shapes, imms, sv),
                    uses=[s for s in slots if s >= 0])
            return 1
        raise KernelError(f"lowering: unsupported op kind {k}")

    # -- execution -----------------------------------------------------------------
    def run(self, inputs: Sequence, libraries) -> List[Tensor]:
        outs = self._run(inputs, libraries)
        if self.post_reduce:
            # gradients no plan reduced (computed by Python segments, or
            # aliases of inputs/constants): reduce copies after the run
            spec = self.collective[0]
            red = spec.comm.allreduce([outs[i] for i in self.post_reduce], spec.scale)
            outs = list(outs)
            for i, t in zip(self.post_reduce, red):
                outs[i] = t
        return outs

    def _run(self, inputs: Sequence, libraries) -> List[Tensor]:
        g = self.__dict__.get("_replay")
        if g is not None and g is not False:
            outs = g.try_run(inputs)
            if outs is not None:
                return outs
        elif g is None and GRAPH_REPLAY and self._replayable():
            calls = self.__dict__["_calls"] = self.__dict__.get("_calls", 0) + 1
            if calls >= 2:  # first call compiled and loaded every kernel
                try:
                    self._replay = _ProgramGraph(self, inputs, libraries)
                except _NotCapturable:
                    self._replay = False
                else:
                    # hand the first replay's outputs over without keeping a
                    # reference (a kept output would mark the graph busy forever)
                    outs, self._replay.first_outputs = self._replay.first_outputs, None
                    return outs
        return self._run_direct(inputs, libraries)

    def _replayable(self) -> bool:
        r = self.__dict__.get("_replayable_flag")
        if r is None:
            r = (not self.has_rng and self.collective is None
                 and self.n_launches >= GRAPH_MIN_LAUNCHES
                 and all(s.op.name in GRAPH_SAFE_OPS for s in self.segments
                         if isinstance(s, _PySegment)))
            self._replayable_flag = r
        return r

    def _single_plan(self):
        """(plan, input positions, output specs) when the whole program is one
        native plan whose outputs are all plan outputs; False otherwise."""
        segs = self.segments
        if len(segs) != 1 or not isinstance(segs[0], _NativeSegment):
            return False
        seg = segs[0]
        pos = {id(lv.root()): i for i, lv in enumerate(self.in_vals)}
        if any(id(r) not in pos for r in seg.in_roots):
            return False
        slot = {id(r): (j, r.nbytes) for j, r in enumerate(seg.out_roots)}
        outs = []
        for lv in self.out_vals:
            s = slot.get(id(lv.root()))
            if s is None:
                return False
            outs.append((s[0], s[1], lv.dtype, lv.shape))
        if len({j for j, _, _, _ in outs}) != len(outs) or len(outs) != len(seg.out_roots):
            return False  # an output returned twice (or unused) shares one buffer
        return seg.plan, [pos[id(r)] for r in seg.in_roots], outs

    def _run_direct(self, inputs: Sequence, libraries) -> List[Tensor]:
        fast = self.__dict__.get("_fast")
        if fast is None:
            fast = self._fast = self._single_plan()
        if fast:
            plan, pos, specs = fast
            ptrs = []
            for i in pos:
                h = inputs[i]
                if type(h) is Tensor:
                    b = h._buf
                    ptrs.append(b.ptr if b is not None else h._ptr())
                elif isinstance(h, Tensor):
                    ptrs.append(h._ptr())
                else:
                    ptrs.append(h._storage_ptr())  # Variable
            raw = plan.run(ptrs)
            dev, device, DB, adopt = self.dev, self.device, _native.DeviceBuffer, Tensor._adopt
            outs = [adopt(dt, shape, device, DB(dev, raw[j], nb)) for j, nb, dt, shape in specs]
            if len(outs) > 1:
                sib = [weakref.ref(t) for t in outs]
                for t in outs:
                    t._sib = sib
            return outs
        env: Dict[int, object] = {}
        for lv, v in zip(self.in_vals, inputs):
            env[id(lv)] = v
        device = self.device
        for seg in self.segments:
            if isinstance(seg, _NativeSegment):
                ptrs = [self._ptr_of(env, r) for r in seg.in_roots]
                outs = seg.plan.run(ptrs)
                dev = self.dev
                for r, p in zip(seg.out_roots, outs):
                    env[id(r)] = _native.DeviceBuffer(dev, p, r.nbytes)
            else:
                self._run_py(seg.op, env, libraries)
        return [self._tensor_of(env, lv) for lv in self.out_vals]

    @staticmethod
    def _ptr_of(env, root: LV) -> int:
        h = env[id(root)]
        t = type(h)
        if t is Tensor:
            b = h._buf
            return b.ptr if b is not None else h._ptr()
        if t is _native.DeviceBuffer:
            return h.ptr
        if isinstance(h, Tensor):
            return h._ptr()
        return h._storage_ptr()  # Variable

    def _tensor_of(self, env, lv: LV) -> Tensor:
        r = lv.root()
        if r.kind == "const":
            t = r.tensor
            host = t._host.reshape(lv.shape) if t._host is not None else None
            if t._buf is None and host is None:
                t._device_buffer()
            return Tensor._adopt(lv.dtype, lv.shape, self.device, t._buf, host)
        h = env[id(r)]
        if isinstance(h, _native.DeviceBuffer):
            return Tensor._adopt(lv.dtype, lv.shape, self.device, h)
        if isinstance(h, Tensor):
            host = h._host.reshape(lv.shape) if h._host is not None else None
            return Tensor._adopt(lv.dtype, lv.shape, self.device, h._buf, host)
        return h  # Variable (only as an input of a py op)

    def _run_py(self, op: LOp, env, libraries) -> None:
        ins = [self._tensor_of(env, x) for x in op.ins]
        kenv = KernelEnv(device=self.device, libraries=tuple(libraries), nested=True)
        try:
            outs = op.op_def.kernel(op.attrs, ins, kenv)
        except _PASSTHROUGH:
            raise
        except StageflowError as e:
            raise KernelError(f"node {op.node_idx} ({op.name}): {e}") from e
        except Exception as e:
            raise KernelError(f"node {op.node_idx} ({op.name}): {e}") from e
        for lv, t in zip(op.outs, outs):
            env[id(lv)] = t


# Small immutable tensors a staged function captured (network weights, masks)
# are specialised into the generated row kernels as literal operands: an
# FFMA with an immediate weight instead of a shared-memory load per use
# (the L2HMC row kernel was bound by shared-memory load latency and the LSU
# pipe, profiles/r02c_l2hmc_rows_full.md).  The compiled program is keyed by
# the identity of those tensors (tensors are immutable; a capture of a trace
# is the same object on every call).  SF_BAKE=0 disables it.
BAKE = __import__("os").environ.get("SF_BAKE", "1") == "1"
# drop x + (+0) whose result only reaches relu (lowering.elide_zero_adds)
ELIDE_ZERO_ADDS = __import__("os").environ.get("SF_ELIDE_ZERO_ADDS", "1") == "1"
BAKE_MAX_NUMEL = 1024
# tensors captured by a ConcreteFunction (staging.py): the same immutable
# object is passed on every call of that function
STABLE_CAPTURES: "weakref.WeakSet" = weakref.WeakSet()


def bakeable(ph, v) -> bool:
    return (BAKE and not ph.is_variable_ref and isinstance(v, Tensor) and v._symbolic is None
            and v.dtype.is_float and 0 < v.size <= BAKE_MAX_NUMEL and v in STABLE_CAPTURES)


_collective_local = threading.local()


@contextmanager
def reduce_outputs(spec, outputs: Sequence[int]):
    """Run graph functions in this block with ``outputs`` summed over the
    ranks of ``spec.comm`` (comm.GradientCollective): the staged backward of
    a data-parallel step."""
    from .comm import output_spec

    prev = _collective_local.__dict__.get("spec")
    _collective_local.spec = (spec, tuple(outputs), output_spec(spec, outputs))
    try:
        yield
    finally:
        _collective_local.spec = prev


def _output_collective():
    return _collective_local.__dict__.get("spec")


def _signature(inputs: Sequence) -> Tuple:
    return tuple((type(v).__name__ == "Variable", v.dtype, v.shape) for v in inputs)


def _bake_key(gf: GraphFunction, inputs: Sequence) -> Tuple:
    return tuple(id(v) for ph, v in zip(gf.inputs, inputs) if bakeable(ph, v))


def _program_for(gf: GraphFunction, inputs, device, libraries) -> Program:
    cache = gf._plan
    if cache is None:
        cache = gf._plan = {}
    # fast path: the same program as last call when every input is either the
    # very same object (its signature cannot have changed: tensors are
    # immutable, a variable's dtype/shape fixed) or has the same signature
    rt = get_runtime()
    opts = rt.options
    # compiled programs depend on the runtime's RNG mode, fusion switch and
    # registry: a program from an earlier runtime is never reused
    pkey = (device, rt.generation, opts.rng, opts.fuse)
    last = gf.__dict__.get("_last_prog")
    if _collective_local.__dict__.get("spec") is not None:
        last = None  # keyed by the collective too (below)
    if (last is not None and last[0] == pkey and len(last[1]) == len(inputs)
            and last[3].collective is None):
        refs, comps, prog = last[1], last[2], last[3]
        baked = prog.baked
        for i, v in enumerate(inputs):
            if refs[i]() is v:
                continue
            if i in baked or (type(v).__name__ == "Variable", v.dtype, v.shape) != comps[i]:
                break
            refs[i] = weakref.ref(v)
        else:
            return prog
    coll = _output_collective()
    key = (pkey, _signature(inputs), _bake_key(gf, inputs),
           None if coll is None else coll[2])
    prog = cache.get(key)
    if prog is not None and any(r() is not inputs[i] for i, r in prog.baked.items()):
        prog = None  # an id reused by a different tensor
    if prog is None:
        if any(k[0][1] != rt.generation for k in cache):
            cache.clear()  # programs of a replaced runtime
        prog = Program(gf, inputs, device, libraries, opts.rng, opts.fuse,
                       None if coll is None else coll[:2])
        cache[key] = prog
    gf._last_prog = (pkey, [weakref.ref(v) for v in inputs], list(key[1]), prog)
    return prog


def _needs_interpretation(gf: GraphFunction, inputs, device, rt) -> bool:
    if len(rt.devices) == 1:
        return False
    if any(n.device is not None and n.device != device for n in gf.nodes):
        return True
    return any(isinstance(v, Tensor) and v.device != device for v in inputs)


# single elementwise ops of at least this many elements get a generated
# (NVRTC) kernel instead of the precompiled eager one
SINGLE_OP_JIT_NUMEL = 1 << 16

# ---------------------------------------------------------------------------
# whole-program CUDA-graph replay
# ---------------------------------------------------------------------------

# Programs with at least this many native launches are recorded into a CUDA
# graph on their second call and replayed with one launch afterwards.
GRAPH_REPLAY = True
GRAPH_MIN_LAUNCHES = 16
# Python-run plugin ops that only enqueue device work on the backend stream
# (no host reads, no host RNG): safe inside a capture.  nn.install() adds the
# ResNet ops.
GRAPH_SAFE_OPS: set = set()


class _NotCapturable(Exception):
    pass


class _GraphBuffer(_native.DeviceBuffer):
    """Device memory owned by a recorded graph: never freed through the
    allocator; holds the replay's liveness token."""

    __slots__ = ("token",)

    def __init__(self, dev, ptr, nbytes, token):
        super().__init__(dev, ptr, nbytes)
        self.token = token

    def __del__(self):
        self.ptr = 0  # the graph owns the memory: nothing to release


class _Token:
    """Liveness of one replay's outputs; keeps the graph (and so the memory
    the outputs live in) alive while any output is."""

    __slots__ = ("graph", "__weakref__")

    def __init__(self, graph):
        self.graph = graph


class _ProgramGraph:
    """A staged program recorded once into a CUDA graph (stream capture of its
    plans and capture-safe Python segments) and replayed with one
    cudaGraphLaunch per call — "CUDA graphs instead of a tracing compiler".

    Inputs: variables and outputs of other recorded programs are *borrowed*
    (their addresses are stable; a replay requires the same addresses);
    every other tensor is copied into a graph-owned buffer each call (skipped
    when it is the same immutable tensor as last time).  Outputs are the
    graph's own buffers, handed out zero-copy; while any output of the last
    replay is alive the graph is busy and the program runs directly instead,
    so a result is never overwritten under its owner."""

    def __init__(self, prog: "Program", inputs, libraries):
        from .state import Variable

        self.prog = prog
        dev = self.dev = prog.dev
        w = self.graph = _native.WhileGraph(dev, plain=True)
        self.kinds: List[tuple] = []
        run_inputs = []
        for lv, v in zip(prog.in_vals, inputs):
            if isinstance(v, Variable):
                self.kinds.append(("borrow", v._storage_ptr()))
                run_inputs.append(v)
            elif isinstance(v, Tensor) and isinstance(v._buf, _GraphBuffer):
                self.kinds.append(("borrow", v._buf.ptr))
                run_inputs.append(v)
            elif isinstance(v, Tensor):
                p = w.buffer(v.nbytes)
                self.kinds.append(("fixed", p, v.nbytes))
                run_inputs.append(Tensor._adopt(v.dtype, v.shape, v.device,
                                                _GraphBuffer(dev, p, v.nbytes, None)))
            else:
                raise _NotCapturable("unsupported input")
        self.last = [None] * len(self.kinds)
        self._copy_in(inputs)
        w.capture_begin(0)
        try:
            outs = prog._run_direct(run_inputs, libraries)
        except BaseException:
            try:
                w.capture_end(0)
            except Exception:
                pass
            raise
        w.capture_end(0)
        inputs_ptrs = {k[1] for k in self.kinds}
        self.outs = []
        owned_bufs = []
        for lv, t in zip(prog.out_vals, outs):
            buf = t._buf
            ptr = buf.ptr if buf is not None else 0
            if lv.root().kind == "const" or buf is None:
                kind = "static"      # a plan-owned constant: returned as is
            elif ptr in inputs_ptrs:
                kind = "copy"        # passes an input through: copied out per call
            else:
                kind = "graph"       # allocated inside the capture: graph-owned
                owned_bufs.append(buf)
            self.outs.append((kind, t, ptr, t.nbytes))
        for buf in owned_bufs:
            buf.ptr = 0              # never freed through the allocator
        self.token_ref = None
        self.first_outputs = self._launch()

    def _copy_in(self, inputs) -> None:
        for i, (k, v) in enumerate(zip(self.kinds, inputs)):
            if k[0] != "fixed":
                continue
            ref = self.last[i]
            if ref is not None and ref() is v:
                continue
            if k[2]:
                _native.copy_d2d(self.dev, k[1], v._ptr(), k[2])
            self.last[i] = weakref.ref(v)

    def _launch(self) -> List[Tensor]:
        self.graph.launch()
        token = _Token(self.graph)
        self.token_ref = weakref.ref(token)
        res = []
        dev, device = self.dev, self.prog.device
        for kind, t, ptr, n in self.outs:
            if kind == "graph":
                res.append(Tensor._adopt(t.dtype, t.shape, device, _GraphBuffer(dev, ptr, n, token)))
            elif kind == "copy":
                buf = _native.alloc(dev, n)
                if n:
                    _native.copy_d2d(dev, buf.ptr, ptr, n)
                res.append(Tensor._adopt(t.dtype, t.shape, device, buf))
            else:
                res.append(t)
        return res

    def try_run(self, inputs) -> Optional[List[Tensor]]:
        if self.token_ref is not None and self.token_ref() is not None:
            return None  # outputs of the last replay still alive
        from .state import Variable

        for k, v in zip(self.kinds, inputs):
            if k[0] == "borrow":
                p = v._storage_ptr() if isinstance(v, Variable) else \
                    (v._buf.ptr if isinstance(v, Tensor) and isinstance(v._buf, _GraphBuffer)
                     else None)
                if p != k[1]:
                    return None
            elif not isinstance(v, Tensor):
                return None
        self._copy_in(inputs)
        return self._launch()


# ---------------------------------------------------------------------------
# device-side while_loop
# ---------------------------------------------------------------------------

DEVICE_WHILE = True
# cond as an IF/ELSE graph: correct (tests/test_gpu_api.py) but, measured on
# B200 (bench extra f1_device_while), 88 us/call against 74 us for the host
# read — one predicate read is cheaper than the graph launch plus the copies
# into its fixed buffers — so it is opt-in
DEVICE_COND = False


def _plain_program(prog: "Program") -> bool:
    """One native segment, no RNG (counters are reserved at enqueue time, so
    a recorded graph would replay the same draws), tensors only."""
    if any(isinstance(s, _PySegment) for s in prog.segments) or len(prog.segments) > 1:
        return False
    if prog.has_rng:
        return False
    return all(lv.kind == "input" for lv in prog.in_vals)


class _WhileProgram:
    """A while_loop whose predicate never leaves the device.

    The cond and body native plans are recorded once, by stream capture, into
    a CUDA graph with a WHILE conditional node (csrc/sf_graph.cu); each call
    copies the loop variables and captures into the graph's fixed buffers,
    launches the graph and copies the final state out.  The kernels are the
    plans' own, so results are bit-identical to the host loop's."""

    def __init__(self, cprog: "Program", bprog: "Program", n_vars: int, dev: int):
        self.n_vars = n_vars
        self.dev = dev
        self.cprog, self.bprog = cprog, bprog
        w = self.graph = _native.WhileGraph(dev)
        self.sizes = [lv.nbytes for lv in cprog.in_vals]
        self.state = [w.buffer(n) for n in self.sizes[:n_vars]]
        self.ccaps = [w.buffer(n) for n in self.sizes[n_vars:]]
        self.bcaps = [w.buffer(lv.nbytes) for lv in bprog.in_vals[n_vars:]]
        self.specs = [(lv.dtype, lv.shape, lv.nbytes) for lv in bprog.in_vals[:n_vars]]
        part = 0
        try:
            w.capture_begin(0)
            w.set_cond(self._run(cprog, self.state + self.ccaps)[0])
            w.capture_end(0)
            part = 1
            w.capture_begin(1)
            new = self._run(bprog, self.state + self.bcaps)
            # a new value that IS an old state buffer must be read before any
            # state buffer is overwritten: stage those through scratch
            staged = []
            for k, p in enumerate(new):
                if p in self.state and p != self.state[k]:
                    tmp = _native.alloc(dev, self.specs[k][2])
                    _native.copy_d2d(dev, tmp.ptr, p, self.specs[k][2])
                    staged.append(tmp)
                    tmp_ptr, tmp.ptr = tmp.ptr, 0  # owned by the graph from now on
                    new[k] = tmp_ptr
            for k, p in enumerate(new):
                if p != self.state[k]:
                    _native.copy_d2d(dev, self.state[k], p, self.specs[k][2])
            w.set_cond(self._run(cprog, self.state + self.ccaps)[0])
            w.capture_end(1)
            part = -1
        except BaseException:
            if part >= 0:
                try:
                    w.capture_end(part)
                except Exception:
                    pass
            raise

    @staticmethod
    def _run(prog: "Program", ptrs: List[int]) -> List[int]:
        """Enqueue prog's plan on fixed pointers; device pointers of its outputs."""
        by_input = {id(lv): p for lv, p in zip(prog.in_vals, ptrs)}
        out_ptr: Dict[int, int] = {}
        for seg in prog.segments:
            outs = seg.plan.run([by_input[id(r)] for r in seg.in_roots])
            for r, p in zip(seg.out_roots, outs):
                out_ptr[id(r)] = p   # graph-owned (allocated inside the capture)
        res = []
        for lv in prog.out_vals:
            r = lv.root()
            if id(r) in out_ptr:
                res.append(out_ptr[id(r)])
            elif id(r) in by_input:
                res.append(by_input[id(r)])
            else:
                prog.keep.append(r.tensor)
                res.append(r.tensor._ptr())
        return res

    def run(self, state, ccaps, bcaps, device) -> List[Tensor]:
        dev = self.dev
        last = self.__dict__.setdefault("last", {})
        for i, (dst, t) in enumerate(zip(self.state + self.ccaps + self.bcaps,
                                         list(state) + list(ccaps) + list(bcaps))):
            if i >= self.n_vars:
                ref = last.get(i)
                if ref is not None and ref() is t:
                    continue  # the same immutable captured tensor: already in place
                last[i] = weakref.ref(t)
            if t.nbytes:
                _native.copy_d2d(dev, dst, t._ptr(), t.nbytes)
        self.graph.launch()
        out = []
        for (dtype, shape, n), src in zip(self.specs, self.state):
            buf = _native.alloc(dev, n)
            if n:
                _native.copy_d2d(dev, buf.ptr, src, n)
            out.append(Tensor._adopt(dtype, shape, device, buf))
        return out


class _CondProgram:
    """cond with the predicate read on the device: one CUDA graph
    [set_cond(pred)] -> IF { then plan -> copy } ELSE { else plan -> copy }
    (csrc/sf_graph.cu), replacing the host read of _cond_kernel."""

    def __init__(self, tprog: "Program", eprog: "Program", n_ops: int, dev: int):
        self.dev = dev
        w = self.graph = _native.WhileGraph(dev, is_if=True)
        self.pred = w.buffer(1)
        self.bufs = [w.buffer(lv.nbytes) for lv in tprog.in_vals[:n_ops]]
        self.bufs += [w.buffer(lv.nbytes) for lv in tprog.in_vals[n_ops:]]
        self.bufs += [w.buffer(lv.nbytes) for lv in eprog.in_vals[n_ops:]]
        self.last = [None] * len(self.bufs)  # weakrefs: immutable inputs copied once
        nt = len(tprog.in_vals)
        self.specs = [(lv.dtype, lv.shape, lv.nbytes) for lv in tprog.out_vals]
        self.outs = [w.buffer(n) for _, _, n in self.specs]
        part = 0
        try:
            w.capture_begin(0)
            w.set_cond(self.pred)
            w.capture_end(0)
            for part, (prog, ins) in enumerate(
                    ((tprog, self.bufs[:nt]), (eprog, self.bufs[:n_ops] + self.bufs[nt:])), 1):
                w.capture_begin(part)
                for dst, src, (_, _, n) in zip(self.outs, _WhileProgram._run(prog, ins),
                                               self.specs):
                    if n:
                        _native.copy_d2d(dev, dst, src, n)
                w.capture_end(part)
            part = -1
        except BaseException:
            if part >= 0:
                try:
                    w.capture_end(part)
                except Exception:
                    pass
            raise

    def run(self, pred, values, device) -> List[Tensor]:
        dev = self.dev
        _native.copy_d2d(dev, self.pred, pred._ptr(), 1)
        for i, (dst, t) in enumerate(zip(self.bufs, values)):
            ref = self.last[i]
            if ref is not None and ref() is t:
                continue  # the same immutable tensor as last call: already in place
            if t.nbytes:
                _native.copy_d2d(dev, dst, t._ptr(), t.nbytes)
            self.last[i] = weakref.ref(t)
        self.graph.launch()
        out = []
        for (dtype, shape, n), src in zip(self.specs, self.outs):
            buf = _native.alloc(dev, n)
            if n:
                _native.copy_d2d(dev, buf.ptr, src, n)
            out.append(Tensor._adopt(dtype, shape, device, buf))
        return out


def device_cond(then_gf: GraphFunction, else_gf: GraphFunction, pred, operands, then_caps,
                else_caps, env: KernelEnv) -> Optional[List[Tensor]]:
    """Run a cond with the predicate on the device, or return None (the caller
    reads it on the host).  Same first-call policy as device_while."""
    values = list(operands) + list(then_caps) + list(else_caps)
    if not DEVICE_COND or not isinstance(pred, Tensor) or pred.dtype is not DType.boolean \
            or pred.size != 1 or any(not isinstance(v, Tensor) for v in values):
        return None
    device = env.device
    cache = then_gf.__dict__.setdefault("_device_cond", {})
    key = (id(else_gf), device, _signature(list(operands) + list(then_caps)),
           _signature(list(else_caps)))
    ent = cache.get(key)
    if ent is None:
        cache[key] = "host-once"
        return None
    if ent == "host-once":
        libs = tuple(env.libraries)
        try:
            tprog = _program_for(then_gf, list(operands) + list(then_caps), device, libs)
            eprog = _program_for(else_gf, list(operands) + list(else_caps), device, libs)
        except Exception:
            tprog = eprog = None
        ok = (tprog is not None and _plain_program(tprog) and _plain_program(eprog)
              and [(v.dtype, v.shape) for v in tprog.out_vals]
              == [(v.dtype, v.shape) for v in eprog.out_vals])
        ent = cache[key] = (_CondProgram(tprog, eprog, len(operands), ordinal_of(device))
                            if ok else "host")
    if ent == "host":
        return None
    get_runtime().stats.count_graph_launch()
    return ent.run(pred, values, device)


def device_while(cond_gf: GraphFunction, body_gf: GraphFunction, state, cond_caps, body_caps,
                 env: KernelEnv) -> Optional[List[Tensor]]:
    """Run a while_loop on the device, or return None (caller loops on the
    host with the same kernels).  The first call of a loop signature runs on
    the host, which also compiles and loads every kernel; the graph is
    recorded on the second call."""
    if not DEVICE_WHILE or any(not isinstance(v, Tensor) for v in
                               list(state) + list(cond_caps) + list(body_caps)):
        return None
    device = env.device
    cache = body_gf.__dict__.setdefault("_device_while", {})
    key = (id(cond_gf), device, _signature(list(state) + list(cond_caps)),
           _signature(list(body_caps)))
    ent = cache.get(key)
    if ent is None:
        cache[key] = "host-once"
        return None
    if ent == "host-once":
        libs = tuple(env.libraries)
        try:
            cprog = _program_for(cond_gf, list(state) + list(cond_caps), device, libs)
            bprog = _program_for(body_gf, list(state) + list(body_caps), device, libs)
        except Exception:
            cprog = bprog = None
        ok = (cprog is not None and _plain_program(cprog) and _plain_program(bprog)
              and len(cprog.out_vals) == 1 and cprog.out_vals[0].dtype is DType.boolean
              and len(bprog.out_vals) == len(state))
        ent = cache[key] = (_WhileProgram(cprog, bprog, len(state), ordinal_of(device))
                            if ok else "host")
    if ent == "host":
        return None
    get_runtime().stats.count_graph_launch()
    return ent.run(state, cond_caps, body_caps, device)


def execute_graph(gf: GraphFunction, inputs: Sequence, env: Optional[KernelEnv] = None,
                  workers: Optional[int] = None) -> List[Tensor]:
    rt = get_runtime()
    _bind_inputs(gf, inputs)
    if env is not None:
        device = env.device
        libraries = (gf.library,) + tuple(env.libraries)
    else:
        device = current_context().scope_device() or rt.devices[0].name
        libraries = (gf.library,)
    if _needs_interpretation(gf, inputs, device, rt):
        return _interpret(gf, inputs, device, libraries)
    prog = _program_for(gf, inputs, device, libraries[1:])
    rt.stats.count_graph_launch()
    return prog.run(inputs, libraries)


def _interpret(gf: GraphFunction, inputs, device, libraries) -> List[Tensor]:
    """Per-node launches with the reference's transparent-copy accounting."""
    rt = get_runtime()
    n_in = len(gf.inputs)
    vals: Dict[Tuple[int, int], object] = {(i, 0): v for i, v in enumerate(inputs)}
    for j, node in enumerate(gf.nodes):
        vid = n_in + j
        if node.op == "constant":
            vals[(vid, 0)] = node.attrs["value"]
            continue
        from .ops import get_op_def

        target = node.device or device
        kenv = KernelEnv(device=target, libraries=libraries, nested=True)
        ins, moved = [], {}
        for r in node.inputs:
            v = vals[r]
            if isinstance(v, Tensor) and v.device != target:
                c = moved.get(id(v))
                if c is None:
                    c = moved[id(v)] = relabel(v, target)
                    rt.stats.count_copy()
                v = c
            ins.append(v)
        try:
            outs = get_op_def(node.op).kernel(node.attrs, ins, kenv)
        except _PASSTHROUGH:
            raise
        except Exception as e:
            raise KernelError(f"node {j} ({node.op}): {e}") from e
        for k, o in enumerate(outs):
            vals[(vid, k)] = o
    return [vals[ref] for _, ref in gf.outputs]


def execute(gf: GraphFunction, inputs: Sequence, captured: Sequence = (),
            workers: Optional[int] = None) -> List[Tensor]:
    """Run a graph function directly (inputs, then captured values)."""
    everything = list(inputs) + list(captured)
    rt = get_runtime()
    device = current_context().scope_device()
    if device is None:
        device = next((v.device for v in everything if isinstance(v, Tensor)), rt.devices[0].name)
    return execute_graph(gf, everything, env=KernelEnv(device=device), workers=workers)


def run_node_for_folding(node: Node, inputs: Sequence[Tensor], library) -> List[Tensor]:
    """Evaluate one stateless node on constant inputs with the GPU kernels."""
    from .ops import get_op_def

    rt = get_runtime()
    env = KernelEnv(device=rt.devices[0].name, libraries=(library,), nested=True)
    try:
        return get_op_def(node.op).kernel(node.attrs, list(inputs), env)
    except StageflowError:
        raise
    except Exception as e:
        raise KernelError(f"folding {node.op}: {e}") from e
