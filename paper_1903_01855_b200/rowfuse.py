"""Row programs: whole per-chain computations fused into ONE kernel.

The staged graphs of samplers (the reference's leapfrog, the L2HMC
transition) are thousands of tiny ops over a batch of independent chains:
every value is either *rowed* — shape (B, w) or (B,), one row per chain — or
*uniform* — weights, time encodings, masks, scalars.  Every op is row-local
(elementwise with row/uniform broadcasting, ``rowed @ uniform`` matmuls,
reductions along the row, per-element RNG).  Such a run of ops lowers to a
single generated kernel in which each thread owns one chain and keeps its
whole trajectory in registers; uniform inputs are staged once per CTA in
shared memory.  This is the "persistent kernel for small-op graphs" of the
north star: the per-op launch cost and all intermediate HBM traffic vanish.

Bit-exactness with the eager kernels is by construction: elementwise ops
call the sf_ops.cuh functions, matmuls use the sequential-k FMA contract of
sf_matmul.cu, row reductions use the canonical reduction order (CRO) of
sf_reduce.cu, and RNG elements use the same Philox counter (offset + flat
index) as sf_misc.cu.
"""
from __future__ import annotations

import hashlib
import re
from typing import Dict, List, Optional, Tuple

from . import dtypes
from .dtypes import DType
from .errors import KernelError
from .lowering import LOp, LV, _CTYPE, _strides_for, c_literal, ew_expr

ROW_KINDS = frozenset(("ew", "matmul", "reduce", "transpose", "rng", "eye"))
MAX_UNIFORM_NUMEL = 1024       # uniform values computed per thread
MAX_MATVEC = 1024              # k*n of a row matmul
MAX_SMEM_BYTES = 40 * 1024     # uniform inputs staged in shared memory
UNIFORM_SMEM_BYTES = 46 * 1024  # uniform kernel: results (static smem)
# uniform kernel: global operands staged once into dynamic shared memory (a
# chain of small layers, like C2's 100 (16,16) weights = 109 KB, then reads
# every operand at shared-memory latency instead of an L2 round trip per layer)
UNIFORM_DYN_BYTES = 200 * 1024
MIN_BATCH = 2


# NVVM compile time grows superlinearly with function size, so a long row
# program is cut into chunks of about this many scalar operations; each
# chunk is its own kernel (rowed values crossing a cut round-trip through
# L2-resident temporaries) and the chunks compile in parallel.
# (B200 sweeps, L2HMC 1e5 chains, before re-rolling:
# 1200 -> 0.38 ms/step, 4800 -> 0.29 ms, 9600 -> 0.28 ms at 3x the compile
# time, 19200+ slower.  With re-rolled loops the whole transition is ~9000
# ops: 4800 -> 2 row kernels, 0.202 ms; 9000 -> 1 row kernel, 0.196 ms, and
# 0.081 -> 0.077 ms at 200 chains, for +1.3 s of one-time compile (cached).)
CHUNK_COST = int(__import__("os").environ.get("SF_CHUNK_COST", "9000"))
# CTAs of 128 threads that must fit per SM (register budget = 64K / (128 *
# MIN_BLOCKS)); 0 = no minimum, ptxas picks (best in the sweep once the
# weights are read with volatile vector loads: ~96 registers, no spills)
MIN_BLOCKS = int(__import__("os").environ.get("SF_MIN_BLOCKS", "0"))
# chains per thread in row kernels: 0 = automatic.  Measured on B200 (L2HMC,
# 1e5 chains): 2 chains/thread halves the shared-memory weight loads per
# chain and doubles the independent work per thread.  With the transition
# split over two row kernels it did not move the step (0.207 vs 0.204 ms);
# with the whole transition in one kernel it does with a warm L2: 0.195 ->
# 0.177 ms (e2e 3.5e8 -> 3.7e8 samples/s; compile 3.7 -> 10 s, cached).  But
# the doubled loop body makes the step sensitive to a cold L2 (instruction
# refetch): with the L2 flushed between steps, as bench.py times the
# headline, 0.204 -> 0.239 ms.  Automatic keeps 1 chain per thread; set
# SF_ROW_REPLICAS=2 (or REPLICA_MIN_BATCH) for warm-cache serving loops.
# Round 2: with two chains per thread, element j of both chains shares one
# float2 (FADD2 / FFMA2 with the weight broadcast, "xpack"); still slower on
# the flushed headline step (0.171 -> 0.192 ms, 168 registers, 10.6 warps/SM).
ROW_REPLICAS = int(__import__("os").environ.get("SF_ROW_REPLICAS", "0"))
REPLICA_MIN_BATCH = 1 << 62
# SMs of the target GPU (B200: 148); set by the executor from the device
SM_COUNT = 148
# matvec weight vectors loaded ahead of their FMAs (latency hiding vs registers)
PREFETCH = int(__import__("os").environ.get("SF_PREFETCH", "4"))
# adjacent fp32 row elements computed as packed pairs (sm_100a FADD2 /
# FFMA2: one instruction for two IEEE operations, bit-identical to the
# scalar ones) in elementwise add/sub and in matvec accumulators.
# Multiplies stay scalar: ptxas (12.9) contracts mul.rn.f32x2 + add.rn.f32x2
# into FFMA2 even under -fmad=false (measured: the fused leapfrog then
# differed from eager in 77% of elements), while a scalar FMUL feeding an
# FADD2 is never fused.
PACK = __import__("os").environ.get("SF_ROW_PACK", "1") == "1"
_PACKED = {"add": "sf::add2", "sub": "sf::sub2"}
# Option: row kernels read their uniform operands (weights, biases, stacked
# per-step uniforms) from a per-module __constant__ pool that the plan
# gathers before each launch, instead of staging them into shared memory in
# every CTA.  Warp-uniform constant loads run on the uniform datapath (LDCU)
# and feed FFMA/FFMA2 as uniform-register operands.  A B200 microbenchmark
# (10x10 relu matvecs per thread, 1.6 KB of weights) ran 94.5 -> 49.8 us;
# but ptxas merges repeated constant loads of one address into long-lived
# registers (4.7 KB of spills), so every use site needs its own copy, and
# the L2HMC transition's 31 KB pool then runs SLOWER than shared memory
# (B200: 64 -> 86 us at 200 chains, 166 -> 176 us at 1e5; ncu: the LDCU
# latency moves the short_scoreboard stall onto the FFMA2s).  Off by
# default; SF_ROW_CONST=1 enables it (tests keep it bit-exact).
CONST_POOL = __import__("os").environ.get("SF_ROW_CONST", "0") == "1"
_CL = {"float": "clf", "double": "cld", "int": "cli", "bool": "clb"}
CPOOL_BYTES = 60 * 1024  # constant bank 3 holds 64 KB
# re-roll repeated blocks of row ops into loops (LoopOp)
REROLL = __import__("os").environ.get("SF_REROLL", "1") == "1"


class RowProgram:
    __slots__ = ("ops", "batch", "gen", "uniform_only", "block", "replicas", "cpool", "teams",
                 "team_width", "min_blocks", "row_threads",
                 "rows_per_cta", "dyn_smem")

    def __init__(self, batch: int):
        self.ops: List[LOp] = []
        self.batch = batch
        self.gen = None  # cached generate_rowprog result
        self.uniform_only = False  # single-CTA kernel for chain-independent ops
        # (pool bytes, [(pointer slot, offset, elements, width, N, Np)]) of a
        # row kernel reading its uniforms from the __constant__ pool
        self.cpool = None
        self.block = 128  # threads per CTA (set by code generation)
        # chains per thread: large batches take 2 (shared weight loads, 2x ILP)
        self.replicas = ROW_REPLICAS if ROW_REPLICAS else (2 if batch >= REPLICA_MIN_BATCH else 1)
        # two teams of warps per CTA, each running one independent half of
        # the program for the same 64 chains (find_teams), or None
        self.teams = None
        self.rows_per_cta = 128  # chains per CTA (set by code generation)
        self.team_width = 0  # threads per team of a team-split kernel
        self.min_blocks = 0  # CTAs per SM the launch bounds ask for
        self.row_threads = 128  # threads of a CTA that own chains
        self.dyn_smem = 0  # dynamic shared memory bytes of the kernel


class LoopOp:
    """``m`` consecutive, structurally identical blocks of row ops run as one loop.

    Tracing unrolls the sampler's Python loop (the reference traces every
    leapfrog step into the graph, stageflow/staging.py), so a row program
    repeats the same block of ops once per step; straight-line code for all
    of them overflows the SM instruction cache (ncu: ``no_instruction`` was
    the top stall, and a cold L2 re-fetches every byte of it from HBM).  The
    blocks are re-rolled into one loop body: rowed values flowing from block
    i-1 into block i become loop-carried registers, per-step uniform operands
    (time encodings, per-step weights) are stacked in shared memory and
    indexed by the iteration, and the last block's values used afterwards
    are exported.  Every element still goes through the identical sequence
    of scalar operations, so results are bit-for-bit those of the unrolled
    code.
    """

    __slots__ = ("kind", "name", "ins", "outs", "attrs", "body", "m", "carried", "stacked",
                 "exports")

    def __init__(self):
        self.kind = "loop"
        self.name = "loop"
        self.attrs = {}
        self.body: List[LOp] = []
        self.m = 0
        self.carried: List[Tuple[LV, LV, LV]] = []    # (synthetic, init value, body source)
        self.stacked: List[Tuple[LV, List[LV]]] = []  # (synthetic, per-iteration roots)
        self.exports: List[Tuple[LV, LV]] = []        # (last block's value, body value)
        self.ins: List[LV] = []
        self.outs: List[LV] = []


_SYN_ID = [1 << 40]


def _synthetic(dtype, shape, kind: str, base: Optional[LV] = None) -> LV:
    _SYN_ID[0] += 1
    v = LV(_SYN_ID[0], dtype, shape, kind)
    v.base = base
    return v


MIN_REPS = 3
MIN_PERIOD = 4
PHASE_SHIFTS = 8  # block starts tried within the first block of a repeat


def _sig(op: LOp, planner) -> tuple:
    ins = []
    for x in op.ins:
        r = x.root()
        imm = repr(r.imm) if (r.kind == "const" and r.imm is not None) else None
        ins.append((tuple(x.shape), x.dtype.value, planner.layout_of(x)[0], imm))
    return (op.kind, op.name, repr(sorted(op.attrs.items())), tuple(ins),
            tuple((tuple(o.shape), o.dtype.value) for o in op.outs))


def reroll(ops: List[LOp], planner, users: Dict[int, List[LOp]], keep: set) -> List:
    """Replace tandem repeats of row-op blocks by LoopOps (recursively on the
    remaining prefix and suffix)."""
    import numpy as np

    n = len(ops)
    if n < MIN_PERIOD * MIN_REPS or any(op.kind == "loop" for op in ops):
        return list(ops)
    table: Dict[tuple, int] = {}
    seq = np.array([table.setdefault(_sig(op, planner), len(table)) for op in ops])
    cands = []
    for p in range(MIN_PERIOD, n // MIN_REPS + 1):
        eq = seq[:-p] == seq[p:]
        cs = np.concatenate(([0], np.cumsum(eq)))
        last = n - 2 * p
        if last < 0:
            break
        starts = np.arange(last + 1)
        good = (cs[starts + p] - cs[starts]) == p
        for s in np.nonzero(good)[0].tolist():
            if s >= p and good[s - p]:
                continue  # not the start of a chain
            reps = 1
            while s + (reps - 1) * p <= last and good[s + (reps - 1) * p]:
                reps += 1
            if reps >= MIN_REPS:
                cands.append(((reps - 1) * p, p, s, reps))
    cands.sort(key=lambda c: (-c[0], c[1]))
    for _score, p, s, reps in cands[:40]:
        # spans that start 0-2 whole blocks in, or a few ops into a block (the
        # first block of a traced loop often reads a value computed before
        # the loop where later blocks compute it themselves; starting the
        # blocks one op later turns that operand into a carried one), with
        # as many blocks as the periodic run from that start allows
        eq = seq[:-p] == seq[p:]
        tried, attempts = set(), []
        for shift in range(min(p, PHASE_SHIFTS)):
            for front in range(3):
                s0 = s + front * p + shift
                if s0 >= len(eq):
                    continue
                stop = np.flatnonzero(~eq[s0:])
                run = int(stop[0]) if len(stop) else len(eq) - s0
                for back in range(3):
                    m = 1 + run // p - back
                    if m >= MIN_REPS and (m, s0) not in tried:
                        tried.add((m, s0))
                        attempts.append((-m, s0))
        for neg_m, s0 in sorted(attempts)[:64]:
            m = -neg_m
            loop = _make_loop(ops[s0:s0 + m * p], p, m, planner, users, keep)
            if loop is not None:
                return (reroll(ops[:s0], planner, users, keep) + [loop]
                        + reroll(ops[s0 + m * p:], planner, users, keep))
    return list(ops)


def _make_loop(span: List[LOp], p: int, m: int, planner, users, keep) -> Optional[LoopOp]:
    blocks = [span[i * p:(i + 1) * p] for i in range(m)]
    if any(op.kind == "rng" for op in blocks[0]):
        return None
    pos: Dict[int, Tuple[int, int, int]] = {}
    for i, blk in enumerate(blocks):
        for j, op in enumerate(blk):
            for oi, o in enumerate(op.outs):
                pos[id(o)] = (i, j, oi)
    in_span = {id(op) for op in span}
    # values of blocks 1..m-1 may only feed their own block or the next one;
    # the last block's values used after the loop are exported
    exports: Dict[int, Tuple[LV, LV]] = {}
    for i, blk in enumerate(blocks):
        for j, op in enumerate(blk):
            for oi, o in enumerate(op.outs):
                outside = id(o) in keep or any(id(u) not in in_span
                                               for u in users.get(id(o), ()))
                if i < m - 1:
                    if outside:
                        return None
                elif outside:
                    exports[id(o)] = (o, blocks[0][j].outs[oi])
    # per-op block index of every user inside the span (for the i/i+1 rule)
    block_of = {}
    for i, blk in enumerate(blocks):
        for op in blk:
            block_of[id(op)] = i
    for o_id, (i, j, oi) in pos.items():
        for u in users.get(o_id, ()):
            bi = block_of.get(id(u))
            if bi is not None and bi not in (i, i + 1):
                return None
    loop = LoopOp()
    loop.m = m
    carried: Dict[Tuple[int, int], LV] = {}   # (j', oi) of the source -> synthetic
    stacked: Dict[tuple, LV] = {}
    ext: Dict[int, LV] = {}
    body: List[LOp] = []
    for j, op0 in enumerate(blocks[0]):
        new_ins = []
        for q, x0 in enumerate(op0.ins):
            xs = [blocks[i][j].ins[q] for i in range(m)]
            roots = [x.root() for x in xs]
            r0 = roots[0]
            if r0.kind == "const" and r0.imm is not None:
                new_ins.append(x0)  # same literal in every block (part of the signature)
                continue
            P = [pos.get(id(r)) for r in roots]
            L = planner.layout_of(x0)
            if L[0] == UNI:
                if any(pp is not None for pp in P):
                    return None
                if all(r is r0 for r in roots):
                    ext[id(r0)] = r0
                    new_ins.append(x0)
                    continue
                if any(x.shape != r.shape for x, r in zip(xs, roots)) or \
                        any(r.shape != r0.shape or r.dtype != r0.dtype for r in roots):
                    return None
                key = tuple(id(r) for r in roots)
                syn = stacked.get(key)
                if syn is None:
                    syn = _synthetic(r0.dtype, r0.shape, "stacked")
                    planner.layout[id(syn)] = (UNI,)
                    stacked[key] = syn
                    loop.stacked.append((syn, roots))
                    for r in roots:
                        ext[id(r)] = r
                new_ins.append(syn)
                continue
            # rowed operand
            if all(pp is not None and pp[0] == i for i, pp in enumerate(P)):
                if any(pp[1:] != P[0][1:] for pp in P):
                    return None
                new_ins.append(x0)                      # internal to the block
                continue
            if all(pp is None for pp in P):
                if any(r is not r0 for r in roots):
                    return None
                ext[id(r0)] = r0
                new_ins.append(x0)                      # loop-invariant
                continue
            if P[0] is None and all(pp is not None and pp[0] == i - 1
                                    for i, pp in enumerate(P) if i):
                src = P[1][1:]
                if any(pp[1:] != src for pp in P[1:]):
                    return None
                if any(x.shape != xs[0].shape for x in xs):
                    return None
                syn = carried.get(src)
                if syn is None:
                    syn = _synthetic(r0.dtype, r0.shape, "carried")
                    planner.layout[id(syn)] = planner.layout_of(r0)
                    carried[src] = syn
                    body_src = blocks[0][src[0]].outs[src[1]]
                    if body_src.shape != r0.shape or body_src.dtype != r0.dtype:
                        return None
                    loop.carried.append((syn, r0, body_src))
                    ext[id(r0)] = r0
                elif any(c[1] is not r0 for c in loop.carried if c[0] is syn):
                    return None
                if x0 is r0:
                    new_ins.append(syn)
                else:
                    al = _synthetic(x0.dtype, x0.shape, "alias", base=syn)
                    if planner.layout_of(al)[0] == BAD:
                        return None
                    new_ins.append(al)
                continue
            return None
        body.append(LOp(op0.kind, op0.name, new_ins, op0.outs, op0.attrs, op0.node_idx,
                        op0.op_def))
    loop.body = body
    loop.exports = list(exports.values())
    loop.ins = list(ext.values())
    loop.outs = [e for e, _ in loop.exports]
    return loop


def _op_cost(op, planner) -> int:
    if op.kind == "loop":
        return sum(_op_cost(b, planner) for b in op.body)
    o = op.outs[0]
    L = planner.layout_of(o)
    width = L[1] if L[0] == ROW else max(1, o.numel)
    if op.kind == "matmul":
        return op.ins[0].shape[-1] * width
    return width


def _split(rp: RowProgram, planner) -> List[RowProgram]:
    chunks, cur, cost = [], RowProgram(rp.batch), 0
    for op in rp.ops:
        c = _op_cost(op, planner)
        if cur.ops and cost + c > CHUNK_COST:
            chunks.append(cur)
            cur, cost = RowProgram(rp.batch), 0
        cur.ops.append(op)
        cost += c
    if cur.ops:
        chunks.append(cur)
    return chunks


ROW, UNI, BAD = "row", "uni", "bad"


def variable_derived(ops: List[LOp]) -> set:
    """ids of chain-independent values: variables, the weight operands of
    matmuls (the B side, traced back to the graph inputs they come from), and
    everything computed from those and constants only.  Such a value stays
    uniform even when its leading extent happens to equal the batch (10
    chains through 10-wide layers: W is (10, 10) and W_out (10, 2) looks like
    the chain state), so the planner does not mistake it for rows."""
    prod: Dict[int, LOp] = {}
    for op in ops:
        for o in getattr(op, "outs", ()):
            prod[id(o)] = op
    vd: set = set()
    stack = [op.ins[1].root() for op in ops
             if getattr(op, "kind", None) == "matmul" and not op.attrs.get("tb")]
    while stack:
        r = stack.pop()
        if id(r) in vd:
            continue
        vd.add(id(r))
        p = prod.get(id(r))
        if p is not None and p.kind in ("ew", "transpose", "matmul", "var_read"):
            stack.extend(x.root() for x in p.ins)
    for op in ops:
        if isinstance(op, tuple) or not getattr(op, "ins", None):
            continue
        if op.kind == "var_read":
            vd.update(id(o) for o in op.outs)
            continue
        srcs = [x.root() for x in op.ins]
        if any(id(r) in vd or r.kind == "var" for r in srcs) and all(
                id(r) in vd or r.kind in ("var", "const") for r in srcs):
            vd.update(id(o) for o in op.outs)
    return vd


class RowPlanner:
    def __init__(self, batch: int, uniform_ids=frozenset()):
        self.B = batch
        self.layout: Dict[int, Tuple] = {}
        self.uniform_ids = uniform_ids  # variable-derived values (see variable_derived)

    def layout_of(self, lv: LV) -> Tuple:
        L = self.layout.get(id(lv))
        if L is not None:
            return L
        if lv.kind == "alias":
            base = self.layout_of(lv.base)
            if base[0] == UNI:
                L = (UNI,)
            elif base[0] == ROW:
                L = self._shape_layout(lv.shape)
                if L[0] != ROW or L[1] != base[1]:
                    L = (BAD,)
            else:
                L = (BAD,)
        elif id(lv) in self.uniform_ids or lv.kind == "var":
            L = (UNI,)
        else:
            L = self._shape_layout(lv.shape)
        self.layout[id(lv)] = L
        return L

    def _shape_layout(self, shape) -> Tuple:
        if len(shape) in (1, 2) and shape[0] == self.B:
            return (ROW, shape[1] if len(shape) == 2 else 1, len(shape))
        return (UNI,)

    def op_layouts(self, op: LOp) -> Optional[List[Tuple]]:
        if op.kind not in ROW_KINDS:
            return None
        ins = [self.layout_of(x) for x in op.ins]
        if any(L[0] == BAD for L in ins):
            return None
        k = op.kind
        out = op.outs[0]
        rowed = [L for L in ins if L[0] == ROW]
        if k == "ew":
            if not rowed:
                return [(UNI,)] if out.numel <= MAX_UNIFORM_NUMEL else None
            oL = self._shape_layout(out.shape)
            if oL[0] != ROW:
                return None
            _, w, rank = oL
            for x, L in zip(op.ins, ins):
                if L[0] == ROW:
                    if L[2] != rank or (L[1] != w and L[1] != 1):
                        return None
                elif not _uniform_broadcasts_into_row(x.shape, w, rank):
                    return None
            return [oL]
        if k == "matmul":
            if op.attrs.get("ta") or op.attrs.get("tb"):
                return None
            (La, Lb), (a, b) = ins, op.ins
            if La[0] == UNI and Lb[0] == UNI:
                return [(UNI,)] if out.numel <= MAX_UNIFORM_NUMEL else None
            if La[0] == ROW and La[2] == 2 and Lb[0] == UNI and b.numel <= MAX_MATVEC:
                return [(ROW, b.shape[1], 2)]
            return None
        if k == "reduce":
            L = ins[0]
            if L[0] == UNI:
                return [(UNI,)] if op.ins[0].numel <= MAX_UNIFORM_NUMEL else None
            if L[2] == 2 and tuple(op.attrs["axes"]) == (1,):
                oL = self._shape_layout(out.shape)
                return [oL] if oL[0] == ROW and oL[1] == 1 else None
            return None
        if k == "transpose":
            return [(UNI,)] if ins[0][0] == UNI and out.numel <= MAX_UNIFORM_NUMEL else None
        if k == "eye":
            return [(UNI,)] if out.numel <= MAX_UNIFORM_NUMEL else None
        if k == "rng":
            oL = self._shape_layout(out.shape)
            return [oL] if oL[0] == ROW else None
        return None


def _uniform_broadcasts_into_row(shape, w: int, rank: int) -> bool:
    if dtypes.element_count(shape) == 1:
        return len(shape) <= rank
    if rank == 1:
        return False
    if len(shape) == 1:
        return shape[0] == w
    if len(shape) == 2:
        return shape[0] == 1 and shape[1] == w
    return False


def choose_batch(ops: List[LOp]) -> int:
    counts: Dict[int, int] = {}
    for op in ops:
        for o in op.outs:
            if len(o.shape) in (1, 2) and o.shape[0] >= MIN_BATCH:
                counts[o.shape[0]] = counts.get(o.shape[0], 0) + 1
    if not counts:
        return 0
    return max(counts.items(), key=lambda kv: (kv[1], kv[0]))[0]


def plan_rows(ops: List[LOp], keep=frozenset()) -> List:
    """Split ops into RowPrograms (runs of row-local ops) and plain ops.

    ``keep``: ids of root values the caller needs afterwards (graph outputs)."""
    batch = choose_batch(ops)
    users: Dict[int, List[LOp]] = {}
    for op in ops:
        for x in op.ins:
            users.setdefault(id(x.root()), []).append(op)
    # no batch dimension (e.g. the C2 chain on (1, 16)): every value is uniform
    # and runs of small ops become one-warp uniform kernels
    planner = RowPlanner(batch if batch >= MIN_BATCH else -1, variable_derived(ops))
    units: List = []
    cur: Optional[RowProgram] = None
    for op in ops:
        Ls = planner.op_layouts(op)
        if Ls is None:
            cur = None
            units.append(op)
            continue
        if cur is None:
            cur = RowProgram(batch)
            units.append(cur)
        cur.ops.append(op)
        for o, L in zip(op.outs, Ls):
            planner.layout[id(o)] = L
    # keep row programs that actually carry rowed work and are worth a kernel
    out: List = []
    for u in units:
        if isinstance(u, RowProgram):
            row_ops = [op for op in u.ops if planner.layout_of(op.outs[0])[0] == ROW]
            if len(row_ops) >= 2:
                # chain-independent (uniform) ops never depend on rowed values, so
                # they are hoisted into one single-CTA kernel run once per call
                uni = RowProgram(u.batch)
                uni.ops = [op for op in u.ops if planner.layout_of(op.outs[0])[0] != ROW]
                uni.uniform_only = True
                body = RowProgram(u.batch)
                body.ops = reroll(row_ops, planner, users, keep) if REROLL else row_ops
                chunks = _split(body, planner)
                if 0 < batch <= team_max_batch():
                    for c in chunks:
                        if c.replicas == 1:
                            c.teams = find_teams(c, planner)
                if (all(_smem_bytes(c, planner) <= MAX_SMEM_BYTES for c in chunks)
                        and _uniform_smem(uni) <= MAX_SMEM_BYTES):
                    if uni.ops:
                        out.append((uni, planner))
                    out.extend((c, planner) for c in chunks)
                    continue
            elif not row_ops and len(u.ops) >= 2 and _uniform_smem(u) <= MAX_SMEM_BYTES:
                u.uniform_only = True
                out.append((u, planner))
                continue
            out.extend(u.ops)
        else:
            out.append(u)
    return out


# Team split (latency-bound batches): a row program whose per-chain work
# falls into independent parts — the L2HMC transition's forward and backward
# trajectories, joined only by the direction select and the MH step — runs
# as two teams of warps per CTA over the same 64 chains, each team executing
# one part; the values the join needs cross through shared memory after one
# barrier.  One thread's serial latency per chain halves, which is what
# bounds small batches (C1: 200 chains, ~60 us of dependent instructions).
# Only while the team-split grid (64 chains per CTA) stays within one CTA per
# SM: measured on B200 (L2HMC, device time per transition), 10 - 2000 chains
# 47 -> 35 us, but 1e4 chains (157 CTAs > 148 SMs) 46 -> 53 us.
# SF_TEAM_MAX_BATCH overrides (0 disables).
_TEAM_ENV = __import__("os").environ.get("SF_TEAM_MAX_BATCH")


def team_max_batch() -> int:
    return int(_TEAM_ENV) if _TEAM_ENV is not None else 64 * SM_COUNT
TEAM_MIN_SHARE = 0.25   # each team carries at least this share of the work
TEAM_MAX_JOIN = 0.10    # at most this share of the work runs after the barrier
DUP_MAX_COST = 32       # ops computed from inputs alone up to this cost are recomputed per team


def _full_cost(op, planner) -> int:
    if op.kind == "loop":
        return op.m * sum(_op_cost(b, planner) for b in op.body)
    return _op_cost(op, planner)


def find_teams(rp: RowProgram, planner) -> Optional[Tuple[List[LOp], List[LOp], List[LOp],
                                                            List[LV], List[LV]]]:
    """(team 0 ops, team 1 ops, join ops, team-0 values the join reads,
    team-1 values the join reads), or None when the program does not split."""
    ops = rp.ops
    n = len(ops)
    if n < 4:
        return None
    prod: Dict[int, int] = {}
    for i, op in enumerate(ops):
        for o in op.outs:
            prod[id(o)] = i
    deps = [set() for _ in ops]
    users = [set() for _ in ops]
    for i, op in enumerate(ops):
        for x in op.ins:
            j = prod.get(id(x.root()))
            if j is not None and j != i:
                deps[i].add(j)
                users[j].add(i)
    cost = [_full_cost(op, planner) for op in ops]
    total = float(sum(cost)) or 1.0
    # cheap ops computed from the program's inputs alone (random draws, the
    # energy and force at the initial state both trajectories start from) are
    # recomputed by every part that uses them instead of linking the parts
    dup = [False] * n
    for i, op in enumerate(ops):
        dup[i] = (op.kind != "loop" and (op.kind == "rng" or cost[i] <= DUP_MAX_COST)
                  and all(dup[j] for j in deps[i]))
    rest = {i for i in range(n) if not dup[i]}
    join: set = set()

    def parts():
        parent = {i: i for i in rest}

        def find(i):
            while parent[i] != i:
                parent[i] = parent[parent[i]]
                i = parent[i]
            return i

        for i in rest:
            for j in deps[i]:
                if j in rest:
                    parent[find(i)] = find(j)
        groups: Dict[int, List[int]] = {}
        for i in rest:
            groups.setdefault(find(i), []).append(i)
        return list(groups.values())

    while True:
        comps = parts()
        if len(comps) >= 2:
            comps.sort(key=lambda g: -sum(cost[i] for i in g))
            sides = [[], []]
            load = [0, 0]
            for g in comps:
                t = 0 if load[0] <= load[1] else 1
                sides[t] += g
                load[t] += sum(cost[i] for i in g)
            if min(load) >= TEAM_MIN_SHARE * total:
                break
        sinks = [i for i in rest if not (users[i] & rest)]
        if not sinks:
            return None
        i = max(sinks)
        rest.discard(i)
        join.add(i)
        if sum(cost[j] for j in join) > TEAM_MAX_JOIN * total:
            return None

    def with_sources(members):
        need = set(members)
        stack = [j for i in members for j in deps[i] if dup[j]]
        while stack:
            j = stack.pop()
            if j not in need:
                need.add(j)
                stack += [d for d in deps[j] if dup[d]]
        return [ops[i] for i in sorted(need)]

    side_of = {i: t for t in (0, 1) for i in sides[t]}
    xfer: List[List[LV]] = [[], []]
    seen: set = set()
    for i in sorted(join):
        for x in ops[i].ins:
            r = x.root()
            j = prod.get(id(r))
            if j is None or j not in side_of or id(r) in seen:
                continue
            if planner.layout_of(r)[0] != ROW:
                return None
            seen.add(id(r))
            xfer[side_of[j]].append(r)
    return (with_sources(sides[0]), with_sources(sides[1]), with_sources(sorted(join)),
            xfer[0], xfer[1])


# re-roll runs of identical uniform-kernel levels (see _uniform_prologue)
UNI_REROLL = __import__("os").environ.get("SF_UNI_REROLL", "1") == "1"
UNI_REROLL_MIN = 3
# extra warps of a uniform kernel that only help stage its operands (C2: 1 -> 4
# warps, 24.7 -> 19.6 us per chain; 8: no further gain)
UNI_MIN_WARPS = int(__import__("os").environ.get("SF_UNI_MIN_WARPS", "4"))
_UNI_TOK = re.compile(r"\bU(\d+)\b|\bdsm \+ (\d+)\b|\ba\.p\[(\d+)\]")


def _stage_loops(loads: List[Tuple[int, int, int, int]]) -> List[str]:
    """cp.async staging of a uniform kernel's global operands: operands of
    one size whose pointer slots and shared offsets advance by fixed strides
    (a traced loop's per-layer weights) are staged by one loop over the slots
    (each line contains "int q": it is a load, see _generate)."""
    by_class: Dict[Tuple[int, int], List[Tuple[int, int]]] = {}
    for k, off, nb, w in loads:
        by_class.setdefault((nb, w), []).append((k, off))
    out = []
    for (nb, w), items in by_class.items():
        i = 0
        while i < len(items):
            m = 1
            if i + 1 < len(items):
                dk = items[i + 1][0] - items[i][0]
                do = items[i + 1][1] - items[i][1]
                while (i + m < len(items) and items[i + m][0] == items[i][0] + dk * m
                       and items[i + m][1] == items[i][1] + do * m):
                    m += 1
            k0, o0 = items[i]
            if m < 3:
                m, dk, do = 1, 0, 0
            # one flattened loop over (operand, 16-byte chunk): independent
            # iterations, so the CTA keeps many copies in flight
            g = 16 if nb % 16 == 0 else w
            ch = nb // g
            out.append(f"  for (int q = threadIdx.x; q < {m * ch}; q += blockDim.x) {{ "
                       f"const int t = q / {ch}, c = q - t * {ch}; "
                       f"sf::stage_chunk<{g}, {w}>(dsm + {o0} + {do} * t + {g} * c, "
                       f"(const unsigned char*)a.p[{k0} + {dk} * t] + {g} * c); }}")
            i += m
    return out


def _uni_canon(code: str, offs) -> Tuple[str, List[int]]:
    """(template, values): the uniform pool arrays U<id>, staged-operand
    offsets `dsm + N` and pointer slots `a.p[k]` of a level's code replaced by
    numbered holes; values[k] fills hole k (U arrays become pool byte
    offsets, tagged by element type in the template)."""
    vals: List[int] = []
    out = []
    last = 0
    for mt in _UNI_TOK.finditer(code):
        out.append(code[last:mt.start()])
        k = len(vals)
        if mt.group(1) is not None:
            off, ct = offs[int(mt.group(1))]
            vals.append(off)
            out.append(f"(({ct}*)(upool + @{k}@))")
        elif mt.group(2) is not None:
            vals.append(int(mt.group(2)))
            out.append(f"dsm + @{k}@")
        else:
            vals.append(int(mt.group(3)))
            out.append(f"a.p[@P{k}@]")
        last = mt.end()
    out.append(code[last:])
    return "".join(out), vals


def _uni_arith(canon, i: int, m: int) -> bool:
    """Levels i .. i+m-1: every hole's value advances by a fixed stride
    (pointer slots must stay fixed: the parameter array is not indexed at
    run time)."""
    t0 = canon[i][0]
    v0, v1 = canon[i][1], canon[i + 1][1]
    if len(v0) != len(v1):
        return False
    d = [b - a for a, b in zip(v0, v1)]
    for k in range(len(v0)):
        if f"@P{k}@" in t0 and d[k] != 0:
            return False
    for q in range(m):
        vq = canon[i + q][1]
        if len(vq) != len(v0) or any(vq[k] != v0[k] + d[k] * q for k in range(len(v0))):
            return False
    return True


def _uni_fill(text: str, vals: List[str]) -> str:
    for k in range(len(vals) - 1, -1, -1):
        text = text.replace(f"@P{k}@", vals[k]).replace(f"@{k}@", vals[k])
    return text


def _uniform_smem(rp: RowProgram) -> int:
    """Shared memory a uniform kernel needs for its computed values."""
    return sum(o.nbytes for op in rp.ops for o in op.outs)


def _smem_bytes(rp: RowProgram, planner: RowPlanner) -> int:
    produced = {id(o) for op in rp.ops for o in op.outs}
    seen, total = set(), 0
    for op in rp.ops:
        for x in op.ins:
            r = x.root()
            if id(r) in produced or id(r) in seen:
                continue
            seen.add(id(r))
            if planner.layout_of(x)[0] == UNI and not (r.kind == "const" and r.imm is not None):
                total += r.nbytes
    return total


# ---------------------------------------------------------------------------
# code generation
# ---------------------------------------------------------------------------


class _Gen:
    def __init__(self, rp: RowProgram, planner: RowPlanner, needed: set):
        self.rp = rp
        self.P = planner
        self.needed = needed
        flat = [b for op in rp.ops for b in (op.body if op.kind == "loop" else (op,))]
        self.produced = {id(o) for op in rp.ops for o in op.outs}
        self.produced |= {id(o) for op in flat for o in op.outs}
        self.ext: List[LV] = []          # root LVs in pointer order (inputs)
        self.ext_kind: List[str] = []    # "row" | "uni"
        self.ptr_of: Dict[int, int] = {}
        self.prologue: List[str] = []
        self.smem: List[str] = []
        self.body: List[str] = []
        self.rowed_names: Dict[int, List[str]] = {}
        self.uni_names: Dict[int, List[str]] = {}
        self.rng_ops: List[Tuple[LOp, int]] = []   # (op, count)
        self.rng_slot: Dict[int, int] = {}          # id(op) -> index in rng_ops
        self.scope_rows: set = set()  # rowed inputs declared in the current C++ scope
        self.outs: List[LV] = []
        self.tmp = 0
        # staged weights of rowed matvecs get a padded [K, Np] shared layout
        # (Np = N rounded up to one 16-byte vector) so a weight row is one or
        # a few vector loads: root id -> (N, Np)
        self.pad: Dict[int, Tuple[int, int]] = {}
        # root id -> (pool array name, stacked per loop iteration?) of staged operands
        self.smem_name: Dict[int, Tuple[str, bool]] = {}
        # row kernels: the shared-memory pool (array -> (byte offset, slice
        # elements, C type, element width)) and its size in bytes
        self.pool: Dict[str, Tuple[int, int, str, int]] = {}
        self.pool_size = 0
        # uniform kernel: staged global operands, CSE table, aliased results
        self.staged: Dict[int, str] = {}
        self.uni_smem = _uniform_smem(rp) if rp.uniform_only else 0
        self.dyn = 0  # dynamic shared memory of the uniform kernel (staged operands)
        self.dyn_loads: List[Tuple[int, int, int, int]] = []  # (slot, dsm offset, bytes, width)
        self.cse: Dict[tuple, LV] = {}
        self.alias: Dict[int, LV] = {}
        self.level: Dict[int, int] = {}
        self.uni_ops: List[Tuple[int, int, str, tuple]] = []  # (level, work, code, out shape)
        self.upool: List[Tuple[int, str, int, int]] = []  # (U id, ctype, elements, width)
        self.upool_offs: Dict[int, Tuple[int, str]] = {}
        self.uni_entry: Dict[int, int] = {}  # uniform op output id -> its uni_ops entry
        self.block = 128
        self.f2vars: set = set()  # names declared float2 (packed row pairs)
        self.cpool = CONST_POOL and not rp.uniform_only
        self.cp_entries: List[Tuple[int, int, int, int, int, int]] = []
        self.cp_arrays: Dict[str, tuple] = {}
        self.cp_first: Dict[str, int] = {}
        self.in_loop = False
        # chains per thread: replica k owns row r + 128 k of the CTA's 128 R
        # rows; the replicas' statements are emitted interleaved, op by op,
        # so they share every weight load and double the ILP
        self.R = 1 if rp.uniform_only else rp.replicas
        self.rep = 0
        self.rowv = ["r"] + [f"rq{k}" for k in range(1, self.R)]
        if not rp.uniform_only:
            seen: Dict[int, object] = {}
            widths: Dict[int, int] = {}
            for op in flat:
                if op.kind != "matmul" or planner.layout_of(op.outs[0])[0] != ROW:
                    continue
                b = op.ins[1]
                r = b.root()
                if planner.layout_of(b)[0] == ROW or id(r) in self.produced:
                    continue
                if (r.kind == "const" and r.imm is not None) or r.vals is not None:
                    continue  # literal weights: scalar FMAs with immediates
                n = b.shape[1]
                prev = seen.get(id(r))
                seen[id(r)] = n if prev in (None, n) else False
                widths[id(r)] = r.dtype.width
            for rid, n in seen.items():
                width = widths[rid]
                if n is False or width not in (4, 8):
                    continue
                vw = 16 // width
                # N dividing the vector: rows pack densely (one load spans rows)
                self.pad[rid] = (n, n if vw % n == 0 else -(-n // vw) * vw)

    @staticmethod
    def sfx(rep: int) -> str:
        return "" if rep == 0 else f"q{rep}"

    def _store(self, lines: List[str], o: LV, names_per_rep: List[List[str]]) -> None:
        """Stores of a needed rowed value (replica k > 0 only if its row exists)."""
        ct = _CTYPE[o.dtype]
        for rep, names in enumerate(names_per_rep):
            w = len(names)
            rv = self.rowv[rep]
            st = " ".join(f"(({ct}*)a.p[@O{o.id}@])[{rv if w == 1 else f'{rv} * {w} + {j}'}]"
                          f" = {nm};" for j, nm in enumerate(names))
            if rep > 0:
                st = f"if (v{rv}) {{ {st} }}"
            elif LOOP_SYNC and not self.rp.uniform_only and self.rp.teams is None:
                st = f"if (live) {{ {st} }}"
            lines.append(st)

    # -- operand access -------------------------------------------------------------
    def _input(self, x: LV) -> None:
        r = x.root()
        if id(r) in self.produced or (r.kind == "const" and r.imm is not None):
            return
        if (r.vals is not None and not self.rp.uniform_only
                and self.P.layout_of(x)[0] == UNI):
            return  # specialised immutable capture: read as literals (uni_elem)
        if id(r) in self.ptr_of:
            k = self.ptr_of[id(r)]
            if (self.P.layout_of(x)[0] == ROW and id(r) in self.rowed_names
                    and id(r) not in self.scope_rows):
                self._declare_row_input(r, k, self.P.layout_of(x)[1])  # a new team scope
                return
            if (self.P.layout_of(x)[0] == UNI and not self.rp.uniform_only
                    and id(r) not in self.uni_names):
                # slot taken by a loop's stacked operand; stage it on its own too
                pidx, _ = self._stage(r, f"s{k}", [k])
                self.uni_names[id(r)] = [self._lds(f"s{k}", p, False) for p in pidx]
                self.smem_name[id(r)] = (f"s{k}", False)
            return
        k = len(self.ext)
        self.ptr_of[id(r)] = k
        self.ext.append(r)
        L = self.P.layout_of(x)
        ct = _CTYPE[r.dtype]
        if L[0] == ROW:
            self.ext_kind.append(ROW)
            self._declare_row_input(r, k, L[1])
        elif self.rp.uniform_only:
            # uniform kernel: every global operand is put in flight at kernel
            # start (cp.async into shared memory), so the op loops that follow
            # never wait on a global load one after the other
            self.ext_kind.append(UNI)
            n = r.numel
            width = r.dtype.width
            off = -(-self.dyn // 16) * 16
            # static (result arrays) + dynamic shared memory <= 227 KB per CTA
            budget = min(UNIFORM_DYN_BYTES, 224 * 1024 - self.uni_smem)
            if width in (4, 8) and off + n * width <= budget:
                self.dyn = off + n * width
                self.staged[id(r)] = f"((const {ct}*)(dsm + {off}))"
                self.dyn_loads.append((k, off, n * width, width))
        else:
            self.ext_kind.append(UNI)
            pidx, _ = self._stage(r, f"s{k}", [k])
            self.uni_names[id(r)] = [self._lds(f"s{k}", p, False) for p in pidx]
            self.smem_name[id(r)] = (f"s{k}", False)

    def _declare_row_input(self, r: LV, k: int, w: int) -> None:
        ct = _CTYPE[r.dtype]
        per_rep = []
        for rep in range(self.R):
            names = [f"i{k}_{j}{self.sfx(rep)}" for j in range(w)]
            per_rep.append(names)
            rv = self.rowv[rep]
            self.body.append("    " + " ".join(
                f"const {ct} {nm} = ((const {ct}*)a.p[{k}])[{rv} * {w} + {j}];" if w > 1 else
                f"const {ct} {nm} = ((const {ct}*)a.p[{k}])[{rv}];"
                for j, nm in enumerate(names)))
        self.rowed_names[id(r)] = per_rep
        self.scope_rows.add(id(r))

    def _stage(self, r: LV, name: str, slots: List[int]):
        """Stage uniform operand(s) of r's shape into shared array ``name``
        (one slice per pointer slot, padded rows for matvec weights).
        Returns (padded index of each flat element, slice size)."""
        ct = _CTYPE[r.dtype]
        n = r.numel
        width = r.dtype.width
        if id(r) in self.pad:
            N, Np = self.pad[id(r)]
            off = f"(q / {N}) * {Np} + q % {N}"
            pidx = [(q // N) * Np + q % N for q in range(n)]
            size = (n // N) * Np
        else:
            off, pidx, size = "q", list(range(n)), n
        if width in (4, 8):
            vw = 16 // width  # slices start 16-byte aligned; vector reads stay inside
            size = -(-size // vw) * vw
        if self.cpool:
            # placed per use site by _fill (each op reading the array gets
            # its own copy, so no two loads share an address)
            N, Np = self.pad.get(id(r), (max(1, n), max(1, n)))
            self.pool[name] = (f"@P{name}@", size, ct, width)
            self.cp_arrays[name] = (list(slots), n, width, N, Np, size)
            return pidx, size
        # one pool per kernel: every array is a fixed byte offset from one base
        # register, so each load is LDS [base + immediate]
        pos = -(-self.pool_size // 16) * 16
        self.pool[name] = (pos, size, ct, width)
        self.pool_size = pos + max(1, size * len(slots)) * width
        head = (f"if (const int q = threadIdx.x; q < {n}) " if n <= self.rp.block else
                f"for (int q = threadIdx.x; q < {n}; q += blockDim.x) ")
        for i, k in enumerate(slots):
            dst = f"smem_pool + {pos + i * size * width} + {width} * ({off})"
            src_q = f"((const {ct}*)a.p[{k}])[q]"
            copy = (f"sf::cp_async<{width}>({dst}, &{src_q});" if width in (4, 8)
                    else f"*({ct}*)({dst}) = {src_q};")
            self.smem.append(f"  {head}{copy}")
        return pidx, size

    def _lds(self, name: str, index: int, stacked: bool) -> str:
        """Scalar load of element ``index`` of pool array ``name`` (of the
        current loop iteration's slice when stacked).  Constant-pool loads
        carry @DEP@ / @SITE@ placeholders, filled per use (_fill)."""
        pos, size, ct, width = self.pool[name]
        if self.cpool:
            fn = "sf::" + _CL[ct]
            if stacked:
                return f"{fn}s<{pos} + {index * width}, @SITE@>(it * {size * width})"
            return f"{fn}<{pos} + {index * width}, @SITE@>(@DEP@)"
        base = f"(sp + it * {size * width})" if stacked else "sp"
        return f"sf::ldp<{ct}, {pos + index * width}>({base})"

    def _lds_vec(self, name: str, index: int, stacked: bool) -> str:
        """16-byte vector load starting at element ``index`` (aligned)."""
        pos, size, ct, width = self.pool[name]
        if self.cpool:
            fn = "sf::clf4" if width == 4 else "sf::cld2"
            if stacked:
                return f"{fn}s<{pos} + {index * width}, @SITE@>(it * {size * width})"
            return f"{fn}<{pos} + {index * width}, @SITE@>(@DEP@)"
        base = f"(sp + it * {size * width})" if stacked else "sp"
        fn = "sf::ldp4" if width == 4 else "sf::ldp2"
        return f"{fn}<{pos + index * width}>({base})"

    def _place(self, name: str) -> int:
        """A fresh copy of pool array ``name`` for one use site; the plan
        gathers every copy before the launch.  Past CPOOL_BYTES the first
        copy is shared."""
        slots, n, width, N, Np, size = self.cp_arrays[name]
        nbytes = max(1, size * len(slots)) * width
        first = self.cp_first.get(name)
        if first is not None and self.pool_size + nbytes > CPOOL_BYTES:
            return first
        pos = -(-self.pool_size // 16) * 16
        self.pool_size = pos + nbytes
        for i, k in enumerate(slots):
            self.cp_entries.append((k, pos + i * size * width, n, width, N, Np))
        self.cp_first.setdefault(name, pos)
        return pos

    def _fill(self, line: str) -> str:
        """Constant-pool load placeholders: the loop counter as the dependency
        inside re-rolled loops (no hoisting), a unique site id per use (no
        merging of repeated loads into long-lived registers)."""
        if "@" not in line:
            return line
        line = line.replace("@DEP@", "it" if self.in_loop else "0")
        for name in dict.fromkeys(re.findall(r"@P(\w+)@", line)):
            line = line.replace(f"@P{name}@", str(self._place(name)))

        def site(_m):
            self.tmp += 1
            return str(self.tmp)

        return re.sub("@SITE@", site, line)

    def _ext_slot(self, r: LV, kind: str) -> int:
        """Pointer slot of an external root without staging it."""
        k = self.ptr_of.get(id(r))
        if k is None:
            k = len(self.ext)
            self.ptr_of[id(r)] = k
            self.ext.append(r)
            self.ext_kind.append(kind)
        return k

    def uni_elem(self, x: LV, flat: int) -> str:
        r = x.root()
        if r.kind == "const" and r.imm is not None:
            return c_literal(r.imm, r.dtype)
        if r.vals is not None and id(r) not in self.uni_names:
            return c_literal(r.vals[flat].item(), r.dtype)
        names = self.uni_names[id(r)]
        return names[flat]

    def uni_ref(self, x: LV, idx: str) -> str:
        """Uniform element at a run-time flat index (uniform-kernel loops)."""
        r = x.root()
        if r.kind == "const" and r.imm is not None:
            return c_literal(r.imm, r.dtype)
        if id(r) in self.ptr_of and id(r) not in self.produced:
            if id(r) in self.staged:
                return f"{self.staged[id(r)]}[{idx}]"
            k = self.ptr_of[id(r)]
            ct = _CTYPE[r.dtype]
            if ct == "bool":
                return f"((const bool*)a.p[{k}])[{idx}]"
            return f"__ldg((const {ct}*)a.p[{k}] + ({idx}))"
        return f"U{self.alias.get(id(r), r).id}[{idx}]"

    def _canon(self, x: LV) -> LV:
        r = x.root()
        return self.alias.get(id(r), r)

    def _cse_key(self, op: LOp):
        if op.kind not in ("ew", "matmul", "transpose", "eye", "reduce"):
            return None
        ins = []
        for x in op.ins:
            r = x.root()
            if r.kind == "const" and r.imm is not None:
                ins.append(("imm", repr(r.imm), r.dtype.value, tuple(x.shape)))
            else:
                ins.append((id(self._canon(x)), tuple(x.shape)))
        o = op.outs[0]
        return (op.kind, op.name, repr(sorted(op.attrs.items())), tuple(ins),
                o.dtype.value, tuple(o.shape))

    def _emit_uniform_loop(self, op: LOp) -> None:
        """Uniform op in the uniform kernel: a generated loop over the output
        elements run by one warp (lanes take consecutive elements), the result
        in shared memory.  Ops are grouped by dependency level; the ops of one
        level are spread over the CTA's warps and levels are separated by
        __syncthreads (see _uniform_prologue)."""
        from .lowering import _index_expr

        o = op.outs[0]
        ct = _CTYPE[o.dtype]
        n = o.numel
        # common subexpressions: a traced graph repeats chain-independent work
        # (the same weight transposes / embeddings at every leapfrog step);
        # within this one kernel launch a repeat aliases the first result
        key = self._cse_key(op)
        if key is not None:
            prev = self.cse.get(key)
            if prev is not None:
                self.alias[id(o)] = prev
                self.uni_names[id(o)] = self.uni_names[id(prev)]
                return
            self.cse[key] = o
        level = 1 + max((self.level.get(id(self._canon(x)), -1) for x in op.ins), default=-1)
        # an elementwise op whose newest operand is element-aligned with one
        # op of the previous level (same output shape, so the same lane
        # computes both elements) joins that op's loop: no barrier, no extra
        # level (a chain like C2's matmul -> add -> tanh is one level per
        # layer instead of three)
        fold = None
        if op.kind == "ew" and level > 0:
            top = [x for x in op.ins if self.level.get(id(self._canon(x)), -1) == level - 1]
            srcs = {id(self._canon(x)) for x in top}
            if len(srcs) == 1 and all(x.shape == o.shape for x in top):
                e = self.uni_entry.get(next(iter(srcs)))
                if e is not None and self.uni_ops[e][3] == o.shape:
                    fold = e
                    level -= 1
        self.level[id(o)] = level
        # computed uniform values live in one shared pool (placed by
        # _uniform_prologue), so re-rolled levels can address them by iteration
        self.upool.append((o.id, ct, max(1, n), o.dtype.width))
        self.uni_names[id(o)] = [f"U{o.id}[{q}]" for q in range(n)]
        k = op.kind
        shape = o.shape
        loop = f"  for (int f = lane; f < {n}; f += 32) {{ "
        if k == "ew":
            args = [self.uni_ref(x, _index_expr(x.shape, shape, "f") if x.numel != 1 else "0")
                    for x in op.ins]
            body = f"U{o.id}[f] = {ew_expr(op.name, args, ct)};"
        elif k == "matmul":
            a, b = op.ins
            m, kk_n = a.shape
            nn = b.shape[1]
            fma = "__fmaf_rn" if o.dtype is DType.float32 else "__fma_rn"
            body = (f"const int i = f / {nn}, j = f % {nn}; {ct} acc = ({ct})0; "
                    f"for (int k = 0; k < {kk_n}; ++k) acc = {fma}("
                    f"{self.uni_ref(a, f'i * {kk_n} + k')}, {self.uni_ref(b, f'k * {nn} + j')}, acc); "
                    f"U{o.id}[f] = acc;")
        elif k == "transpose":
            x = op.ins[0]
            rows, cols = x.shape
            body = (f"const int j = f / {rows}, i = f % {rows}; "
                    f"U{o.id}[f] = {self.uni_ref(x, f'i * {cols} + j')};")
        elif k == "eye":
            m = shape[0]
            body = f"U{o.id}[f] = ({ct})(f / {m} == f % {m} ? 1 : 0);"
        elif k == "reduce":
            x = op.ins[0]
            axes = tuple(op.attrs["axes"])
            xs = x.shape
            kept = [d for d in range(len(xs)) if d not in axes]
            red = [d for d in range(len(xs)) if d in axes]
            xst = _strides_for(xs, xs)
            count = dtypes.element_count([xs[d] for d in red])
            # offset of reduced element g (row-major over reduced dims) for output f
            terms, inner = [], 1
            for d in reversed(kept):
                terms.append(f"((f / {inner}) % {xs[d]}) * {xst[d]}")
                inner *= xs[d]
            inner = 1
            for d in reversed(red):
                terms.append(f"((g / {inner}) % {xs[d]}) * {xst[d]}")
                inner *= xs[d]
            off = " + ".join(terms) if terms else "0"
            p = min(count, 32)
            scale = f" / ({ct}){float(count)!r}" if op.name == "reduce_mean" else ""
            body = (f"{ct} acc[32]; "
                    f"for (int l = 0; l < {p}; ++l) {{ int g = l; acc[l] = {self.uni_ref(x, off)}; "
                    f"for (g = l + 32; g < {count}; g += 32) acc[l] = sf::add(acc[l], "
                    f"{self.uni_ref(x, off)}); }} "
                    f"for (int s = 16; s >= 1; s >>= 1) for (int l = 0; l < s; ++l) "
                    f"if (l + s < {p}) acc[l] = sf::add(acc[l], acc[l + s]); "
                    f"U{o.id}[f] = acc[0]{scale};")
        else:
            raise KernelError(f"uniform kernel: unsupported op {k}")
        work = n * (op.ins[0].shape[-1] if k == "matmul" else 1)
        if k == "reduce":
            work = op.ins[0].numel
        if fold is not None:
            lv, wk, code, shp = self.uni_ops[fold]
            # same loop: insert the body before the loop's closing brace
            self.uni_ops[fold] = (lv, wk + work, code[:-2] + " " + body + " }", shp)
            self.uni_entry[id(o)] = fold
            return
        self.uni_entry[id(o)] = len(self.uni_ops)
        self.uni_ops.append((level, work, loop + body + " }", shape))

    def _uniform_prologue(self) -> None:
        """Level-by-level schedule of the uniform ops over up to 32 warps.

        Computed values sit in one shared pool (`upool`).  Runs of at least
        UNI_REROLL_MIN consecutive levels whose code is identical up to pool
        offsets and staged-operand offsets that advance by a fixed stride (a
        traced loop's layers: C2's 100 x tanh(x W_i + b_i)) are emitted as
        one loop over the level index: each iteration executes exactly the
        straight-line level's statements at the same addresses, so results
        are unchanged, while the kernel's code shrinks ~m-fold (the
        straight-line C2 kernel was instruction-fetch bound: one warp
        walking ~100 KB of SASS once per call)."""
        self.smem += _stage_loops(self.dyn_loads)
        if not self.uni_ops:
            return
        offs: Dict[int, Tuple[int, str]] = {}
        pos = 0
        for uid, ct, n, width in self.upool:
            pos = -(-pos // 16) * 16
            offs[uid] = (pos, ct)
            pos += n * width
        if pos:
            self.smem.append(f"  __shared__ __align__(16) unsigned char upool[{pos}];")
        self.upool_offs = offs
        levels: Dict[int, List[Tuple[int, str]]] = {}
        for level, work, code, _shape in self.uni_ops:
            levels.setdefault(level, []).append((work, code))
        warps = max(1, min(32, max(len(v) for v in levels.values())))
        # extra warps only stage operands (more cp.async in flight)
        nw = max(warps, UNI_MIN_WARPS if self.dyn_loads else 1)
        self.block = 32 * nw
        blocks = []
        for level in sorted(levels):
            load = [0] * warps
            assign: List[List[str]] = [[] for _ in range(warps)]
            for work, code in sorted(levels[level], key=lambda wc: -wc[0]):
                w = load.index(min(load))
                load[w] += work + 32
                assign[w].append(code)
            parts = []
            for w, codes in enumerate(assign):
                if codes:
                    cond = "" if nw == 1 else f"if (warp == {w}) "
                    parts.append(f"  {cond}{{\n  " + "\n  ".join(codes) + "\n  }")
            blocks.append("\n".join(parts))
        canon = [_uni_canon(b, offs) for b in blocks]
        out = ["  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;"]
        i = 0
        while i < len(blocks):
            m = 1
            while (i + m < len(blocks) and canon[i + m][0] == canon[i][0]
                   and _uni_arith(canon, i, m + 1)):
                m += 1
            last = i + m == len(blocks)
            if UNI_REROLL and m >= UNI_REROLL_MIN:
                text, vals = canon[i]
                d = [b - a for a, b in zip(vals, canon[i + 1][1])]
                body = _uni_fill(text, [f"({v} + {dv} * it)" if dv else str(v)
                                        for v, dv in zip(vals, d)])
                out.append(f"#pragma unroll 1\n  for (int it = 0; it < {m}; ++it) {{\n{body}"
                           "\n  __syncthreads();\n  }")
            else:
                for q in range(i, i + m):
                    out.append(_uni_fill(canon[q][0], [str(v) for v in canon[q][1]]))
                    if q + 1 < len(blocks):
                        out.append("  __syncthreads();")
            i += m
            del last
        self.prologue = out

    def row_elem(self, x: LV, j: int, out_w: int, out_rank: int) -> str:
        """Element of operand x for output column j of a rowed op."""
        r = x.root()
        if r.kind == "const" and r.imm is not None:
            return c_literal(r.imm, r.dtype)
        L = self.P.layout_of(x)
        if L[0] == ROW:
            names = self.rowed_names[id(r)][self.rep]
            return names[0] if L[1] == 1 else names[j]
        n = x.numel
        if n == 1:
            return self.uni_elem(x, 0)
        return self.uni_elem(x, j)

    # -- emission ---------------------------------------------------------------------
    def _emit_ops(self, ops) -> None:
        for op in ops:
            if op.kind == "loop":
                self._emit_loop(op)
                continue
            for x in op.ins:
                self._input(x)
            L = self.P.layout_of(op.outs[0])
            if L[0] == UNI:
                if not self.rp.uniform_only:
                    raise KernelError("row program: uniform ops belong in the uniform kernel")
                self._emit_uniform_loop(op)
            else:
                self._emit_rowed(op, L)
                self._maybe_sync(op)

    def _maybe_sync(self, op) -> None:
        """With LOOP_SYNC: a CTA barrier after about SYNC_EVERY scalar ops of
        straight-line (or loop-body) code."""
        if not LOOP_SYNC or SYNC_EVERY <= 0 or self.rp.uniform_only or self.rp.teams is not None:
            return
        self.since_sync = getattr(self, "since_sync", 0) + _op_cost(op, self.P)
        if self.since_sync >= SYNC_EVERY:
            self.since_sync = 0
            self.body.append("    __syncthreads();")

    def _emit_teams(self) -> None:
        """Team 0 / team 1 bodies and the join body (see find_teams): team 0
        hands its values to the join in registers (tk*), team 1 through
        shared memory (xf*, one slot per chain of the CTA)."""
        t0, t1, join, x0, x1 = self.rp.teams
        # Philox counter ranges are reserved in program order (as the eager
        # draws consume them), not in the teams' emission order
        for op in self.rp.ops:
            for b in (op.body if op.kind == "loop" else (op,)):
                if b.kind == "rng" and id(b) not in self.rng_slot:
                    self.rng_ops.append((b, b.outs[0].numel))
                    self.rng_slot[id(b)] = len(self.rng_ops) - 1
        self.team_decls: List[str] = []
        bodies = []
        for t, (ops, xfer) in enumerate(((t0, x0), (t1, x1))):
            self.body, self.scope_rows = [], set()
            self._emit_ops(ops)
            for lv in xfer:
                ct = _CTYPE[lv.dtype]
                for j, nm in enumerate(self.rowed_names[id(lv)][0]):
                    if t == 0:
                        self.team_decls.append(f"  {ct} tk{lv.id}_{j};")
                        self.body.append(f"    tk{lv.id}_{j} = {nm};")
                    else:
                        self.team_decls.append(
                            f"  __shared__ {ct} xf{lv.id}_{j}[{self.rp.team_width}];")
                        self.body.append(f"    xf{lv.id}_{j}[lid] = {nm};")
            bodies.append(self.body)
        self.body, self.scope_rows = [], set()
        for t, xfer in enumerate((x0, x1)):
            for lv in xfer:
                ct = _CTYPE[lv.dtype]
                names = []
                for j in range(len(self.rowed_names[id(lv)][0])):
                    nm = f"j{lv.id}_{j}"
                    src = f"tk{lv.id}_{j}" if t == 0 else f"xf{lv.id}_{j}[lid]"
                    self.body.append(f"    const {ct} {nm} = {src};")
                    names.append(nm)
                self.rowed_names[id(lv)] = [names]
        self._emit_ops(join)
        self.team_bodies = (bodies[0], bodies[1], self.body)
        self.body = []

    def emit(self) -> None:
        if self.rp.teams is not None and not self.rp.uniform_only and self.R == 1:
            self._emit_teams()
        else:
            self.rp.teams = None
            self._emit_ops(self.rp.ops)
        if self.rp.uniform_only:
            self._uniform_prologue()
        for op in self.rp.ops:
            for o in op.outs:
                if id(o) in self.needed:
                    self.outs.append(o)

    def _emit_loop(self, lp: LoopOp) -> None:
        """for (it = 0; it < m; ++it) { body } with carried/exported registers."""
        stacked_ids = {id(r) for _, roots in lp.stacked for r in roots}
        for x in lp.ins:
            if id(x) not in stacked_ids:
                self._input(x)
        for syn, roots in lp.stacked:
            name = f"S{syn.id}"
            slots = [self._ext_slot(r, UNI) for r in roots]
            pidx, size = self._stage(syn, name, slots)
            self.uni_names[id(syn)] = [self._lds(name, p, True) for p in pidx]
            self.smem_name[id(syn)] = (name, True)
        pre = []
        for syn, init, _src in lp.carried:
            _, w, rank = self.P.layout_of(syn)
            ct = _CTYPE[syn.dtype]
            per_rep = []
            for rep in range(self.R):
                self.rep = rep
                names = [f"c{syn.id}_{j}{self.sfx(rep)}" for j in range(w)]
                pre.append(" ".join(f"{ct} {nm} = {self.row_elem(init, j, w, rank)};"
                                    for j, nm in enumerate(names)))
                per_rep.append(names)
            self.rep = 0
            self.rowed_names[id(syn)] = per_rep
        exp_names = []
        for e, _b in lp.exports:
            _, w, _rank = self.P.layout_of(e)
            ct = _CTYPE[e.dtype]
            per_rep = [[f"e{e.id}_{j}{self.sfx(rep)}" for j in range(w)] for rep in range(self.R)]
            pre.append(" ".join(f"{ct} {nm} = ({ct})0;" for names in per_rep for nm in names))
            exp_names.append(per_rep)
        pre.append(f"#pragma unroll 1\n    for (int it = 0; it < {lp.m}; ++it) {{")
        if LOOP_SYNC and self.rp.teams is None:
            pre.append("__syncthreads();")
        self.body.append(self._fill("    " + "\n    ".join(pre)))
        self.in_loop = True
        self.since_sync = 0
        for op in lp.body:
            self._emit_rowed(op, self.P.layout_of(op.outs[0]))
            self._maybe_sync(op)
        self.since_sync = 0
        self.in_loop = False
        post = []
        for (e, b), per_rep in zip(lp.exports, exp_names):
            for names, src in zip(per_rep, self.rowed_names[id(b)]):
                post.append(" ".join(f"{nm} = {s};" for nm, s in zip(names, src)))
        for syn, _init, b in lp.carried:
            for names, src in zip(self.rowed_names[id(syn)], self.rowed_names[id(b)]):
                post.append(" ".join(f"{nm} = {s};" for nm, s in zip(names, src)))
        post.append("}")
        for (e, _b), per_rep in zip(lp.exports, exp_names):
            self.rowed_names[id(e)] = per_rep
            if id(e) in self.needed:
                self._store(post, e, per_rep)
        self.body.append("    " + "\n    ".join(post))

    def _new_tmp(self) -> str:
        self.tmp += 1
        return f"t{self.tmp}"

    def _cro(self, elems: List[str], ct: str, sink: List[str]) -> str:
        """Canonical reduction order over elems (see sf_ops.cuh)."""
        n = len(elems)
        if n == 0:
            return f"({ct})0"
        acc = []
        for lane in range(min(32, n)):
            nm = self._new_tmp()
            expr = elems[lane]
            k = lane + 32
            while k < n:
                expr = f"sf::add({expr}, {elems[k]})" if ct != "int" else f"sf::add({expr}, {elems[k]})"
                k += 32
            sink.append(f"{ct} {nm} = {expr};")
            acc.append(nm)
        p = len(acc)
        off = 16
        while off >= 1:
            for lane in range(off):
                if lane + off < p:
                    sink.append(f"{acc[lane]} = sf::add({acc[lane]}, {acc[lane + off]});")
            off //= 2
        return acc[0]

    def _vector_operands(self, op: LOp, w: int, lines: List[str]) -> Dict[int, List[str]]:
        """A row-wide uniform operand of an elementwise op (a bias, a scale
        vector) read with 16-byte vector loads instead of one load per
        element: operand index -> element expressions."""
        out: Dict[int, List[str]] = {}
        if w < 2:
            return out
        for q, x in enumerate(op.ins):
            r = x.root()
            if (self.P.layout_of(x)[0] != UNI or x.numel != w or r.numel != w
                    or id(r) not in self.smem_name or id(r) in self.pad
                    or r.dtype.width not in (4, 8)):
                continue
            name, stacked = self.smem_name[id(r)]
            vw = 16 // r.dtype.width
            vt = "float4" if vw == 4 else "double2"
            elems = []
            for g in range(0, w, vw):
                t = self._new_tmp()
                lines.append(f"const {vt} {t} = {self._lds_vec(name, g, stacked)};")
                elems += [f"{t}.{c}" for c in "xyzw"[:min(vw, w - g)]]
            out[q] = elems
        return out

    def _pair(self, e0: str, e1: str, lines: List[str]) -> str:
        """float2 operand from two element expressions: a packed variable's
        own pair, a scalar broadcast, or a fresh make_float2."""
        if e0.endswith(".x") and e1.endswith(".y") and e0[:-2] == e1[:-2] \
                and e0[:-2] in self.f2vars:
            return e0[:-2]
        if e0 == e1:
            if "(" in e0 and not e0.startswith("__int_as_float("):
                t = self._new_tmp()  # a shared-memory load: issue it once
                lines.append(f"const float {t} = {e0};")
                e0 = t
            return f"make_float2({e0}, {e0})"
        return f"make_float2({e0}, {e1})"

    def _emit_rowed(self, op: LOp, L) -> None:
        _, w, rank = L
        o = op.outs[0]
        ct = _CTYPE[o.dtype]
        base = f"r{o.id}"
        per_rep = [[f"{base}_{j}{self.sfx(rep)}" for j in range(w)] for rep in range(self.R)]
        self.rowed_names[id(o)] = per_rep
        lines = []
        k = op.kind
        xpack = PACK and self.R == 2 and o.dtype is DType.float32
        if k == "ew" and xpack and op.name in _PACKED:
            # two chains per thread: element j of both chains in one float2
            vec = self._vector_operands(op, w, lines)
            fn = _PACKED[op.name]
            for j in range(w):
                args = []
                for rep in range(2):
                    self.rep = rep
                    args.append([vec[q][j] if q in vec else self.row_elem(x, j, w, rank)
                                 for q, x in enumerate(op.ins)])
                pn = f"{base}_{j}x"
                ops2 = [self._pair(a0, a1, lines) for a0, a1 in zip(args[0], args[1])]
                lines.append(f"const float2 {pn} = {fn}({ops2[0]}, {ops2[1]});")
                self.f2vars.add(pn)
                per_rep[0][j], per_rep[1][j] = pn + ".x", pn + ".y"
        elif k == "ew" and PACK and op.name in _PACKED and o.dtype is DType.float32 and w >= 2:
            vec = self._vector_operands(op, w, lines)
            fn = _PACKED[op.name]
            for rep in range(self.R):
                self.rep = rep
                names = per_rep[rep]
                for j in range(w):
                    args = [vec[q][j] if q in vec else self.row_elem(x, j, w, rank)
                            for q, x in enumerate(op.ins)]
                    if j % 2 == 0 and j + 1 < w:
                        args1 = [vec[q][j + 1] if q in vec else self.row_elem(x, j + 1, w, rank)
                                 for q, x in enumerate(op.ins)]
                        pn = f"{base}_p{j // 2}{self.sfx(rep)}"
                        ops2 = [self._pair(a0, a1, lines) for a0, a1 in zip(args, args1)]
                        lines.append(f"const float2 {pn} = {fn}({ops2[0]}, {ops2[1]});")
                        self.f2vars.add(pn)
                        names[j], names[j + 1] = pn + ".x", pn + ".y"
                    elif j % 2 == 0:
                        lines.append(f"const {ct} {names[j]} = {ew_expr(op.name, args, ct)};")
        elif k == "ew":
            vec = self._vector_operands(op, w, lines)
            for j in range(w):
                for rep in range(self.R):
                    self.rep = rep
                    args = [vec[q][j] if q in vec else self.row_elem(x, j, w, rank)
                            for q, x in enumerate(op.ins)]
                    lines.append(f"const {ct} {per_rep[rep][j]} = {ew_expr(op.name, args, ct)};")
        elif k == "matmul":
            a, b = op.ins
            kk_n = a.shape[1]
            n = b.shape[1]
            fma = "__fmaf_rn" if o.dtype is DType.float32 else "__fma_rn"
            xs_rep = []
            for rep in range(self.R):
                self.rep = rep
                xs_rep.append([self.row_elem(a, kk, kk_n, 2) for kk in range(kk_n)])
            # compiler-only memory fence: keeps NVVM from merging this matvec's
            # weight loads with other uses of the same weights (which would pin
            # hundreds of weights in registers for the whole chunk)
            lines.append('asm volatile("" ::: "memory");')
            br = b.root()
            if id(br) in self.pad:
                # k-outer: weight row k arrives in 16-byte vector loads and the
                # n accumulators advance together (same sequential-k FMA chain
                # per output as the nested form / the eager kernel)
                N, Np = self.pad[id(br)]
                sname, stacked = self.smem_name[id(br)]
                vw = 16 // br.dtype.width
                vt = "float4" if vw == 4 else "double2"
                comp = "xyzw"
                # packed accumulators: output pairs (c, c + 1) whose weights
                # sit in one vector's .xy or .zw for every k
                pk = (PACK and o.dtype is DType.float32 and not xpack and
                      all(((kk * Np + c) % vw) % 2 == 0 for kk in range(kk_n)
                          for c in range(0, n - 1, 2)))
                npair = n // 2 if pk else 0
                if xpack:
                    # two chains per thread: output c of both chains in one
                    # float2, the weight broadcast to both halves
                    lines.append(" ".join(f"float2 {base}_{c}x = make_float2(0.0f, 0.0f);"
                                          for c in range(n)))
                    self.f2vars.update(f"{base}_{c}x" for c in range(n))
                for rep in range(self.R if not xpack else 0):
                    names = per_rep[rep]
                    decl = []
                    for c in range(n):
                        if c < 2 * npair:
                            if c % 2 == 0:
                                pn = f"{base}_p{c // 2}{self.sfx(rep)}"
                                self.f2vars.add(pn)
                                decl.append(f"float2 {pn} = make_float2(0.0f, 0.0f);")
                        else:
                            decl.append(f"{ct} {names[c]} = ({ct})0;")
                    lines.append(" ".join(decl))
                # weight vectors in first-use order, issued PREFETCH vectors
                # ahead of the FMAs that consume them (volatile loads keep
                # program order, so this is the issue order)
                order: List[int] = []
                for kk in range(kk_n):
                    for c in range(n):
                        v = (kk * Np + c) // vw
                        if not order or order[-1] != v:
                            if v not in order:
                                order.append(v)
                vecs: Dict[int, str] = {}
                issued = 0

                def issue_upto(limit, stmt):
                    nonlocal issued
                    while issued < min(limit, len(order)):
                        v = order[issued]
                        t = self._new_tmp()
                        stmt.append(f"const {vt} {t} = {self._lds_vec(sname, v * vw, stacked)};")
                        vecs[v] = t
                        issued += 1

                for kk in range(kk_n):
                    stmt = []
                    for c in range(n):
                        f = kk * Np + c
                        v = f // vw
                        issue_upto(order.index(v) + 1 + PREFETCH, stmt)
                        if xpack:
                            xp = self._pair(xs_rep[0][kk], xs_rep[1][kk], stmt)
                            wv = f"{vecs[v]}.{comp[f % vw]}"
                            stmt.append(f"{base}_{c}x = sf::fma2({xp}, make_float2({wv}, {wv}), "
                                        f"{base}_{c}x);")
                            continue
                        if c < 2 * npair:
                            if c % 2:
                                continue
                            for rep in range(self.R):
                                pn = f"{base}_p{c // 2}{self.sfx(rep)}"
                                x = xs_rep[rep][kk]
                                stmt.append(f"{pn} = sf::fma2(make_float2({x}, {x}), make_float2("
                                            f"{vecs[v]}.{comp[f % vw]}, {vecs[v]}.{comp[f % vw + 1]}"
                                            f"), {pn});")
                            continue
                        for rep in range(self.R):
                            nm = per_rep[rep][c]
                            stmt.append(f"{nm} = {fma}({xs_rep[rep][kk]}, "
                                        f"{vecs[v]}.{comp[f % vw]}, {nm});")
                    lines.append(" ".join(stmt))
                for rep in range(self.R):
                    for c in range(2 * npair):
                        per_rep[rep][c] = f"{base}_p{c // 2}{self.sfx(rep)}.{'xy'[c % 2]}"
                    if xpack:
                        for c in range(n):
                            per_rep[rep][c] = f"{base}_{c}x.{'xy'[rep]}"
            elif xpack:
                # two chains per thread, weights specialised as literals:
                # output j of both chains in one float2, FFMA2 with the weight
                # as a broadcast immediate (one instruction per weight for two
                # chains; the same sequential-k FMA chain per lane)
                xps = [self._pair(xs_rep[0][kk], xs_rep[1][kk], lines) for kk in range(kk_n)]
                for j in range(n):
                    acc = "make_float2(0.0f, 0.0f)"
                    for kk in range(kk_n):
                        wv = self._pair(self.uni_elem(b, kk * n + j), self.uni_elem(b, kk * n + j),
                                        lines)
                        acc = f"sf::fma2({xps[kk]}, {wv}, {acc})"
                    pn = f"{base}_{j}x"
                    lines.append(f"const float2 {pn} = {acc};")
                    self.f2vars.add(pn)
                    per_rep[0][j], per_rep[1][j] = pn + ".x", pn + ".y"
            else:
                for j in range(n):
                    for rep in range(self.R):
                        acc = f"({ct})0"
                        for kk in range(kk_n):
                            acc = f"{fma}({xs_rep[rep][kk]}, {self.uni_elem(b, kk * n + j)}, {acc})"
                        lines.append(f"const {ct} {per_rep[rep][j]} = {acc};")
        elif k == "reduce":
            x = op.ins[0]
            xw = self.P.layout_of(x)[1]
            for rep in range(self.R):
                self.rep = rep
                elems = [self.row_elem(x, j, xw, 2) for j in range(xw)]
                red = self._cro(elems, ct, lines)
                nm = per_rep[rep][0]
                if op.name == "reduce_mean":
                    lines.append(f"const {ct} {nm} = {red} / ({ct}){float(xw)!r};")
                else:
                    lines.append(f"const {ct} {nm} = {red};")
        elif k == "rng":
            slot = self.rng_slot.get(id(op))
            if slot is None:  # (a draw recomputed by two teams uses the same counters)
                self.rng_ops.append((op, o.numel))
                slot = self.rng_slot[id(op)] = len(self.rng_ops) - 1
            for rep in range(self.R):
                rv = self.rowv[rep]
                for j in range(w):
                    ctr = f"(a.off[{slot}] + (unsigned long long){rv} * {w}ull + {j}ull)"
                    if op.attrs["kind"] == 0:
                        val = f"({ct})sf::normal_f64({ctr}, a.seed)"
                    else:
                        val = (f"sf::uniform_f32({ctr}, a.seed)" if o.dtype is DType.float32
                               else f"sf::uniform_f64({ctr}, a.seed)")
                    lines.append(f"const {ct} {per_rep[rep][j]} = {val};")
        else:
            raise KernelError(f"row program: unsupported rowed op {k}")
        self.rep = 0
        if id(o) in self.needed:
            # store right at the definition so the value's registers free up
            self._store(lines, o, per_rep)
        self.body.append(self._fill("    " + "\n    ".join(lines)))


def _unflatten(f: int, shape) -> List[int]:
    idx = []
    for d in reversed(shape):
        idx.append(f % d)
        f //= d
    return idx[::-1]


def generate_rowprog(rp: RowProgram, planner: RowPlanner, needed: set):
    """Returns (name, source, in_roots, out_lvs, rng_counts, n_ptr); cached on rp."""
    if rp.gen is None:
        rp.gen = _generate(rp, planner, needed)
    return rp.gen


# Row-kernel grid: "balanced" spreads the chains evenly over a grid that is a
# whole multiple of the SM count (each CTA gets ceil(batch / CTAs) chains, so
# every SM carries the same number of chains); "legacy" = 128 (64 per team)
# chains per CTA, whatever the remainder.  Measured on B200, L2HMC 1e5 chains:
# 782 legacy CTAs put 6 CTAs on 42 SMs and 5 on the rest (ncu: SM active
# cycles only 80% of elapsed).
# (B200, L2HMC 1e5 chains, device time per transition, warm L2: legacy
# 128-chain CTAs 137 us; balanced 256-thread CTAs 120 us; balanced with one
# 704-thread CTA per SM and LOOP_SYNC 108 us.)
ROW_GRID = __import__("os").environ.get("SF_ROW_GRID", "balanced")
# a CTA barrier at the top of every re-rolled loop iteration: keeps the
# CTA's warps within one loop body of each other (shared instruction fetch)
# (1e5 chains: 704-thread CTAs 119.7 -> 108 us; 256-thread 119.7 -> 112 us;
# extra barriers in straight-line code every 150-600 scalar ops: no gain)
LOOP_SYNC = __import__("os").environ.get("SF_ROW_LOOPSYNC", "1") == "1"
SYNC_EVERY = int(__import__("os").environ.get("SF_ROW_SYNC_EVERY", "0"))
# most threads per CTA of a balanced row kernel (704 = 22 warps: 1e5 chains
# as one CTA per SM at <= 93 registers per thread)
ROW_CTA_THREADS = int(__import__("os").environ.get("SF_ROW_CTA_THREADS", "704"))


def _geometry(rp: RowProgram, teams: bool) -> None:
    """Sets rp.rows_per_cta, rp.row_threads, rp.block, rp.team_width and
    rp.min_blocks (the launch bounds' CTAs per SM)."""
    rp.team_width = 0
    rp.min_blocks = 0
    if rp.uniform_only:
        rp.rows_per_cta = 128
        return
    R = rp.replicas
    b = rp.batch
    if teams:
        # small batches: 64 chains per CTA spreads the latency-bound chains
        # over as many SMs as possible
        rpc = 64
    elif ROW_GRID == "balanced" and b >= 32 * SM_COUNT * R:
        tmax = ROW_CTA_THREADS // R
        per_sm = -(-(-(-b // (tmax * R))) // SM_COUNT)
        rpc = -(-b // (SM_COUNT * per_sm))
    else:
        rpc = 128 * R
    per_sm = -(-(-(-b // rpc)) // SM_COUNT)
    rp.rows_per_cta = rpc
    rp.row_threads = -(-rpc // R)          # threads with a chain (replica 0's rows)
    width = 32 * -(-rp.row_threads // 32)  # threads per team (or per CTA)
    rp.block = 2 * width if teams else width
    if teams:
        rp.team_width = width
    # fit the whole batch in ONE wave when a register cap allows it (and
    # leaves ~80 registers per chain): with 1e5 chains in 128-chain CTAs,
    # 6 CTAs per SM need <= 80 registers (an 87-register kernel ran 5/SM
    # and spilled 42 CTAs into a second wave)
    if 2 <= per_sm <= 7 and rp.block * per_sm * 80 * R <= 65536:
        rp.min_blocks = per_sm


def _generate(rp: RowProgram, planner: RowPlanner, needed: set):
    _geometry(rp, rp.teams is not None and not rp.uniform_only and rp.replicas == 1)
    g = _Gen(rp, planner, needed)
    g.emit()
    stores = []
    k0 = len(g.ext)
    uni_stores = []
    for t, o in enumerate(g.outs):
        ct = _CTYPE[o.dtype]
        L = planner.layout_of(o)
        if L[0] == ROW:
            token = f"@O{o.id}@"
            g.body = [b.replace(token, str(k0 + t)) for b in g.body]
        else:
            n = o.numel
            src_arr = g.uni_names[id(o)][0].split("[")[0]
            uni_stores.append(f"for (int q = threadIdx.x; q < {n}; q += blockDim.x) "
                              f"(({ct}*)a.p[{k0 + t}])[q] = {src_arr}[q];")
    if rp.teams is not None:
        bodies = []
        for body in g.team_bodies:
            for t, o in enumerate(g.outs):
                body = [b.replace(f"@O{o.id}@", str(k0 + t)) for b in body]
            bodies.append(body)
        g.team_bodies = bodies
    n_ptr = k0 + len(g.outs)
    n_rng = max(1, len(g.rng_ops))
    if rp.uniform_only:
        rp.block = g.block
    mb = MIN_BLOCKS or (0 if rp.uniform_only else rp.min_blocks)
    bounds = str(rp.block) if rp.uniform_only or mb == 0 else f"{rp.block}, {mb}"
    src = [f"struct Params {{ void* p[{max(1, n_ptr)}]; long long rows; "
           f"unsigned long long seed; unsigned long long off[{n_rng}]; }};",
           f"extern \"C\" __global__ void __launch_bounds__({bounds}) KNAME(const "
           "__grid_constant__ Params a) {"]
    loads = [x for x in g.smem if "int q" in x]
    decls = [x for x in g.smem if "int q" not in x]
    if g.pool_size and g.cpool:
        # keep the pool symbol in the module (it is referenced only from asm)
        decls.append('  asm volatile("" :: "l"((const void*)cpool));')
    elif g.pool_size:
        decls.append(f"  __shared__ __align__(16) unsigned char smem_pool[{g.pool_size}];\n"
                     "  const unsigned sp = sf::saddr(smem_pool);")
    src += decls + loads
    if loads:
        src.append("  sf::cp_wait();\n  __syncthreads();")
    src += g.prologue
    if g.prologue:
        src.append("  __syncthreads();")
    if uni_stores:
        if g.upool_offs:
            uni_stores = [_uni_fill(t, [str(v) for v in vs])
                          for t, vs in (_uni_canon(x, g.upool_offs) for x in uni_stores)]
        src.append("  if (blockIdx.x == 0) {\n    " + "\n    ".join(uni_stores) + "\n  }")
    if rp.uniform_only:
        src.append("}\n")
        rp.dyn_smem = g.dyn
        if g.dyn:
            src.insert(2, "  extern __shared__ __align__(16) unsigned char dsm[];")
        core = "\n".join(src)
        name = "sf_uni_" + hashlib.sha1(core.encode()).hexdigest()[:16]
        source = '#include "sf_ops.cuh"\n' + core.replace("KNAME", name)
        return name, source, list(g.ext), list(g.outs), [c for _, c in g.rng_ops], n_ptr
    if rp.teams is not None:
        # two teams of two warps over the CTA's 64 chains (find_teams)
        tw, rpc = rp.team_width, rp.rows_per_cta
        src.append(f"  const int team = threadIdx.x >= {tw}, lid = threadIdx.x - team * {tw};")
        src.append(f"  const long long r = (long long)blockIdx.x * {rpc} + lid;")
        src.append(f"  const bool live = lid < {rpc} && r < a.rows;")
        src += g.team_decls
        src.append("  if (live && team == 0) {")
        src += g.team_bodies[0]
        src.append("  }\n  if (live && team == 1) {")
        src += g.team_bodies[1]
        src.append("  }\n  __syncthreads();\n  if (live && team == 0) {")
        src += g.team_bodies[2]
        src.append("  }\n}\n")
        core = "\n".join(src)
        name = "sf_rows_" + hashlib.sha1(core.encode()).hexdigest()[:16]
        source = '#include "sf_ops.cuh"\n' + core.replace("KNAME", name)
        return name, source, list(g.ext), list(g.outs), [c for _, c in g.rng_ops], n_ptr
    # R chains per thread (rows r + 128 k of the CTA's 128 R rows; a replica
    # past the end computes on the last row and does not store)
    # replica k of a thread owns row r + k T of its CTA's rows (T = threads
    # with a chain); a replica past the CTA's rows computes on row r and does
    # not store
    rpc, T = rp.rows_per_cta, rp.row_threads
    if LOOP_SYNC:
        # every thread reaches the per-iteration barriers: a thread without
        # a chain computes on its CTA's first row and does not store
        src.append(f"  const long long r0 = (long long)blockIdx.x * {rpc} + threadIdx.x;")
        src.append(f"  const bool live = threadIdx.x < {T} && r0 < a.rows;")
        src.append(f"  const long long r = live ? r0 : (long long)blockIdx.x * {rpc};")
    else:
        src.append(f"  const long long r = (long long)blockIdx.x * {rpc} + threadIdx.x;")
    if LOOP_SYNC:
        pass
    elif T < rp.block:
        src.append(f"  if (threadIdx.x >= {T} || r >= a.rows) return;")
    else:
        src.append("  if (r >= a.rows) return;")
    if g.R > 1:
        src.append(f"  const long long rend = min((long long)blockIdx.x * {rpc} + {rpc}, a.rows);")
    for k in range(1, g.R):
        src.append(f"  const bool vrq{k} = r + {T * k} < rend;")
        src.append(f"  const long long rq{k} = vrq{k} ? r + {T * k} : r;")
    src.append("  {")
    src += g.body
    if stores:
        src.append("    " + "\n    ".join(stores))
    src.append("  }\n}\n")
    head = ""
    rp.cpool = None
    if g.cpool and g.pool_size:
        size = -(-g.pool_size // 16) * 16
        head = ("#define SF_CPOOL 1\n"
                f"__constant__ __align__(16) unsigned char cpool[{size}];\n")
        rp.cpool = (size, list(g.cp_entries))
    core = head + "\n".join(src)
    name = "sf_rows_" + hashlib.sha1(core.encode()).hexdigest()[:16]
    source = head + '#include "sf_ops.cuh"\n' + "\n".join(src).replace("KNAME", name)
    return name, source, list(g.ext), list(g.outs), [c for _, c in g.rng_ops], n_ptr
