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
from typing import Dict, List, Optional, Tuple

from . import dtypes
from .dtypes import DType
from .errors import KernelError
from .lowering import LOp, LV, _CTYPE, _strides_for, c_literal, ew_expr

ROW_KINDS = frozenset(("ew", "matmul", "reduce", "transpose", "rng", "eye"))
MAX_UNIFORM_NUMEL = 1024       # uniform values computed per thread
MAX_MATVEC = 1024              # k*n of a row matmul
MAX_SMEM_BYTES = 40 * 1024     # uniform inputs staged in shared memory
MIN_BATCH = 2


class RowProgram:
    __slots__ = ("ops", "batch")

    def __init__(self, batch: int):
        self.ops: List[LOp] = []
        self.batch = batch


ROW, UNI, BAD = "row", "uni", "bad"


class RowPlanner:
    def __init__(self, batch: int):
        self.B = batch
        self.layout: Dict[int, Tuple] = {}

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


def plan_rows(ops: List[LOp]) -> List:
    """Split ops into RowPrograms (runs of row-local ops) and plain ops."""
    batch = choose_batch(ops)
    if batch < MIN_BATCH:
        return list(ops)
    planner = RowPlanner(batch)
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
            n_row = sum(1 for op in u.ops if planner.layout_of(op.outs[0])[0] == ROW)
            if n_row >= 2 and _smem_bytes(u, planner) <= MAX_SMEM_BYTES:
                out.append((u, planner))
                continue
            out.extend(u.ops)
        else:
            out.append(u)
    return out


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
        self.produced = {id(o) for op in rp.ops for o in op.outs}
        self.ext: List[LV] = []          # root LVs in pointer order (inputs)
        self.ext_kind: List[str] = []    # "row" | "uni"
        self.ptr_of: Dict[int, int] = {}
        self.prologue: List[str] = []
        self.smem: List[str] = []
        self.body: List[str] = []
        self.rowed_names: Dict[int, List[str]] = {}
        self.uni_names: Dict[int, List[str]] = {}
        self.rng_ops: List[Tuple[LOp, int]] = []   # (op, count)
        self.outs: List[LV] = []
        self.tmp = 0

    # -- operand access -------------------------------------------------------------
    def _input(self, x: LV) -> None:
        r = x.root()
        if id(r) in self.ptr_of or id(r) in self.produced:
            return
        if r.kind == "const" and r.imm is not None:
            return
        k = len(self.ext)
        self.ptr_of[id(r)] = k
        self.ext.append(r)
        L = self.P.layout_of(x)
        ct = _CTYPE[r.dtype]
        if L[0] == ROW:
            w = L[1]
            self.ext_kind.append(ROW)
            names = [f"i{k}_{j}" for j in range(w)]
            self.rowed_names[id(r)] = names
            idx = "r" if w == 1 else f"r * {w}"
            self.body.append("    " + " ".join(
                f"const {ct} {nm} = ((const {ct}*)a.p[{k}])[{idx} + {j}];" if w > 1 else
                f"const {ct} {nm} = ((const {ct}*)a.p[{k}])[r];" for j, nm in enumerate(names)))
        else:
            self.ext_kind.append(UNI)
            n = r.numel
            self.smem.append(f"  __shared__ {ct} s{k}[{max(1, n)}];\n"
                             f"  for (int q = threadIdx.x; q < {n}; q += blockDim.x) "
                             f"s{k}[q] = ((const {ct}*)a.p[{k}])[q];")
            self.uni_names[id(r)] = [f"s{k}[{q}]" for q in range(n)]

    def uni_elem(self, x: LV, flat: int) -> str:
        r = x.root()
        if r.kind == "const" and r.imm is not None:
            return c_literal(r.imm, r.dtype)
        names = self.uni_names[id(r)]
        return names[flat]

    def row_elem(self, x: LV, j: int, out_w: int, out_rank: int) -> str:
        """Element of operand x for output column j of a rowed op."""
        r = x.root()
        if r.kind == "const" and r.imm is not None:
            return c_literal(r.imm, r.dtype)
        L = self.P.layout_of(x)
        if L[0] == ROW:
            names = self.rowed_names[id(r)]
            return names[0] if L[1] == 1 else names[j]
        n = x.numel
        if n == 1:
            return self.uni_elem(x, 0)
        return self.uni_elem(x, j)

    # -- emission ---------------------------------------------------------------------
    def emit(self) -> None:
        for op in self.rp.ops:
            for x in op.ins:
                self._input(x)
            L = self.P.layout_of(op.outs[0])
            if L[0] == UNI:
                self._emit_uniform(op)
            else:
                self._emit_rowed(op, L)
        for op in self.rp.ops:
            for o in op.outs:
                if id(o) in self.needed:
                    self.outs.append(o)

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

    def _emit_rowed(self, op: LOp, L) -> None:
        _, w, rank = L
        o = op.outs[0]
        ct = _CTYPE[o.dtype]
        base = f"r{o.id}"
        names = [f"{base}_{j}" for j in range(w)]
        self.rowed_names[id(o)] = names
        lines = []
        k = op.kind
        if k == "ew":
            for j in range(w):
                args = [self.row_elem(x, j, w, rank) for x in op.ins]
                lines.append(f"const {ct} {names[j]} = {ew_expr(op.name, args, ct)};")
        elif k == "matmul":
            a, b = op.ins
            kk_n = a.shape[1]
            n = b.shape[1]
            fma = "__fmaf_rn" if o.dtype is DType.float32 else "__fma_rn"
            xs = [self.row_elem(a, kk, kk_n, 2) for kk in range(kk_n)]
            for j in range(n):
                acc = f"({ct})0"
                for kk in range(kk_n):
                    acc = f"{fma}({xs[kk]}, {self.uni_elem(b, kk * n + j)}, {acc})"
                lines.append(f"const {ct} {names[j]} = {acc};")
        elif k == "reduce":
            x = op.ins[0]
            xw = self.P.layout_of(x)[1]
            elems = [self.row_elem(x, j, xw, 2) for j in range(xw)]
            red = self._cro(elems, ct, lines)
            if op.name == "reduce_mean":
                lines.append(f"const {ct} {names[0]} = {red} / ({ct}){float(xw)!r};")
            else:
                lines.append(f"const {ct} {names[0]} = {red};")
        elif k == "rng":
            self.rng_ops.append((op, o.numel))
            slot = len(self.rng_ops) - 1
            for j in range(w):
                ctr = f"(a.off[{slot}] + (unsigned long long)r * {w}ull + {j}ull)"
                if op.attrs["kind"] == 0:
                    val = f"({ct})sf::normal_f64({ctr}, a.seed)"
                else:
                    val = (f"sf::uniform_f32({ctr}, a.seed)" if o.dtype is DType.float32
                           else f"sf::uniform_f64({ctr}, a.seed)")
                lines.append(f"const {ct} {names[j]} = {val};")
        else:
            raise KernelError(f"row program: unsupported rowed op {k}")
        self.body.append("    " + "\n    ".join(lines))

    def _emit_uniform(self, op: LOp) -> None:
        o = op.outs[0]
        ct = _CTYPE[o.dtype]
        n = o.numel
        names = [f"u{o.id}_{q}" for q in range(n)]
        self.uni_names[id(o)] = names
        lines = []
        k = op.kind
        shape = o.shape
        if k == "ew":
            strides = [(_strides_for(x.shape, shape) if x.numel != 1 else None) for x in op.ins]
            for f in range(n):
                idx = _unflatten(f, shape)
                args = []
                for x, st in zip(op.ins, strides):
                    src = 0 if st is None else sum(i * s for i, s in zip(idx, st))
                    args.append(self.uni_elem(x, src))
                lines.append(f"const {ct} {names[f]} = {ew_expr(op.name, args, ct)};")
        elif k == "matmul":
            a, b = op.ins
            m, kk_n = a.shape
            nn = b.shape[1]
            fma = "__fmaf_rn" if o.dtype is DType.float32 else "__fma_rn"
            for i in range(m):
                for j in range(nn):
                    acc = f"({ct})0"
                    for kk in range(kk_n):
                        acc = f"{fma}({self.uni_elem(a, i * kk_n + kk)}, {self.uni_elem(b, kk * nn + j)}, {acc})"
                    lines.append(f"const {ct} {names[i * nn + j]} = {acc};")
        elif k == "transpose":
            x = op.ins[0]
            rows, cols = x.shape
            for i in range(rows):
                for j in range(cols):
                    lines.append(f"const {ct} {names[j * rows + i]} = {self.uni_elem(x, i * cols + j)};")
        elif k == "eye":
            m = shape[0]
            for f in range(n):
                lines.append(f"const {ct} {names[f]} = ({ct}){1 if f // m == f % m else 0};")
        elif k == "reduce":
            x = op.ins[0]
            axes = tuple(op.attrs["axes"])
            xs = x.shape
            kept = [d for d in range(len(xs)) if d not in axes]
            red = [d for d in range(len(xs)) if d in axes]
            xst = _strides_for(xs, xs)
            for f in range(n):
                # output flat f -> kept coordinates
                kshape = [xs[d] for d in kept]
                kidx = _unflatten(f, kshape) if kshape else []
                rshape = [xs[d] for d in red]
                count = dtypes.element_count(rshape)
                elems = []
                for g in range(count):
                    ridx = _unflatten(g, rshape) if rshape else []
                    full = [0] * len(xs)
                    for d, v in zip(kept, kidx):
                        full[d] = v
                    for d, v in zip(red, ridx):
                        full[d] = v
                    elems.append(self.uni_elem(x, sum(i * s for i, s in zip(full, xst))))
                total = self._cro(elems, ct, lines)
                if op.name == "reduce_mean":
                    lines.append(f"const {ct} {names[f]} = {total} / ({ct}){float(count)!r};")
                else:
                    lines.append(f"const {ct} {names[f]} = {total};")
        else:
            raise KernelError(f"row program: unsupported uniform op {k}")
        self.prologue.append("  " + "\n  ".join(lines))


def _unflatten(f: int, shape) -> List[int]:
    idx = []
    for d in reversed(shape):
        idx.append(f % d)
        f //= d
    return idx[::-1]


def generate_rowprog(rp: RowProgram, planner: RowPlanner, needed: set):
    """Returns (name, source, in_roots, out_lvs, rng_counts)."""
    g = _Gen(rp, planner, needed)
    g.emit()
    stores = []
    k0 = len(g.ext)
    uni_stores = []
    for t, o in enumerate(g.outs):
        ct = _CTYPE[o.dtype]
        L = planner.layout_of(o)
        if L[0] == ROW:
            w = L[1]
            for j, nm in enumerate(g.rowed_names[id(o)]):
                idx = "r" if w == 1 else f"r * {w} + {j}"
                stores.append(f"(({ct}*)a.p[{k0 + t}])[{idx}] = {nm};")
        else:
            for q, nm in enumerate(g.uni_names[id(o)]):
                uni_stores.append(f"(({ct}*)a.p[{k0 + t}])[{q}] = {nm};")
    n_ptr = k0 + len(g.outs)
    n_rng = max(1, len(g.rng_ops))
    src = [f"struct Params {{ void* p[{max(1, n_ptr)}]; long long rows; "
           f"unsigned long long seed; unsigned long long off[{n_rng}]; }};",
           "extern \"C\" __global__ void __launch_bounds__(128) KNAME(const __grid_constant__ Params a) {"]
    src += g.smem
    if g.smem:
        src.append("  __syncthreads();")
    src += g.prologue
    if uni_stores:
        src.append("  if (blockIdx.x == 0 && threadIdx.x == 0) {\n    " +
                   "\n    ".join(uni_stores) + "\n  }")
    src.append("  const long long stride = (long long)gridDim.x * blockDim.x;")
    src.append("  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; "
               "r < a.rows; r += stride) {")
    src += g.body
    if stores:
        src.append("    " + "\n    ".join(stores))
    src.append("  }\n}\n")
    core = "\n".join(src)
    name = "sf_rows_" + hashlib.sha1(core.encode()).hexdigest()[:16]
    source = '#include "sf_ops.cuh"\n' + core.replace("KNAME", name)
    return name, source, list(g.ext), list(g.outs), [c for _, c in g.rng_ops], n_ptr
