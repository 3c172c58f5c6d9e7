"""Host logic of the row-program compiler (paper_1903_01855_b200/rowfuse.py):
loop re-rolling of repeated op blocks and the generated source (compiled with
NVRTC, which needs no GPU)."""
import numpy as np
import pytest

from paper_1903_01855_b200 import _native, rowfuse
from paper_1903_01855_b200.dtypes import DType
from paper_1903_01855_b200.lowering import LOp, LV

B = 64


class _Prog:
    def __init__(self):
        self.n = 0
        self.ops = []

    def lv(self, shape, kind="op"):
        self.n += 1
        return LV(self.n, DType.float32, shape, kind)

    def op(self, kind, name, ins, shape):
        o = self.lv(shape)
        self.ops.append(LOp(kind, name, list(ins), [o]))
        o.producer = self.ops[-1]
        return o


def _steps(n_steps, per_step_weights=True, leak_mid=False):
    """x <- tanh(x @ W_i + b) * c, n_steps times (the shape of a traced leapfrog loop)."""
    P = _Prog()
    x0 = P.lv((B, 4), "input")
    b = P.lv((4,), "input")
    Ws = [P.lv((4, 4), "input") for _ in range(n_steps if per_step_weights else 1)]
    c = P.lv((1,), "const")
    c.imm = 0.5
    x = x0
    mids = []
    for i in range(n_steps):
        W = Ws[i] if per_step_weights else Ws[0]
        h = P.op("matmul", "matmul", [x, W], (B, 4))
        h = P.op("ew", "add", [h, b], (B, 4))
        h = P.op("ew", "tanh", [h], (B, 4))
        x = P.op("ew", "mul", [h, c], (B, 4))
        mids.append(x)
    keep = {id(x)}
    if leak_mid:
        keep.add(id(mids[1]))
    return P, keep, x


def test_reroll_finds_loop_with_carried_and_stacked_operands():
    P, keep, out = _steps(6)
    units = rowfuse.plan_rows(P.ops, keep)
    rows = [u for u in units if isinstance(u, tuple) and not u[0].uniform_only]
    loops = [op for rp, _ in rows for op in rp.ops if op.kind == "loop"]
    assert len(loops) == 1
    lp = loops[0]
    assert lp.m >= rowfuse.MIN_REPS and len(lp.body) == 4
    assert len(lp.carried) == 1 and len(lp.stacked) == 1
    assert [e for e, _ in lp.exports] == [out]


def test_reroll_shared_weights_are_not_stacked():
    P, keep, _ = _steps(5, per_step_weights=False)
    units = rowfuse.plan_rows(P.ops, keep)
    lp = [op for u in units if isinstance(u, tuple) for op in u[0].ops if op.kind == "loop"][0]
    assert lp.stacked == [] and lp.m == 5


def test_reroll_refuses_when_an_intermediate_step_escapes():
    # step 2's value is a graph output: only blocks after it may be rolled
    P, keep, _ = _steps(6, leak_mid=True)
    units = rowfuse.plan_rows(P.ops, keep)
    loops = [op for u in units if isinstance(u, tuple) for op in u[0].ops if op.kind == "loop"]
    for lp in loops:
        body_outs = {id(o) for op in lp.body for o in op.outs}
        assert all(id(v) not in body_outs for v in P.ops[7].outs)


def test_batch_equal_to_layer_width_keeps_weights_uniform():
    """4 chains through 4-wide layers: the (4, 4) weights read from variables
    have the batch's leading extent but are chain-independent — they must be
    uniform operands of one row program, not rows."""
    P = _Prog()
    x = P.lv((4, 4), "input")
    wv = P.lv((4, 4), "var")
    w = P.op("var_read", "var_read", [wv], (4, 4))
    wt = P.op("ew", "mul", [w, w], (4, 4))  # a weight transform: still uniform
    h = P.op("matmul", "matmul", [x, wt], (4, 4))
    y = P.op("ew", "tanh", [h], (4, 4))
    assert rowfuse.choose_batch(P.ops) == 4
    units = rowfuse.plan_rows(P.ops, {id(y)})
    rows = [u for u in units if isinstance(u, tuple) and not u[0].uniform_only]
    assert len(rows) == 1
    names = [op.name for op in rows[0][0].ops]
    assert "matmul" in names and "tanh" in names


def test_rerolled_program_generates_and_compiles():
    P, keep, out = _steps(6)
    units = rowfuse.plan_rows(P.ops, keep)
    for u in units:
        if isinstance(u, tuple):
            name, src = rowfuse.generate_rowprog(u[0], u[1], keep)[:2]
            if not u[0].uniform_only:
                assert "for (int it = 0; it <" in src
            _native.jit_compile(name, src)


def test_two_chains_per_thread_codegen(monkeypatch):
    """Replicated codegen (2 chains per thread) shares the weight loads and
    guards the second replica's stores."""
    monkeypatch.setattr(rowfuse, "ROW_REPLICAS", 2)
    P, keep, out = _steps(6)
    units = rowfuse.plan_rows(P.ops, keep)
    for u in units:
        if isinstance(u, tuple) and not u[0].uniform_only:
            assert u[0].replicas == 2
            name, src = rowfuse.generate_rowprog(u[0], u[1], keep)[:2]
            assert "rq1" in src and "if (vrq1)" in src
            _native.jit_compile(name, src)
