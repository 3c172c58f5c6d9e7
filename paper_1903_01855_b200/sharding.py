"""Chain sharding below the trace cache.

The sampler graphs are row-separable: every op works on each chain's row on
its own (elementwise ops, ``rows @ weights`` matmuls, reductions along a
row), so a batch of B chains can be cut into contiguous shards that run
independently — on several GPUs of one process, or one after another on one
GPU — and concatenated, with every element computed by exactly the same
sequence of operations as in the unsharded run (bit-identical; the survey
measured the same property on the reference, §8(e)).

Sharding must not retrace: the reference's trace key holds the argument
shapes (stageflow/staging.py:258-264), so tracing per shard would change
the trace counts.  ``ShardedFunction`` therefore traces once through the
staged function's own cache at the full batch, then rewrites the traced
graph's batch extent B -> b (``rebatch``) and runs the rewritten graph per
shard through the normal executor (one compiled program per device and
shard size).  A graph that is not row-separable (a reduction or transpose
across chains, a per-chain constant baked into the graph) raises
``NotShardable``.  Random draws inside the graph take per-shard Philox
counter ranges, so a sampler that draws on the device matches its
unsharded run only statistically; with its draws passed in as inputs
(``L2HMCSampler(draws="inputs")``) it is bit-identical.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Set, Tuple

import numpy as np

from . import _native, dtypes
from .errors import StageflowError
from .graph import GraphFunction, Node, Placeholder
from .tensor import Tensor


class NotShardable(StageflowError):
    """The graph couples chains (or its batch dimension is ambiguous)."""


_EW_BUILTIN = frozenset(("add", "sub", "mul", "div", "neg", "exp", "log", "softplus", "relu",
                         "step_positive", "greater", "identity"))


def _is_elementwise(op: str) -> bool:
    if op in _EW_BUILTIN:
        return True
    from .ops import get_op_def

    try:
        low = get_op_def(op).lowering
    except StageflowError:
        return False
    return bool(low) and low[0] in ("ew", "cast")


def _rows(shape, b: int):
    return (b,) + tuple(shape[1:])


def rebatch(gf: GraphFunction, B: int, b: int, rowed_inputs: Set[int]) -> Tuple[GraphFunction,
                                                                                 List[bool]]:
    """``gf`` with its batch extent B replaced by b.  ``rowed_inputs``:
    placeholder indices whose leading dimension is the batch.  Returns the
    new graph and, per output, whether it is rowed (sharded) or uniform."""
    n_in = len(gf.inputs)
    rowed: Set[Tuple[int, int]] = set()
    inputs = []
    for i, ph in enumerate(gf.inputs):
        if i in rowed_inputs:
            if not ph.shape or ph.shape[0] != B:
                raise NotShardable(f"input {ph.name} has no batch dimension {B}")
            rowed.add((i, 0))
            inputs.append(Placeholder(ph.name, ph.dtype, _rows(ph.shape, b), ph.is_variable_ref))
        else:
            inputs.append(ph)

    def ambiguous_uniform(ref, out_rank) -> bool:
        dt, shape = gf.spec_of(ref)
        return len(shape) == out_rank and out_rank > 0 and shape[0] == B and B != 1

    nodes: List[Node] = []
    for j, node in enumerate(gf.nodes):
        vid = n_in + j
        op = node.op
        ins_rowed = [r in rowed for r in node.inputs]
        attrs = dict(node.attrs)
        out_rowed = False
        if op == "constant":
            t = node.attrs["value"]
            if t.shape and t.shape[0] == B and B != 1:
                flat = t.raw().reshape(-1)
                if flat.size and not np.all(flat == flat[0]):
                    raise NotShardable(f"node {j}: a per-chain constant is baked into the graph")
                arr = np.full(_rows(t.shape, b), flat[0] if flat.size else 0,
                              dtype=t.dtype.np_dtype)
                arr.flags.writeable = False
                attrs["value"] = Tensor(t.dtype, arr.shape, t.device, array=arr)
                out_rowed = True
        elif _is_elementwise(op):
            out_rowed = any(ins_rowed)
            if out_rowed:
                rank = len(node.out_specs[0][1])
                for r, rr in zip(node.inputs, ins_rowed):
                    if not rr and ambiguous_uniform(r, rank):
                        raise NotShardable(f"node {j} ({op}): a uniform operand spans the batch")
        elif op == "matmul":
            if ins_rowed[1]:
                raise NotShardable(f"node {j}: matmul with a per-chain right operand")
            out_rowed = ins_rowed[0]
        elif op in ("reduce_sum", "reduce_mean"):
            if ins_rowed[0]:
                rank = len(gf.spec_of(node.inputs[0])[1])
                axes = node.attrs.get("axes")
                axes = tuple(range(rank)) if axes is None else tuple(a % rank for a in axes)
                if 0 in axes:
                    raise NotShardable(f"node {j}: {op} across chains")
                out_rowed = True
        elif op in ("reshape", "broadcast_to"):
            target = tuple(node.attrs["shape"])
            if ins_rowed[0] or (op == "broadcast_to" and target and target[0] == B):
                if not target or target[0] != B:
                    raise NotShardable(f"node {j}: {op} moves the batch dimension")
                attrs["shape"] = _rows(target, b)
                out_rowed = True
        elif op in ("random_normal", "random_uniform"):
            shape = tuple(node.attrs["shape"])
            if shape and shape[0] == B and B != 1:
                attrs["shape"] = _rows(shape, b)
                out_rowed = True
        elif any(ins_rowed):
            raise NotShardable(f"node {j}: {op} is not row-separable")
        specs = node.out_specs
        if out_rowed:
            specs = tuple((dt, _rows(shape, b)) for dt, shape in specs)
            for k in range(len(specs)):
                rowed.add((vid, k))
        nodes.append(Node(op, node.inputs, attrs, node.device, specs))
    out = GraphFunction(f"{gf.name}__rows{b}", inputs, nodes, gf.outputs, gf.library)
    return out, [ref in rowed for _, ref in gf.outputs]


def _slice_rows(t: Tensor, lo: int, hi: int, dev: int, device) -> Tensor:
    row = t.nbytes // t.shape[0] if t.shape[0] else 0
    n = (hi - lo) * row
    buf = _native.alloc(dev, n)
    src = t._device_buffer()
    if n:
        if src.dev == dev:
            _native.copy_d2d(dev, buf.ptr, src.ptr + lo * row, n)
        else:
            _native.copy_p2p(dev, buf.ptr, src.dev, src.ptr + lo * row, n)
    return Tensor._adopt(t.dtype, (hi - lo,) + tuple(t.shape[1:]), device, buf)


def _to_device(t, dev: int, device):
    from .kernels import relabel

    return t if not isinstance(t, Tensor) or t.device == device else relabel(t, device)


def _concat_rows(parts: Sequence[Tensor], dev: int, device) -> Tensor:
    total = sum(p.shape[0] for p in parts)
    first = parts[0]
    row = first.nbytes // first.shape[0] if first.shape[0] else 0
    buf = _native.alloc(dev, total * row)
    off = 0
    for p in parts:
        n = p.nbytes
        if n:
            src = p._device_buffer()
            if src.dev == dev:
                _native.copy_d2d(dev, buf.ptr + off, src.ptr, n)
            else:
                _native.copy_p2p(dev, buf.ptr + off, src.dev, src.ptr, n)
        off += n
    return Tensor._adopt(first.dtype, (total,) + tuple(first.shape[1:]), device, buf)


class ShardedFunction:
    """Run a staged function with its batch cut into contiguous shards, one
    per entry of ``devices`` (device names; repeats run sequentially on the
    same GPU), tracing once at the full batch."""

    def __init__(self, staged, devices: Optional[Sequence] = None, shards: Optional[int] = None):
        from .runtime import get_runtime

        self.staged = staged
        rt = get_runtime()
        if devices is None:
            devices = [d.name for d in rt.devices]
            if shards is not None:
                devices = [devices[i % len(devices)] for i in range(shards)]
        self.devices = list(devices)
        self._graphs: Dict[Tuple[int, int, int], Tuple[GraphFunction, List[bool]]] = {}
        self._caps: Dict[Tuple[int, object], list] = {}

    def __call__(self, *args):
        from .executor import execute_graph
        from .kernels import KernelEnv
        from .runtime import get_runtime

        pf = self.staged
        bound = pf._bind(args, {})
        cf = pf._concrete_for(bound)  # one trace at the full batch
        explicit = [v for _, v, _ in bound if isinstance(v, Tensor)]
        if len(explicit) != len([v for _, v, _ in bound if v is not None and
                                 not isinstance(v, (int, float, str, bool))]):
            raise NotShardable("sharded calls take tensor arguments only")
        B = explicit[0].shape[0]
        rowed_inputs = {i for i, t in enumerate(explicit) if t.shape and t.shape[0] == B}
        G = len(self.devices)
        per = -(-B // G)
        ranges = [(lo, min(B, lo + per)) for lo in range(0, B, per)]
        rt = get_runtime()
        caps = cf.materialize_captured()
        results = []
        for g, (lo, hi) in enumerate(ranges):
            device = self.devices[g]
            dev = rt.ordinals[device]
            b = hi - lo
            key = (id(cf), b)
            entry = self._graphs.get(key)
            if entry is None:
                entry = self._graphs[key] = rebatch(cf.graph, B, b, rowed_inputs)
            gf_b, out_rowed = entry
            ck = (id(cf), device)
            caps_g = self._caps.get(ck)
            if caps_g is None:
                caps_g = self._caps[ck] = [_to_device(c, dev, device) for c in caps]
            ins = [(_slice_rows(t, lo, hi, dev, device) if i in rowed_inputs
                    else _to_device(t, dev, device)) for i, t in enumerate(explicit)]
            results.append(execute_graph(gf_b, ins + caps_g,
                                         KernelEnv(device=device, libraries=(gf_b.library,))))
        dev0 = rt.ordinals[self.devices[0]]
        outs = []
        for k, rowed in enumerate(out_rowed):
            if rowed:
                outs.append(_concat_rows([r[k] for r in results], dev0, self.devices[0]))
            else:
                outs.append(results[0][k])
        return cf.unpack(outs)


def shard(staged, devices: Optional[Sequence] = None, shards: Optional[int] = None):
    """``ShardedFunction(staged, devices, shards)``."""
    return ShardedFunction(staged, devices, shards)
