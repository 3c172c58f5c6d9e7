"""The SGF1 graph-function container (reference: stageflow/serial.py).

Byte-compatible with the reference's format, which makes ``serialize`` the
structure-parity probe: a graph traced by this backend and the same program
traced by the reference must serialize to identical bytes (constant
payloads included).  Layout (little-endian): ``SGF1`` | u32 version |
five length-prefixed sections — string table (id 0 = ""), inputs, nodes,
outputs, nested library (sorted by name).  Node output specs are not stored
and are re-inferred on load — here through the live op registry, so graphs
with registered plugin ops load too (the reference's global INFERENCE table
cannot, stageflow/serial.py:384-401).
"""
from __future__ import annotations

import struct
from typing import Dict, List, Tuple

import numpy as np

from .dtypes import DTYPE_TAGS, TAG_DTYPES, DType
from .errors import CorruptGraph, FormatVersionMismatch, NotSerializable
from .graph import GraphFunction, Node, Placeholder
from .tensor import Tensor, tensor_from_host

MAGIC = b"SGF1"
VERSION = 1
_VAR_BIT = 0x80
(T_INT, T_FLOAT, T_BOOL, T_STRING, T_DTYPE, T_SHAPE, T_FUNCTION, T_TENSOR, T_INT_LIST,
 T_NONE) = range(1, 11)


class _Out:
    def __init__(self):
        self.buf = bytearray()

    def put(self, fmt: str, *vals):
        self.buf += struct.pack("<" + fmt, *vals)

    def raw(self, b: bytes):
        self.buf += b


class _In:
    def __init__(self, data: bytes):
        self.data = data
        self.pos = 0

    def get(self, fmt: str):
        fmt = "<" + fmt
        try:
            vals = struct.unpack_from(fmt, self.data, self.pos)
        except struct.error:
            raise CorruptGraph("truncated container") from None
        self.pos += struct.calcsize(fmt)
        return vals[0] if len(vals) == 1 else vals

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.data):
            raise CorruptGraph("truncated container")
        b = self.data[self.pos:self.pos + n]
        self.pos += n
        return b

    def section(self) -> "_In":
        return _In(self.take(self.get("I")))


class _Strings:
    def __init__(self):
        self.ids: Dict[str, int] = {"": 0}
        self.items: List[str] = [""]

    def __call__(self, s: str) -> int:
        sid = self.ids.get(s)
        if sid is None:
            sid = self.ids[s] = len(self.items)
            self.items.append(s)
        return sid


def _put_shape(w: _Out, shape) -> None:
    w.put("H", len(shape))
    for d in shape:
        w.put("q", -1 if d is None else d)


def _get_shape(r: _In):
    return tuple(None if d == -1 else d for d in (r.get("q") for _ in range(r.get("H"))))


def _put_attr(w: _Out, strings: _Strings, v) -> None:
    if v is None:
        w.put("B", T_NONE)
    elif isinstance(v, bool):
        w.put("BB", T_BOOL, 1 if v else 0)
    elif isinstance(v, int):
        w.put("Bq", T_INT, v)
    elif isinstance(v, float):
        w.put("Bd", T_FLOAT, v)
    elif isinstance(v, str):
        w.put("BI", T_STRING, strings(v))
    elif isinstance(v, DType):
        w.put("BB", T_DTYPE, DTYPE_TAGS[v])
    elif isinstance(v, Tensor):
        w.put("BB", T_TENSOR, DTYPE_TAGS[v.dtype])
        _put_shape(w, v.shape)
        w.raw(v.raw().tobytes())
    elif isinstance(v, tuple) and any(d is None for d in v):
        w.put("B", T_SHAPE)
        _put_shape(w, v)
    elif isinstance(v, tuple):
        w.put("BH", T_INT_LIST, len(v))
        for d in v:
            w.put("q", d)
    else:
        raise NotSerializable(f"attr value {v!r} has no wire encoding")


def _get_attr(r: _In, strings: List[str]):
    tag = r.get("B")
    if tag == T_NONE:
        return None
    if tag == T_BOOL:
        return bool(r.get("B"))
    if tag == T_INT:
        return r.get("q")
    if tag == T_FLOAT:
        return r.get("d")
    if tag == T_STRING:
        return strings[r.get("I")]
    if tag == T_DTYPE:
        dt = TAG_DTYPES.get(r.get("B"))
        if dt is None:
            raise CorruptGraph("bad dtype tag in attr")
        return dt
    if tag == T_TENSOR:
        dt = TAG_DTYPES.get(r.get("B"))
        if dt is None:
            raise CorruptGraph("bad dtype tag")
        shape = _get_shape(r)
        if None in shape:
            raise CorruptGraph("constant tensors cannot have wildcard dims")
        n = int(np.prod(shape, dtype=np.int64)) if shape else 1
        arr = np.frombuffer(r.take(n * dt.width), dtype=dt.np_dtype)
        return tensor_from_host(arr, shape, dt)
    if tag == T_SHAPE:
        return _get_shape(r)
    if tag == T_INT_LIST:
        return tuple(r.get("q") for _ in range(r.get("H")))
    raise CorruptGraph(f"unknown attr tag {tag}")


def serialize(gf: GraphFunction) -> bytes:
    if not gf.serializable:
        raise NotSerializable(f"{gf.name} contains a host_call (directly or in its library) and "
                              "cannot be serialized")
    return _encode(gf)


def _encode(gf: GraphFunction) -> bytes:
    strings = _Strings()
    for ph in gf.inputs:
        strings(ph.name)
    for node in gf.nodes:
        strings(node.op)
        for k in sorted(node.attrs):
            strings(k)
            if isinstance(node.attrs[k], str):
                strings(node.attrs[k])
        if node.device is not None:
            strings(node.device.render())
    for name, _ in gf.outputs:
        strings(name)
    lib = sorted(gf.library.items())
    for name, _ in lib:
        strings(name)

    sec_in = _Out()
    sec_in.put("I", len(gf.inputs))
    for ph in gf.inputs:
        sec_in.put("IB", strings(ph.name), DTYPE_TAGS[ph.dtype] | (_VAR_BIT if ph.is_variable_ref else 0))
        _put_shape(sec_in, ph.shape)
    sec_nodes = _Out()
    sec_nodes.put("I", len(gf.nodes))
    for node in gf.nodes:
        sec_nodes.put("II", strings(node.op), len(node.inputs))
        for vid, k in node.inputs:
            sec_nodes.put("IH", vid, k)
        sec_nodes.put("I", len(node.attrs))
        for k in sorted(node.attrs):
            sec_nodes.put("I", strings(k))
            _put_attr(sec_nodes, strings, node.attrs[k])
        sec_nodes.put("I", strings(node.device.render()) if node.device else 0)
    sec_out = _Out()
    sec_out.put("I", len(gf.outputs))
    for name, (vid, k) in gf.outputs:
        sec_out.put("IIH", strings(name), vid, k)
    sec_lib = _Out()
    sec_lib.put("I", len(lib))
    for name, sub in lib:
        body = _encode(sub)
        sec_lib.put("II", strings(name), len(body))
        sec_lib.raw(body)
    sec_str = _Out()
    sec_str.put("I", len(strings.items))
    for s in strings.items:
        b = s.encode("utf-8")
        sec_str.put("I", len(b))
        sec_str.raw(b)

    w = _Out()
    w.raw(MAGIC)
    w.put("I", VERSION)
    for sec in (sec_str, sec_in, sec_nodes, sec_out, sec_lib):
        w.put("I", len(sec.buf))
        w.raw(bytes(sec.buf))
    return bytes(w.buf)


def deserialize(data: bytes, name: str = "loaded") -> GraphFunction:
    from .kernels import KernelEnv
    from .ops import get_op_def
    from .runtime import get_runtime

    r = _In(data)
    if r.take(4) != MAGIC:
        raise CorruptGraph("not a graph-function container (bad magic)")
    version = r.get("I")
    if version != VERSION:
        raise FormatVersionMismatch(f"container version {version}, this runtime reads {VERSION}")
    sr = r.section()
    strings = [sr.take(sr.get("I")).decode("utf-8") for _ in range(sr.get("I"))]

    def s_at(i: int) -> str:
        if i >= len(strings):
            raise CorruptGraph(f"string id {i} out of range")
        return strings[i]

    ir = r.section()
    placeholders = []
    for _ in range(ir.get("I")):
        pname = s_at(ir.get("I"))
        b = ir.get("B")
        dt = TAG_DTYPES.get(b & ~_VAR_BIT)
        if dt is None:
            raise CorruptGraph("bad placeholder dtype")
        placeholders.append(Placeholder(pname, dt, _get_shape(ir), bool(b & _VAR_BIT)))
    nr = r.section()
    raw_nodes = []
    for _ in range(nr.get("I")):
        op = s_at(nr.get("I"))
        ins = tuple(nr.get("IH") for _ in range(nr.get("I")))
        attrs = {}
        for _ in range(nr.get("I")):
            k = s_at(nr.get("I"))
            attrs[k] = _get_attr(nr, strings)
        dev_id = nr.get("I")
        device = None
        if dev_id:
            from .devices import DeviceName

            device = DeviceName.parse(s_at(dev_id))
        raw_nodes.append((op, ins, attrs, device))
    orr = r.section()
    outputs = [(s_at(orr.get("I")), orr.get("IH")) for _ in range(orr.get("I"))]
    lr = r.section()
    library: Dict[str, GraphFunction] = {}
    for _ in range(lr.get("I")):
        lname = s_at(lr.get("I"))
        library[lname] = deserialize(lr.take(lr.get("I")), name=lname)

    env = KernelEnv(device=get_runtime().devices[0].name, libraries=(library,))
    specs: List[list] = [[(ph.dtype, ph.shape)] for ph in placeholders]
    nodes = []
    for op, ins, attrs, device in raw_nodes:
        in_specs = []
        for vid, k in ins:
            if vid >= len(specs):
                raise CorruptGraph("node references a later value")
            if k >= len(specs[vid]):
                raise CorruptGraph("node references a missing output")
            in_specs.append(specs[vid][k])
        out_specs = tuple(get_op_def(op).infer(attrs, in_specs, env))
        nodes.append(Node(op, tuple(tuple(x) for x in ins), attrs, device, out_specs))
        specs.append(list(out_specs))
    outputs = [(nm, tuple(ref)) for nm, ref in outputs]
    return GraphFunction(name, placeholders, nodes, outputs, library)
