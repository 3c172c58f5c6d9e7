"""Binding of the native eager front-end, ``_lib/_sfeager*.so`` (csrc/sf_eager.cpp).

The extension provides the storage types the front-end is built on
(``TensorBase`` — the slot layout and arithmetic operators of ``Tensor`` —
and ``DeviceBuffer``) and a C implementation of ``dispatch`` and of the op
wrappers for the common eager case: built-in/plugin elementwise ops, tiny
matmuls, transposes, identity, reshape and broadcast_to on a single-device
runtime outside traces.  Each such op is one descriptor handed to the
device's launch queue (sf_queue_push); everything else — and every error —
runs the reference-semantics Python dispatcher ``ops._dispatch_py``
(reference: stageflow/ops.py:294-362).

Which ops may take the native path is declared on their kernels: a kernel
function carrying ``_sf_fast = (kind, opcode, flags)`` (set by
``mark_fast``) is one the C code reproduces exactly.  User kernels have no
mark and always run through Python.

Without a GPU (the CPU test container) the extension may be absent; the
package then uses pure-Python stand-ins for the storage types.  On a machine
with a GPU a missing extension is an error (``require_native``): there is
no slow eager path on a GPU box.
"""
from __future__ import annotations

import importlib.machinery
import importlib.util
import os
import sysconfig
import weakref
from typing import Optional

_LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
EXT_PATH = os.path.join(_LIB_DIR, "_sfeager" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def _load():
    if not os.path.exists(EXT_PATH):
        return None, f"{EXT_PATH} is not built"
    # make sure the ctypes binding loads libsfb200.so first (one instance)
    from . import _native

    try:
        _native.load_library()
    except Exception as e:  # pragma: no cover - library missing
        return None, f"libsfb200.so failed to load: {e}"
    try:
        loader = importlib.machinery.ExtensionFileLoader("_sfeager", EXT_PATH)
        spec = importlib.util.spec_from_file_location("_sfeager", EXT_PATH, loader=loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        return mod, None
    except ImportError as e:
        return None, str(e)


ext, LOAD_ERROR = _load()
NATIVE = ext is not None

if NATIVE:
    TensorBase = ext.TensorBase
    DeviceBuffer = ext.DeviceBuffer
    K_EW1, K_EW2, K_MATMUL = ext.K_EW1, ext.K_EW2, ext.K_MATMUL
    K_TRANSPOSE, K_IDENTITY, K_RESHAPE, K_BROADCAST_TO = (
        ext.K_TRANSPOSE, ext.K_IDENTITY, ext.K_RESHAPE, ext.K_BROADCAST_TO)
    F_FLOATS_ONLY, F_OUT_BOOL = ext.F_FLOATS_ONLY, ext.F_OUT_BOOL
else:
    K_EW1, K_EW2, K_MATMUL, K_TRANSPOSE, K_IDENTITY, K_RESHAPE, K_BROADCAST_TO = range(1, 8)
    F_FLOATS_ONLY, F_OUT_BOOL = 1, 2

    class TensorBase:
        """Pure-Python stand-in (no extension: host-only use, no GPU)."""

        __slots__ = ("dtype", "shape", "device", "_buf", "_host", "_symbolic", "_born_trace",
                     "_sib", "_pend", "__weakref__")

    class DeviceBuffer:
        """Pure-Python stand-in of _sfeager.DeviceBuffer (no extension)."""

        __slots__ = ("dev", "ptr", "nbytes", "__weakref__")

        def __init__(self, dev: int, ptr, nbytes: int):
            self.dev = dev
            self.ptr = ptr or 0
            self.nbytes = nbytes

        def __del__(self):
            ptr = self.ptr
            if ptr:
                self.ptr = 0
                try:
                    from . import _native

                    _native._lib.sf_free(self.dev, ptr)
                except Exception:  # interpreter shutdown
                    pass


if NATIVE:
    from . import _native as _nat

    _nat.DeviceBuffer = ext.DeviceBuffer  # one allocator block, sf_free in C


def require_native() -> None:
    """Called when a runtime with a GPU starts: the native front-end is part
    of the backend, not an optional accelerator."""
    if not NATIVE:
        from .errors import DeviceUnavailable

        raise DeviceUnavailable(f"native eager front-end unavailable: {LOAD_ERROR}; run "
                                "`python -c 'import __graft_entry__ as g; g.build()'`")


def mark_fast(kernel, kind: int, opcode: int = 0, flags: int = 0):
    """Declare that `kernel` is reproduced exactly by the native fast path."""
    kernel._sf_fast = (kind, opcode, flags)
    return kernel


def fast_spec(op_def):
    return getattr(op_def.kernel, "_sf_fast", None)


# ---------------------------------------------------------------------------
# binding to the live runtime
# ---------------------------------------------------------------------------

_bound: Optional[weakref.ref] = None


def drain_into(rt) -> None:
    """Fold the native dispatch counters of `rt` into its RuntimeStats."""
    if NATIVE and rt is not None:
        counts = ext.drain(rt)
        if counts:
            rt.stats._absorb(counts)


def pending(rt) -> int:
    return ext.pending(rt) if NATIVE else 0


def configure(rt) -> None:
    """(Re)bind the native fast path to runtime `rt` (called by the
    extension when the live runtime changed, e.g. after init_runtime)."""
    global _bound
    from . import ops, runtime, tensor
    from .dtypes import DType
    from .errors import KernelError

    old = _bound() if _bound is not None else None
    if old is not None and old is not rt:
        drain_into(old)
    fast = []
    for d in rt.registry.all_defs():
        spec = fast_spec(d)
        if spec is not None:
            fast.append((d.name, d) + tuple(spec))
        elif d.name == "call_function":
            fast.append((d.name, d, 0, 0, 0))  # counted by the staged-call path
    dev = rt.devices[0]
    # (no GPU: the fast path stays off and the Python path reports it)
    single = len(rt.devices) == 1 and rt.backend_available
    ext.configure(rt, rt.registry, single, dev.ordinal, dev.name, tensor.Tensor,
                  (DType.float32, DType.float64, DType.int32, DType.boolean),
                  runtime.ExecutionContext, ops._dispatch_py, ops._notify_tapes, KernelError,
                  ops._operator_slow, fast)
    _bound = weakref.ref(rt)


def on_register(registry, op_def) -> None:
    """A plugin op registered after the fast path was bound to the runtime."""
    spec = fast_spec(op_def)
    if NATIVE and spec is not None:
        ext.add_op(registry, op_def.name, op_def, *spec)


def bootstrap() -> None:
    if NATIVE:
        from . import ops, runtime

        ext.bootstrap(vars(runtime), runtime._local, configure, ops._dispatch_py,
                      ops._operator_slow, host_scalar)


def host_scalar(value, dtype):
    """The read-only 0-d host array the reference's ``_as_operand(value,
    like)`` builds for a Python scalar (ops.py:370-383 -> tensor.py:138-162)."""
    import numpy as np

    from .tensor import _checked_host_array

    arr = np.asarray(value, dtype=dtype.np_dtype)
    return _checked_host_array(arr.reshape(-1), arr.shape, dtype)


def wrap(name: str, arity: int, slow):
    """The native wrapper of `slow` (a reference-semantics op wrapper)."""
    if not NATIVE:
        return slow
    return ext.FastWrapper(name, arity, slow)


def set_enabled(on: bool) -> bool:
    """Enable/disable the native fast path (tests compare both); returns the
    previous state."""
    return ext.set_enabled(on) if NATIVE else False


def staged_fast(rt, cf, prog, args, structure: str):
    """The native repeat-call path of a staged function (ext.StagedFast) for
    calls like `args` (positional tensors), or None when the program is not
    one native plan or a capture is not a plain tensor."""
    if not NATIVE or len(rt.devices) != 1 or not rt.backend_available:
        return None
    from .tensor import Tensor

    fast = prog._single_plan() if prog.__dict__.get("_fast") is None else prog._fast
    if not fast or prog.__dict__.get("_replay"):
        return None
    plan, pos, specs = fast
    caps = cf.materialize_captured()
    everything = list(args) + caps
    if not all(type(v) is Tensor for v in everything):
        return None
    n_args = len(args)
    in_src, in_ptr = [], []
    for i in pos:
        if i < n_args:
            in_src.append(i)
            in_ptr.append(0)
        else:
            in_src.append(-1)
            in_ptr.append(everything[i]._ptr())
    code = {"none": 0, "single": 1, "tuple": 2, "list": 3}[structure]
    return ext.StagedFast(rt, (prog, plan, tuple(caps), cf), plan._lock, plan.handle, prog.dev,
                          prog.device, tuple(a.dtype for a in args),
                          tuple(a.shape for a in args), in_src, in_ptr,
                          [j for j, _, _, _ in specs], [nb for _, nb, _, _ in specs],
                          tuple(dt for _, _, dt, _ in specs),
                          tuple(tuple(sh) for _, _, _, sh in specs), code)


MISS = ext.MISS if NATIVE else object()
