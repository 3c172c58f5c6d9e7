"""ctypes binding of libsfb200.so (the C-ABI declared in include/sfb200.h).

This is the only module that talks to the native library.  Every call
checks the returned status and raises: ``DeviceUnavailable`` when no GPU or
no built library is present, ``KernelError`` for any other native failure.
There is no host fallback anywhere behind these functions.
"""
from __future__ import annotations

import ctypes
import os
import struct
import threading
from typing import List, Optional, Sequence

import numpy as np

from .errors import DeviceUnavailable, KernelError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libsfb200.so")

# ---- opcodes: must match csrc/sf_ops.cuh ------------------------------------
OP = dict(
    identity=0, neg=1, exp=2, log=3, softplus=4, relu=5, step_positive=6, tanh=7,
    sqrt=8, rsqrt=9, sigmoid=10, abs=11, square=12, isfinite=13, logical_not=14,
    reciprocal=15, cos=16, sin=17,
    add=32, sub=33, mul=34, div=35, greater=36, maximum=37, minimum=38, less=39,
    equal=40, greater_equal=41,
    select=64,
)
BOOL_RESULT_OPS = frozenset(("greater", "less", "equal", "greater_equal", "isfinite",
                             "logical_not"))

SF_OK, SF_ERR_NO_DEVICE = 0, 6
MAX_DIMS = 8

_lib: Optional[ctypes.CDLL] = None
_lib_lock = threading.Lock()
_load_error: Optional[str] = None
_tls = threading.local()

_VP = ctypes.c_void_p
_I64 = ctypes.c_int64
_PVP = ctypes.POINTER(ctypes.c_void_p)


def _declare(lib: ctypes.CDLL) -> None:
    sig = {
        "sf_last_error": (ctypes.c_char_p, []),
        "sf_version": (ctypes.c_int, []),
        "sf_init": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
        "sf_device_info": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_size_t)]),
        "sf_set_stream": (ctypes.c_int, [ctypes.c_int, _VP]),
        "sf_get_stream": (ctypes.c_int, [ctypes.c_int, _PVP]),
        "sf_device_sync": (ctypes.c_int, [ctypes.c_int]),
        "sf_alloc": (ctypes.c_int, [ctypes.c_int, ctypes.c_size_t, _PVP]),
        "sf_free": (ctypes.c_int, [ctypes.c_int, _VP]),
        "sf_mem_stats": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_size_t),
                                         ctypes.POINTER(ctypes.c_size_t)]),
        "sf_trim": (ctypes.c_int, [ctypes.c_int]),
        "sf_reduce_counters": (ctypes.c_int, [ctypes.c_int, _PVP]),
        "sf_host_alloc": (ctypes.c_int, [ctypes.c_size_t, _PVP]),
        "sf_host_free": (ctypes.c_int, [_VP]),
        "sf_memcpy_h2d": (ctypes.c_int, [ctypes.c_int, _VP, _VP, ctypes.c_size_t]),
        "sf_memcpy_h2d_immutable": (ctypes.c_int, [ctypes.c_int, _VP, _VP, ctypes.c_size_t,
                                                   ctypes.POINTER(ctypes.c_int)]),
        "sf_memcpy_d2h_enqueue": (ctypes.c_int, [ctypes.c_int, _VP, _VP, ctypes.c_size_t]),
        "sf_memcpy_d2h": (ctypes.c_int, [ctypes.c_int, _VP, _VP, ctypes.c_size_t]),
        "sf_memcpy_d2d": (ctypes.c_int, [ctypes.c_int, _VP, _VP, ctypes.c_size_t]),
        "sf_memcpy_p2p": (ctypes.c_int, [ctypes.c_int, _VP, ctypes.c_int, _VP, ctypes.c_size_t]),
        "sf_elementwise": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, _PVP]),
        "sf_reduce": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_char_p, ctypes.c_uint32, _VP, _PVP]),
        "sf_matmul": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64, _I64, _I64, _VP,
                                      ctypes.c_int, _VP, ctypes.c_int, _PVP]),
        "sf_transpose2d": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64, _I64, _VP, _PVP]),
        "sf_fill": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64, ctypes.c_double, _PVP]),
        "sf_eye": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64, _PVP]),
        "sf_cast": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _I64, _VP, _PVP]),
        "sf_rng_seed": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64]),
        "sf_rng_reserve": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64,
                                           ctypes.POINTER(ctypes.c_uint64)]),
        "sf_rng": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _I64,
                                   ctypes.c_uint64, _PVP]),
        "sf_dropout": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64, _VP, _VP, ctypes.c_int,
                                       ctypes.c_double, _PVP, _PVP]),
        "sf_im2col": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, _VP, _PVP]),
        "sf_col2im": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, _VP, _PVP]),
        "sf_maxpool2d": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, _VP, _PVP]),
        "sf_conv2d_tc": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, _I64, _VP, _VP, _PVP]),
        "sf_maxpool2d_grad": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, _VP,
                                              _VP, _PVP]),
        "sf_softmax_xent": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64, _I64, _VP, _VP,
                                            _PVP]),
        "sf_softmax_xent_grad": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64, _I64, _VP,
                                                 _VP, _VP, _PVP]),
        "sf_gemm_tf32x3": (ctypes.c_int, [ctypes.c_int, _I64, _I64, _I64, _VP, _VP, _VP, _VP,
                                           _PVP]),
        "sf_gemm_tf32x3_ex": (ctypes.c_int, [ctypes.c_int, _I64, _I64, _I64, ctypes.c_int,
                                              ctypes.c_int, _I64, _I64, _VP, _VP, _VP, _VP,
                                              _PVP]),
        "sf_im2col_split": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, _I64, _VP, _PVP, _PVP]),
        "sf_split_tf32": (ctypes.c_int, [ctypes.c_int, _I64, _I64, _I64, ctypes.c_int, _VP, _PVP,
                                          _PVP]),
        "sf_jit_compile": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, _PVP]),
        "sf_jit_log": (ctypes.c_char_p, []),
        "sf_jit_launch": (ctypes.c_int, [ctypes.c_int, _VP, ctypes.c_uint, ctypes.c_uint,
                                          ctypes.c_uint, ctypes.c_char_p, ctypes.c_size_t]),
        "sf_plan_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t, _PVP]),
        "sf_plan_run": (ctypes.c_int, [_VP, _VP, _VP]),
        "sf_plan_info": (ctypes.c_int, [_VP] + [ctypes.POINTER(ctypes.c_int)] * 4),
        "sf_plan_destroy": (ctypes.c_int, [_VP]),
        "sf_plan_profile": (ctypes.c_int, [_VP, ctypes.c_int]),
        "sf_plan_step_stats": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                               ctypes.POINTER(ctypes.c_double),
                                               ctypes.POINTER(ctypes.c_uint64)]),
        "sf_launch_count": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]),
        "sf_comm_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
        "sf_comm_init": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_char_p, _PVP]),
        "sf_comm_destroy": (ctypes.c_int, [_VP]),
        "sf_allreduce": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_void_p),
                                         ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                         ctypes.c_int, ctypes.c_double]),
        "sf_nccl_version": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
        "sf_queue_push": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, _PVP]),
        "sf_queue_flush": (ctypes.c_int, [ctypes.c_int]),
        "sf_queue_config": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64]),
        "sf_queue_stats": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                                           ctypes.POINTER(ctypes.c_uint64)]),
        "sf_while_create": (ctypes.c_int, [ctypes.c_int, _PVP]),
        "sf_cond_create": (ctypes.c_int, [ctypes.c_int, _PVP]),
        "sf_graph_create": (ctypes.c_int, [ctypes.c_int, _PVP]),
        "sf_while_buffer": (ctypes.c_int, [_VP, ctypes.c_size_t, _PVP]),
        "sf_while_capture_begin": (ctypes.c_int, [_VP, ctypes.c_int]),
        "sf_while_set_cond": (ctypes.c_int, [_VP, _VP]),
        "sf_while_capture_end": (ctypes.c_int, [_VP, ctypes.c_int]),
        "sf_while_launch": (ctypes.c_int, [_VP]),
        "sf_while_destroy": (ctypes.c_int, [_VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


EXPORTED_SYMBOLS = (
    "sf_last_error", "sf_version", "sf_init", "sf_device_info", "sf_set_stream",
    "sf_get_stream", "sf_device_sync", "sf_alloc", "sf_free", "sf_mem_stats", "sf_trim",
    "sf_reduce_counters", "sf_host_alloc", "sf_host_free",
    "sf_memcpy_h2d", "sf_memcpy_h2d_immutable", "sf_memcpy_d2h", "sf_memcpy_d2h_enqueue",
    "sf_memcpy_d2d",
    "sf_memcpy_p2p", "sf_elementwise",
    "sf_reduce", "sf_matmul", "sf_transpose2d", "sf_fill", "sf_eye", "sf_cast", "sf_rng_seed",
    "sf_rng_reserve", "sf_rng", "sf_dropout", "sf_jit_compile", "sf_jit_log", "sf_jit_launch",
    "sf_plan_create", "sf_plan_run", "sf_plan_info", "sf_plan_destroy", "sf_launch_count",
    "sf_plan_profile", "sf_plan_step_stats", "sf_im2col", "sf_col2im", "sf_maxpool2d",
    "sf_maxpool2d_grad", "sf_softmax_xent", "sf_softmax_xent_grad", "sf_gemm_tf32x3",
    "sf_gemm_tf32x3_ex", "sf_conv2d_tc",
    "sf_split_tf32", "sf_im2col_split", "sf_while_create", "sf_cond_create", "sf_graph_create",
    "sf_while_buffer",
    "sf_while_capture_begin", "sf_while_set_cond", "sf_while_capture_end", "sf_while_launch",
    "sf_while_destroy", "sf_queue_push", "sf_queue_flush", "sf_queue_config", "sf_queue_stats",
    "sf_comm_unique_id", "sf_comm_init", "sf_comm_destroy", "sf_allreduce", "sf_nccl_version",
)


def im2col_split(dev: int, geom: bytes, m: int, kp: int, src: int):
    L = require_device()
    hi, lo = ctypes.c_void_p(0), ctypes.c_void_p(0)
    rc = L.sf_im2col_split(dev, geom, kp, src, ctypes.byref(hi), ctypes.byref(lo))
    if rc:
        raise _err(L, rc, "sf_im2col_split")
    return DeviceBuffer(dev, hi.value, m * kp * 4), DeviceBuffer(dev, lo.value, m * kp * 4)


def im2col_raw(dev: int, geom: bytes, m: int, kp: int, src: int) -> DeviceBuffer:
    """(m, kp) raw fp32 im2col rows, K zero-padded to kp (no lo part: for
    GEMMs that derive it in shared memory)."""
    L = require_device()
    hi = ctypes.c_void_p(0)
    rc = L.sf_im2col_split(dev, geom, kp, src, ctypes.byref(hi), None)
    if rc:
        raise _err(L, rc, "sf_im2col_split")
    return DeviceBuffer(dev, hi.value, m * kp * 4)


def gemm_tf32x3(dev: int, m: int, n: int, k: int, a_hi: int, a_lo: int, b_hi: int,
                b_lo: int) -> "DeviceBuffer":
    """C[m,n] = A[m,k] . B[n,k]^T on tcgen05 (3xTF32); operands pre-split."""
    return nn_call("sf_gemm_tf32x3", dev, m, n, k, a_hi, a_lo, b_hi, b_lo, out_nbytes=m * n * 4)


def gemm_tf32x3_ex(dev: int, m: int, n: int, k: int, a_mn: bool, b_mn: bool, ak: int, bk: int,
                   a_hi: int, a_lo: int, b_hi: int, b_lo: int) -> "DeviceBuffer":
    """C[m,n] on tcgen05 with per-operand majorness (see sf_gemm_tf32x3_ex)."""
    return nn_call("sf_gemm_tf32x3_ex", dev, m, n, k, int(a_mn), int(b_mn), ak, bk, a_hi, a_lo,
                   b_hi, b_lo, out_nbytes=m * n * 4)


class RawRef:
    """A borrowed device pointer (the caller keeps its owner alive)."""

    __slots__ = ("ptr",)

    def __init__(self, ptr: int):
        self.ptr = ptr


def split_tf32(dev: int, rows: int, cols: int, src: int, transpose: bool = False,
               ldo: int = 0):
    """(hi, lo) of an fp32 matrix (optionally transposed/padded).  Without
    transpose the hi operand is the source itself (RawRef): the tensor cores
    ignore the low 13 mantissa bits, so only lo is materialised."""
    L = require_device()
    ldo = ldo or (rows if transpose else cols)
    raw_hi = not transpose and ldo == cols
    hi, lo = ctypes.c_void_p(0), ctypes.c_void_p(0)
    rc = L.sf_split_tf32(dev, rows, cols, ldo, int(transpose), src,
                         None if raw_hi else ctypes.byref(hi), ctypes.byref(lo))
    if rc:
        raise _err(L, rc, "sf_split_tf32")
    n = (cols if transpose else rows) * ldo * 4
    hi_ref = RawRef(src) if raw_hi else DeviceBuffer(dev, hi.value, n)
    return hi_ref, DeviceBuffer(dev, lo.value, n)


def nn_call(name: str, dev: int, *args, out_nbytes: int) -> "DeviceBuffer":
    """Call one of the NN entry points whose last argument is `void** out`."""
    L = require_device()
    out, ref = _outslot()
    rc = getattr(L, name)(dev, *args, ref)
    if rc:
        raise _err(L, rc, name)
    return DeviceBuffer(dev, out.value, out_nbytes)


def load_library() -> ctypes.CDLL:
    """Load libsfb200.so (no device needed for the load itself)."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                _load_error = (f"native library {LIB_PATH} is not built; run "
                               "`python -c 'import __graft_entry__ as g; g.build()'`")
                raise DeviceUnavailable(_load_error)
            lib = ctypes.CDLL(LIB_PATH)
            _declare(lib)
            _lib = lib
    return _lib


def _err(lib, rc: int, what: str):
    msg = (lib.sf_last_error() or b"").decode(errors="replace")
    if rc == SF_ERR_NO_DEVICE:
        return DeviceUnavailable(f"{what}: {msg}")
    return KernelError(f"{what}: {msg}")


def lib() -> ctypes.CDLL:
    return load_library()


_device_count: Optional[int] = None


def device_count() -> int:
    """Number of usable CUDA devices; 0 if the library or GPU is missing."""
    global _device_count
    if _device_count is None:
        try:
            L = load_library()
        except (DeviceUnavailable, OSError):
            _device_count = 0
            return 0
        n = ctypes.c_int(0)
        _device_count = n.value if L.sf_init(ctypes.byref(n)) == SF_OK else 0
    return _device_count


def require_device():
    if device_count() == 0:
        L = None
        try:
            L = load_library()
        except DeviceUnavailable:
            raise
        n = ctypes.c_int(0)
        rc = L.sf_init(ctypes.byref(n))
        raise _err(L, rc if rc else SF_ERR_NO_DEVICE, "GPU backend unavailable")
    return lib()


def _outslot():
    p = getattr(_tls, "out", None)
    if p is None:
        p = _tls.out = ctypes.c_void_p(0)
        _tls.outref = ctypes.byref(p)
        _tls.out2 = ctypes.c_void_p(0)
        _tls.out2ref = ctypes.byref(_tls.out2)
    p.value = None
    return p, _tls.outref


# ---------------------------------------------------------------- buffers
class DeviceBuffer:
    """Owns one allocation from the device's caching allocator."""

    __slots__ = ("dev", "ptr", "nbytes", "__weakref__")

    def __init__(self, dev: int, ptr: int, nbytes: int):
        self.dev = dev
        self.ptr = ptr
        self.nbytes = nbytes

    def __del__(self):
        ptr = self.ptr
        if ptr:
            self.ptr = 0
            try:
                _lib.sf_free(self.dev, ptr)
            except Exception:  # interpreter shutdown
                pass


def alloc(dev: int, nbytes: int) -> DeviceBuffer:
    L = require_device()
    out, ref = _outslot()
    rc = L.sf_alloc(dev, max(1, nbytes), ref)
    if rc:
        raise _err(L, rc, "sf_alloc")
    return DeviceBuffer(dev, out.value, nbytes)


def upload(dev: int, arr: np.ndarray) -> DeviceBuffer:
    arr = np.ascontiguousarray(arr)
    buf = alloc(dev, arr.nbytes)
    if arr.nbytes:
        rc = _lib.sf_memcpy_h2d(dev, buf.ptr, arr.ctypes.data, arr.nbytes)
        if rc:
            raise _err(_lib, rc, "sf_memcpy_h2d")
    return buf


def frozen_pinned(arr: np.ndarray) -> bool:
    """True when arr views a block of the pinned result pool through a
    read-only memoryview the runtime put there (``freeze_pinned``): nothing
    can make it writable again, and its memory is only reused by a later
    copy on a device stream, or freed after a device sync (_PinnedPool)."""
    b, ro = arr, False
    while True:
        if isinstance(b, np.ndarray):
            b = b.base
        elif isinstance(b, memoryview):
            ro = ro or b.readonly
            b = b.obj
        else:
            break
    return ro and getattr(b, "_blk", None) is not None


def freeze_pinned(arr: np.ndarray) -> np.ndarray:
    """A permanently read-only view of a pinned-pool download (Tensor.raw):
    its WRITEABLE flag can never be set again, so uploading it may alias it."""
    b = arr
    while isinstance(b, np.ndarray):
        b = b.base
    if getattr(b, "_blk", None) is None or not arr.flags.c_contiguous:
        arr.flags.writeable = False
        return arr
    return np.frombuffer(memoryview(arr).toreadonly(), dtype=arr.dtype).reshape(arr.shape)


def upload_immutable(dev: int, arr: np.ndarray) -> DeviceBuffer:
    """Upload a read-only C-contiguous array that the caller keeps alive (the
    new tensor holds it as its host copy): page-locked memory is DMA'd
    without waiting for the copy.  Later work on the device's stream is
    ordered after it; a pooled pinned block only returns to the pool when the
    array dies, and its next use is a copy on the same stream."""
    buf = alloc(dev, arr.nbytes)
    if arr.nbytes:
        flag = ctypes.c_int(0)
        rc = _lib.sf_memcpy_h2d_immutable(dev, buf.ptr, arr.ctypes.data, arr.nbytes,
                                          ctypes.byref(flag))
        if rc:
            raise _err(_lib, rc, "sf_memcpy_h2d_immutable")
    return buf


class _PinnedBlock:
    """A page-locked host block; returns itself to the pool when the numpy
    array built over it is collected."""

    __slots__ = ("ptr", "cap")

    def __init__(self, ptr: int, cap: int):
        self.ptr, self.cap = ptr, cap

    def __del__(self):
        try:
            _PINNED.put(self)
        except Exception:  # interpreter shutdown
            pass


class _PinnedPool:
    """Size-class pool of page-locked host blocks for device->host results:
    the DMA lands directly in the array the caller receives (no staging
    copy).  At most LIMIT bytes stay cached."""

    LIMIT = 256 << 20
    MIN = 64 << 10
    MAX_ARRAY = 64 << 20  # larger results use pageable memory (page-locking is scarce)

    def __init__(self):
        self.free: dict = {}
        self.cached = 0
        self.lock = threading.Lock()
        # blocks over LIMIT waiting to be unpinned.  put() runs from a
        # finalizer (any allocation can trigger it, including one inside a
        # stream capture), so it never syncs or frees: drain() does, from
        # get() -- called only outside captures.
        self.pending: list = []

    def get(self, nbytes: int) -> Optional["_PinnedBlock"]:
        cap = self.MIN
        while cap < nbytes:
            cap <<= 1
        if self.pending:
            self.drain()
        ptr = 0
        with self.lock:
            lst = self.free.get(cap)
            if lst:
                self.cached -= cap
                ptr = lst.pop()
        if not ptr:
            p = ctypes.c_void_p(0)
            if _lib.sf_host_alloc(cap, ctypes.byref(p)):
                return None
            ptr = p.value
        return _PinnedBlock(ptr, cap)  # created outside the lock (see put)

    def put(self, blk: "_PinnedBlock") -> None:
        ptr, blk.ptr = blk.ptr, 0
        if not ptr:
            return
        with self.lock:
            if self.cached + blk.cap <= self.LIMIT:
                self.free.setdefault(blk.cap, []).append(ptr)
                self.cached += blk.cap
            else:
                self.pending.append(ptr)

    def drain(self) -> None:
        with self.lock:
            ptrs, self.pending = self.pending, []
        if not ptrs:
            return
        # a block may still be the source of an asynchronous upload
        # (upload_immutable): let every device drain before unpinning it
        for dev in range(device_count()):
            _lib.sf_device_sync(dev)
        for ptr in ptrs:
            _lib.sf_host_free(ptr)


_PINNED = _PinnedPool()


def download(buf: DeviceBuffer, np_dtype, shape) -> np.ndarray:
    nbytes = int(np.prod(shape, dtype=np.int64)) * np.dtype(np_dtype).itemsize
    if _PinnedPool.MIN <= nbytes <= _PinnedPool.MAX_ARRAY:
        blk = _PINNED.get(nbytes)
        if blk is not None:
            # the array lives in page-locked memory: the copy DMAs straight into it
            cbuf = (ctypes.c_char * nbytes).from_address(blk.ptr)
            cbuf._blk = blk  # the block is freed to the pool with the array
            out = np.frombuffer(cbuf, dtype=np_dtype).reshape(shape)
            rc = _lib.sf_memcpy_d2h(buf.dev, blk.ptr, buf.ptr, nbytes)
            if rc:
                raise _err(_lib, rc, "sf_memcpy_d2h")
            return out
    out = np.empty(shape, dtype=np_dtype)
    if out.nbytes:
        rc = _lib.sf_memcpy_d2h(buf.dev, out.ctypes.data, buf.ptr, out.nbytes)
        if rc:
            raise _err(_lib, rc, "sf_memcpy_d2h")
    return out


def download_enqueue(buf: DeviceBuffer, np_dtype, shape) -> Optional[np.ndarray]:
    """Enqueue a device->host copy into a pooled page-locked array without
    waiting; the array is valid once a later synchronising call on the
    device's stream has returned.  None when no pinned block is available."""
    nbytes = int(np.prod(shape, dtype=np.int64)) * np.dtype(np_dtype).itemsize
    if not (_PinnedPool.MIN <= nbytes <= _PinnedPool.MAX_ARRAY):
        return None
    blk = _PINNED.get(nbytes)
    if blk is None:
        return None
    cbuf = (ctypes.c_char * nbytes).from_address(blk.ptr)
    cbuf._blk = blk
    out = np.frombuffer(cbuf, dtype=np_dtype).reshape(shape)
    if _lib.sf_memcpy_d2h_enqueue(buf.dev, blk.ptr, buf.ptr, nbytes):
        return None
    return out


def copy_d2d(dev: int, dst: int, src: int, nbytes: int) -> None:
    rc = _lib.sf_memcpy_d2d(dev, dst, src, nbytes)
    if rc:
        raise _err(_lib, rc, "sf_memcpy_d2d")


def copy_p2p(dst_dev: int, dst: int, src_dev: int, src: int, nbytes: int) -> None:
    rc = _lib.sf_memcpy_p2p(dst_dev, dst, src_dev, src, nbytes)
    if rc:
        raise _err(_lib, rc, "sf_memcpy_p2p")



def device_name(dev: int) -> str:
    """Short device description for reports, e.g. "sm_100 148SM 178GB"."""
    L = require_device()
    sms, ma, mi, mem = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0), ctypes.c_size_t(0)
    rc = L.sf_device_info(dev, ctypes.byref(sms), ctypes.byref(ma), ctypes.byref(mi),
                          ctypes.byref(mem))
    if rc:
        raise _err(L, rc, "sf_device_info")
    return f"sm_{ma.value}{mi.value} {sms.value}SM {mem.value >> 30}GB"

def sync(dev: int) -> None:
    L = require_device()
    rc = L.sf_device_sync(dev)
    if rc:
        raise _err(L, rc, "sf_device_sync")


def stream_of(dev: int) -> int:
    L = require_device()
    p = ctypes.c_void_p(0)
    rc = L.sf_get_stream(dev, ctypes.byref(p))
    if rc:
        raise _err(L, rc, "sf_get_stream")
    return p.value or 0


def set_stream(dev: int, stream: int) -> None:
    L = require_device()
    rc = L.sf_set_stream(dev, stream or None)
    if rc:
        raise _err(L, rc, "sf_set_stream")


_COUNTERS: dict = {}


def reduce_counters(dev: int) -> int:
    """Device address of the reduction arrival counters (fixed per process)."""
    p = _COUNTERS.get(dev)
    if p is None:
        L = require_device()
        out = ctypes.c_void_p(0)
        rc = L.sf_reduce_counters(dev, ctypes.byref(out))
        if rc:
            raise _err(L, rc, "sf_reduce_counters")
        p = _COUNTERS[dev] = out.value
    return p


def mem_stats(dev: int):
    L = require_device()
    a, b = ctypes.c_size_t(0), ctypes.c_size_t(0)
    L.sf_mem_stats(dev, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def launch_count(dev: int) -> int:
    L = load_library()
    c = ctypes.c_uint64(0)
    L.sf_launch_count(dev, ctypes.byref(c))
    return c.value


def comm_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (rank 0 of a communicator creates it)."""
    buf = ctypes.create_string_buffer(128)
    rc = require_device().sf_comm_unique_id(buf)
    if rc:
        raise _err(_lib, rc, "sf_comm_unique_id")
    return buf.raw


def comm_init(dev: int, nranks: int, rank: int, uid: bytes) -> int:
    h = ctypes.c_void_p(0)
    rc = require_device().sf_comm_init(dev, nranks, rank, uid, ctypes.byref(h))
    if rc:
        raise _err(_lib, rc, "sf_comm_init")
    return h.value


def comm_destroy(handle: int) -> None:
    if handle and _lib is not None:
        _lib.sf_comm_destroy(handle)


def allreduce(handle: int, ptrs: Sequence[int], counts: Sequence[int], dtype_tag: int,
              scale: float = 1.0) -> None:
    n = len(ptrs)
    parr = (ctypes.c_void_p * max(1, n))(*ptrs)
    carr = (ctypes.c_size_t * max(1, n))(*counts)
    rc = lib().sf_allreduce(handle, parr, carr, n, dtype_tag, scale)
    if rc:
        raise _err(_lib, rc, "sf_allreduce")


def nccl_version() -> int:
    v = ctypes.c_int(0)
    rc = require_device().sf_nccl_version(ctypes.byref(v))
    if rc:
        raise _err(_lib, rc, "sf_nccl_version")
    return v.value


def queue_flush(dev: int) -> None:
    """Launch what the eager launch queue holds (csrc/sf_queue.cu)."""
    rc = lib().sf_queue_flush(dev)
    if rc:
        raise _err(_lib, rc, "sf_queue_flush")


def queue_config(dev: int, max_ops: int, max_numel: int = 16384) -> None:
    """Ops per queue launch (0 disables queueing) and the largest queued op."""
    rc = lib().sf_queue_config(dev, max_ops, max_numel)
    if rc:
        raise _err(_lib, rc, "sf_queue_config")


def queue_stats(dev: int):
    """(ops pushed into the queue, queue launches) since sf_init."""
    a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
    rc = lib().sf_queue_stats(dev, ctypes.byref(a), ctypes.byref(b))
    if rc:
        raise _err(_lib, rc, "sf_queue_stats")
    return a.value, b.value


def rng_seed(dev: int, seed: int) -> None:
    rc = lib().sf_rng_seed(dev, seed & 0xFFFFFFFFFFFFFFFF)
    if rc:
        raise _err(_lib, rc, "sf_rng_seed")


# ---------------------------------------------------------------- launches
# sf_ew_desc header: op, dtype, ndim, n_in, in[3], imm[3]; the geometry
# (shape[8], strides[3][8]) is packed once per shape signature by the caller.
EW_HEAD = struct.Struct("<iiii3Q3d")
EW_GEOM = struct.Struct("<8q24q")


def pack_geometry(out_shape: Sequence[int], strides: Sequence[Sequence[int]]) -> bytes:
    nd = len(out_shape)
    shp = list(out_shape) + [1] * (MAX_DIMS - nd)
    flat: List[int] = []
    for j in range(3):
        s = list(strides[j]) if j < len(strides) else []
        s = s + [0] * (MAX_DIMS - len(s))
        flat.extend(s)
    return EW_GEOM.pack(*shp, *flat)


def elementwise(dev: int, op: int, dtype_tag: int, ndim: int, n_in: int, ptrs, imms,
                geometry: bytes, out_nbytes: int) -> DeviceBuffer:
    desc = EW_HEAD.pack(op, dtype_tag, ndim, n_in, *ptrs, *imms) + geometry
    out, ref = _outslot()
    rc = _lib.sf_elementwise(dev, desc, ref)
    if rc:
        raise _err(_lib, rc, "elementwise")
    return DeviceBuffer(dev, out.value, out_nbytes)


def elementwise_into(dev: int, op: int, dtype_tag: int, ndim: int, n_in: int, ptrs, imms,
                     geometry: bytes, out_ptr: int) -> None:
    """Elementwise launch writing into an existing buffer (in-place updates)."""
    desc = EW_HEAD.pack(op, dtype_tag, ndim, n_in, *ptrs, *imms) + geometry
    out = ctypes.c_void_p(out_ptr)
    rc = _lib.sf_elementwise(dev, desc, ctypes.byref(out))
    if rc:
        raise _err(_lib, rc, "elementwise")


def reduce(dev: int, op: int, dtype_tag: int, shape, axes_mask: int, src: int,
           out_nbytes: int) -> DeviceBuffer:
    shp = struct.pack("<%dq" % len(shape), *shape) if shape else b"\0" * 8
    out, ref = _outslot()
    rc = _lib.sf_reduce(dev, op, dtype_tag, len(shape), shp, axes_mask, src, ref)
    if rc:
        raise _err(_lib, rc, "reduce")
    return DeviceBuffer(dev, out.value, out_nbytes)


def matmul(dev: int, dtype_tag: int, m: int, n: int, k: int, a: int, ta: int, b: int, tb: int,
           out_nbytes: int) -> DeviceBuffer:
    out, ref = _outslot()
    rc = _lib.sf_matmul(dev, dtype_tag, m, n, k, a, ta, b, tb, ref)
    if rc:
        raise _err(_lib, rc, "matmul")
    return DeviceBuffer(dev, out.value, out_nbytes)


def transpose2d(dev: int, dtype_tag: int, rows: int, cols: int, src: int,
                out_nbytes: int) -> DeviceBuffer:
    out, ref = _outslot()
    rc = _lib.sf_transpose2d(dev, dtype_tag, rows, cols, src, ref)
    if rc:
        raise _err(_lib, rc, "transpose")
    return DeviceBuffer(dev, out.value, out_nbytes)


def fill(dev: int, dtype_tag: int, n: int, value: float, out_nbytes: int) -> DeviceBuffer:
    require_device()
    out, ref = _outslot()
    rc = _lib.sf_fill(dev, dtype_tag, n, value, ref)
    if rc:
        raise _err(_lib, rc, "fill")
    return DeviceBuffer(dev, out.value, out_nbytes)


def eye(dev: int, dtype_tag: int, n: int, out_nbytes: int) -> DeviceBuffer:
    require_device()
    out, ref = _outslot()
    rc = _lib.sf_eye(dev, dtype_tag, n, ref)
    if rc:
        raise _err(_lib, rc, "eye")
    return DeviceBuffer(dev, out.value, out_nbytes)


def cast(dev: int, src_tag: int, dst_tag: int, n: int, src: int, out_nbytes: int) -> DeviceBuffer:
    out, ref = _outslot()
    rc = _lib.sf_cast(dev, src_tag, dst_tag, n, src, ref)
    if rc:
        raise _err(_lib, rc, "cast")
    return DeviceBuffer(dev, out.value, out_nbytes)


def rng(dev: int, kind: int, dtype_tag: int, n: int, out_nbytes: int) -> DeviceBuffer:
    require_device()
    out, ref = _outslot()
    rc = _lib.sf_rng(dev, kind, dtype_tag, n, 0xFFFFFFFFFFFFFFFF, ref)
    if rc:
        raise _err(_lib, rc, "rng")
    return DeviceBuffer(dev, out.value, out_nbytes)


def dropout(dev: int, dtype_tag: int, n: int, x: int, u: int, u_tag: int, rate: float,
            nbytes: int):
    out, ref = _outslot()
    m2 = _tls.out2
    m2.value = None
    rc = _lib.sf_dropout(dev, dtype_tag, n, x, u or None, u_tag, rate, ref, _tls.out2ref)
    if rc:
        raise _err(_lib, rc, "dropout")
    return DeviceBuffer(dev, out.value, nbytes), DeviceBuffer(dev, m2.value, nbytes)


# ---------------------------------------------------------------- JIT + plans
def jit_compile(name: str, source: str) -> int:
    L = load_library()
    out = ctypes.c_void_p(0)
    rc = L.sf_jit_compile(name.encode(), source.encode(), ctypes.byref(out))
    if rc:
        raise _err(L, rc, f"jit compile {name}")
    return out.value


class NativePlan:
    """Owns a sf_plan handle (a lowered graph segment on one device)."""

    __slots__ = ("handle", "dev", "n_in", "n_out", "_in_arr", "_out_arr", "n_launches",
                 "_lock")

    def __init__(self, dev: int, desc: bytes, n_in: int, n_out: int):
        L = require_device()
        h = ctypes.c_void_p(0)
        rc = L.sf_plan_create(dev, desc, len(desc), ctypes.byref(h))
        if rc:
            raise _err(L, rc, "plan create")
        self.handle = h.value
        self.dev = dev
        self.n_in = n_in
        self.n_out = n_out
        self._in_arr = (ctypes.c_void_p * max(1, n_in))()
        self._out_arr = (ctypes.c_void_p * max(1, n_out))()
        info = [ctypes.c_int(0) for _ in range(4)]
        L.sf_plan_info(self.handle, *[ctypes.byref(x) for x in info])
        self.n_launches = info[3].value
        self._lock = threading.Lock()

    def run(self, in_ptrs: Sequence[int]) -> List[int]:
        with self._lock:
            arr = self._in_arr
            arr[:len(in_ptrs)] = in_ptrs  # one slice store (per-item stores cost ~0.15 us each)
            outs = self._out_arr
            rc = _lib.sf_plan_run(self.handle, arr, outs)
            if rc:
                raise _err(_lib, rc, "plan run")
            return outs[: self.n_out]

    def profile(self, enable: bool) -> None:
        rc = _lib.sf_plan_profile(self.handle, int(enable))
        if rc:
            raise _err(_lib, rc, "plan profile")

    def step_stats(self) -> List[tuple]:
        """[(step kind, total ms, runs)] accumulated while profiling."""
        n = ctypes.c_int(0)
        _lib.sf_plan_info(self.handle, None, None, ctypes.byref(n), None)
        out = []
        kind, ms, runs = ctypes.c_int(0), ctypes.c_double(0), ctypes.c_uint64(0)
        for s in range(n.value):
            _lib.sf_plan_step_stats(self.handle, s, ctypes.byref(kind), ctypes.byref(ms),
                                    ctypes.byref(runs))
            out.append((kind.value, ms.value, runs.value))
        return out

    def __del__(self):
        h = self.handle
        if h:
            self.handle = 0
            try:
                _lib.sf_plan_destroy(h)
            except Exception:
                pass


class WhileGraph:
    """Device-side control flow (csrc/sf_graph.cu): fixed buffers plus a CUDA
    graph with a WHILE conditional node, or (is_if) an IF node with an else
    branch for cond."""

    def __init__(self, dev: int, is_if: bool = False, plain: bool = False):
        L = require_device()
        h = ctypes.c_void_p(0)
        create = L.sf_graph_create if plain else L.sf_cond_create if is_if else L.sf_while_create
        rc = create(dev, ctypes.byref(h))
        if rc:
            raise _err(L, rc, "while create")
        self.handle = h.value
        self.dev = dev

    def buffer(self, nbytes: int) -> int:
        p = ctypes.c_void_p(0)
        rc = _lib.sf_while_buffer(self.handle, max(1, nbytes), ctypes.byref(p))
        if rc:
            raise _err(_lib, rc, "while buffer")
        return p.value

    def capture_begin(self, part: int) -> None:
        rc = _lib.sf_while_capture_begin(self.handle, part)
        if rc:
            raise _err(_lib, rc, "while capture begin")

    def set_cond(self, pred_ptr: int) -> None:
        rc = _lib.sf_while_set_cond(self.handle, pred_ptr)
        if rc:
            raise _err(_lib, rc, "while set cond")

    def capture_end(self, part: int) -> None:
        rc = _lib.sf_while_capture_end(self.handle, part)
        if rc:
            raise _err(_lib, rc, "while capture end")

    def launch(self) -> None:
        rc = _lib.sf_while_launch(self.handle)
        if rc:
            raise _err(_lib, rc, "while launch")

    def __del__(self):
        h = self.handle
        if h:
            self.handle = 0
            try:
                _lib.sf_while_destroy(h)
            except Exception:
                pass
