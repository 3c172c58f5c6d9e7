"""Data-parallel communication (config C5) without torch.

One process per GPU.  ``Communicator`` wraps an NCCL communicator created
through the C-ABI (sf_comm_init, csrc/sf_comm.cpp); rank 0's unique id
reaches the other ranks over a plain TCP rendezvous (``rendezvous``), the
way torchrun's environment describes the job (RANK, WORLD_SIZE,
MASTER_ADDR, MASTER_PORT; the id travels on MASTER_PORT + 1 unless
SF_COMM_PORT says otherwise).

The gradient exchange is folded into the staged backward: inside
``gradient_allreduce(comm, variables)``, a tape's staged backward that
produces gradients of those variables is compiled with its gradient outputs
marked, and the executor issues one grouped in-place all-reduce per bucket
(``plan_buckets``) right after the plan step that produced the bucket's
last gradient — the transfer overlaps the rest of the backward, and the
plan joins it back before returning.  Sampler chains (C1/C3) shard with no
collective at all.  The reference has no distribution.
"""
from __future__ import annotations

import os
import socket
import struct
import threading
import time
from contextlib import contextmanager
from typing import Iterable, List, Optional, Sequence, Tuple

BUCKET_BYTES = 25 << 20
UID_BYTES = 128


def _recv_exact(sock: socket.socket, n: int) -> bytes:
    buf = b""
    while len(buf) < n:
        chunk = sock.recv(n - len(buf))
        if not chunk:
            raise ConnectionError("rendezvous peer closed the connection")
        buf += chunk
    return buf


def rendezvous(rank: int, world: int, addr: str, port: int, make_id,
               timeout: float = 120.0) -> bytes:
    """Rank 0 calls ``make_id()`` and serves the bytes to ranks 1..world-1
    over TCP; every rank returns the same id.  (A length-prefixed payload,
    so any id size works; the tests use it with world 2 on CPU.)"""
    if world == 1:
        return make_id()
    deadline = time.monotonic() + timeout
    if rank == 0:
        uid = make_id()
        srv = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        srv.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        srv.bind((addr, port))
        srv.listen(world)
        srv.settimeout(timeout)
        try:
            served = 0
            while served < world - 1:
                conn, _ = srv.accept()
                with conn:
                    conn.sendall(struct.pack("<I", len(uid)) + uid)
                    _recv_exact(conn, 1)  # ack
                served += 1
        finally:
            srv.close()
        return uid
    while True:
        try:
            with socket.create_connection((addr, port), timeout=5.0) as c:
                n = struct.unpack("<I", _recv_exact(c, 4))[0]
                uid = _recv_exact(c, n)
                c.sendall(b"k")
                return uid
        except OSError:
            if time.monotonic() > deadline:
                raise
            time.sleep(0.05)


class Communicator:
    """An NCCL communicator of one rank (device ``dev``)."""

    def __init__(self, world: int, rank: int, dev: int = 0, uid: Optional[bytes] = None):
        from . import _native

        if uid is None:
            if world != 1:
                raise ValueError("a multi-rank communicator needs the rank-0 unique id")
            uid = _native.comm_unique_id()
        self.world = world
        self.rank = rank
        self.dev = dev
        self.handle = _native.comm_init(dev, world, rank, uid)

    @classmethod
    def from_env(cls, dev: Optional[int] = None) -> "Communicator":
        """Rank / world / rendezvous address from the torchrun environment."""
        from . import _native

        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if dev is None:
            dev = int(os.environ.get("LOCAL_RANK", "0"))
        addr = os.environ.get("MASTER_ADDR", "127.0.0.1")
        port = int(os.environ.get("SF_COMM_PORT", int(os.environ.get("MASTER_PORT", "29500")) + 1))
        uid = rendezvous(rank, world, addr, port, _native.comm_unique_id)
        return cls(world, rank, dev, uid)

    def allreduce(self, tensors: Sequence, scale: float = 1.0) -> List:
        """Sum over ranks (times ``scale``) of each tensor, as new tensors
        (the inputs are immutable: each is copied once, reduced in place)."""
        from . import _native
        from .tensor import Tensor

        outs, ptrs, counts = [], [], []
        for t in tensors:
            buf = _native.alloc(self.dev, t.nbytes)
            _native.copy_d2d(self.dev, buf.ptr, t._ptr(), t.nbytes)
            outs.append(Tensor._adopt(t.dtype, t.shape, t.device, buf))
            ptrs.append(buf.ptr)
            counts.append(t.size)
        if outs:
            _native.allreduce(self.handle, ptrs, counts, tensors[0].dtype.tag, scale)
        return outs

    def close(self) -> None:
        from . import _native

        h, self.handle = self.handle, 0
        _native.comm_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def plan_buckets(sizes: Sequence[int], bucket_bytes: int = BUCKET_BYTES) -> List[List[int]]:
    """Split items, in the order a backward produces them, into consecutive
    buckets of about ``bucket_bytes`` (an item larger than that is a bucket
    of its own).  Returns lists of indices into ``sizes``."""
    buckets: List[List[int]] = []
    cur: List[int] = []
    size = 0
    for i, nb in enumerate(sizes):
        if cur and size + nb > bucket_bytes:
            buckets.append(cur)
            cur, size = [], 0
        cur.append(i)
        size += nb
    if cur:
        buckets.append(cur)
    return buckets


# ---------------------------------------------------------------------------
# gradient all-reduce folded into the staged backward
# ---------------------------------------------------------------------------


class GradientCollective:
    __slots__ = ("comm", "ids", "bucket_bytes", "scale")

    def __init__(self, comm: Communicator, variables: Iterable, bucket_bytes: int, scale: float):
        self.comm = comm
        self.ids = frozenset(id(v) for v in variables)
        self.bucket_bytes = bucket_bytes
        self.scale = scale


_local = threading.local()


def active_collective() -> Optional[GradientCollective]:
    return getattr(_local, "spec", None)


@contextmanager
def gradient_allreduce(comm: Communicator, variables: Iterable, bucket_bytes: int = BUCKET_BYTES,
                       scale: float = 1.0):
    """Within the block, staged backwards that produce gradients of
    ``variables`` all-reduce them across ``comm`` (sum, times ``scale``),
    bucket by bucket as the backward produces them."""
    prev = active_collective()
    _local.spec = GradientCollective(comm, variables, bucket_bytes, scale)
    try:
        yield _local.spec
    finally:
        _local.spec = prev


def output_spec(spec: GradientCollective, outputs: Sequence[int]) -> Tuple:
    """Program-cache key part for a backward whose ``outputs`` are reduced."""
    return (spec.comm.handle, tuple(outputs), spec.bucket_bytes, float(spec.scale))
