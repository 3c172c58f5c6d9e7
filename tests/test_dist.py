"""Host logic of the data-parallel exchange (paper_1903_01855_b200/comm.py),
on CPU: the TCP rendezvous that hands rank 0's NCCL unique id to the other
ranks (world 2, two processes) and the bucket planning of the gradient
all-reduce."""
import multiprocessing as mp
import os
import socket

import pytest

from paper_1903_01855_b200.comm import plan_buckets, rendezvous


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q):
    uid = rendezvous(rank, world, "127.0.0.1", port, lambda: os.urandom(128), timeout=60)
    q.put((rank, uid))


@pytest.mark.parametrize("world", [2, 3])
def test_rendezvous_hands_rank0_id_to_every_rank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=90) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    assert len(got) == world and len(set(got.values())) == 1
    assert len(got[0]) == 128


def test_rendezvous_world1_is_local():
    assert rendezvous(0, 1, "127.0.0.1", 1, lambda: b"x" * 128) == b"x" * 128


def test_plan_buckets_in_production_order():
    assert plan_buckets([40, 40, 40, 40], bucket_bytes=80) == [[0, 1], [2, 3]]
    assert plan_buckets([400, 4], bucket_bytes=8) == [[0], [1]]  # oversized: own bucket
    assert plan_buckets([], bucket_bytes=8) == []
    sizes = [4 * n for n in (9408, 64, 64, 4096, 64, 64, 36864, 64)]
    buckets = plan_buckets(sizes, bucket_bytes=64 << 10)
    assert [i for b in buckets for i in b] == list(range(len(sizes)))
    assert all(sum(sizes[i] for i in b[:-1]) < 64 << 10 for b in buckets)
