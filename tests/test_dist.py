"""Host logic of the C5 data-parallel gradient exchange (paper_1903_01855_b200/dist.py),
run on CPU with the gloo backend at world_size 2."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_01855_b200.dist import BucketAllReduce

SHAPES = [(7, 7, 3, 8), (8,), (8,), (3, 3, 8, 16), (16,), (1000,), (16, 1000)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, bucket_bytes, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(rank)
        grads = [torch.randn(s, generator=g) for s in SHAPES]
        red = BucketAllReduce([t.numel() for t in grads], torch.float32, "cpu",
                              bucket_bytes=bucket_bytes)
        red(grads)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), nb=len(red.buckets),
                 *[t.numpy() for t in grads])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bucket_bytes", [64, 4096, 25 << 20])
def test_bucket_allreduce_gloo_world2(tmp_path, bucket_bytes):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), bucket_bytes, str(tmp_path)), nprocs=world,
             join=True)
    per_rank = []
    for r in range(world):
        g = torch.Generator().manual_seed(r)
        per_rank.append([torch.randn(s, generator=g) for s in SHAPES])
    expect = [sum(p[i] for p in per_rank).numpy() for i in range(len(SHAPES))]
    # sum order over ranks is fixed for two ranks up to commutativity: exact
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npz")
        for i, e in enumerate(expect):
            np.testing.assert_allclose(got[f"arr_{i}"], e, rtol=1e-6, atol=1e-6)
        if bucket_bytes == 64:
            assert int(got["nb"]) >= len(SHAPES) - 2
        if bucket_bytes == 25 << 20:
            assert int(got["nb"]) == 1


def test_bucket_assignment_reverse_order():
    red = BucketAllReduce([10, 10, 10, 10], torch.float32, "cpu", bucket_bytes=80)
    assert red.buckets == [[3, 2], [1, 0]]
    assert [f.numel() for f in red.flat] == [20, 20]
    red = BucketAllReduce([100, 1], torch.float32, "cpu", bucket_bytes=8)
    assert red.buckets == [[1], [0]]  # an oversized tensor gets its own bucket
