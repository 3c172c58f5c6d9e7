"""Data parallelism across GPUs (BASELINE config C5).

One process per GPU, ``torch.distributed`` over NCCL for the plumbing.  The
only exchange step in the whole build is the ResNet-50 gradient
all-reduce: after each rank's staged forward + backward, the 161 gradient
buffers are packed into ~25 MB flat buckets, sum-reduced with NCCL on the
backend's own CUDA stream (so it orders with our kernels without host
syncs), unpacked in place, and applied by the staged update with the
learning rate divided by the world size.  Sampler chains (C1/C3) shard with
no collective at all.

``torch_view`` exposes a backend tensor's HBM buffer to torch without a
copy (CUDA array interface); ``BucketAllReduce`` works on any list of torch
tensors, so its host logic is tested on CPU with gloo (tests/test_dist.py).
"""
from __future__ import annotations

from typing import List, Sequence

BUCKET_BYTES = 25 << 20


def torch_view(t):
    """A torch CUDA tensor aliasing the backend tensor's device buffer."""
    import torch

    from .tensor import Tensor

    assert isinstance(t, Tensor) and not t.is_symbolic
    buf = t._device_buffer()
    typestr = {"float32": "<f4", "float64": "<f8", "int32": "<i4", "boolean": "|b1"}[t.dtype.value]

    class _Iface:
        __cuda_array_interface__ = {"shape": (t.size,), "typestr": typestr,
                                    "data": (buf.ptr, False), "version": 3, "stream": None}

    view = torch.as_tensor(_Iface(), device=f"cuda:{buf.dev}")
    return view


class BucketAllReduce:
    """Sum-all-reduce a fixed list of tensors through flat buckets.

    Tensors are assigned to buckets in reverse order (the backward pass
    produces the last layers' gradients first, so late buckets could start
    early); each bucket is one collective.
    """

    def __init__(self, numels: Sequence[int], dtype, device, bucket_bytes: int = BUCKET_BYTES):
        import torch

        itemsize = torch.empty((), dtype=dtype).element_size()
        self.buckets: List[List[int]] = []
        cur, size = [], 0
        for i in reversed(range(len(numels))):
            nb = numels[i] * itemsize
            if cur and size + nb > bucket_bytes:
                self.buckets.append(cur)
                cur, size = [], 0
            cur.append(i)
            size += nb
        if cur:
            self.buckets.append(cur)
        self.flat = [torch.empty(sum(numels[i] for i in b), dtype=dtype, device=device)
                     for b in self.buckets]

    def __call__(self, tensors: Sequence, group=None) -> None:
        import torch.distributed as dist

        for b, flat in zip(self.buckets, self.flat):
            off = 0
            for i in b:
                n = tensors[i].numel()
                flat[off:off + n].copy_(tensors[i].reshape(-1))
                off += n
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
            off = 0
            for i in b:
                n = tensors[i].numel()
                tensors[i].reshape(-1).copy_(flat[off:off + n])
                off += n


def run_on_backend_stream(dev: int = 0):
    """Make torch's current stream the backend's stream (NCCL orders with our kernels)."""
    import torch

    from . import _native

    stream = torch.cuda.ExternalStream(_native.stream_of(dev))
    torch.cuda.set_stream(stream)
    return stream


class ResNetDataParallel:
    """C5: ResNet-50 DP step — local staged fwd/bwd, bucketed NCCL all-reduce,
    staged SGD with lr / world_size."""

    def __init__(self, sf, batch_per_rank: int, rank: int, world: int, image: int = 224,
                 width_div: int = 1):
        import numpy as np
        import torch

        from . import dtypes
        from .workloads import resnet

        self.sf = sf
        self.world = world
        # identical weights on every rank (same model seed); per-rank data below
        self.train = resnet.ResNetTrain(sf, batch=1, mode="staged", image=image, seed=0,
                                        width_div=width_div)
        rng = np.random.default_rng(1000 + rank)
        shape = (batch_per_rank, image, image, 3)
        self.x = sf.tensor_from_host(rng.standard_normal(shape).astype(np.float32), shape,
                                     sf.float32)
        self.labels = sf.tensor_from_host(rng.integers(0, 1000, size=(batch_per_rank,)),
                                          (batch_per_rank,), sf.int32)
        params = self.train.model.params
        self.reducer = BucketAllReduce([dtypes.element_count(p.shape) for p in params],
                                       torch.float32, "cuda")
        scale = -resnet.ResNetTrain.LR / world

        def apply_mean(*grads):
            for v, g in zip(params, grads):
                v.assign_add(sf.mul(g, scale))

        self.apply = sf.stage(apply_mean, name="resnet50_apply_mean_updates")

    def step(self):
        sf = self.sf
        with sf.Tape() as t:
            loss = self.train.forward_loss(self.x, self.labels)
        grads = t.gradient(loss, self.train.model.params)
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            self.reducer([torch_view(g) for g in grads])
        self.apply(*grads)
        return loss
