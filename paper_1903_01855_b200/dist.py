"""Data-parallel ResNet-50 training (BASELINE config C5).

One process per GPU; no torch anywhere on this path.  Every rank holds the
same weights (same model seed) and its own minibatch.  The step is the
reference's mlp_train pattern (stageflow/bench.py:131-144) — staged
forward + loss under a tape, the tape's staged backward, a staged update —
with the only exchange of the build folded into the backward: inside
``comm.gradient_allreduce`` the backward's plan sums each ~25 MB bucket of
weight gradients over the ranks with NCCL as soon as the bucket's last
gradient kernel has run (csrc/sf_comm.cpp, plan step 12), overlapping the
remaining backward; the update applies ``-lr / world * sum``.  BN statistics
stay per rank (standard DP).  The reference has no distribution
(SPEC.md:11).
"""
from __future__ import annotations

from .comm import BUCKET_BYTES, Communicator, gradient_allreduce


class ResNetDataParallel:
    """C5 step: local staged fwd/bwd with the bucketed all-reduce inside the
    backward plan, then the staged SGD update with lr / world."""

    def __init__(self, sf, batch_per_rank: int, comm: Communicator, image: int = 224,
                 width_div: int = 1, bucket_bytes: int = BUCKET_BYTES, seed: int = 0,
                 grad_scale: float = 1.0):
        import numpy as np

        from .workloads import resnet

        self.sf = sf
        self.comm = comm
        self.bucket_bytes = bucket_bytes
        self.grad_scale = grad_scale
        # identical weights on every rank (same model seed); per-rank data below
        self.train = resnet.ResNetTrain(sf, batch=1, mode="staged", image=image, seed=seed,
                                        width_div=width_div)
        rng = np.random.default_rng(1000 + comm.rank)
        shape = (batch_per_rank, image, image, 3)
        self.x = sf.tensor_from_host(rng.standard_normal(shape).astype(np.float32), shape,
                                     sf.float32)
        self.labels = sf.tensor_from_host(rng.integers(0, 1000, size=(batch_per_rank,)),
                                          (batch_per_rank,), sf.int32)
        params = self.train.model.params
        scale = -resnet.ResNetTrain.LR / comm.world

        def apply_mean(*grads):
            for v, g in zip(params, grads):
                v.assign_add(sf.mul(g, scale))

        self.apply = sf.stage(apply_mean, name="resnet50_apply_mean_updates")

    def step(self, x=None, labels=None):
        sf = self.sf
        params = self.train.model.params
        with sf.Tape() as t:
            loss = self.train.forward_loss(self.x if x is None else x,
                                           self.labels if labels is None else labels)
        with gradient_allreduce(self.comm, params, self.bucket_bytes, self.grad_scale):
            grads = t.gradient(loss, params)
        self.apply(*grads)
        return loss

    def backward_plans(self):
        """The native plans of the staged backward this step ran (tests read
        their step kinds to check where the all-reduce steps sit)."""
        from . import _native
        from .executor import _NativeSegment

        plans = []
        for pf in self.train.staged_functions:
            for cf in pf.cached_functions():
                fb = getattr(cf.graph, "_fwd_bwd", None)
                if not fb:
                    continue
                bwd = fb[1]
                graphs = [bwd.graph] + [c.graph for c in bwd.__dict__.get("_selected", {}).values()]
                for g in graphs:
                    for prog in (g._plan or {}).values():
                        if prog.collective is None:
                            continue
                        plans += [s.plan for s in prog.segments if isinstance(s, _NativeSegment)]
        return plans
