"""Generate golden fixtures by running the REFERENCE itself (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports the reference package from /root/reference/pkg/src (read-only) and
records, through its own public API and stock code paths:

* leapfrog (stageflow/bench.py:147-183): q,p after 1 and 10 trajectories,
  eager and staged, for B in {10, 200, 1000}; checksums for 1e4 / 1e5;
* mlp_train (bench.py:103-144): per-iteration losses, 10 iterations,
  B in {8, 32, 256};
* C2 microbenchmark (builder-defined, tanh registered with register_op):
  chain output and d sum / dx;
* the SGF1 bytes (serial.serialize) of the traced graphs and their trace
  counts — the structure-parity oracle;
* L2HMC sampler outputs (builder-defined; plugin ops registered with numpy
  kernels) — see paper_1903_01855_b200/workloads/l2hmc.py.

The fixtures travel to the GPU box; /root/reference does not.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import stageflow as ref  # noqa: E402
from stageflow import bench as ref_bench  # noqa: E402
from stageflow.ops import OpDef, register_op  # noqa: E402
from stageflow.serial import serialize  # noqa: E402


def _fresh(workers=1, seed=0):
    ref.init_runtime(ref.RuntimeOptions(executor_workers=workers, seed=seed))


def leapfrog_fixtures(out):
    for b in (10, 200, 1000, 10000, 100000):
        for mode in ("eager", "staged"):
            if mode == "eager" and b > 10000:
                continue
            _fresh()
            cfg = ref_bench.BenchConfig(workload="leapfrog", mode=mode, batch_size=b)
            wl = ref_bench._Leapfrog(cfg, mode)
            v1 = wl.run_iteration()
            for _ in range(9):
                v10 = wl.run_iteration()
            if b <= 1000:
                out[f"leapfrog_{mode}_{b}_t1"] = v1
                out[f"leapfrog_{mode}_{b}_t10"] = v10
            else:
                out[f"leapfrog_{mode}_{b}_t10_sum"] = np.array([np.sum(v10.astype(np.float64)),
                                                                 np.sum(np.square(v10.astype(np.float64)))])
                out[f"leapfrog_{mode}_{b}_t10_head"] = v10[:64]
            if mode == "staged":
                pf = wl.staged_functions[0]
                gf = pf.cached_functions()[0].graph
                out[f"leapfrog_graph_{b}"] = np.frombuffer(serialize(gf), dtype=np.uint8)
                out[f"leapfrog_trace_count_{b}"] = np.array([pf.trace_count])


def mlp_fixtures(out):
    for b in (8, 32, 256):
        for mode in ("eager", "staged"):
            _fresh()
            cfg = ref_bench.BenchConfig(workload="mlp_train", mode=mode, batch_size=b)
            wl = ref_bench._MLPTrain(cfg, mode)
            losses = [wl.run_iteration() for _ in range(10)]
            out[f"mlp_{mode}_{b}_losses"] = np.array(losses, dtype=np.float64)
            out[f"mlp_{mode}_{b}_w1_after"] = wl.w1.numpy()
            if mode == "staged":
                stats = ref.get_runtime().stats.snapshot()
                out[f"mlp_staged_{b}_counts"] = np.array(
                    [wl.forward_loss.trace_count, wl.apply_updates.trace_count,
                     stats["derived_traces"]])
                gf = wl.forward_loss.cached_functions()[0].graph
                out[f"mlp_fwd_graph_{b}"] = np.frombuffer(serialize(gf), dtype=np.uint8)
                bwd = gf._fwd_bwd[1].graph
                out[f"mlp_bwd_graph_{b}"] = np.frombuffer(serialize(bwd), dtype=np.uint8)


def register_ref_plugins():
    """numpy plugin ops in the reference runtime (same names/semantics as
    paper_1903_01855_b200/plugins.py)."""
    from oracle.ref_plugins import register_all

    register_all(ref, OpDef, register_op)


def c2_fixtures(out):
    from oracle import workloads_np

    _fresh()
    register_ref_plugins()
    x, ws, bs = workloads_np.c2_params(0)
    tx = ref.constant(x)
    tws = [ref.constant(w) for w in ws]
    tbs = [ref.constant(b) for b in bs]

    def chain(v):
        for w, b in zip(tws, tbs):
            v = ref.dispatch("tanh", [ref.add(ref.matmul(v, w), b)])[0]
        return v

    eager = chain(tx).numpy()
    pf = ref.stage(chain)
    staged = pf(tx).numpy()
    with ref.Tape() as t:
        t.watch(tx)
        y = ref.reduce_sum(chain(tx))
    grad = t.gradient(y, tx).numpy()
    out["c2_eager"] = eager
    out["c2_staged"] = staged
    out["c2_grad"] = grad
    gf = pf.cached_functions()[0].graph
    out["c2_graph"] = np.frombuffer(serialize(gf), dtype=np.uint8)


def l2hmc_fixtures(out):
    from paper_1903_01855_b200.workloads import l2hmc

    for b in (16, 200):
        for mode in ("eager", "staged"):
            ref.init_runtime(ref.RuntimeOptions(executor_workers=1, seed=0))
            register_ref_plugins()
            sampler = l2hmc.L2HMCSampler(ref, batch=b, mode=mode, seed=0)
            res = [sampler.run_iteration() for _ in range(3)]
            out[f"l2hmc_{mode}_{b}"] = np.stack(res)
            if mode == "staged":
                pf = sampler.staged_functions[0]
                out[f"l2hmc_trace_count_{b}"] = np.array([pf.trace_count])


def resnet_fixtures(out):
    """ResNet-50 (full widths) at 64x64, batch 4: 3 SGD steps on the reference."""
    from paper_1903_01855_b200.workloads import resnet

    for tag, dt in (("grad0", ref.float32), ("grad64", ref.float64)):
        ref.init_runtime(ref.RuntimeOptions(executor_workers=1, seed=0))
        register_ref_plugins()
        tr = resnet.ResNetTrain(ref, batch=4, mode="eager", image=64, seed=0, dtype=dt)
        with ref.Tape() as t:
            loss = tr.forward_loss(tr.x, tr.labels)
        grads = t.gradient(loss, tr.model.params)
        out[f"resnet_{tag}_loss"] = np.array([float(loss)])
        for i in (0, 1, 2, 3, 10, 100, 159, 160):
            out[f"resnet_{tag}_{i}"] = grads[i].numpy().ravel()[:4096]  # keep fixtures small
    ref.init_runtime(ref.RuntimeOptions(executor_workers=1, seed=0))
    register_ref_plugins()
    tr = resnet.ResNetTrain(ref, batch=4, mode="staged", image=64, seed=0, dtype=ref.float64)
    out["resnet_f64_losses"] = np.array([tr.run_iteration() for _ in range(3)])
    for mode in ("eager", "staged"):
        ref.init_runtime(ref.RuntimeOptions(executor_workers=1, seed=0))
        register_ref_plugins()
        tr = resnet.ResNetTrain(ref, batch=4, mode=mode, image=64, seed=0)
        out[f"resnet_{mode}_losses"] = np.array([tr.run_iteration() for _ in range(3)])
        out[f"resnet_{mode}_fc_b"] = tr.model.fc_b.numpy()
        out[f"resnet_{mode}_stem_w"] = tr.model.stem[0].numpy()[:, :, :, :4]
        if mode == "staged":
            out["resnet_trace_counts"] = np.array([tr.forward_loss.trace_count,
                                                   tr.apply_updates.trace_count])


def main():
    out = {}
    leapfrog_fixtures(out)
    mlp_fixtures(out)
    c2_fixtures(out)
    if "--no-l2hmc" not in sys.argv:
        l2hmc_fixtures(out)
    resnet_fixtures(out)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    meta = {"reference": "/root/reference/pkg/src/stageflow", "numpy": np.__version__,
            "keys": sorted(out)}
    with open(os.path.join(HERE, "golden_meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
