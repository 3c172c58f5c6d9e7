"""Round-2 golden fixtures, produced by running the REFERENCE itself at the
benchmarked configurations (build container only; ~minutes of CPU):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_r2.py [--skip-resnet]

Imports the reference package from /root/reference/pkg/src (read-only) and
records, through its own public API (stage / Tape / dispatch, numpy plugin
ops registered with its ``register_op``, oracle/ref_plugins.py):

* ``l2hmc_graph_runtime_200`` / ``l2hmc_graph_inputs_200``: the SGF1 bytes
  (stageflow/serial.py serialize) of the traced L2HMC transition — draws
  inside the program, and draws passed in — and their trace counts;
* ``l2hmc_inputs_1e5_t{1,2,3}_*``: the L2HMC sampler (draws passed in, drawn
  from default_rng(0) in the runtime's order) staged on the reference at the
  headline batch, 100,000 chains, for three transitions: the first 4096
  chains of the state and accept probabilities, and float64 sums over all
  chains;
* ``microop_*``: the reference's microop_loop workload — values, the staged
  graph's SGF1 bytes, and run_benchmark's trace/cache/copy counters;
* ``resnet_c4_{f32,f64}_*``: ResNet-50 at config C4 (batch 32, 224x224x3,
  seed 0) — the loss and the gradients of all 161 parameters of one tape
  step, in float32 and float64: per-parameter float64 norms and sums, and the
  first 2048 values of 12 parameters spread from the stem to the classifier.

The fixtures travel to the GPU box; /root/reference does not.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import stageflow as ref  # noqa: E402
from stageflow.ops import OpDef, register_op  # noqa: E402
from stageflow.serial import serialize  # noqa: E402

L2HMC_B = 100_000
HEAD = 4096
RESNET_SLICE = 2048
# stem conv, stem bn, layer1.0 conv1/conv2, layer1 down, layer2, layer3 (x3),
# layer4 conv3 / bn, fc weight and bias
RESNET_PARAMS = (0, 1, 3, 6, 12, 40, 80, 100, 120, 150, 157, 159, 160)


def _fresh():
    from oracle.ref_plugins import register_all  # includes the nn ops

    ref.init_runtime(ref.RuntimeOptions(executor_workers=1, seed=0))
    register_all(ref, OpDef, register_op)


def l2hmc_graphs(out):
    from paper_1903_01855_b200.workloads import l2hmc

    for draws in ("runtime", "inputs"):
        _fresh()
        s = l2hmc.L2HMCSampler(ref, batch=200, mode="staged", seed=0, draws=draws)
        s.step()
        s.step()
        pf = s.staged_functions[0]
        gf = pf.cached_functions()[0].graph
        out[f"l2hmc_graph_{draws}_200"] = np.frombuffer(serialize(gf), dtype=np.uint8)
        out[f"l2hmc_graph_{draws}_200_trace_count"] = np.array([pf.trace_count])


def l2hmc_headline(out):
    from paper_1903_01855_b200.workloads import l2hmc

    _fresh()
    s = l2hmc.L2HMCSampler(ref, batch=L2HMC_B, mode="staged", seed=0, draws="inputs")
    for t in (1, 2, 3):
        t0 = time.time()
        s.step()
        x, a = s.x.numpy(), s.accept.numpy()
        out[f"l2hmc_inputs_1e5_t{t}_x_head"] = x[:HEAD]
        out[f"l2hmc_inputs_1e5_t{t}_acc_head"] = a[:HEAD]
        x64, a64 = x.astype(np.float64), a.astype(np.float64)
        out[f"l2hmc_inputs_1e5_t{t}_sums"] = np.array(
            [x64.sum(), np.square(x64).sum(), a64.sum(), np.square(a64).sum()])
        print(f"l2hmc 1e5 transition {t}: {time.time() - t0:.1f}s", flush=True)


def resnet_c4(out):
    from paper_1903_01855_b200.workloads import resnet

    for tag, dt in (("f32", ref.float32), ("f64", ref.float64)):
        t0 = time.time()
        _fresh()
        tr = resnet.ResNetTrain(ref, batch=32, mode="eager", image=224, seed=0, dtype=dt)
        with ref.Tape() as t:
            loss = tr.forward_loss(tr.x, tr.labels)
        grads = t.gradient(loss, tr.model.params)
        out[f"resnet_c4_{tag}_loss"] = np.array([float(loss)])
        norms, sums = [], []
        for g in grads:
            a = g.numpy().astype(np.float64).ravel()
            norms.append(np.sqrt(np.square(a).sum()))
            sums.append(a.sum())
        out[f"resnet_c4_{tag}_grad_norms"] = np.array(norms)
        out[f"resnet_c4_{tag}_grad_sums"] = np.array(sums)
        for i in RESNET_PARAMS:
            out[f"resnet_c4_{tag}_grad_{i}"] = grads[i].numpy().ravel()[:RESNET_SLICE]
        del grads, loss, t, tr
        print(f"resnet c4 {tag}: {time.time() - t0:.1f}s", flush=True)
    out["resnet_c4_params"] = np.array(RESNET_PARAMS)


def microop_fixtures(out):
    """_MicroOpLoop (stageflow/bench.py:186-206): values, graph bytes, and the
    reference harness's trace/copy counters (run_benchmark, :237-273)."""
    from stageflow import bench as ref_bench

    for mode in ("eager", "staged"):
        _fresh()
        cfg = ref_bench.BenchConfig(workload="microop_loop", mode=mode, batch_size=1,
                                    iterations=3, warmup=1, repeats=2)
        wl = ref_bench._MicroOpLoop(cfg, mode)
        out[f"microop_{mode}_values"] = np.array([wl.run_iteration() for _ in range(3)])
        if mode == "staged":
            gf = wl.staged_functions[0].cached_functions()[0].graph
            out["microop_graph"] = np.frombuffer(serialize(gf), dtype=np.uint8)
        _fresh()
        rep = ref_bench.run_benchmark(cfg)
        out[f"microop_{mode}_report"] = np.array([rep.trace_count, rep.cache_size, rep.copies])


def main():
    out = {}
    microop_fixtures(out)
    l2hmc_graphs(out)
    l2hmc_headline(out)
    if "--skip-resnet" not in sys.argv:
        resnet_c4(out)
    path = os.path.join(HERE, "golden_r2.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
