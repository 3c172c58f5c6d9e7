"""Benchmark driver (one JSON line on rank 0).

Headline (BASELINE.json metric "L2HMC samples/s ... staged vs eager"):
the L2HMC sampler (workloads/l2hmc.py) on the 2-D strongly-correlated
Gaussian, 10 leapfrog steps, staged, 100,000 chains per GPU (config C3's
largest chain count; weak scaling: N GPUs sample N x 1e5 independent chains,
no collective).  A step = one full transition (forward + backward
trajectories, direction draw, MH accept) of every chain.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--chains B]
    python bench.py --impl reference ...     # the CPU reference arm

``value``: samples/s with the chain state resident in HBM, timed per step
with CUDA events on the backend's stream (L2 flushed between steps), max
over ranks.  ``e2e``: the same metric through the public API with the chain
state uploaded from host memory and the new state + accept probabilities
read back every step.  Extra keys report config C1 (200 chains) staged and
eager, the reference-pinned leapfrog workload, and the C2 microbenchmark.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

_OPENBLAS_ENV = os.environ.get("OPENBLAS_NUM_THREADS")
FFMA_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # derived nominal FP32 SIMT peak


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--chains", type=int, default=100000)
    ap.add_argument("--quick", action="store_true", help="skip the extra workloads")
    ap.add_argument("--no-gate", action="store_true",
                    help="skip the same-seed eager==staged gate before timing")
    # the reference's benchmark contract (stageflow/cli.py bench): with
    # --workload, run paper_1903_01855_b200.benchmark instead of the headline
    from paper_1903_01855_b200.benchmark import add_bench_args

    add_bench_args(ap, required=False, warmup=False)
    return ap.parse_args()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def _compute_peaks():
    """FP32 SIMT and tcgen05 peaks measured on a B200 by tools/peaks.cu
    (profiles/r02_peaks.json); MEASURED_PEAKS.json has HBM and bf16 only."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_peaks.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class Clocks:
    """SM clock + throttle reasons sampled DURING the timed region.

    The timed region of the headline is a few ms, far below nvidia-smi's
    100 ms loop, so NVML is polled in-process every ~2 ms from a helper
    thread (ctypes releases the GIL); nvidia-smi is the fallback."""
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits
    NVML_BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
                 "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = (pynvml, h, reasons, mx)
            self.stop = threading.Event()

            def poll():
                while True:
                    self._nvml_row()
                    if self.stop.wait(0.002):
                        break

            self._nvml_row()
            self.reader = threading.Thread(target=poll, daemon=True)
            self.reader.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.reader = threading.Thread(target=self._read, daemon=True)
            self.reader.start()
            # the timed region can be a few ms: make sure the sampler is live
            # (first row in) before it starts, and take one more row at exit
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5 and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _nvml_row(self):
        pynvml, h, reasons, mx = self.nvml
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        bits = reasons(h)
        self.rows.append([str(sm), str(mx)] + ["Active" if bits & b else "Not Active"
                                               for b in self.NVML_BITS.values()])

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.reader.join(timeout=5)
            self._nvml_row()
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=10).stdout
                for line in out.splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# algorithmic work of a traced graph (SURVEY.md §8(d) definition)
# ---------------------------------------------------------------------------


def graph_work(gf):
    import numpy as np

    flops = 0
    n_ops = 0
    for n in gf.nodes:
        if n.op in ("constant", "reshape", "identity", "transpose", "broadcast_to"):
            continue
        n_ops += 1
        out = n.out_specs[0][1] if n.out_specs else ()
        if n.op == "matmul":
            (m, k), (_, nn) = gf.spec_of(n.inputs[0])[1], gf.spec_of(n.inputs[1])[1]
            flops += 2 * m * k * nn
        elif n.op in ("reduce_sum", "reduce_mean"):
            flops += int(np.prod(gf.spec_of(n.inputs[0])[1], dtype=np.int64))
        else:
            flops += int(np.prod(out, dtype=np.int64)) if out else 1
    return flops, n_ops


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port on host cores
# ---------------------------------------------------------------------------


_PORT = None


def _port_init(chains, seed):
    global _PORT
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import workloads_np

    _PORT = workloads_np.L2HMC(chains, seed=seed, runtime_seed=seed)


def _port_step(_=None):
    t = time.perf_counter()
    _PORT.transition()
    return time.perf_counter() - t


class PortPool:
    """The NumPy oracle port of the L2HMC transition (oracle/workloads_np.py),
    chains sharded contiguously over `workers` persistent processes (created
    once, before any timed step; each holds its shard's state)."""

    def __init__(self, chains: int, workers: int):
        import multiprocessing as mp

        self.chains, self.workers = chains, workers
        per = -(-chains // workers)
        sizes = [min(per, chains - i * per) for i in range(workers)]
        sizes = [n for n in sizes if n > 0]
        self.pools = []
        if len(sizes) == 1:
            _port_init(sizes[0], 1000)
        else:
            ctx = mp.get_context("fork")
            self.pools = [ctx.Pool(1, initializer=_port_init, initargs=(n, 1000 + i))
                          for i, n in enumerate(sizes)]
            for p in self.pools:  # fork + build the shard before timing
                p.apply(os.getpid)

    def step(self) -> float:
        """One transition of every chain; returns the wall time."""
        t = time.perf_counter()
        if not self.pools:
            _port_step()
        else:
            for r in [p.apply_async(_port_step) for p in self.pools]:
                r.get()
        return time.perf_counter() - t

    def close(self):
        for p in self.pools:
            p.terminate()


def host_info() -> dict:
    import numpy as np

    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")),
                         "")
    except OSError:
        pass
    blas = ""
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg["Build Dependencies"]["blas"]
        blas = f"{b.get('name')} {b.get('version')}"
    except Exception:  # noqa: BLE001 - informational only
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "numpy": np.__version__, "blas": blas,
            "OPENBLAS_NUM_THREADS": _OPENBLAS_ENV or "unset; 1 per port process (bench.py)"}


def cpu_port_rates(chains: int, steps: int, warmup: int = 1):
    """All-cores and one-process samples/s of the port at `chains` chains."""
    cores = os.cpu_count() or 1
    pool = PortPool(chains, cores)
    try:
        for _ in range(warmup):
            pool.step()
        dts = [pool.step() for _ in range(steps)]
    finally:
        pool.close()
    all_cores = chains * steps / sum(dts)
    one = PortPool(chains, 1)
    dt1 = one.step()
    return {"all_cores": all_cores, "all_cores_s_per_step": sum(dts) / steps,
            "workers_1": chains / dt1, "workers_1_s_per_step": dt1, "cores": cores}


def run_reference(a, rank, world):
    if rank != 0:
        return
    r = cpu_port_rates(a.chains, a.steps, a.warmup)
    value = r["all_cores"]
    sample = (f"the full config: {a.chains} chains x {a.steps} transitions (1 transition per "
              f"step), numpy oracle port (oracle/workloads_np.py L2HMC, pinned to the reference "
              f"run at 1e5 chains) sharded over {r['cores']} persistent processes")
    line = {
        "impl": "reference", "metric": "l2hmc_samples_per_sec", "value": value,
        "unit": "samples/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": r["all_cores_s_per_step"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "l2hmc_sampler_staged", "chains_per_gpu": a.chains,
                   "leapfrog_steps": 10, "x_dim": 2, "hidden": 10, "same_config": True},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": r["cores"], "kind": "port",
                         "sample": sample, "workers_1": r["workers_1"], "host": host_info()},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def gate_headline(sf, plugins, l2hmc, chains, seed, rank, transitions=1):
    """Eager and staged runs of the benchmarked program (same seeds, device
    Philox) must agree bit for bit before anything is timed."""
    import numpy as np

    outs = {}
    for mode in ("eager", "staged"):
        sf.init_runtime(sf.RuntimeOptions(seed=seed))
        plugins.install()
        s = l2hmc.L2HMCSampler(sf, chains, mode, seed=rank)
        outs[mode] = np.stack([s.run_iteration() for _ in range(transitions)])
    diff = float(np.max(np.abs(outs["eager"].astype(np.float64) - outs["staged"])))
    return {"passed": outs["eager"].tobytes() == outs["staged"].tobytes(),
            "transitions": transitions, "chains": chains, "max_abs_diff": diff,
            "criterion": "bitwise (reference gate: 1e-5)"}


def run_ours(a, rank, world, dist):
    import numpy as np
    import torch

    import paper_1903_01855_b200 as sf
    from paper_1903_01855_b200 import _native, plugins
    from paper_1903_01855_b200.workloads import l2hmc

    assert _native.device_count() > 0, "no CUDA device"
    gate = None
    if not a.no_gate:
        # the reference refuses to time without a same-seed eager == staged
        # check (stageflow/bench.py:216-234); here on the timed config itself
        gate = gate_headline(sf, plugins, l2hmc, a.chains, 1234 + rank, rank)
        if not gate["passed"]:
            if rank == 0:
                print(json.dumps({"metric": "l2hmc_samples_per_sec", "error": "gate failed",
                                  "gate": gate}), flush=True)
            sys.exit(2)
    sf.init_runtime(sf.RuntimeOptions(seed=1234 + rank))
    plugins.install()
    dev = 0
    stream = torch.cuda.ExternalStream(_native.stream_of(dev))
    peaks, peak_kind = _peaks()

    B = a.chains
    sampler = l2hmc.L2HMCSampler(sf, B, "staged", seed=rank)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        _native.sync(dev)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    t0 = time.perf_counter()
    for _ in range(a.warmup):
        sampler.step()
    _native.sync(dev)
    warm_s = time.perf_counter() - t0
    cf = sampler.transition.cached_functions()[0]
    prog = next(iter(cf.graph._plan.values()))
    flops_per_step, n_graph_ops = graph_work(cf.graph)

    # -- value: device-resident state, per-step CUDA events, L2 flushed between steps
    barrier()
    launches0 = _native.launch_count(dev)
    times = []
    with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for _ in range(a.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)  # > L2 (126 MB)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            sampler.step()
            e1.record(stream)
            times.append((e0, e1))
        _native.sync(dev)
        torch.cuda.synchronize()
    launches = _native.launch_count(dev) - launches0 - 0
    step_ms = [e0.elapsed_time(e1) for e0, e1 in times]
    total_s = sum(step_ms) / 1e3
    if dist is not None:
        t = torch.tensor([total_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_s = float(t.item())
    barrier()
    value = B * world * a.steps / total_s
    ms_per_step = total_s * 1e3 / a.steps

    # -- roofline of the dominant kernel: per-launch GPU time from plan events
    # (the same L2 flush before every profiled step as in the timed region:
    # the row kernel then refetches its code and weights as it does there)
    seg = prog.segments[0]
    seg.plan.profile(True)
    for _ in range(5):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        sampler.step()
    stats = seg.plan.step_stats()
    seg.plan.profile(False)
    jit_ms = [ms / runs for kind, ms, runs in stats if kind == 1 and runs]
    kern_ms = sum(jit_ms)
    achieved = flops_per_step / (kern_ms / 1e3) / 1e12 if kern_ms else 0.0
    # DRAM bytes per launch of the row kernel, from the committed ncu --set
    # full capture of this configuration (profiles/r01i_l2hmc_rows_full.md)
    traffic = None
    try:
        for name in ("r02_rows_traffic.json", "r01i_rows_traffic.json"):
            tp = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
            if os.path.exists(tp):
                with open(tp) as fh:
                    traffic = json.load(fh)["dram_bytes_per_launch"]
                break
    except (OSError, ValueError, KeyError):
        pass
    cpk = _compute_peaks()
    ffma_peak = cpk.get("ffma_tflops", FFMA_PEAK_TFLOPS)
    roofline = {"bound": "fp32", "achieved": achieved, "peak": ffma_peak,
                "unit": "TFLOP/s", "frac": achieved / ffma_peak, "traffic": traffic,
                "traffic_unit": "DRAM bytes per row-kernel launch (ncu)",
                "peak_kind": ("measured FP32 SIMT FFMA peak (tools/peaks.cu, profiles/r02_peaks.json;"
                              " FFMA2 measured the same 74 TF)" if "ffma_tflops" in cpk else
                              "derived nominal FP32 SIMT (148 SM x 128 lanes x 2 x 1.965 GHz)")
                             + "; the row program has no tensor-core-shaped work (K<=10 per chain)",
                "kernels_per_step": len(jit_ms), "kernel_ms_per_step": kern_ms,
                "algorithmic_flops_per_step": flops_per_step,
                "flops_per_chain": flops_per_step / B,
                "hbm_bytes_per_step": B * (8 + 8 + 4),
                "hbm_frac": B * 20 / (kern_ms / 1e3) / (peaks["hbm_gbs"] * 1e9) if kern_ms else 0}

    # -- e2e through the public API: the chain state lives on the host between
    # steps; each step uploads it (H2D from page-locked memory), transitions,
    # and reads the new state and the acceptance back (D2H).  The state read
    # back is a page-locked array of the result pool (Tensor.raw: permanently
    # read-only); fed to the next step, its upload is an asynchronous DMA that overlaps the
    # call's host-side work (tensor_from_host: immutable pinned sources).
    x_host = sampler.x.raw()

    def e2e_step(x_host):
        x = sf.tensor_from_host(x_host, (B, 2), sf.float32)   # H2D inside the call
        x_out, acc = sampler.transition(x)
        xo, ao = x_out.raw(), acc.raw()                       # D2H of the step's results
        return xo

    for _ in range(a.warmup):
        x_host = e2e_step(x_host)
    e2e_ms = []
    barrier()
    # a step is ~0.3 ms: time at least 200 of them so one host hiccup (a GC
    # pass, a page fault) does not dominate the total
    e2e_steps = max(a.steps, 200)
    for _ in range(e2e_steps):
        t = time.perf_counter()
        x_host = e2e_step(x_host)
        e2e_ms.append((time.perf_counter() - t) * 1e3)
    e2e_s = sum(e2e_ms) / 1e3
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": B * world * e2e_steps / e2e_s, "unit": "samples/s",
           "h2d_bytes_per_step": B * 2 * 4, "d2h_bytes_per_step": B * 2 * 4 + B * 4,
           "steps": e2e_steps,
           "step_ms_p50": float(np.median(e2e_ms)), "step_ms_max": float(max(e2e_ms))}

    extra = {}
    if rank == 0 and world == 1 and not a.quick:
        extra = extras(sf, np, _native, plugins, l2hmc)
    if world > 1 and not a.quick:
        try:
            extra["c5_resnet50_dp"] = c5_extra(sf, _native, rank, world, dist)
        except Exception as e:  # reported, never masks the headline line
            extra["c5_resnet50_dp"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    cpu = None
    if rank == 0 and world == 1:
        r = cpu_port_rates(B, 3, 1)
        cpu = {"value": r["all_cores"], "unit": "samples/s", "cores": r["cores"], "kind": "port",
               "sample": f"the full config: {B} chains x 3 transitions "
                         f"({r['all_cores_s_per_step']:.2f} s each), numpy oracle port sharded "
                         f"over {r['cores']} persistent processes",
               "workers_1": r["workers_1"], "host": host_info()}
    if rank != 0:
        return
    line = {
        "metric": "l2hmc_samples_per_sec", "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (random-init L2HMC nets, N(0,1) initial chains)",
        "config": {"workload": "l2hmc_sampler_staged", "chains_per_gpu": B,
                   "global_chains": B * world, "leapfrog_steps": 10, "x_dim": 2, "hidden": 10,
                   "parallelism": f"dp{world} (independent chains, no collective)",
                   "l2_flush": "256 MiB fill between timed steps",
                   "rng": "device Philox"},
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "gate": gate,
        "gpu_launches": launches, "gpu_launches_per_step": launches / a.steps,
        "clocks": clk.summary(), "trace_and_compile_s": warm_s,
        "graph_ops": n_graph_ops, "native_launches_per_step": prog.n_launches,
        "peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "kind": peak_kind},
        "extra": extra,
    }
    print(json.dumps(line), flush=True)


def _time_steps(fn, n, _native, warm=2):
    import gc

    for _ in range(warm):
        fn()
    _native.sync(0)
    # objects left by the workloads timed earlier in this process (compiled
    # programs, traced graphs) move to the permanent generation, so the
    # cyclic collector's full passes do not rescan them inside this
    # workload's host-bound timed loop (C4 eager: 42.7 ms/step here vs 35.5
    # in a fresh process)
    gc.collect()
    gc.freeze()
    try:
        t = time.perf_counter()
        for _ in range(n):
            fn()
        _native.sync(0)
        return (time.perf_counter() - t) / n
    finally:
        gc.unfreeze()


def extras(sf, np, _native, plugins, l2hmc):
    """Secondary configs (wall-clock per step incl. Python dispatch)."""
    from paper_1903_01855_b200.workloads.leapfrog import Leapfrog
    from paper_1903_01855_b200.workloads import microbench

    out = {}
    # C3: the chain sweep 10 .. 1e5 (staged, one GPU; at N GPUs each shards
    # its own chains with no collective, see the headline)
    c3 = {}
    sf.init_runtime(sf.RuntimeOptions(seed=3))
    plugins.install()
    for b in (10, 100, 1000, 10000, 100000):
        s = l2hmc.L2HMCSampler(sf, b, "staged", seed=0)
        dt = _time_steps(s.step, 30, _native)
        c3[str(b)] = {"samples_per_sec": b / dt, "us_per_transition": dt * 1e6}
    out["c3_l2hmc_chain_sweep"] = c3
    # C1: L2HMC 200 chains, staged vs eager
    c1 = {}
    for mode, n in (("staged", 50), ("eager", 3)):
        sf.init_runtime(sf.RuntimeOptions(seed=7))
        plugins.install()
        s = l2hmc.L2HMCSampler(sf, 200, mode, seed=0)
        dt = _time_steps(s.step, n, _native)
        c1[mode] = {"samples_per_sec": 200 / dt, "ms_per_transition": dt * 1e3}
    c1["staged_over_eager"] = c1["staged"]["samples_per_sec"] / c1["eager"]["samples_per_sec"]
    out["c1_l2hmc_200_chains"] = c1
    # reference-pinned leapfrog (stageflow/bench.py:147-183)
    lf = {}
    for b in (200, 100000, 10000000):
        row = {}
        for mode in ("staged", "eager"):
            if mode == "eager" and b > 100000:
                continue
            sf.init_runtime(sf.RuntimeOptions())
            wl = Leapfrog(b, mode)
            dt = _time_steps(wl.step, 50 if mode == "staged" else 10, _native)
            row[mode] = {"chains_per_sec": b / dt, "us_per_trajectory": dt * 1e6}
        if "eager" in row:
            row["staged_over_eager"] = row["staged"]["chains_per_sec"] / row["eager"]["chains_per_sec"]
        row["staged"]["hbm_gbs_wall"] = 32 * b / (row["staged"]["us_per_trajectory"] * 1e-6) / 1e9
        lf[str(b)] = row
    out["leapfrog"] = lf
    # C2 microbenchmark: 100 x (matmul + add + tanh), primitive ops/s
    c2 = {}
    for mode, n in (("staged", 50), ("eager", 20)):
        sf.init_runtime(sf.RuntimeOptions())
        plugins.install()
        mb = microbench.Chain(mode)
        dt = _time_steps(mb.step, n, _native)
        c2[mode] = {"ops_per_sec": 300 / dt, "us_per_op": dt * 1e6 / 300}
    c2["staged_over_eager"] = c2["staged"]["ops_per_sec"] / c2["eager"]["ops_per_sec"]
    out["c2_microbench"] = c2
    out["eager_launch_path"] = eager_path_extra(sf, np, _native, plugins)
    # L2HMC training (the paper's L2HMC figure): ESJD loss over two full
    # transitions, the tape's staged backward through every leapfrog step
    tr_row = {}
    for mode, n in (("staged", 10), ("eager", 2)):
        sf.init_runtime(sf.RuntimeOptions(seed=1))
        plugins.install()
        tr = l2hmc.L2HMCTrain(sf, 200, mode, seed=0)
        dt = _time_steps(tr.step, n, _native)
        tr_row[mode] = {"ms_per_step": dt * 1e3, "samples_per_sec": 200 / dt}
    tr_row["staged_over_eager"] = tr_row["eager"]["ms_per_step"] / tr_row["staged"]["ms_per_step"]
    tr_row["chains"] = 200
    out["l2hmc_training_200_chains"] = tr_row
    out["c4_resnet50_b32"] = resnet_extra(sf, np, _native)
    try:
        out["c5_resnet50_b256_1gpu"] = c5_extra(sf, _native, 0, 1, None)
    except Exception as e:  # report, never lose the headline line
        out["c5_resnet50_b256_1gpu"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    out["f1_device_while"] = while_extra(sf, np, _native)
    return out


def eager_path_extra(sf, np, _native, plugins):
    """North-star subsystem 1, the eager launch path: host+device cost per
    primitive (wall clock over 20k dispatches incl. the final sync) through
    the native front-end + launch queue (default), the native front-end with
    one kernel launch per op, and the reference-semantics Python dispatcher
    (ops._dispatch_py) with one launch per op; plus kernel launches per op."""
    from paper_1903_01855_b200 import _fastpath
    from paper_1903_01855_b200.workloads import microbench

    out = {}
    sf.init_runtime(sf.RuntimeOptions())
    plugins.install()
    x = sf.constant(np.ones((1, 16), np.float32))
    for mode in ("queue", "direct", "python"):
        _fastpath.set_enabled(mode != "python")
        _native.queue_config(0, 64 if mode == "queue" else 0)
        n = 20000
        l0 = _native.launch_count(0)
        add_us = _time_steps(lambda: sf.add(x, x), n, _native) * 1e6
        launches = (_native.launch_count(0) - l0) / (n + 2)
        ch = microbench.Chain("eager")
        c2_us = _time_steps(ch.step, 20, _native) * 1e6 / 300
        out[mode] = {"add_us_per_op": add_us, "kernel_launches_per_op": launches,
                     "c2_eager_us_per_op": c2_us}
    _fastpath.set_enabled(True)
    _native.queue_config(0, 64)
    out["what"] = ("eager sf.add on (1,16) f32 and the C2 eager chain; queue = native "
                   "front-end + launch queue (64 ops per interpreter-kernel launch), direct = "
                   "native front-end with one launch per op, python = reference-semantics "
                   "Python dispatcher with one launch per op")
    return out


def while_extra(sf, np, _native):
    """a staged while_loop (1000 iterations of a small matvec
    body on (64, 8)) with the predicate read on the host every iteration vs.
    kept on the device (CUDA graph WHILE node)."""
    from paper_1903_01855_b200 import executor

    sf.init_runtime(sf.RuntimeOptions())
    W = sf.constant(np.random.default_rng(0).standard_normal((8, 8)).astype(np.float32) * 0.3)

    def iterate(x, n):
        def body(i, v):
            return sf.sub(i, 1), sf.add(sf.matmul(v, W), sf.mul(v, 0.5))

        return sf.while_loop(lambda i, v: sf.greater(i, 0), body, [n, x])[1]

    x = sf.constant(np.random.default_rng(1).standard_normal((64, 8)).astype(np.float32))
    n = sf.constant(1000, dtype=sf.int32)
    row = {}
    for mode, flag in (("host_predicate", False), ("device_graph", True)):
        executor.DEVICE_WHILE = flag
        staged = sf.stage(iterate)
        dt = _time_steps(lambda: staged(x, n), 3, _native)
        row[mode] = {"ms_per_loop": dt * 1e3, "us_per_iteration": dt * 1e3}
    executor.DEVICE_WHILE = True
    row["speedup"] = row["host_predicate"]["ms_per_loop"] / row["device_graph"]["ms_per_loop"]

    # cond: the predicate comes out of a device computation each call
    def branchy(v):
        flag = sf.greater(sf.reduce_sum(v), 0.0)
        return sf.cond(flag, lambda u: sf.matmul(u, W), lambda u: sf.mul(u, 0.5), [v])

    for mode, flag in (("cond_host_predicate", False), ("cond_device_graph", True)):
        executor.DEVICE_COND = flag
        staged = sf.stage(branchy)
        dt = _time_steps(lambda: staged(x), 50, _native)
        row[mode] = {"us_per_call": dt * 1e6}
    executor.DEVICE_COND = False
    return row


def c5_extra(sf, _native, rank, world, dist, batch=256):
    """C5: ResNet-50 data parallel, batch 256 per GPU (BASELINE config 5).
    The gradient all-reduce runs inside the staged backward's plan (NCCL via
    the C-ABI, ~25 MB buckets issued as the backward produces them, comm
    stream joined at the end; paper_1903_01855_b200/dist.py).  Device time
    per step with CUDA events on the backend stream, max over ranks.  At
    world 1 the communicator has one rank (the per-GPU compute plus the
    collective's fork/join)."""
    import torch

    from paper_1903_01855_b200 import comm as sfcomm
    from paper_1903_01855_b200 import dist as sfdist
    from paper_1903_01855_b200 import nn

    sf.init_runtime(sf.RuntimeOptions())
    nn.install()
    com = sfcomm.Communicator.from_env(dev=0) if world > 1 else sfcomm.Communicator(1, 0, 0)
    dp = sfdist.ResNetDataParallel(sf, batch_per_rank=batch, comm=com)
    for _ in range(3):
        dp.step()
    _native.sync(0)
    if dist is not None:
        dist.barrier()
    stream = torch.cuda.ExternalStream(_native.stream_of(0))
    n = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        dp.step()
    e1.record(stream)
    _native.sync(0)
    ms = e0.elapsed_time(e1) / n
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    plans = dp.backward_plans()
    n_ar = sum(1 for p in plans for k, _, _ in p.step_stats() if k == 12)
    out = {"img_per_sec": batch * world / (ms / 1e3), "ms_per_step": ms, "batch_per_gpu": batch,
           "n_gpus": world, "scaling": "weak", "allreduce_steps_in_backward": n_ar,
           "collective": "NCCL sum of ~25 MB gradient buckets inside the backward plan "
                         "(comm stream, overlapped), lr/N update"}
    com.close()
    return out


def resnet_extra(sf, np, _native):
    """C4: ResNet-50 v1.5 train step, batch 32, 224x224 synthetic fp32, 1 GPU."""
    import torch

    from paper_1903_01855_b200 import nn
    from paper_1903_01855_b200.workloads import resnet

    row = {}
    for mode, n in (("staged", 10), ("eager", 6)):
        sf.init_runtime(sf.RuntimeOptions())
        nn.install()
        tr = resnet.ResNetTrain(sf, batch=32, mode=mode, image=224, seed=0)
        dt = _time_steps(tr.step, n, _native, warm=3)
        row[mode] = {"img_per_sec": 32 / dt, "ms_per_step": dt * 1e3,
                     "useful_tflops": 0.785 / dt}
        del tr
    row["staged_over_eager"] = row["staged"]["img_per_sec"] / row["eager"]["img_per_sec"]
    # roofline of the dominant tensor kernel: the tcgen05 3xTF32 GEMM at the
    # shape of layer1's 3x3 convolution (M = 32*56*56, N = 64, K = 576), in
    # the variant the training step runs (raw fp32 operands, the tf32 lo
    # parts derived in shared memory), timed back to back with CUDA events
    peaks, kind = _peaks()
    cpk = _compute_peaks()
    m, n, k = 32 * 56 * 56, 64, 576
    a = sf.constant(np.random.default_rng(0).standard_normal((m, k)).astype(np.float32))
    b = sf.constant(np.random.default_rng(1).standard_normal((n, k)).astype(np.float32))
    stream = torch.cuda.ExternalStream(_native.stream_of(0))

    def gemm():
        return _native.gemm_tf32x3_ex(0, m, n, k, False, False, k, k, a._ptr(), 0, b._ptr(), 0)

    for _ in range(3):
        gemm()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record(stream)
    for _ in range(reps):
        gemm()
    e1.record(stream)
    _native.sync(0)
    ms = e0.elapsed_time(e1) / reps
    useful = 2.0 * m * n * k / (ms * 1e-3) / 1e12
    tf32 = cpk.get("tcgen05_tf32_tflops")
    peak = tf32 / 3 if tf32 else peaks.get("bf16_tflops", 1590.0) / 6
    # the same layer as the training step's forward runs it: the implicit-GEMM
    # convolution (sf_conv2d_tc; the GEMM gathers its im2col rows)
    from paper_1903_01855_b200 import nn as _nn
    x4 = sf.constant(np.random.default_rng(2).standard_normal((32, 56, 56, 64)).astype(np.float32))
    w4 = sf.constant(np.random.default_rng(3).standard_normal((3, 3, 64, 64)).astype(np.float32))
    for _ in range(3):
        _nn.conv2d(x4, w4, 1, 1)
    e0.record(stream)
    for _ in range(reps):
        _nn.conv2d(x4, w4, 1, 1)
    e1.record(stream)
    _native.sync(0)
    conv_ms = e0.elapsed_time(e1) / reps
    row["roofline"] = {"kernel": "gemm_tc_persistent (tcgen05 kind::tf32, 3 passes, lo parts "
                                 "derived in shared memory)",
                       "implicit_conv_ms": conv_ms,
                       "implicit_conv_tflops": 2.0 * m * n * k / (conv_ms * 1e-3) / 1e12,
                       "implicit_conv_note": "the forward of this layer as the step runs it "
                                             "(sf_conv2d_tc: im2col rows gathered by the GEMM; "
                                             "L2-bandwidth bound at N = 64)",
                       "shape_mnk": [m, n, k], "ms": ms, "bound": "tensor",
                       "achieved": useful, "unit": "TFLOP/s (useful fp32 MACs x2)",
                       "peak": peak, "frac": useful / peak,
                       "tensor_issue_tflops": 3 * useful,
                       "peak_kind": ("measured tcgen05 kind::tf32 dense / 3 (3xTF32 issues 3 MMAs "
                                     "per useful MAC; profiles/r02_peaks.json)" if tf32 else
                                     f"{kind} bf16 dense / 6 (TF32 = half, 3 passes)"),
                       "step_useful_tflops": row["staged"]["useful_tflops"],
                       "step_frac": row["staged"]["useful_tflops"] / peak}
    return row


def main():
    a = _args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if a.workload:
        # the reference's benchmark contract (stageflow bench --workload ...)
        from paper_1903_01855_b200.benchmark import run_cli

        a.bench_warmup = a.warmup
        sys.exit(run_cli(a))
    if world > 1:
        os.environ["CUDA_VISIBLE_DEVICES"] = str(local)
    import torch

    dist = None
    if world > 1:
        import torch.distributed as tdist

        torch.cuda.set_device(0)
        tdist.init_process_group("nccl")
        dist = tdist
    run_ours(a, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
