"""The reference's benchmark contract on this backend
(stageflow/bench.py:40-297 and stageflow/cli.py:18-60).

* ``BenchConfig`` / ``run_benchmark`` / ``emit_csv`` keep the reference's
  fields, validation errors, same-seed eager-vs-staged gate (raises
  ``NumericalDivergence`` before any timing; 1e-6 for trajectories, 1e-5
  otherwise — this backend is in fact bit-exact between the modes), the
  repeats / mean / population-stddev statistics and the CSV columns, plus
  two trailing columns: ``gpus`` and ``device``.
* Workloads: the reference's three (``mlp_train``, ``leapfrog``,
  ``microop_loop``) and the BASELINE configs' builder-defined ones
  (``l2hmc`` — C1/C3, ``c2_chain`` — C2, ``resnet50`` — C4 at batch
  ``--batch``).
* Timing is wall clock around ``run_iteration``, which ends in a host fetch
  of the iteration's result (reference :181-183), so device work is
  included.  The bench.py headline reports device-event timings instead.

    python -m paper_1903_01855_b200.benchmark bench --workload leapfrog \
        --mode staged --batch 200 [--iters 10 --warmup 2 --repeats 3 --out r.csv]

Exit codes as the reference CLI: 0 ok, 2 gate failure, 1 other errors.
"""
from __future__ import annotations

import argparse
import csv
import statistics
import sys
import time
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .errors import ConfigError, NumericalDivergence, StageflowError, StorageError
from .runtime import RuntimeOptions, get_runtime, init_runtime

WORKLOADS = ("mlp_train", "leapfrog", "microop_loop", "l2hmc", "c2_chain", "resnet50")
MODES = ("eager", "staged")
CSV_HEADER = "workload,mode,batch,iters,examples_per_sec,stddev,trace_count,copies,gpus,device"


@dataclass(frozen=True)
class BenchConfig:
    workload: str
    mode: str
    batch_size: int = 8
    iterations: int = 10
    warmup: int = 2
    repeats: int = 3
    workers: Optional[int] = None
    seed: int = 0

    def validate(self) -> None:
        if self.workload not in WORKLOADS:
            raise ConfigError(f"unknown workload {self.workload!r}; choose from {WORKLOADS}")
        if self.mode not in MODES:
            raise ConfigError(f"unknown mode {self.mode!r}; choose from {MODES}")
        if self.iterations < 1:
            raise ConfigError("iterations must be >= 1")
        if self.batch_size < 1:
            raise ConfigError("batch size must be >= 1")
        if self.warmup < 0 or self.repeats < 1:
            raise ConfigError("warmup must be >= 0 and repeats >= 1")


@dataclass
class BenchReport:
    config: BenchConfig
    wall_times: List[float]
    examples_per_sec_runs: List[float]
    examples_per_sec: float
    stddev: float
    trace_count: int
    cache_size: int
    copies: int
    setup_time: float  # tracing, lowering and JIT compile: excluded from timing
    gpus: int = 1
    device: str = ""


class _C2:
    """C2 chain adapter: one chain per iteration, 300 primitive ops."""

    gate_tol = 1e-5

    def __init__(self, mode, seed):
        from .workloads import microbench

        self.c = microbench.Chain(mode, seed=seed)
        self.staged_functions = [self.c.fn] if mode == "staged" else []

    def run_iteration(self):
        return self.c.step().numpy()

    def cache_size(self):
        return sum(pf.cache_size for pf in self.staged_functions)


class _ResNet:
    gate_tol = 1e-5

    def __init__(self, mode, seed, batch):
        from . import nn
        from .workloads import resnet

        nn.install()
        self.t = resnet.ResNetTrain(__import__("paper_1903_01855_b200"), batch=batch, mode=mode,
                                    seed=seed)
        self.staged_functions = self.t.staged_functions

    def run_iteration(self):
        return self.t.run_iteration()

    def cache_size(self):
        return sum(pf.cache_size for pf in self.staged_functions)


def _make(cfg: BenchConfig, mode: str):
    import paper_1903_01855_b200 as sf

    get_runtime().reseed(cfg.seed)
    w = cfg.workload
    if w == "mlp_train":
        from .workloads.mlp import MLPTrain

        return MLPTrain(cfg.batch_size, mode, seed=cfg.seed)
    if w == "leapfrog":
        from .workloads.leapfrog import Leapfrog

        return Leapfrog(cfg.batch_size, mode, seed=cfg.seed)
    if w == "microop_loop":
        from .workloads.microop import MicroOpLoop

        return MicroOpLoop(mode, seed=cfg.seed)
    if w == "l2hmc":
        from . import plugins
        from .workloads.l2hmc import L2HMCSampler

        plugins.install()
        return L2HMCSampler(sf, cfg.batch_size, mode, seed=cfg.seed)
    if w == "c2_chain":
        return _C2(mode, cfg.seed)
    return _ResNet(mode, cfg.seed, cfg.batch_size)


def gate(cfg: BenchConfig) -> None:
    """Same seed, both modes, every iteration: results must agree
    (reference bench.py:216-234).  Each mode runs from a reseeded runtime
    (the reference interleaves the two; with device RNG draws in the
    workload the interleaving would hand the modes different counters)."""
    eager = _make(cfg, "eager")
    tol = getattr(eager, "gate_tol", 1e-5)
    ves = [np.asarray(eager.run_iteration(), dtype=np.float64) for _ in range(cfg.iterations)]
    staged = _make(cfg, "staged")
    for i, ve in enumerate(ves):
        vs = np.asarray(staged.run_iteration(), dtype=np.float64)
        diff = float(np.max(np.abs(ve - vs))) if ve.size else 0.0
        if not np.isfinite(diff) or diff > tol:
            raise NumericalDivergence(
                f"{cfg.workload}: eager and staged diverge at iteration {i} "
                f"(max abs diff {diff:.3e} > {tol:g})")


def run_benchmark(cfg: BenchConfig) -> BenchReport:
    cfg.validate()
    gate(cfg)
    rt = get_runtime()
    before = rt.stats.snapshot()
    walls: List[float] = []
    rates: List[float] = []
    setup = 0.0
    cache = 0
    for _ in range(cfg.repeats):
        t0 = time.perf_counter()
        wl = _make(cfg, cfg.mode)
        for _ in range(cfg.warmup):
            wl.run_iteration()
        setup += time.perf_counter() - t0
        t1 = time.perf_counter()
        for _ in range(cfg.iterations):
            wl.run_iteration()
        dt = time.perf_counter() - t1
        walls.append(dt)
        rates.append(cfg.batch_size * cfg.iterations / dt)
        cache = wl.cache_size()
    after = rt.stats.snapshot()
    return BenchReport(
        config=cfg, wall_times=walls, examples_per_sec_runs=rates,
        examples_per_sec=statistics.fmean(rates),
        stddev=statistics.pstdev(rates) if len(rates) > 1 else 0.0,
        trace_count=after["traces"] - before["traces"], cache_size=cache,
        copies=after["transparent_copies"] - before["transparent_copies"],
        setup_time=setup, gpus=len(rt.devices), device=_device_name())


def _device_name() -> str:
    from . import _native

    try:
        return _native.device_name(0)
    except Exception:  # noqa: BLE001 - informational only
        return ""


def emit_csv(report: BenchReport, path: str) -> None:
    """One row per repeat plus a mean row (reference :276-297 columns, then
    gpus and device); UTF-8, LF line endings."""
    cfg = report.config
    tail = [report.gpus, report.device]
    try:
        with open(path, "w", encoding="utf-8", newline="\n") as f:
            w = csv.writer(f, lineterminator="\n")
            w.writerow(CSV_HEADER.split(","))
            head = [cfg.workload, cfg.mode, cfg.batch_size, cfg.iterations]
            for eps in report.examples_per_sec_runs:
                w.writerow(head + [f"{eps:.3f}", "0.000", report.trace_count, report.copies] + tail)
            w.writerow(head + [f"{report.examples_per_sec:.3f}", f"{report.stddev:.3f}",
                               report.trace_count, report.copies] + tail)
    except OSError as e:
        raise StorageError(f"cannot write report to {path}: {e}") from e


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_1903_01855_b200.benchmark",
                                description="eager-vs-staged benchmarks on the B200 backend")
    sub = p.add_subparsers(dest="command", required=True)
    b = sub.add_parser("bench", help="run an eager-vs-staged benchmark")
    add_bench_args(b, required=True)
    return p


def add_bench_args(b: argparse.ArgumentParser, required: bool, warmup: bool = True) -> None:
    """The reference CLI's bench flags; bench.py keeps its own --warmup (the
    driver's W) and passes it through."""
    b.add_argument("--workload", choices=WORKLOADS, required=required)
    b.add_argument("--mode", choices=MODES, default="staged")
    b.add_argument("--batch", type=int, default=8)
    b.add_argument("--iters", type=int, default=10)
    if warmup:
        b.add_argument("--warmup", dest="bench_warmup", type=int, default=2)
    b.add_argument("--repeats", type=int, default=3)
    b.add_argument("--workers", type=int, default=None)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--out", default=None, help="write the CSV report here")


def run_cli(args) -> int:
    init_runtime(RuntimeOptions(executor_workers=args.workers, seed=args.seed))
    cfg = BenchConfig(workload=args.workload, mode=args.mode, batch_size=args.batch,
                      iterations=args.iters, warmup=args.bench_warmup, repeats=args.repeats,
                      workers=args.workers, seed=args.seed)
    try:
        report = run_benchmark(cfg)
    except NumericalDivergence as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except StageflowError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    print(f"{cfg.workload} [{cfg.mode}] batch={cfg.batch_size} iters={cfg.iterations}: "
          f"{report.examples_per_sec:.1f} examples/s (stddev {report.stddev:.1f}, "
          f"{report.trace_count} traces, {report.copies} copies, "
          f"setup {report.setup_time * 1e3:.1f} ms, {report.gpus} GPU {report.device})")
    if args.out:
        emit_csv(report, args.out)
        print(f"report written to {args.out}")
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return run_cli(args)


if __name__ == "__main__":
    sys.exit(main())
