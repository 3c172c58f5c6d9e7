"""The reference's benchmark contract (stageflow/bench.py:40-297,
stageflow/cli.py) on this backend: config validation, CSV layout, the
same-seed gate, counters, and the microop_loop workload."""
import os

import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import benchmark as bm
from paper_1903_01855_b200.errors import ConfigError, NumericalDivergence, StorageError

GOLD2 = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_r2.npz"))


@pytest.mark.parametrize("kw,msg", [
    (dict(workload="nope", mode="eager"), "unknown workload"),
    (dict(workload="leapfrog", mode="lazy"), "unknown mode"),
    (dict(workload="leapfrog", mode="eager", iterations=0), "iterations"),
    (dict(workload="leapfrog", mode="eager", batch_size=0), "batch size"),
    (dict(workload="leapfrog", mode="eager", repeats=0), "repeats"),
])
def test_config_validation(kw, msg):
    with pytest.raises(ConfigError, match=msg):
        bm.BenchConfig(**kw).validate()


def _report():
    cfg = bm.BenchConfig(workload="leapfrog", mode="staged", batch_size=200, iterations=10)
    return bm.BenchReport(config=cfg, wall_times=[0.1, 0.2], examples_per_sec_runs=[100.0, 300.0],
                          examples_per_sec=200.0, stddev=100.0, trace_count=2, cache_size=1,
                          copies=0, setup_time=0.5, gpus=1, device="sm_100 148SM")


def test_csv_layout(tmp_path):
    path = tmp_path / "r.csv"
    bm.emit_csv(_report(), str(path))
    raw = path.read_bytes()
    assert b"\r" not in raw
    lines = raw.decode().splitlines()
    # the reference's columns, then gpus and device
    assert lines[0] == ("workload,mode,batch,iters,examples_per_sec,stddev,trace_count,copies,"
                        "gpus,device")
    assert len(lines) == 1 + 2 + 1  # header, one row per repeat, the mean row
    assert lines[1] == "leapfrog,staged,200,10,100.000,0.000,2,0,1,sm_100 148SM"
    assert lines[3] == "leapfrog,staged,200,10,200.000,100.000,2,0,1,sm_100 148SM"


def test_csv_unwritable_path_is_storage_error(tmp_path):
    with pytest.raises(StorageError):
        bm.emit_csv(_report(), str(tmp_path / "missing" / "r.csv"))


def test_cli_parser():
    args = bm.build_parser().parse_args(
        ["bench", "--workload", "microop_loop", "--mode", "eager", "--iters", "3"])
    assert (args.workload, args.mode, args.iters, args.batch, args.repeats) == \
        ("microop_loop", "eager", 3, 8, 3)


# ---------------------------------------------------------------- on the GPU
@pytest.mark.gpu
def test_microop_loop_matches_reference():
    from paper_1903_01855_b200.serial import serialize
    from paper_1903_01855_b200.workloads.microop import MicroOpLoop

    for mode in ("eager", "staged"):
        wl = MicroOpLoop(mode)
        got = np.array([wl.run_iteration() for _ in range(3)])
        assert got.tobytes() == GOLD2[f"microop_{mode}_values"].tobytes()  # 1000, 2000, 3000
    wl = MicroOpLoop("staged")
    wl.step()
    gf = wl.chain.cached_functions()[0].graph
    assert serialize(gf) == GOLD2["microop_graph"].tobytes()
    prog = next(iter(gf._plan.values()))
    assert prog.n_launches == 1  # 1000 adds in one kernel


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["eager", "staged"])
def test_run_benchmark_counters_match_reference(mode):
    cfg = bm.BenchConfig(workload="microop_loop", mode=mode, batch_size=1, iterations=3,
                         warmup=1, repeats=2)
    rep = bm.run_benchmark(cfg)
    assert [rep.trace_count, rep.cache_size, rep.copies] == \
        list(GOLD2[f"microop_{mode}_report"])
    assert len(rep.examples_per_sec_runs) == 2 and rep.examples_per_sec > 0


@pytest.mark.gpu
def test_gate_rejects_divergence(monkeypatch):
    from paper_1903_01855_b200.workloads import leapfrog

    orig = leapfrog.Leapfrog.run_iteration

    def skewed(self):
        out = orig(self)
        return out + (1e-3 if self.mode == "staged" else 0.0)

    monkeypatch.setattr(leapfrog.Leapfrog, "run_iteration", skewed)
    with pytest.raises(NumericalDivergence, match="diverge at iteration 0"):
        bm.run_benchmark(bm.BenchConfig(workload="leapfrog", mode="staged", batch_size=10,
                                        iterations=2))
    assert bm.main(["bench", "--workload", "leapfrog", "--batch", "10", "--iters", "2"]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("workload,batch", [("leapfrog", 200), ("mlp_train", 32), ("l2hmc", 200),
                                            ("c2_chain", 1)])
def test_run_benchmark_workloads(workload, batch, tmp_path):
    out = tmp_path / "r.csv"
    rc = bm.main(["bench", "--workload", workload, "--mode", "staged", "--batch", str(batch),
                  "--iters", "3", "--repeats", "2", "--out", str(out)])
    assert rc == 0
    rows = out.read_text().splitlines()
    assert len(rows) == 4 and rows[-1].startswith(f"{workload},staged,{batch},3,")
