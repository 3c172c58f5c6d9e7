"""GPU parity of the benchmark workloads against the reference's golden
vectors and the NumPy oracle.

Floating-point bar (north star): rtol 1e-4 vs the reference; eager vs
staged on this backend must be bit-exact.
"""
import os

import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import plugins
from paper_1903_01855_b200.workloads import l2hmc
from paper_1903_01855_b200.workloads.leapfrog import Leapfrog
from oracle import workloads_np

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
RTOL = 1e-4


@pytest.mark.parametrize("b", [10, 200, 1000])
def test_leapfrog_matches_reference_golden(b):
    for mode in ("eager", "staged"):
        wl = Leapfrog(b, mode)
        v1 = wl.run_iteration()
        for _ in range(9):
            v10 = wl.run_iteration()
        np.testing.assert_allclose(v1, GOLD[f"leapfrog_{mode}_{b}_t1"], rtol=RTOL, atol=1e-6)
        np.testing.assert_allclose(v10, GOLD[f"leapfrog_{mode}_{b}_t10"], rtol=RTOL, atol=1e-6)


@pytest.mark.parametrize("b", [10000, 100000])
def test_leapfrog_large_staged(b):
    wl = Leapfrog(b, "staged")
    for _ in range(10):
        v = wl.run_iteration()
    head = GOLD[f"leapfrog_staged_{b}_t10_head"]
    np.testing.assert_allclose(v[:64], head, rtol=RTOL, atol=1e-6)
    want = workloads_np.leapfrog(b, seed=0, trajectories=10)
    np.testing.assert_allclose(v, want, rtol=RTOL, atol=1e-6)


def test_leapfrog_eager_equals_staged_bitwise():
    e, s = Leapfrog(200, "eager"), Leapfrog(200, "staged")
    for _ in range(3):
        assert e.run_iteration().tobytes() == s.run_iteration().tobytes()


def test_leapfrog_staged_is_one_fused_launch():
    wl = Leapfrog(1000, "staged")
    wl.step()
    prog = next(iter(wl.trajectory.cached_functions()[0].graph._plan.values()))
    assert prog.n_launches == 1
    assert wl.trajectory.trace_count == 1


@pytest.mark.parametrize("b", [16, 200])
def test_l2hmc_matches_reference_golden_host_rng(b):
    """Host-RNG parity mode reproduces the reference's PCG64 draws."""
    for mode in ("staged", "eager"):
        sf.init_runtime(sf.RuntimeOptions(rng="host", seed=0))
        plugins.install()
        s = l2hmc.L2HMCSampler(sf, b, mode, seed=0)
        got = np.stack([s.run_iteration() for _ in range(3)])
        np.testing.assert_allclose(got, GOLD[f"l2hmc_{mode}_{b}"], rtol=RTOL, atol=1e-5)


@pytest.mark.parametrize("b", [2, 10, 200, 5000])
def test_l2hmc_eager_equals_staged_device_rng(b):
    # b = 2 and 10 equal the sampler's layer widths: weights then have the
    # batch's leading extent and must still be planned as uniform operands
    outs = {}
    for mode in ("eager", "staged"):
        sf.init_runtime(sf.RuntimeOptions(seed=3))
        plugins.install()
        s = l2hmc.L2HMCSampler(sf, b, mode, seed=0)
        outs[mode] = np.stack([s.run_iteration() for _ in range(2)])
    assert outs["eager"].tobytes() == outs["staged"].tobytes()


def test_l2hmc_staged_row_program():
    plugins.install()
    s = l2hmc.L2HMCSampler(sf, 512, "staged", seed=0)
    s.step()
    prog = next(iter(s.transition.cached_functions()[0].graph._plan.values()))
    n_nodes = len(s.transition.cached_functions()[0].graph.nodes)
    # ~3300 graph nodes -> one uniform kernel + a few row-program chunks (the
    # unrolled leapfrog steps re-rolled into loops)
    assert prog.n_launches <= 8 < n_nodes, (prog.n_launches, n_nodes)
    assert len(prog.segments) == 1


@pytest.mark.parametrize("replicas,const_pool", [(1, False), (2, False), (1, True), (2, True)])
def test_rerolled_loop_bitwise_equals_eager(replicas, const_pool, monkeypatch):
    """A traced Python loop with per-step weights and a shared bias: the staged
    row program re-rolls it (carried rows, stacked per-step weights, exported
    last step) and must match the eager per-op kernels bit for bit — with one
    or two chains per thread (1000 rows: the second replica of the last CTA
    runs past the end and must not store)."""
    from paper_1903_01855_b200 import rowfuse

    monkeypatch.setattr(rowfuse, "ROW_REPLICAS", replicas)
    monkeypatch.setattr(rowfuse, "CONST_POOL", const_pool)
    plugins.install()
    rng = np.random.default_rng(3)
    B, D, steps = 1000, 6, 7
    Ws = [sf.constant(rng.standard_normal((D, D)).astype(np.float32) * 0.5) for _ in range(steps)]
    bias = sf.constant(rng.standard_normal((D,)).astype(np.float32))
    x0 = sf.constant(rng.standard_normal((B, D)).astype(np.float32))

    def f(x):
        acc = sf.reduce_sum(x, axes=(1,))
        for i in range(steps):
            h = plugins.tanh(sf.add(sf.matmul(x, Ws[i]), bias))
            x = sf.add(sf.mul(h, 0.5), sf.mul(x, 0.5))
            acc = sf.add(acc, sf.reduce_sum(x, axes=(1,)))
        return x, acc

    want = [t.numpy() for t in f(x0)]
    staged = sf.stage(f)
    got = [t.numpy() for t in staged(x0)]
    for g, w in zip(got, want):
        assert g.tobytes() == w.tobytes()
    prog = next(iter(staged.cached_functions()[0].graph._plan.values()))
    assert prog.n_launches <= 3


def test_l2hmc_oracle_host_rng_long_run():
    sf.init_runtime(sf.RuntimeOptions(rng="host", seed=0))
    plugins.install()
    s = l2hmc.L2HMCSampler(sf, 64, "staged", seed=0)
    m = workloads_np.L2HMC(64, seed=0, runtime_seed=0)
    for _ in range(5):
        np.testing.assert_allclose(s.run_iteration(), m.transition(), rtol=RTOL, atol=1e-5)
