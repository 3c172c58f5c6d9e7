"""Pin the NumPy oracle against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""
import os

import numpy as np
import pytest

from oracle import workloads_np

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


@pytest.mark.parametrize("b", [10, 200, 1000])
def test_leapfrog_oracle_bit_exact(b):
    for t in (1, 10):
        want = GOLD[f"leapfrog_staged_{b}_t{t}"]
        assert GOLD[f"leapfrog_eager_{b}_t{t}"].tobytes() == want.tobytes()
        got = workloads_np.leapfrog(b, seed=0, trajectories=t)
        assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("b", [10000, 100000])
def test_leapfrog_oracle_large(b):
    got = workloads_np.leapfrog(b, seed=0, trajectories=10).astype(np.float64)
    np.testing.assert_array_equal(got[:64], GOLD[f"leapfrog_staged_{b}_t10_head"])
    np.testing.assert_allclose([got.sum(), np.square(got).sum()],
                               GOLD[f"leapfrog_staged_{b}_t10_sum"], rtol=1e-12)


@pytest.mark.parametrize("b", [8, 32, 256])
def test_mlp_oracle(b):
    want = GOLD[f"mlp_staged_{b}_losses"]
    np.testing.assert_allclose(GOLD[f"mlp_eager_{b}_losses"], want, rtol=1e-6)
    got = workloads_np.mlp_losses(b, 10)
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-7)


def test_c2_oracle():
    x, ws, bs = workloads_np.c2_params(0)
    np.testing.assert_allclose(workloads_np.c2_chain(x, ws, bs), GOLD["c2_eager"], rtol=1e-6,
                               atol=1e-7)
    assert GOLD["c2_eager"].tobytes() == GOLD["c2_staged"].tobytes()
    np.testing.assert_allclose(workloads_np.c2_chain_grad(x, ws, bs), GOLD["c2_grad"], rtol=1e-5,
                               atol=1e-6)


@pytest.mark.parametrize("b", [16, 200])
def test_l2hmc_reference_eager_equals_staged(b):
    np.testing.assert_array_equal(GOLD[f"l2hmc_eager_{b}"], GOLD[f"l2hmc_staged_{b}"])
    assert int(GOLD[f"l2hmc_trace_count_{b}"][0]) == 1


@pytest.mark.parametrize("b", [16, 200])
def test_l2hmc_oracle(b):
    want = GOLD[f"l2hmc_staged_{b}"]
    m = workloads_np.L2HMC(b, seed=0, runtime_seed=0)
    got = np.stack([m.transition() for _ in range(3)])
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6)


# ---------------------------------------------------------------- device RNG oracle
def test_philox_oracle_known_answers():
    """oracle/philox_np.py reproduces the published Random123 philox4x32_10
    known-answer vectors (the device generator is pinned to this oracle in
    tests/test_gpu_rng.py)."""
    from oracle import philox_np

    for ctr, key, want in philox_np.KAT:
        got = philox_np.philox4x32_10(*ctr, *key)
        assert [int(w) for w in got] == list(want)


def test_philox_oracle_draw_mapping():
    from oracle import philox_np

    u = philox_np.uniform_f32(4, seed=0, offset=0)
    assert u[0] == np.float32((0x6627E8D5 >> 8) * 2.0 ** -24)
    assert u.dtype == np.float32 and np.all((u >= 0) & (u < 1))
    z = philox_np.normal_f64(200000, seed=5, offset=7)
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1) < 0.02
    # offset shifts the stream: element i of (offset k) == element i+k of (offset 0)
    a = philox_np.uniform_f64(10, seed=9, offset=3)
    b = philox_np.uniform_f64(13, seed=9, offset=0)
    assert a.tobytes() == b[3:].tobytes()


# ---------------------------------------------------------------- L2HMC at the headline batch
GOLD2 = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_r2.npz"))


def test_l2hmc_oracle_matches_reference_at_1e5():
    """The oracle (draws passed in) against the reference run at 1e5 chains
    (tests/golden/make_golden_r2.py): first 4096 chains of each of three
    transitions, and float64 sums over all chains."""
    b = 100_000
    m = workloads_np.L2HMC(b, seed=0)
    rng = np.random.default_rng(0)
    for t in (1, 2, 3):
        draws = (rng.standard_normal((b, 2)).astype(np.float32),
                 rng.standard_normal((b, 2)).astype(np.float32),
                 rng.random((b,)).astype(np.float32), rng.random((b,)).astype(np.float32))
        m.x, acc = m.transition_with(m.x, *draws)
        np.testing.assert_allclose(m.x[:4096], GOLD2[f"l2hmc_inputs_1e5_t{t}_x_head"],
                                   rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(acc[:4096], GOLD2[f"l2hmc_inputs_1e5_t{t}_acc_head"],
                                   rtol=1e-5, atol=1e-6)
        x64, a64 = m.x.astype(np.float64), acc.astype(np.float64)
        np.testing.assert_allclose([np.square(x64).sum(), a64.sum()],
                                   GOLD2[f"l2hmc_inputs_1e5_t{t}_sums"][[1, 2]], rtol=1e-5)
