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
