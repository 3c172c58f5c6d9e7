"""Device RNG (Philox4x32-10, csrc/sf_ops.cuh) against its oracle
(oracle/philox_np.py, pinned to the Random123 known-answer vectors in
tests/test_oracle.py), its distributions, and counter bookkeeping.

The reference draws from a locked host PCG64 stream
(stageflow/runtime.py:124-127; kernels stageflow/kernels.py:372-404); that
stream is reproduced by ``RuntimeOptions(rng="host")`` and pinned by the
golden tests.  The default device mode is what the staged L2HMC headline
runs, so its generator is pinned here: values bit-exact with the oracle
(uniforms; normals within f64 Box-Muller ulps), moments and Kolmogorov-
Smirnov at 1e7 draws, and counter ranges that never overlap — eagerly,
inside staged programs (fused row kernels), and across the two.
"""
import math

import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import plugins
from oracle import philox_np

pytestmark = pytest.mark.gpu


def _normal(shape, dt=sf.float32):
    return sf.random_normal(shape, dtype=dt)


def _uniform(shape, dt=sf.float32):
    return plugins.random_uniform(shape, dtype=dt)


def _fresh(seed):
    sf.init_runtime(sf.RuntimeOptions(seed=seed))
    plugins.install()


def test_device_uniform_known_answer():
    """Counter 0 / key 0 is the first Random123 KAT: the first f32 uniform of
    a seed-0 runtime is its first word >> 8 times 2^-24."""
    _fresh(0)
    u = _uniform((4,)).numpy()
    assert u[0] == np.float32((0x6627E8D5 >> 8) * 2.0 ** -24)
    assert u.tobytes() == philox_np.uniform_f32(4, 0, 0).tobytes()


@pytest.mark.parametrize("seed", [0, 12345, (7 << 32) | 99])
def test_device_draws_match_oracle(seed):
    n = 1 << 20
    _fresh(seed)
    u32 = _uniform((n,)).numpy()
    u64 = _uniform((n,), sf.float64).numpy()
    z64 = _normal((n,), sf.float64).numpy()
    z32 = _normal((n,)).numpy()
    assert u32.tobytes() == philox_np.uniform_f32(n, seed, 0).tobytes()
    assert u64.tobytes() == philox_np.uniform_f64(n, seed, n).tobytes()
    want = philox_np.normal_f64(n, seed, 2 * n)
    np.testing.assert_allclose(z64, want, rtol=1e-12, atol=1e-13)
    want32 = philox_np.normal_f64(n, seed, 3 * n).astype(np.float32)
    # f32 rounding of (nearly) the same f64: equal except at rounding ties
    diff = np.abs(z32.astype(np.float64) - want32.astype(np.float64))
    assert np.count_nonzero(diff) <= 8
    np.testing.assert_allclose(z32, want32, rtol=2e-7, atol=1e-7)


def _ks_normal(x):
    from scipy.special import erf

    x = np.sort(x.astype(np.float64))
    n = x.size
    cdf = 0.5 * (1.0 + erf(x / math.sqrt(2.0)))
    i = np.arange(1, n + 1, dtype=np.float64)
    return max(np.max(i / n - cdf), np.max(cdf - (i - 1) / n))


def _ks_uniform(x):
    x = np.sort(x.astype(np.float64))
    n = x.size
    i = np.arange(1, n + 1, dtype=np.float64)
    return max(np.max(i / n - x), np.max(x - (i - 1) / n))


def test_device_normal_distribution_1e7():
    n = 10_000_000
    _fresh(2024)
    z = _normal((n,)).numpy().astype(np.float64)
    se = 1.0 / math.sqrt(n)
    assert abs(z.mean()) < 5 * se
    assert abs(z.var() - 1.0) < 5 * math.sqrt(2.0) * se
    m3 = np.mean(z ** 3)
    m4 = np.mean(z ** 4)
    assert abs(m3) < 5 * math.sqrt(15.0) * se          # skewness, var(z^3) = 15
    assert abs(m4 - 3.0) < 5 * math.sqrt(96.0) * se    # kurtosis, var(z^4) = 96
    # Kolmogorov-Smirnov: critical value at alpha = 0.001 is 1.95 / sqrt(n)
    assert _ks_normal(z) < 1.95 * se
    assert np.all(np.isfinite(z))


def test_device_uniform_distribution_1e7():
    n = 10_000_000
    _fresh(77)
    for dt in (sf.float32, sf.float64):
        u = _uniform((n,), dt).numpy().astype(np.float64)
        assert u.min() >= 0.0 and u.max() < 1.0
        se = 1.0 / math.sqrt(n)
        assert abs(u.mean() - 0.5) < 5 * math.sqrt(1 / 12) * se
        assert abs(u.var() - 1 / 12) < 5 * math.sqrt(1 / 180) * se
        assert _ks_uniform(u) < 1.95 * se
        # serial correlation of consecutive counters
        r = np.corrcoef(u[:-1], u[1:])[0, 1]
        assert abs(r) < 5 * se


def test_eager_draws_consume_disjoint_counter_ranges():
    """Two eager draws of n equal one draw of 2n: each draw reserves exactly
    its element count, so consecutive draws never reuse a counter; normals
    and uniforms share the counter space."""
    n = 100003
    _fresh(5)
    a = _normal((n,)).numpy()
    b = _uniform((n,)).numpy()
    c = _normal((7, 11)).numpy()
    _fresh(5)
    whole_z = _normal((2 * n + 77,)).numpy()
    _fresh(5)
    whole_u = _uniform((2 * n + 77,)).numpy()
    assert a.tobytes() == whole_z[:n].tobytes()
    assert b.tobytes() == whole_u[n:2 * n].tobytes()
    assert c.reshape(-1).tobytes() == whole_z[2 * n:].tobytes()


@pytest.mark.parametrize("b", [1000, 100000])
def test_staged_and_eager_draws_share_one_counter_sequence(b):
    """A staged function whose draws are fused into its row kernel reserves
    the same counter ranges, in program order, as the eager ops would; an
    eager draw after the staged call continues after them."""

    def f(x):
        v = sf.random_normal((b, 2))
        u = plugins.random_uniform((b,))
        w = sf.add(sf.mul(v, 2.0), x)
        return w, sf.mul(u, 3.0)

    x0 = np.random.default_rng(1).standard_normal((b, 2)).astype(np.float32)
    outs = {}
    for mode in ("eager", "staged"):
        _fresh(11)
        fn = sf.stage(f) if mode == "staged" else f
        x = sf.constant(x0)
        r1 = [t.numpy() for t in fn(x)]
        r2 = [t.numpy() for t in fn(x)]
        tail = _uniform((5,)).numpy()
        outs[mode] = (r1, r2, tail)
    for (ga, gb), (wa, wb) in zip(outs["staged"][:2], outs["eager"][:2]):
        assert ga.tobytes() == wa.tobytes() and gb.tobytes() == wb.tobytes()
    assert outs["staged"][2].tobytes() == outs["eager"][2].tobytes()
    # and the counters are exactly the oracle's: call k draws 2b normals then b uniforms
    off = 0
    for (w, u) in outs["eager"][:2]:
        v = philox_np.normal_f64(2 * b, 11, off).astype(np.float32).reshape(b, 2)
        np.testing.assert_allclose(w, v * np.float32(2.0) + x0, rtol=1e-6, atol=1e-6)
        uu = philox_np.uniform_f32(b, 11, off + 2 * b)
        assert u.tobytes() == (uu * np.float32(3.0)).tobytes()
        off += 3 * b
    assert outs["eager"][2].tobytes() == philox_np.uniform_f32(5, 11, off).tobytes()
