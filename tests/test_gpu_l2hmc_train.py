"""Training the L2HMC sampler (workloads/l2hmc.py L2HMCTrain): the tape's
staged backward runs through both full transitions — every leapfrog step,
the networks, the potential's own tape gradient and the MH step — and must
equal the eager tape bit for bit; the update must move the parameters.
The reference has no L2HMC: this is eager-vs-staged parity
on this backend, with the loss's finite-difference check at small size."""
import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import plugins
from paper_1903_01855_b200.workloads import l2hmc

pytestmark = pytest.mark.gpu


def _run(mode, steps, batch=16):
    sf.init_runtime(sf.RuntimeOptions(seed=11))
    plugins.install()
    tr = l2hmc.L2HMCTrain(sf, batch, mode, seed=0)
    before = [p.read_value().numpy() for p in tr.params]
    losses = [tr.run_iteration() for _ in range(steps)]
    after = [p.read_value().numpy() for p in tr.params]
    return losses, before, after, tr


def test_l2hmc_training_eager_equals_staged_bitwise():
    le, be, ae, _ = _run("eager", 2)
    ls, bs, as_, tr = _run("staged", 2)
    assert np.float32(le).tobytes() == np.float32(ls).tobytes()
    for a, b in zip(ae, as_):
        assert a.tobytes() == b.tobytes()
    assert any(np.any(a != b) for a, b in zip(as_, bs))  # the update moved something
    assert [pf.cache_size for pf in tr.staged_functions] == [1, 1]


def test_l2hmc_training_gradient_matches_finite_difference():
    """d loss / d (one network bias) against a central difference of the
    staged loss, with the draws fixed by reseeding (same Philox counters)."""
    sf.init_runtime(sf.RuntimeOptions(seed=5))
    plugins.install()
    tr = l2hmc.L2HMCTrain(sf, 64, "staged", seed=0)
    p = tr.sampler.position_fn.h[1]      # hidden-layer bias, (1, 10)
    rt = sf.get_runtime()

    def loss_at(delta):
        rt.reseed(5)
        base = p.read_value().numpy()
        p.assign(sf.constant((base + delta).astype(np.float32)))
        loss, _ = tr.forward_loss(tr.x)
        p.assign(sf.constant(base))
        return float(loss)

    rt.reseed(5)
    with sf.Tape() as t:
        loss, _ = tr.forward_loss(tr.x)
    g = t.gradient(loss, [p])[0].numpy().ravel()
    h = 1e-2
    j = int(np.argmax(np.abs(g)))
    e = np.zeros((1, 10), np.float32)
    e[0, j] = h
    fd = (loss_at(e) - loss_at(-e)) / (2 * h)
    assert abs(fd - g[j]) <= 0.05 * abs(g[j]) + 1e-3, (fd, g[j])
