"""NumPy restatements of the benchmark workloads (oracle; test-only).

Each follows the op order of the reference program it restates, in the
same dtype, so with NumPy underneath it reproduces the reference's own
results bit-for-bit (pinned by tests/test_oracle.py against the golden
vectors generated from the reference).
"""
from __future__ import annotations

import numpy as np

F32 = np.float32


# ---------------------------------------------------------------------------
# leapfrog — stageflow/bench.py:147-183
# ---------------------------------------------------------------------------

def _leapfrog_force(q):
    # Tape gradient of U = 0.5 * sum(q*q): the mul rule contributes
    # up*q twice (gradients.py:125-132) with up = broadcast(0.5), accumulated
    # by add (tape.py:200-211).
    half = F32(0.5) * F32(1.0)
    g = np.full(q.shape, half, dtype=F32)
    return np.add(g * q, g * q)


def leapfrog_init(batch, seed=0):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((batch, 2)).astype(F32)
    p = rng.standard_normal((batch, 2)).astype(F32)
    return q, p


def leapfrog_trajectory(q, p, n_steps=10, step=0.1):
    half = F32(step / 2.0)
    eps = F32(step)
    for _ in range(n_steps):
        p = p - _leapfrog_force(q) * half
        q = q + p * eps
        p = p - _leapfrog_force(q) * half
    return q, p


def leapfrog(batch, seed=0, trajectories=1):
    """Concatenated (q, p) after `trajectories` trajectories (run_iteration output)."""
    q, p = leapfrog_init(batch, seed)
    for _ in range(trajectories):
        q, p = leapfrog_trajectory(q, p)
    return np.concatenate([q.ravel(), p.ravel()])


# ---------------------------------------------------------------------------
# mlp_train — stageflow/bench.py:103-144
# ---------------------------------------------------------------------------

class MLPTrain:
    IN, HIDDEN, OUT = 128, 256, 1
    LR = 1e-3

    def __init__(self, batch, seed=0):
        rng = np.random.default_rng(seed)
        self.x = (rng.standard_normal((batch, self.IN)) * 0.5).astype(F32)
        self.y = rng.standard_normal((batch, self.OUT)).astype(F32)
        self.w1 = (rng.standard_normal((self.IN, self.HIDDEN)) * 0.05).astype(F32)
        self.b1 = np.zeros(self.HIDDEN, dtype=F32)
        self.w2 = (rng.standard_normal((self.HIDDEN, self.OUT)) * 0.05).astype(F32)
        self.b2 = np.zeros(self.OUT, dtype=F32)

    def step(self):
        x, y = self.x, self.y
        pre = np.matmul(x, self.w1) + self.b1
        h = np.maximum(pre, 0).astype(F32)
        pred = np.matmul(h, self.w2) + self.b2
        err = pred - y
        loss = np.mean(err * err)
        count = err.size
        g = np.full(err.shape, F32(1.0) * F32(1.0 / count), dtype=F32)
        g_err = np.add(g * err, g * err)
        g_b2 = np.sum(g_err, axis=0).astype(F32)
        g_h = np.matmul(g_err, np.ascontiguousarray(self.w2.T))
        g_w2 = np.matmul(np.ascontiguousarray(h.T), g_err)
        g_pre = g_h * (pre > 0).astype(F32)
        g_b1 = np.sum(g_pre, axis=0).astype(F32)
        g_w1 = np.matmul(np.ascontiguousarray(x.T), g_pre)
        lr = F32(-self.LR)
        self.w1 = self.w1 + g_w1 * lr
        self.b1 = self.b1 + g_b1 * lr
        self.w2 = self.w2 + g_w2 * lr
        self.b2 = self.b2 + g_b2 * lr
        return float(loss)


def mlp_losses(batch, iterations, seed=0):
    m = MLPTrain(batch, seed)
    return np.array([m.step() for _ in range(iterations)], dtype=np.float64)


# ---------------------------------------------------------------------------
# L2HMC sampler — builder-defined (paper_1903_01855_b200/workloads/l2hmc.py)
# ---------------------------------------------------------------------------

class L2HMC:
    """NumPy restatement of workloads/l2hmc.py op for op, in float32.

    Random draws follow the reference runtime's host stream
    (``default_rng(runtime_seed)``): per transition standard_normal((B,2))
    for the forward and the backward kernels, then random((B,)) for the
    direction and random((B,)) for the accept test.
    """

    X_DIM, N_HIDDEN, N_STEPS, EPS = 2, 10, 10, 0.1

    def __init__(self, batch, seed=0, runtime_seed=0, x0=None):
        import math

        rng = np.random.default_rng(seed)
        self.batch = batch

        def dense(n_in, n_out, f):
            w = (rng.standard_normal((n_in, n_out)) * math.sqrt(2.0 * f / n_in)).astype(F32)
            return w, np.zeros((1, n_out), dtype=F32)

        def net(factor):
            return dict(v=dense(2, 10, 1 / 3), x=dense(2, 10, factor / 3), t=dense(2, 10, 1 / 3),
                        h=dense(10, 10, 1.0), scale=dense(10, 2, 0.001), transl=dense(10, 2, 0.001),
                        transf=dense(10, 2, 0.001), cs=np.zeros((1, 2), F32),
                        ct=np.zeros((1, 2), F32))

        self.pos_net = net(2.0)
        self.mom_net = net(1.0)
        sigma = np.array([[50.05, -49.95], [-49.95, 50.05]])
        self.A = np.linalg.inv(sigma).astype(F32)
        self.ts = [np.array([[math.cos(2 * math.pi * i / 10), math.sin(2 * math.pi * i / 10)]],
                            dtype=F32) for i in range(10)]
        self.masks = []
        for _ in range(10):
            idx = rng.permutation(2)[:1]
            m = np.zeros((1, 2))
            m[0, idx] = 1.0
            self.masks.append((m.astype(F32), (1.0 - m).astype(F32)))
        x = rng.standard_normal((batch, 2)).astype(F32)
        self.x = x if x0 is None else np.asarray(x0, dtype=F32)
        self.rt = np.random.default_rng(runtime_seed)

    @staticmethod
    def _dense(layer, x):
        w, b = layer
        return np.matmul(x, w) + b

    def _net(self, n, v, x, t):
        h = (self._dense(n["v"], v) + self._dense(n["x"], x)) + self._dense(n["t"], t)
        h = np.maximum(h, 0).astype(F32)
        h = np.maximum(self._dense(n["h"], h), 0).astype(F32)
        scale = np.tanh(self._dense(n["scale"], h)) * np.exp(n["cs"])
        transl = self._dense(n["transl"], h)
        transf = np.tanh(self._dense(n["transf"], h)) * np.exp(n["ct"])
        return scale, transl, transf

    def potential(self, x):
        return np.sum(np.matmul(x, self.A) * x, axis=1).astype(F32) * F32(0.5)

    def grad_potential(self, x):
        g = np.full(x.shape, F32(1.0) * F32(0.5), dtype=F32)
        xa = np.matmul(x, self.A)
        return np.add(g * xa, np.matmul(g * x, np.ascontiguousarray(self.A.T)))

    def hamiltonian(self, x, v):
        return self.potential(x) + np.sum(v * v, axis=1).astype(F32) * F32(0.5)

    def _mom(self, x, v, t, fwd):
        e = F32(self.EPS)
        grad = self.grad_potential(x)
        scale, transl, transf = self._net(self.mom_net, x, grad, t)
        scale = scale * (F32(0.5 * self.EPS) if fwd else F32(-0.5 * self.EPS))
        transf = transf * e
        inner = (np.exp(transf) * grad - transl) * F32(0.5 * self.EPS)
        v = v * np.exp(scale) - inner if fwd else np.exp(scale) * (v + inner)
        return v, np.sum(scale, axis=1).astype(F32)

    def _pos(self, x, v, t, mask, mask_inv, fwd):
        e = F32(self.EPS)
        scale, transl, transf = self._net(self.pos_net, v, mask * x, t)
        scale = scale * (e if fwd else F32(-self.EPS))
        transf = transf * e
        if fwd:
            moved = x * np.exp(scale) + (np.exp(transf) * v + transl) * e
            x = mask * x + mask_inv * moved
        else:
            back = x - (np.exp(transf) * v + transl) * e
            x = mask * x + mask_inv * (np.exp(scale) * back)
        return x, np.sum(mask_inv * scale, axis=1).astype(F32)

    def _lf(self, x, v, i, fwd):
        j = i if fwd else self.N_STEPS - i - 1
        t = self.ts[j]
        m, mi = self.masks[j]
        v, l1 = self._mom(x, v, t, fwd)
        if fwd:
            x, l2 = self._pos(x, v, t, m, mi, True)
            x, l3 = self._pos(x, v, t, mi, m, True)
        else:
            x, l2 = self._pos(x, v, t, mi, m, False)
            x, l3 = self._pos(x, v, t, m, mi, False)
        v, l4 = self._mom(x, v, t, fwd)
        return x, v, (l1 + l2) + (l3 + l4)

    def _kernel(self, x, fwd, v=None):
        if v is None:
            v = self.rt.standard_normal((self.batch, 2)).astype(F32)
        xp, vp, logdet = x, v, None
        for i in range(self.N_STEPS):
            xp, vp, ld = self._lf(xp, vp, i, fwd)
            logdet = ld if logdet is None else logdet + ld
        delta = (self.hamiltonian(x, v) - self.hamiltonian(xp, vp)) + logdet
        with np.errstate(over="ignore", invalid="ignore"):
            prob = np.exp(np.minimum(delta, F32(0.0)))
        prob = np.where(np.isfinite(prob), prob, F32(0.0)).astype(F32)
        return xp, prob

    def transition(self):
        x = self.x
        b = self.batch
        vf = self.rt.standard_normal((b, 2)).astype(F32)
        vb = self.rt.standard_normal((b, 2)).astype(F32)
        u_dir = self.rt.random((b,)).astype(F32)
        u_acc = self.rt.random((b,)).astype(F32)
        self.x, acc_prob = self.transition_with(x, vf, vb, u_dir, u_acc)
        return np.concatenate([self.x.ravel(), acc_prob.ravel()])

    def transition_with(self, x, vf, vb, u_dir, u_acc):
        """One transition of state x with the four draws given (the
        ``draws="inputs"`` program); returns (x_out, accept_prob)."""
        b = x.shape[0]
        xf, pf = self._kernel(x, True, vf)
        xb, pb = self._kernel(x, False, vb)
        fwd = (u_dir > F32(0.5)).astype(F32)
        bwd = F32(1.0) - fwd
        x_post = fwd.reshape(b, 1) * xf + bwd.reshape(b, 1) * xb
        acc_prob = fwd * pf + bwd * pb
        acc = (acc_prob > u_acc).astype(F32)
        x_out = acc.reshape(b, 1) * x_post + (F32(1.0) - acc).reshape(b, 1) * x
        return x_out, acc_prob


# ---------------------------------------------------------------------------
# C2 microbenchmark — builder-defined
# ---------------------------------------------------------------------------

C2_LAYERS, C2_WIDTH = 100, 16


def c2_params(seed=0, layers=C2_LAYERS, width=C2_WIDTH):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((1, width)).astype(F32)
    ws, bs = [], []
    for _ in range(layers):
        ws.append((rng.standard_normal((width, width)) * 0.3).astype(F32))
        bs.append((rng.standard_normal((1, width)) * 0.1).astype(F32))
    return x, ws, bs


def c2_chain(x, ws, bs):
    for w, b in zip(ws, bs):
        x = np.tanh(np.matmul(x, w) + b)
    return x


def c2_chain_grad(x, ws, bs):
    """d sum(chain(x)) / dx via the tanh rule up*(1 - y*y)."""
    ys = []
    h = x
    for w, b in zip(ws, bs):
        h = np.tanh(np.matmul(h, w) + b)
        ys.append(h)
    g = np.ones_like(h)
    for w, y in zip(reversed(ws), reversed(ys)):
        g = g * (F32(1.0) - y * y)
        g = np.matmul(g, np.ascontiguousarray(w.T))
    return g
