"""L2HMC sampler on the 2-D strongly-correlated Gaussian (BASELINE config C1/C3).

Builder-defined, following the structure of the paper's public TF example
(l2hmc Dynamics + GenericNet): the generalized leapfrog with learned
scale / translation / transformation nets, forward and backward
trajectories, a uniformly drawn direction and a Metropolis-Hastings accept
step.  The reference has no L2HMC; its ops that are missing
there (tanh, minimum, select, is_finite, cast, random_uniform) are plugin
ops registered through ``register_op`` on both sides.

The program is written against an API module ``sf`` so the SAME user code
runs on this backend (``paper_1903_01855_b200``) and on the reference
(``stageflow`` + oracle/ref_plugins.py) — that run is the oracle for the
golden fixtures.  Energy: U(x) = 1/2 x^T Sigma^-1 x with
Sigma = [[50.05, -49.95], [-49.95, 50.05]]; eps = 0.1; 10 leapfrog steps;
hidden width 10.
"""
from __future__ import annotations

import math

import numpy as np

X_DIM = 2
N_HIDDEN = 10
N_STEPS = 10
EPS = 0.1
SIGMA = np.array([[50.05, -49.95], [-49.95, 50.05]])


def _f32(sf, arr):
    arr = np.asarray(arr, dtype=np.float32)
    return sf.tensor_from_host(arr.reshape(-1), arr.shape, sf.float32)


class _Net:
    """GenericNet: h = relu(relu(V v + X x + T t) H); three heads.
    ``trainable``: the weights are Variables (L2HMCTrain) instead of
    immutable tensors."""

    def __init__(self, sf, rng, factor, trainable: bool = False):
        def param(arr):
            t = _f32(sf, arr)
            if trainable:
                t = sf.Variable(t)
                self.variables.append(t)
            return t

        self.variables = []

        def dense(n_in, n_out, f):
            w = rng.standard_normal((n_in, n_out)) * math.sqrt(2.0 * f / n_in)
            return param(w), param(np.zeros((1, n_out)))

        self.v = dense(X_DIM, N_HIDDEN, 1.0 / 3.0)
        self.x = dense(X_DIM, N_HIDDEN, factor / 3.0)
        self.t = dense(2, N_HIDDEN, 1.0 / 3.0)
        self.h = dense(N_HIDDEN, N_HIDDEN, 1.0)
        self.scale = dense(N_HIDDEN, X_DIM, 0.001)
        self.transl = dense(N_HIDDEN, X_DIM, 0.001)
        self.transf = dense(N_HIDDEN, X_DIM, 0.001)
        self.coeff_scale = param(np.zeros((1, X_DIM)))
        self.coeff_transf = param(np.zeros((1, X_DIM)))


class L2HMCSampler:
    """apply_transition(x) -> (x_out, accept_prob); staged or eager.

    ``draws="runtime"`` (the benchmarked program): the momenta and the two
    uniforms come from the runtime's random ops inside the transition (device
    Philox fused into the row kernel, or the host PCG64 stream).
    ``draws="inputs"``: the same program with the four draws passed in as
    arguments, ``apply_transition(x, v_fwd, v_bwd, u_dir, u_acc)``; they are
    drawn on the host from ``default_rng(draw_seed)`` in the reference
    runtime's order (oracle/workloads_np.py L2HMC) — the staged program is then
    still one fused row kernel, and comparable with the oracle at any batch.
    """

    gate_tol = 1e-5

    def __init__(self, sf, batch: int, mode: str = "staged", seed: int = 0,
                 draws: str = "runtime", draw_seed: int = 0, trainable: bool = False):
        if draws not in ("runtime", "inputs"):
            raise ValueError(f"draws must be 'runtime' or 'inputs', got {draws!r}")
        self.sf = sf
        self.batch = batch
        self.draws = draws
        self.draw_rng = np.random.default_rng(draw_seed)
        rng = np.random.default_rng(seed)
        self.position_fn = _Net(sf, rng, 2.0, trainable)
        self.momentum_fn = _Net(sf, rng, 1.0, trainable)
        self.variables = self.position_fn.variables + self.momentum_fn.variables
        self.sigma_inv = _f32(sf, np.linalg.inv(SIGMA))
        self.ts = [_f32(sf, [[math.cos(2 * math.pi * i / N_STEPS),
                              math.sin(2 * math.pi * i / N_STEPS)]]) for i in range(N_STEPS)]
        self.masks = []
        for _ in range(N_STEPS):
            idx = rng.permutation(X_DIM)[:X_DIM // 2]
            m = np.zeros((1, X_DIM))
            m[0, idx] = 1.0
            self.masks.append((_f32(sf, m), _f32(sf, 1.0 - m)))
        self.x = _f32(sf, rng.standard_normal((batch, X_DIM)))
        self.mode = mode
        fn = self.apply_transition
        self.transition = sf.stage(fn, name="l2hmc_transition") if mode == "staged" else fn
        self.staged_functions = [self.transition] if mode == "staged" else []

    # -- ops helpers -----------------------------------------------------------
    def _op(self, name, *xs, **attrs):
        return self.sf.dispatch(name, list(xs), attrs or None)[0]

    def _dense(self, layer, x):
        w, b = layer
        return self.sf.add(self.sf.matmul(x, w), b)

    def _net(self, net: _Net, v, x, t):
        sf = self.sf
        h = sf.add(sf.add(self._dense(net.v, v), self._dense(net.x, x)), self._dense(net.t, t))
        h = sf.relu(h)
        h = sf.relu(self._dense(net.h, h))
        scale = sf.mul(self._op("tanh", self._dense(net.scale, h)), sf.exp(net.coeff_scale))
        transl = self._dense(net.transl, h)
        transf = sf.mul(self._op("tanh", self._dense(net.transf, h)), sf.exp(net.coeff_transf))
        return scale, transl, transf

    # -- energy -------------------------------------------------------------------
    def potential(self, x):
        sf = self.sf
        return sf.mul(sf.reduce_sum(sf.mul(sf.matmul(x, self.sigma_inv), x), axes=(1,)), 0.5)

    def grad_potential(self, x):
        sf = self.sf
        with sf.Tape() as tape:
            tape.watch(x)
            u = sf.reduce_sum(self.potential(x))
        return tape.gradient(u, x)

    def hamiltonian(self, x, v):
        sf = self.sf
        return sf.add(self.potential(x), sf.mul(sf.reduce_sum(sf.mul(v, v), axes=(1,)), 0.5))

    # -- leapfrog updates ------------------------------------------------------------
    def _momentum_fwd(self, x, v, t):
        sf = self.sf
        grad = self.grad_potential(x)
        scale, transl, transf = self._net(self.momentum_fn, x, grad, t)
        scale = sf.mul(scale, 0.5 * EPS)
        transf = sf.mul(transf, EPS)
        v = sf.sub(sf.mul(v, sf.exp(scale)),
                   sf.mul(sf.sub(sf.mul(sf.exp(transf), grad), transl), 0.5 * EPS))
        return v, sf.reduce_sum(scale, axes=(1,))

    def _position_fwd(self, x, v, t, mask, mask_inv):
        sf = self.sf
        scale, transl, transf = self._net(self.position_fn, v, sf.mul(mask, x), t)
        scale = sf.mul(scale, EPS)
        transf = sf.mul(transf, EPS)
        moved = sf.add(sf.mul(x, sf.exp(scale)),
                       sf.mul(sf.add(sf.mul(sf.exp(transf), v), transl), EPS))
        x = sf.add(sf.mul(mask, x), sf.mul(mask_inv, moved))
        return x, sf.reduce_sum(sf.mul(mask_inv, scale), axes=(1,))

    def _momentum_bwd(self, x, v, t):
        sf = self.sf
        grad = self.grad_potential(x)
        scale, transl, transf = self._net(self.momentum_fn, x, grad, t)
        scale = sf.mul(scale, -0.5 * EPS)
        transf = sf.mul(transf, EPS)
        v = sf.mul(sf.exp(scale),
                   sf.add(v, sf.mul(sf.sub(sf.mul(sf.exp(transf), grad), transl), 0.5 * EPS)))
        return v, sf.reduce_sum(scale, axes=(1,))

    def _position_bwd(self, x, v, t, mask, mask_inv):
        sf = self.sf
        scale, transl, transf = self._net(self.position_fn, v, sf.mul(mask, x), t)
        scale = sf.mul(scale, -EPS)
        transf = sf.mul(transf, EPS)
        back = sf.sub(x, sf.mul(sf.add(sf.mul(sf.exp(transf), v), transl), EPS))
        x = sf.add(sf.mul(mask, x), sf.mul(mask_inv, sf.mul(sf.exp(scale), back)))
        return x, sf.reduce_sum(sf.mul(mask_inv, scale), axes=(1,))

    def _lf(self, x, v, i, forward):
        sf = self.sf
        if forward:
            t = self.ts[i]
            mask, mask_inv = self.masks[i]
            v, l1 = self._momentum_fwd(x, v, t)
            x, l2 = self._position_fwd(x, v, t, mask, mask_inv)
            x, l3 = self._position_fwd(x, v, t, mask_inv, mask)
            v, l4 = self._momentum_fwd(x, v, t)
        else:
            j = N_STEPS - i - 1
            t = self.ts[j]
            mask, mask_inv = self.masks[j]
            v, l1 = self._momentum_bwd(x, v, t)
            x, l2 = self._position_bwd(x, v, t, mask_inv, mask)
            x, l3 = self._position_bwd(x, v, t, mask, mask_inv)
            v, l4 = self._momentum_bwd(x, v, t)
        return x, v, sf.add(sf.add(l1, l2), sf.add(l3, l4))

    def transition_kernel(self, x, forward, v=None):
        sf = self.sf
        if v is None:
            v = sf.random_normal((self.batch, X_DIM))
        x_post, v_post = x, v
        logdet = None
        for i in range(N_STEPS):
            x_post, v_post, ld = self._lf(x_post, v_post, i, forward)
            logdet = ld if logdet is None else sf.add(logdet, ld)
        delta = sf.add(sf.sub(self.hamiltonian(x, v), self.hamiltonian(x_post, v_post)), logdet)
        prob = sf.exp(self._op("minimum", delta, _f32(sf, 0.0)))
        finite = self._op("is_finite", prob)
        prob = self._op("select", finite, prob, _f32(sf, 0.0))
        return x_post, v_post, prob

    def apply_transition(self, x, v_fwd=None, v_bwd=None, u_dir=None, u_acc=None):
        x_out, accept_prob, _x_post = self.propose(x, v_fwd, v_bwd, u_dir, u_acc)
        return x_out, accept_prob

    def propose(self, x, v_fwd=None, v_bwd=None, u_dir=None, u_acc=None):
        """(state after the MH step, acceptance probability, the proposal)."""
        sf = self.sf
        b = self.batch
        x_f, _v_f, p_f = self.transition_kernel(x, True, v_fwd)
        x_b, _v_b, p_b = self.transition_kernel(x, False, v_bwd)
        if u_dir is None:
            u_dir = self._op("random_uniform", shape=(b,), dtype=sf.float32)
        fwd = self._op("cast", sf.greater(u_dir, 0.5), dtype=sf.float32)
        bwd = sf.sub(1.0, fwd)
        fwd2, bwd2 = sf.reshape(fwd, (b, 1)), sf.reshape(bwd, (b, 1))
        x_post = sf.add(sf.mul(fwd2, x_f), sf.mul(bwd2, x_b))
        accept_prob = sf.add(sf.mul(fwd, p_f), sf.mul(bwd, p_b))
        if u_acc is None:
            u_acc = self._op("random_uniform", shape=(b,), dtype=sf.float32)
        acc = self._op("cast", sf.greater(accept_prob, u_acc), dtype=sf.float32)
        acc2 = sf.reshape(acc, (b, 1))
        x_out = sf.add(sf.mul(acc2, x_post), sf.mul(sf.reshape(sf.sub(1.0, acc), (b, 1)), x))
        return x_out, accept_prob, x_post

    # -- harness -------------------------------------------------------------------
    def host_draws(self):
        """The four draws of one transition, in the reference runtime's
        order: normal (B,2) forward, normal (B,2) backward, uniform (B,)
        direction, uniform (B,) accept (f64 draws rounded to f32)."""
        r, b = self.draw_rng, self.batch
        return (r.standard_normal((b, X_DIM)).astype(np.float32),
                r.standard_normal((b, X_DIM)).astype(np.float32),
                r.random((b,)).astype(np.float32), r.random((b,)).astype(np.float32))

    def step(self, draws=None):
        if self.draws == "inputs":
            if draws is None:
                draws = self.host_draws()
            ts = [self.sf.tensor_from_host(d.reshape(-1), d.shape, self.sf.float32)
                  for d in draws]
            self.x, self.accept = self.transition(self.x, *ts)
        else:
            self.x, self.accept = self.transition(self.x)
        return self.x

    def run_iteration(self):
        self.step()
        return np.concatenate([self.x.numpy().ravel(), self.accept.numpy().ravel()])

    def cache_size(self) -> int:
        return sum(pf.cache_size for pf in self.staged_functions)


class L2HMCTrain:
    """Training the L2HMC sampler (the paper's L2HMC figure: PAPER.md, the
    TF Eager l2hmc example's ``compute_loss``): the networks are Variables;
    one step draws z ~ N(0, I), proposes from the chains x and from z, and
    minimises

        l = mean(scale / d_x + scale / d_z - (d_x + d_z) / scale),
        d = |x - x'|^2 * A(x' | x) + eps

    (expected squared jump distance, both samples), then applies
    ``v += -lr * grad``.  Staged mode mirrors the reference's mlp_train
    pattern (stageflow/bench.py:131-144): the loss (both full transitions,
    with the potential's tape gradient inside each leapfrog step) is one
    staged function, the tape derives its staged backward — through every
    leapfrog step, the networks and the MH step — and the update is a
    second staged function."""

    SCALE, EPS, LR = 0.1, 1e-4, 1e-3
    gate_tol = 1e-5

    def __init__(self, sf, batch: int, mode: str = "staged", seed: int = 0):
        self.sf = sf
        self.sampler = L2HMCSampler(sf, batch, "eager", seed=seed, trainable=True)
        self.params = self.sampler.variables
        s, b = self.sampler, batch

        def forward_loss(x):
            z = sf.random_normal((b, X_DIM))
            x_out, x_acc, x_prop = s.propose(x)
            _z_out, z_acc, z_prop = s.propose(z)

            def jump(a, a_prop, acc):
                d = sf.sub(a, a_prop)
                return sf.add(sf.mul(sf.reduce_sum(sf.mul(d, d), axes=(1,)), acc), self.EPS)

            dx, dz = jump(x, x_prop, x_acc), jump(z, z_prop, z_acc)
            inv = sf.add(sf.div(1.0, dx), sf.div(1.0, dz))
            per_chain = sf.sub(sf.mul(inv, self.SCALE), sf.div(sf.add(dx, dz), self.SCALE))
            return sf.reduce_mean(per_chain), x_out

        def apply_updates(*grads):
            for v, g in zip(self.params, grads):
                v.assign_add(sf.mul(g, -self.LR))

        if mode == "staged":
            self.forward_loss = sf.stage(forward_loss, name="l2hmc_train_loss")
            self.apply_updates = sf.stage(apply_updates, name="l2hmc_train_apply")
            self.staged_functions = [self.forward_loss, self.apply_updates]
        else:
            self.forward_loss = forward_loss
            self.apply_updates = apply_updates
            self.staged_functions = []
        self.x = s.x

    def step(self):
        sf = self.sf
        with sf.Tape() as t:
            loss, x_out = self.forward_loss(self.x)
        grads = t.gradient(loss, self.params)
        self.apply_updates(*grads)
        self.x = x_out
        return loss

    def run_iteration(self) -> float:
        return float(self.step())
