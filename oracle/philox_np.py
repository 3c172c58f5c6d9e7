"""TEST INFRASTRUCTURE ONLY — never imported by the product path.

NumPy restatement of the backend's device RNG (csrc/sf_ops.cuh ``philox``,
``uniform_f32``, ``uniform_f64``, ``normal_f64``), the generator behind the
``random_normal`` / ``random_uniform`` / ``dropout`` kernels in device-RNG
mode.  The reference draws from a host PCG64 stream instead
(stageflow/runtime.py:124-127, stageflow/kernels.py:372-404); its stream is
reproduced by the backend's ``rng="host"`` mode and checked against golden
vectors elsewhere.  This file pins the *device* generator:

* Philox4x32-10 (Salmon et al., SC'11, "Parallel random numbers: as easy as
  1, 2, 3"; Random123 ``philox4x32_10``) — checked against the published
  Random123 known-answer vectors (``KAT`` below, tests/test_oracle.py);
* element ``i`` of a draw with (seed, offset) uses counter
  ``(offset + i, 0, 0, 0)`` (low/high 32 bits of the 64-bit counter in words
  0/1) and key ``(seed_lo, seed_hi)``;
* uniform f32 = (x >> 8) * 2^-24; uniform f64 = ((x >> 5) << 26 | y >> 6) *
  2^-53; normal = Box-Muller on two 53-bit uniforms, u1 in (0, 1].
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)

# Random123 philox4x32_10 known-answer vectors: (counter, key, output)
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 over uint32-valued arrays; returns 4 uint64
    arrays holding 32-bit words."""
    c = [np.asarray(x, dtype=np.uint64) & _MASK for x in (c0, c1, c2, c3)]
    k = [np.asarray(x, dtype=np.uint64) & _MASK for x in (k0, k1)]
    m0, m1 = np.uint64(M0), np.uint64(M1)
    s = np.uint64(32)
    for _ in range(10):
        p0 = m0 * c[0]
        p1 = m1 * c[2]
        c = [(p1 >> s) ^ c[1] ^ k[0], p1 & _MASK, (p0 >> s) ^ c[3] ^ k[1], p0 & _MASK]
        k = [(k[0] + np.uint64(W0)) & _MASK, (k[1] + np.uint64(W1)) & _MASK]
    return c


def _words(n, seed, offset):
    ctr = np.uint64(offset) + np.arange(n, dtype=np.uint64)
    seed = np.uint64(seed)
    return philox4x32_10(ctr & _MASK, ctr >> np.uint64(32), 0, 0, seed & _MASK,
                         seed >> np.uint64(32))


def uniform_f32(n, seed=0, offset=0):
    x = _words(n, seed, offset)[0]
    return (x >> np.uint64(8)).astype(np.float32) * np.float32(2.0 ** -24)


def _u53(a, b):
    return ((a >> np.uint64(5)) << np.uint64(26)) | (b >> np.uint64(6))


def uniform_f64(n, seed=0, offset=0):
    x, y, _, _ = _words(n, seed, offset)
    return _u53(x, y).astype(np.float64) * 2.0 ** -53


def normal_f64(n, seed=0, offset=0):
    """f64 Box-Muller; the device rounds this once to the output dtype.  The
    device uses cospi(2 u2); numpy's cos(2 pi u2) differs from it by ulps."""
    x, y, z, w = _words(n, seed, offset)
    u1 = (_u53(x, y).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = _u53(z, w).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
