"""The tcgen05 3xTF32 GEMM (csrc/sf_gemm_tc.cu) against float64 numpy."""
import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k", [(128, 128, 32), (256, 128, 64), (200, 96, 36), (1000, 64, 148),
                                   (5000, 256, 576), (130, 1000, 2048), (33, 7, 4)])
def test_gemm_tf32x3_vs_float64(m, n, k):
    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((n, k)).astype(np.float32)
    ta, tb = sf.constant(a), sf.constant(b)
    ahi, alo = _native.split_tf32(0, m, k, ta._ptr())
    bhi, blo = _native.split_tf32(0, n, k, tb._ptr())
    c = _native.gemm_tf32x3(0, m, n, k, ahi.ptr, alo.ptr, bhi.ptr, blo.ptr)
    got = _native.download(c, np.float32, (m, n))
    want = a.astype(np.float64) @ b.astype(np.float64).T
    err = np.abs(got - want).max() / (np.abs(a).max() * np.abs(b).max() * np.sqrt(k))
    assert err < 1e-5, err
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-4 * np.sqrt(k))


@pytest.mark.parametrize("m,n,k", [(512, 64, 576), (300, 128, 147), (1000, 256, 64)])
def test_gemm_with_transposed_split_b(m, n, k):
    """C = A @ W with W (k x n) row-major: B = W^T via the transposing split."""
    rng = np.random.default_rng(1)
    a = rng.standard_normal((m, k)).astype(np.float32)
    w = rng.standard_normal((k, n)).astype(np.float32)
    kp = (k + 3) // 4 * 4
    ap = np.zeros((m, kp), np.float32)
    ap[:, :k] = a
    ta, tw = sf.constant(ap), sf.constant(w)
    ahi, alo = _native.split_tf32(0, m, kp, ta._ptr())
    bhi, blo = _native.split_tf32(0, k, n, tw._ptr(), transpose=True, ldo=kp)
    c = _native.gemm_tf32x3(0, m, n, kp, ahi.ptr, alo.ptr, bhi.ptr, blo.ptr)
    got = _native.download(c, np.float32, (m, n))
    np.testing.assert_allclose(got, a.astype(np.float64) @ w, rtol=1e-4, atol=1e-4 * np.sqrt(k))


def test_split_transpose_padding():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((37, 20)).astype(np.float32)
    tx = sf.constant(x)  # keep the source alive while the kernel reads it
    hi, lo = _native.split_tf32(0, 37, 20, tx._ptr(), transpose=True, ldo=40)
    h = _native.download(hi, np.float32, (20, 40))
    l_ = _native.download(lo, np.float32, (20, 40))
    np.testing.assert_array_equal(h[:, :37] + l_[:, :37], x.T)
    assert not np.any(h[:, 37:]) and not np.any(l_[:, 37:])
    assert np.all((h.view(np.uint32) & 0x1FFF) == 0)


@pytest.mark.parametrize("a_mn,b_mn", [(False, True), (True, False), (True, True)])
@pytest.mark.parametrize("m,n,k,ak,bk", [(128, 64, 64, 64, 64), (200, 96, 100, 100, 97),
                                         (516, 256, 3000, 3000, 3000), (36, 128, 33, 33, 33),
                                         (9600, 512, 96, 96, 96)])  # 256-wide tiles
def test_gemm_mn_major_operands(a_mn, b_mn, m, n, k, ak, bk):
    """MN-major operands (A stored k x m, B stored k x n) read straight by TMA,
    no transposed copies; an operand holding fewer than k contraction rows
    reads zeros beyond them.  Must equal the K-major GEMM on the same data."""
    rng = np.random.default_rng(m * 7 + n + k)
    a = np.zeros((m, k), np.float32)
    b = np.zeros((n, k), np.float32)
    a[:, :ak] = rng.standard_normal((m, ak))
    b[:, :bk] = rng.standard_normal((n, bk))
    if not a_mn and ak % 4:
        pytest.skip("K-major leading dimension must be a multiple of 4")
    if not b_mn and bk % 4:
        pytest.skip("K-major leading dimension must be a multiple of 4")
    a_store = np.ascontiguousarray(a[:, :ak].T if a_mn else a[:, :ak])
    b_store = np.ascontiguousarray(b[:, :bk].T if b_mn else b[:, :bk])
    ta, tb = sf.constant(a_store), sf.constant(b_store)
    ah, al = _native.split_tf32(0, *a_store.shape, ta._ptr())
    bh, bl = _native.split_tf32(0, *b_store.shape, tb._ptr())
    c = _native.gemm_tf32x3_ex(0, m, n, k, a_mn, b_mn, ak, bk, ah.ptr, al.ptr, bh.ptr, bl.ptr)
    got = _native.download(c, np.float32, (m, n))
    want = a.astype(np.float64) @ b.astype(np.float64).T
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-4 * np.sqrt(k))
    if k % 4 == 0 and ak == k and bk == k:
        # same products, same accumulation order as the K-major path: same bits
        ta2, tb2 = sf.constant(a), sf.constant(b)
        ah2, al2 = _native.split_tf32(0, m, k, ta2._ptr())
        bh2, bl2 = _native.split_tf32(0, n, k, tb2._ptr())
        ref = _native.gemm_tf32x3(0, m, n, k, ah2.ptr, al2.ptr, bh2.ptr, bl2.ptr)
        assert _native.download(ref, np.float32, (m, n)).tobytes() == got.tobytes()


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("lo_a,lo_b", [(True, True), (True, False), (False, True)])
@pytest.mark.parametrize("m,n,k,ak,bk", [(128, 64, 64, 64, 64), (200, 96, 100, 100, 97),
                                         (516, 256, 3000, 3000, 3000), (1000, 200, 36, 36, 33),
                                         (9600, 512, 96, 96, 96)])  # 256-wide tiles
def test_gemm_lo_in_shared_memory_bitwise(a_mn, b_mn, lo_a, lo_b, m, n, k, ak, bk):
    """A NULL lo pointer makes the GEMM derive that operand's tf32 lo part in
    shared memory from the raw fp32 tile (converter warps) instead of reading
    a precomputed lo matrix: same lo values, same MMA sequence, same bits."""
    if (not a_mn and ak % 4) or (not b_mn and bk % 4):
        pytest.skip("K-major leading dimension must be a multiple of 4")
    rng = np.random.default_rng(m + 3 * n + k)
    a = rng.standard_normal((m, ak)).astype(np.float32)
    b = rng.standard_normal((n, bk)).astype(np.float32)
    a_store = np.ascontiguousarray(a.T if a_mn else a)
    b_store = np.ascontiguousarray(b.T if b_mn else b)
    ta, tb = sf.constant(a_store), sf.constant(b_store)
    ah, al = _native.split_tf32(0, *a_store.shape, ta._ptr())
    bh, bl = _native.split_tf32(0, *b_store.shape, tb._ptr())
    ref = _native.gemm_tf32x3_ex(0, m, n, k, a_mn, b_mn, ak, bk, ah.ptr, al.ptr, bh.ptr, bl.ptr)
    got = _native.gemm_tf32x3_ex(0, m, n, k, a_mn, b_mn, ak, bk, ta._ptr(),
                                 0 if lo_a else al.ptr, tb._ptr(), 0 if lo_b else bl.ptr)
    r = _native.download(ref, np.float32, (m, n))
    assert _native.download(got, np.float32, (m, n)).tobytes() == r.tobytes()


@pytest.mark.parametrize("shape,filt,s,p", [
    ((2, 14, 14, 64), (3, 3, 64, 64), 1, 1),       # layer1-like 3x3, partial last tile
    ((3, 9, 11, 32), (3, 3, 32, 96), 1, 1),        # odd spatial extents, BN=128 path
    ((2, 16, 16, 128), (3, 3, 128, 128), 2, 1),    # strided 3x3 (layer2 entry)
    ((2, 14, 14, 256), (1, 1, 256, 512), 2, 0),    # strided 1x1 downsample
    ((2, 15, 15, 64), (5, 5, 64, 32), 3, 2),       # other window / stride / pad
    ((4, 28, 28, 64), (3, 3, 64, 256), 1, 1),      # BN=256 tiles
    ((1, 7, 7, 512), (3, 3, 512, 512), 1, 1),      # late layer: K = 4608, few tiles
])
def test_implicit_conv_equals_explicit_im2col_gemm(shape, filt, s, p, monkeypatch):
    """sf_conv2d_tc (the GEMM gathers its im2col rows with cp.async) is
    bit-identical to the explicit im2col + GEMM path, and fp32-accurate
    against a float64 convolution."""
    from paper_1903_01855_b200 import nn
    from oracle import nn_np

    nn.install()
    rng = np.random.default_rng(sum(shape) + sum(filt))
    x = rng.standard_normal(shape).astype(np.float32)
    w = (rng.standard_normal(filt) / np.sqrt(filt[0] * filt[1] * filt[2])).astype(np.float32)
    tx, tw = sf.constant(x), sf.constant(w)
    monkeypatch.setattr(nn, "IMPLICIT_CONV", True)
    monkeypatch.setattr(nn, "IMPLICIT_MAX_K", 1 << 30)
    launches0 = _native.launch_count(0)
    got = nn.conv2d(tx, tw, stride=s, pad=p).numpy()
    implicit_launches = _native.launch_count(0) - launches0
    monkeypatch.setattr(nn, "IMPLICIT_CONV", False)
    ref = nn.conv2d(tx, tw, stride=s, pad=p).numpy()
    np.testing.assert_array_equal(got, ref)
    assert implicit_launches <= 2  # the GEMM (+ a split-K reduce), no im2col kernel
    want = nn_np.conv2d(x.astype(np.float64), w.astype(np.float64), s, p)
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-4)
