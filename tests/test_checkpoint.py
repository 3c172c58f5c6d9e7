"""SCK1 checkpoints (paper_1903_01855_b200/checkpoint.py) against files the
reference itself wrote (tests/golden/make_ckpt_golden.py)."""
import os

import numpy as np
import pytest

import paper_1903_01855_b200 as sf
from paper_1903_01855_b200.errors import StorageError
from ckpt_graph import build

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _ref_bytes(name):
    with open(os.path.join(GOLD, name), "rb") as f:
        return f.read()


def test_decode_reference_checkpoint():
    ck = sf.Checkpoint.from_bytes(_ref_bytes("ckpt_ref.sck1"))
    paths = [n.path for n in ck.nodes]
    assert paths[0] == "" and "dense/kernel" in paths and "data" in paths
    kernel = ck.payloads["dense/kernel"]
    assert kernel.dtype is sf.float32 and kernel.shape == (3, 4)
    np.testing.assert_array_equal(kernel.numpy(), np.arange(12, dtype=np.float32).reshape(3, 4))
    assert ck.payloads["dense/bias"].dtype is sf.float64
    assert int(ck.payloads["step"].numpy()) == 7 and bool(ck.payloads["flag"].numpy())
    assert int(np.frombuffer(ck.payloads["data"], dtype=np.int64)[0]) == 2
    # re-encoding the decoded checkpoint reproduces the reference's bytes
    assert ck.to_bytes() == _ref_bytes("ckpt_ref.sck1")


def test_encode_matches_reference_bytes_without_variables():
    assert sf.save(build(sf, with_variables=False)).to_bytes() == \
        _ref_bytes("ckpt_ref_novars.sck1")


def test_restore_blobs_and_iterator_state(tmp_path):
    path = tmp_path / "c.sck1"
    path.write_bytes(_ref_bytes("ckpt_ref_novars.sck1"))
    live = build(sf, with_variables=False, scale=3.0)
    assert live.data.position == 0
    report = sf.restore(live, str(path))
    assert live.data.position == 2 and next(live.data) == 30
    np.testing.assert_array_equal(live.table, np.arange(6, dtype=np.int64).reshape(2, 3))
    assert report.conflicts == [] and report.unmatched_in_checkpoint == []
    assert "dense" in report.matched and "data" in report.matched


def test_corrupt_and_missing_files(tmp_path):
    with pytest.raises(StorageError):
        sf.Checkpoint.from_bytes(b"XXXX")
    with pytest.raises(StorageError):
        sf.Checkpoint.from_bytes(_ref_bytes("ckpt_ref.sck1")[:40])
    with pytest.raises(StorageError):
        sf.load_checkpoint(str(tmp_path / "missing.sck1"))


@pytest.mark.gpu
def test_variables_round_trip_bitwise_with_reference_file(tmp_path):
    sf.init_runtime(sf.RuntimeOptions())
    live = build(sf)
    # device-resident variables snapshot to the reference's exact bytes
    assert sf.save(live).to_bytes() == _ref_bytes("ckpt_ref.sck1")
    other = build(sf, scale=2.0)
    assert float(other.dense.kernel.numpy()[0, 1]) == 2.0
    path = str(tmp_path / "r.sck1")
    with open(path, "wb") as f:
        f.write(_ref_bytes("ckpt_ref.sck1"))
    report = sf.restore(other, path)
    assert report.conflicts == []
    np.testing.assert_array_equal(other.dense.kernel.numpy(), live.dense.kernel.numpy())
    assert other.dense.bias.numpy().tobytes() == live.dense.bias.numpy().tobytes()
    assert int(other.step.numpy()) == 7 and bool(other.flag.numpy())
    # a dtype/shape conflict is reported, not applied
    bad = build(sf)
    bad.dense.kernel = sf.Variable(sf.constant(np.zeros((2, 2), np.float32)))
    rep = sf.restore(bad, path)
    assert any(p == "dense/kernel" for p, _ in rep.conflicts)
