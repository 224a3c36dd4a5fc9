"""Operator files: reference IVOP v1 interchange (CPU) and the compressed
byte-plane v2 format (GPU round trip)."""

import struct
import sys

import numpy as np
import pytest

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import cache


def test_dense_and_quantized_v1_round_trip(tmp_path):
    m = invop.DenseMatrix(n=3, entries=np.arange(9.0).reshape(3, 3) / 7.0)
    p = tmp_path / "d.ivop"
    invop.write_matrix(p, m)
    back = invop.read_matrix(p)
    assert back.entries.tobytes() == m.entries.tobytes()
    q = invop.QuantizedMatrix(n=3, scale_digits=4, mantissas=np.arange(-4, 5).reshape(3, 3))
    invop.write_matrix(tmp_path / "q.ivop", q)
    q2 = invop.read_matrix(tmp_path / "q.ivop")
    assert (q2.mantissas == q.mantissas).all() and q2.scale_digits == 4


def test_v1_files_match_the_reference_layout(tmp_path):
    q = invop.QuantizedMatrix(n=2, scale_digits=3, mantissas=np.array([[1, -2], [3, 40000]]))
    invop.write_matrix(tmp_path / "q.ivop", q)
    data = (tmp_path / "q.ivop").read_bytes()
    expect = struct.pack("<4sBBII", b"IVOP", 1, 1, 2, 2) + struct.pack("<b", 3) + \
        np.array([1, -2, 3, 40000], "<i8").tobytes()
    assert data == expect


@pytest.mark.parametrize("blob,msg", [(b"IVO", "truncated"), (b"XXXX" + bytes(10), "magic"),
                                      (struct.pack("<4sBBII", b"IVOP", 9, 0, 1, 1), "version"),
                                      (struct.pack("<4sBBII", b"IVOP", 1, 7, 1, 1) + bytes(8), "kind"),
                                      (struct.pack("<4sBBII", b"IVOP", 1, 0, 1, 2), "non-square"),
                                      (struct.pack("<4sBBII", b"IVOP", 1, 0, 2, 2) + bytes(8), "expected")])
def test_read_rejects_corrupt_files(tmp_path, blob, msg):
    p = tmp_path / "bad.ivop"
    p.write_bytes(blob)
    with pytest.raises(invop.CacheError) as exc:
        invop.read_matrix(p)
    assert msg in str(exc.value)


def test_vectors_and_entries(tmp_path):
    v = np.array([0.1, -1e-300, 3.0, np.pi])
    invop.write_vector(tmp_path / "v.txt", v)
    assert invop.read_vector(tmp_path / "v.txt").tobytes() == v.tobytes()
    e = invop.entry_for(tmp_path, 41, 41, "uniform", 3)
    assert e.key == "inv-uniform-41x41-m3" and e.kind == "quantized"


@pytest.mark.gpu
def test_v2_planes_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    for lo, hi in ((0, 200), (-30000, 30000), (0, 9_000_000)):
        mant = rng.integers(lo, hi + 1, size=(37, 37))
        q = invop.QuantizedMatrix(n=37, scale_digits=5, mantissas=mant)
        p = tmp_path / "p.ivop"
        invop.write_matrix(p, q, compressed=True)
        assert p.stat().st_size == 14 + 12 + q.device_plan().code_bytes * 37 * 37
        q2 = invop.read_matrix(p)
        assert (q2.mantissas == mant).all()
        x = rng.standard_normal(37)
        y1, c1 = invop.apply(invop.build_plan(q), x)
        y2, c2 = invop.apply(invop.build_plan(q2), x)
        assert y1.tobytes() == y2.tobytes() and c1 == c2
    # row shard of a constructed inverse
    st = invop.uniform_interior(12)
    shard = invop.DeviceOperator(st).factor().quantized_rows(4, 40, 50)
    cache.write_planes(tmp_path / "s.ivop", shard)
    back = invop.read_matrix(tmp_path / "s.ivop")
    assert back.row0 == 40 and back.rows == 50
    assert (back.decode().cpu().numpy() == shard.decode().cpu().numpy()).all()
