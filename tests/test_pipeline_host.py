"""Host-side pieces of the file pipeline (no GPU): I/O chunking, H2D range
coalescing, ranged reads and the pinned-staging layout rules."""

import os

import numpy as np
import pytest

from paper_2406_18820_b200 import api, codec
from paper_2406_18820_b200.spec import DType


def test_chunks_cover_exactly():
    for nb in (0, 1, 4095, 16 << 20, (16 << 20) + 1, 100 << 20):
        ch = api._chunks(nb, 16 << 20)
        assert sum(n for _, n in ch) == nb
        assert len(ch) == 1 or all(n <= 16 << 20 for _, n in ch)
        offs = [o for o, _ in ch]
        assert offs == sorted(offs) and offs[0] == 0
        assert all(a + n == b for (a, n), (b, _) in zip(ch, ch[1:]))
    assert api._chunks(10, -1) == [(0, 10)]  # chunking off: whole ranges


def test_coalesce_merges_small_holes_only():
    assert api._coalesce([], 4096) == []
    assert api._coalesce([(256, 100), (0, 100)], 4096) == [[0, 356]]
    assert api._coalesce([(0, 100), (100 + 5000, 10)], 4096) == [[0, 100], [5100, 10]]
    # contained / overlapping ranges never shrink a run
    assert api._coalesce([(0, 1000), (10, 20)], 0) == [[0, 1000]]
    # a sent chunk (>= SEND_MIN) can never sit inside a mergeable hole
    assert api.SEND_MIN > api.ALIGN_GAP


def test_read_range_into_and_truncation(tmp_path):
    a = np.arange(1 << 16, dtype=np.float32)
    path = str(tmp_path / "t.ucpt")
    codec.write_raw(path, DType.F32, a.shape, memoryview(a).cast("B"))
    hdr = codec.read_header(path)
    out = np.zeros(a.size, dtype=np.float32)
    mv = memoryview(out.view(np.uint8))
    for c, n in api._chunks(hdr.nbytes, 10000):
        codec.read_range_into(path, hdr.offset + c, mv[c:c + n])
    assert np.array_equal(out, a)
    os.truncate(path, hdr.offset + 100)
    with pytest.raises(Exception) as ei:
        codec.read_range_into(path, hdr.offset, mv[:1000])
    assert type(ei.value).__name__ == "TruncatedPayloadError"


def test_create_raw_write_range_round_trip(tmp_path):
    a = np.arange(3000, dtype=np.float32).reshape(30, 100)
    path = str(tmp_path / "w.ucpt")
    off = codec.create_raw(path, DType.F32, a.shape, a.nbytes)
    b = memoryview(a.reshape(-1).view(np.uint8))
    for c, n in api._chunks(a.nbytes, 4096):
        codec.write_range(path, off + c, b[c:c + n])
    t = codec.read_tensor(path)
    assert t.shape == (30, 100) and np.array_equal(t.data, a)
    ref = str(tmp_path / "r.ucpt")
    codec.write_raw(ref, DType.F32, a.shape, b)
    assert open(ref, "rb").read() == open(path, "rb").read()
