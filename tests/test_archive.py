"""LKG1 archives: host header/CRC checks (CPU) and device loading (GPU)
against files written by the reference itself (tests/golden/*.lkg, made by
tests/golden/make_golden_archive.py)."""

import struct
import zlib
from pathlib import Path

import numpy as np
import pytest

from paper_2604_18913_b200 import archive as ar
from paper_2604_18913_b200.errors import (
    ArchiveError,
    BadMagicError,
    ChecksumError,
    TruncatedError,
    VersionError,
)
from oracle import khop_oracle as orc

GOLDEN = Path(__file__).resolve().parent / "golden"


def _bytes(name):
    return (GOLDEN / f"{name}.lkg").read_bytes()


def _recrc(body: bytes) -> bytes:
    body = body[:-4]
    return body + struct.pack("<I", zlib.crc32(body))


def test_header_of_reference_archives():
    assert ar.parse_header(_bytes("tiny")) == (4, 3, 3, 4)
    assert ar.parse_header(_bytes("c1")) == (4, 10_000, 16, 49_737)


def test_every_single_byte_flip_is_detected():
    data = _bytes("tiny")
    for i in range(len(data)):
        bad = bytearray(data)
        bad[i] ^= 0x5A
        with pytest.raises(ArchiveError):
            ar.parse_header(bytes(bad))


def test_header_errors():
    data = _bytes("tiny")
    with pytest.raises(TruncatedError):
        ar.parse_header(data[:20])
    with pytest.raises(TruncatedError):
        ar.parse_header(data + b"\0")
    with pytest.raises(BadMagicError):
        ar.parse_header(_recrc(b"LKG2" + data[4:]))
    with pytest.raises(VersionError):
        ar.parse_header(_recrc(data[:4] + struct.pack("<H", 2) + data[6:]))
    with pytest.raises(ChecksumError):
        ar.parse_header(data[:-1] + bytes([data[-1] ^ 1]))


def _payload_edit(data: bytes, fn) -> bytes:
    """Rewrite the payload arrays with fn(indptr, tids, obj, rel), fix the CRC."""
    width, E, R, T = ar.parse_header(data)
    dt = "<u4" if width == 4 else "<u8"
    off = 40
    ip = np.frombuffer(data, "<u8", E + 1, off).copy()
    off += (E + 1) * 8
    cols = []
    for _ in range(3):
        cols.append(np.frombuffer(data, dt, T, off).copy())
        off += T * width
    fn(ip, *cols)
    body = data[:40] + ip.tobytes() + b"".join(c.tobytes() for c in cols)
    return body + struct.pack("<I", zlib.crc32(body))


def _widen(data: bytes) -> bytes:
    """Same graph with 8-byte ids (valid for the reference loader too)."""
    width, E, R, T = ar.parse_header(data)
    off = 40 + (E + 1) * 8
    cols = [np.frombuffer(data, "<u4", T, off + i * T * 4).astype("<u8") for i in range(3)]
    payload = data[40:off] + b"".join(c.tobytes() for c in cols)
    header = struct.pack("<4sHBBQQQQ", b"LKG1", 1, 1, 8, E, R, T, len(payload))
    body = header + payload
    return body + struct.pack("<I", zlib.crc32(body))


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name,E,R", [("tiny", 3, 3), ("c1", 10_000, 16)])
@pytest.mark.parametrize("wide", [False, True])
def test_device_load_matches_reference_csr(cuda_device, name, E, R, wide):
    import paper_2604_18913_b200 as th

    data = _bytes(name)
    if wide:
        data = _widen(data)
    g = ar.graph_from_bytes(data)
    z = np.load(GOLDEN / f"{name}.npz")
    og = orc.build_csr(z["subj"], z["rel"], z["obj"], E, R)
    assert np.array_equal(g.indptr, og.indptr)
    assert np.array_equal(g.tids, og.tids)
    assert np.array_equal(g.obj, og.obj)
    assert np.array_equal(g.rel, og.rel)
    assert np.array_equal(g.subj, og.subj)
    if not wide:
        assert ar.graph_to_bytes(g) == data  # bit-identical round trip
    seeds = np.arange(min(E, 40))
    res = th.retrieve(g, seeds, 2, semantics="frontier")
    for i, s in enumerate(seeds.tolist()):
        ref = orc.retrieve_one(og, s, 2, "frontier")
        for h in range(2):
            assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h])


@pytest.mark.gpu
def test_device_validation_errors(cuda_device):
    data = _bytes("c1")

    def nonmono(ip, tids, obj, rel):
        ip[5], ip[6] = ip[6] + 1, ip[5]

    def dup(ip, tids, obj, rel):
        tids[1] = tids[0]

    def objrange(ip, tids, obj, rel):
        obj[7] = 10_000

    def unsorted(ip, tids, obj, rel):
        r = int(np.argmax(np.diff(ip) >= 2))  # a row with two slots
        a = int(ip[r])
        tids[a], tids[a + 1] = tids[a + 1], tids[a]

    cases = [(nonmono, "corrupt sub row offsets"),
             (dup, "not a permutation"),
             (objrange, "out of range"),
             (unsorted, "not strictly sorted")]
    for fn, msg in cases:
        with pytest.raises(ArchiveError, match=msg):
            ar.graph_from_bytes(_payload_edit(data, fn))
