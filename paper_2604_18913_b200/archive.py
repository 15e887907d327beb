"""LKG1 graph archives straight onto the device.

Same file format as the reference (archive.py:1-24): header
``<4sHBBQQQQ`` (magic "LKG1", version 1, endianness 1, id width 4|8,
entity/relation/triple counts, payload length), payload = indptr u64[E+1],
row-ordered triple ids, obj and rel in triple-id order (u32 or u64), then a
CRC32 over header + payload.  Archives written by the reference load here
and vice versa (tests/test_archive.py pins a reference-written file).

Loading checks the header and CRC32 on the host (archive.py:84-105; a
single corrupted byte is always detected), copies the raw payload to the
device once, and lets ``th_graph_create_lkg`` narrow, validate
(archive.py:121-133) and build the device graph -- no numpy rebuild of the
incidence structure.
"""

from __future__ import annotations

import ctypes
import struct
import zlib
from pathlib import Path

import numpy as np

from . import _lib
from .errors import ArchiveError, BadMagicError, ChecksumError, TruncatedError, VersionError

MAGIC = b"LKG1"
VERSION = 1
_HEADER = struct.Struct("<4sHBBQQQQ")
_CRC = struct.Struct("<I")


def _id_width(*counts: int) -> int:
    return 4 if max(counts) <= 0xFFFFFFFF else 8


def graph_to_bytes(g) -> bytes:
    """Serialise a device ``IncidenceGraph`` (archive.py:66-81 layout)."""
    width = _id_width(g.n_entities, g.n_relations, g.n_triples)
    dtype = "<u4" if width == 4 else "<u8"
    payload = b"".join([
        np.asarray(g.indptr).astype("<u8").tobytes(),
        np.asarray(g.tids).astype(dtype).tobytes(),
        np.asarray(g.obj).astype(dtype).tobytes(),
        np.asarray(g.rel).astype(dtype).tobytes(),
    ])
    header = _HEADER.pack(MAGIC, VERSION, 1, width, g.n_entities, g.n_relations, g.n_triples,
                          len(payload))
    body = header + payload
    return body + _CRC.pack(zlib.crc32(body))


def parse_header(data) -> tuple:
    """Host checks of archive.py:84-102; returns (width, E, R, T)."""
    if len(data) < _HEADER.size + _CRC.size:
        raise TruncatedError(f"archive too short ({len(data)} bytes)")
    magic, version, endian, width, n_e, n_r, n_t, payload_len = _HEADER.unpack_from(data)
    if magic != MAGIC:
        raise BadMagicError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if version != VERSION:
        raise VersionError(f"unsupported archive version {version}")
    total = _HEADER.size + payload_len + _CRC.size
    if len(data) != total:
        raise TruncatedError(f"expected {total} bytes, file has {len(data)}")
    (stored,) = _CRC.unpack_from(data, total - _CRC.size)
    if zlib.crc32(memoryview(data)[: total - _CRC.size]) != stored:
        raise ChecksumError("archive checksum mismatch")
    if endian != 1:
        raise ArchiveError(f"unsupported endianness flag {endian}")
    if width not in (4, 8):
        raise ArchiveError(f"unsupported id width {width}")
    if payload_len != (n_e + 1) * 8 + 3 * n_t * width:
        raise ArchiveError("payload length inconsistent with counts")
    return width, n_e, n_r, n_t


def graph_from_bytes(data, *, reverse: bool = True, stream=None):
    """Device ``IncidenceGraph`` from LKG1 bytes."""
    import torch

    from .device_graph import IncidenceGraph, _require_cuda

    _require_cuda()
    width, E, R, T = parse_header(data)
    dev = torch.device("cuda", torch.cuda.current_device())
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    payload = np.frombuffer(data, dtype=np.uint8, count=len(data) - _HEADER.size - _CRC.size,
                            offset=_HEADER.size)
    d = torch.from_numpy(payload.copy()).to(dev, non_blocking=False)  # one H2D of the payload
    base = d.data_ptr()
    o_ip = 0
    o_tid = o_ip + (E + 1) * 8
    o_obj = o_tid + T * width
    o_rel = o_obj + T * width
    lib = _lib.load()
    h = ctypes.c_void_p()
    flags = 0 if reverse else _lib.TH_GRAPH_NO_REVERSE
    _lib.check(lib.th_graph_create_lkg(base + o_ip, base + o_tid, base + o_obj, base + o_rel, width, T, E,
                                       R, flags, ctypes.c_void_p(st.cuda_stream), ctypes.byref(h)))
    del d
    return IncidenceGraph(h.value, E, R, T, dev, st)


def save_graph(g, path) -> None:
    Path(path).write_bytes(graph_to_bytes(g))


def load_graph(path, **kw):
    """archive.py:140-144: a missing file is an IntegrityError."""
    from .errors import IntegrityError

    p = Path(path)
    if not p.exists():
        raise IntegrityError(f"no such archive: {p}")
    return graph_from_bytes(p.read_bytes(), **kw)
