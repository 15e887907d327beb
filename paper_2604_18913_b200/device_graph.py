"""Device-resident incidence graph: ``build_incidence`` / ``IncidenceGraph``.

Mirrors incidence.py:121-196 of the reference: same constructor arguments
(a ``Sequence[Triple]`` or a ``(subject, relation, object)`` column tuple,
``n_entities``, ``n_relations``), same ``ValueError`` on out-of-range ids,
same read-only int64 host views (``indptr``, ``tids``, ``obj``, ``rel``,
``subj``) -- but the structure itself is built and kept on the B200 by the
K1 kernels of ``csrc/graph.cu`` (int32 CSR offsets and ids, uint16
relations, plus the reverse CSR used by pull hops).
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib
from .core_types import Triple


def _require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2604_18913_b200 needs a CUDA device (B200); no CPU fallback exists")
    return torch


def _column_to_device(col, name: str, bound: int, torch, device):
    """Validate one id column on its own side (host or device) and narrow to int32."""
    if isinstance(col, torch.Tensor):
        t = col.to(device=device)
        if t.numel():
            lo, hi = int(t.min().item()), int(t.max().item())
            if lo < 0 or hi >= bound:
                raise ValueError(f"{name} id out of range (bound {bound})")
        return t.to(torch.int32).contiguous()
    arr = np.asarray(col).reshape(-1)
    if arr.size:
        if not np.issubdtype(arr.dtype, np.integer):
            arr = arr.astype(np.int64)
        if int(arr.min()) < 0 or int(arr.max()) >= bound:
            raise ValueError(f"{name} id out of range (bound {bound})")
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32)).to(device)


class IncidenceGraph:
    """Immutable device incidence structures for one graph."""

    def __init__(self, handle, n_entities: int, n_relations: int, n_triples: int, device, stream):
        self._handle = handle
        self.n_entities = int(n_entities)
        self.n_relations = int(n_relations)
        self.n_triples = int(n_triples)
        self.device = device
        self._stream = stream
        self._host = {}
        self._default_retriever = None
        lib = _lib.load()
        self._finalizer = weakref.finalize(self, lib.th_graph_destroy, handle)

    # -- device views -------------------------------------------------------
    def info(self) -> _lib.GraphInfo:
        info = _lib.GraphInfo()
        _lib.check(_lib.load().th_graph_info_get(self._handle, ctypes.byref(info)))
        return info

    def device_column(self, name: str):
        """Zero-copy torch view of a device array (indptr, csr_tid, csr_obj,
        csr_rel, subj, obj, rel, rindptr, rsrc, rrel)."""
        info = self.info()
        E, T = self.n_entities, self.n_triples
        shapes = {"indptr": (E + 1, "<i4"), "rindptr": (E + 1, "<i4"), "csr_tid": (T, "<i4"),
                  "csr_obj": (T, "<i4"), "subj": (T, "<i4"), "obj": (T, "<i4"), "rsrc": (T, "<i4"),
                  "csr_rel": (T, "<i2"), "rel": (T, "<i2"), "rrel": (T, "<i2")}
        n, ts = shapes[name]
        return _lib.as_tensor(getattr(info, name), (n,), ts, owner=self)

    def _host_col(self, name: str) -> np.ndarray:
        if name not in self._host:
            t = self.device_column(name)
            arr = t.cpu().numpy()
            if arr.dtype == np.int16:  # uint16 relation ids are exported as int16 views
                arr = arr.view(np.uint16)
            arr = arr.astype(np.int64)
            arr.setflags(write=False)
            self._host[name] = arr
        return self._host[name]

    # -- reference field names (incidence.py:125-151) ------------------------
    @property
    def indptr(self) -> np.ndarray:
        return self._host_col("indptr")

    @property
    def tids(self) -> np.ndarray:
        return self._host_col("csr_tid")

    @property
    def obj(self) -> np.ndarray:
        return self._host_col("obj")

    @property
    def rel(self) -> np.ndarray:
        return self._host_col("rel")

    @property
    def subj(self) -> np.ndarray:
        return self._host_col("subj")

    def sub_row(self, entity: int) -> np.ndarray:
        ip = self.indptr
        return self.tids[ip[entity] : ip[entity + 1]]

    def out_degrees(self) -> np.ndarray:
        return np.diff(self.indptr)

    def triple(self, tid: int) -> Triple:
        return Triple(int(self.subj[tid]), int(self.rel[tid]), int(self.obj[tid]))

    def stats(self) -> dict:
        i = self.info()
        return {"n_entities": i.n_entities, "n_triples": i.n_triples, "n_relations": i.n_relations,
                "max_out_degree": i.max_out_degree, "max_in_degree": i.max_in_degree,
                "n_heavy_in": i.n_heavy_in, "device_bytes": int(i.device_bytes)}

    def retriever(self):
        from .retriever import Retriever

        if self._default_retriever is None:
            self._default_retriever = Retriever(self)
        return self._default_retriever


def build_incidence(triples, n_entities: int, n_relations: int, *, reverse: bool = True,
                    stream=None) -> IncidenceGraph:
    """Build the device incidence graph (incidence.py:154-196).

    ``triples`` is a sequence of ``Triple``/3-tuples or a (subject, relation,
    object) tuple of numpy arrays / torch tensors, in triple-id order.
    """
    torch = _require_cuda()
    device = torch.device("cuda", torch.cuda.current_device())
    if isinstance(triples, tuple) and len(triples) == 3 and not isinstance(triples[0], (int, np.integer)):
        cols = triples
    else:
        rows = list(triples)
        a = np.asarray(rows, dtype=np.int64).reshape(-1, 3) if rows else np.empty((0, 3), np.int64)
        cols = (a[:, 0], a[:, 1], a[:, 2])
    s = _column_to_device(cols[0], "subject", n_entities, torch, device)
    r = _column_to_device(cols[1], "relation", n_relations, torch, device)
    o = _column_to_device(cols[2], "object", n_entities, torch, device)
    if not (s.numel() == r.numel() == o.numel()):
        raise ValueError("subject/relation/object columns differ in length")
    st = stream if stream is not None else torch.cuda.current_stream(device)
    lib = _lib.load()
    handle = ctypes.c_void_p()
    flags = 0 if reverse else _lib.TH_GRAPH_NO_REVERSE
    _lib.check(lib.th_graph_create(s.data_ptr(), r.data_ptr(), o.data_ptr(), s.numel(), int(n_entities),
                                   int(n_relations), flags, ctypes.c_void_p(st.cuda_stream),
                                   ctypes.byref(handle)))
    return IncidenceGraph(handle.value, n_entities, n_relations, s.numel(), device, st)
