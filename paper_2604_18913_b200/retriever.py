"""Batched k-hop retrieval on the device, behind the reference's retriever API.

Public entry points (reference citations are /root/reference/pkg/src/triplehop):

* :func:`k_hop`             incidence.py:319-330 (seed-set query, HopTrace)
* :func:`one_hop`           incidence.py:224-232
* :func:`reconstruct_paths` incidence.py:391-408
* :meth:`Retriever.retrieve` / :func:`retrieve` -- the north-star batch call
  ``retrieve(seeds, k, relation_filter)``: one independent query per seed,
  defined as ``[(k_hop([s], k, g_f, sem), reconstruct_paths([s], k, g_f))
  for s in seeds]`` on the relation-filtered graph g_f.

All hops of all seeds run on the B200 in one ``th_run`` call (csrc/engine.cu);
results come back as device tensors (per-query CSR offsets + ids), with
host conversions for the reference container types.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core_types import (
    DEFAULT_MAX_PATHS,
    EntityVector,
    HopSemantics,
    HopStep,
    HopTrace,
    PathResult,
    Triple,
    TripleVector,
)


def _torch():
    import torch

    return torch


@dataclass
class RetrievalResult:
    """Device-resident results of one batch (``k`` hops x ``n_queries``).

    frontier ids of query q at hop h (1-based):
        frontier_ids[frontier_off[h-1, q] : frontier_off[h-1, q] + frontier_len[h-1, q]]
    ``edges[h-1, q]`` = |activated triples| = the reference's per-hop
    ``triple_count`` (service/app.py:97).  Paths of query q:
        path_tids[path_off[q] : path_off[q] + path_count[q]]   (shape [n, k])
    """

    n_queries: int
    k: int
    semantics: HopSemantics
    frontier_off: object = None
    frontier_len: object = None
    frontier_ids: object = None
    edges: object = None
    act_off: object = None
    act_len: object = None
    act_ids: object = None
    path_off: object = None
    path_count: object = None
    path_truncated: object = None
    path_tids: object = None
    push_hops: int = 0
    pull_hops: int = 0
    _graph: object = None
    _host: dict = None

    # -- host accessors ------------------------------------------------------
    def _h(self, name):
        if self._host is None:
            self._host = {}
        if name not in self._host:
            t = getattr(self, name)
            self._host[name] = None if t is None else t.cpu().numpy()
        return self._host[name]

    def frontier(self, q: int, hop: int) -> np.ndarray:
        off, ln, ids = self._h("frontier_off"), self._h("frontier_len"), self._h("frontier_ids")
        o, n = int(off[hop - 1, q]), int(ln[hop - 1, q])
        return ids[o : o + n].astype(np.int64)

    def activated(self, q: int, hop: int) -> np.ndarray:
        off, ln, ids = self._h("act_off"), self._h("act_len"), self._h("act_ids")
        o, n = int(off[hop - 1, q]), int(ln[hop - 1, q])
        return ids[o : o + n].astype(np.int64)

    def edges_traversed(self, q: int | None = None) -> int:
        e = self._h("edges")
        return int(e.sum()) if q is None else int(e[:, q].sum())

    def path_tid_tuples(self, q: int) -> list[tuple[int, ...]]:
        off, cnt, tids = self._h("path_off"), self._h("path_count"), self._h("path_tids")
        o, n = int(off[q]), int(cnt[q])
        return [tuple(int(t) for t in row) for row in tids[o : o + n]]

    def paths(self, q: int) -> list[tuple[Triple, ...]]:
        g = self._graph
        return [tuple(g.triple(t) for t in p) for p in self.path_tid_tuples(q)]

    def truncated(self, q: int) -> bool:
        return bool(self._h("path_truncated")[q])

    def trace(self, q: int, seeds) -> HopTrace:
        g = self._graph
        steps = []
        for h in range(1, self.k + 1):
            act = self.activated(q, h) if self.act_ids is not None else np.empty(0, np.int64)
            steps.append(HopStep(EntityVector(self.frontier(q, h), g.n_entities, _canonical=True),
                                 TripleVector(act, g.n_triples, _canonical=True)))
        return HopTrace(self.semantics, EntityVector(seeds, g.n_entities), steps)


def _relation_masks(relation_filter, n_queries: int, n_relations: int):
    """Normalise a relation filter to uint32 words [B, ceil(R/32)] (bit r = allowed)."""
    if relation_filter is None:
        return None
    torch = _torch()
    mw = max(1, (n_relations + 31) // 32)

    def words_from_ids(ids) -> np.ndarray:
        ids = np.asarray(list(ids), dtype=np.int64).reshape(-1)
        if ids.size and (ids.min() < 0 or ids.max() >= n_relations):
            raise ValueError(f"relation id out of range (bound {n_relations})")
        bits = np.zeros(mw * 32, dtype=bool)
        bits[ids] = True
        return np.packbits(bits, bitorder="little").view(np.uint32)

    if isinstance(relation_filter, torch.Tensor):
        relation_filter = relation_filter.detach().cpu().numpy()
    if isinstance(relation_filter, np.ndarray) and relation_filter.ndim == 2:
        if relation_filter.shape[0] != n_queries:
            raise ValueError("per-seed relation filter needs one row per seed")
        if relation_filter.dtype == np.bool_:
            if relation_filter.shape[1] != n_relations:
                raise ValueError("boolean relation filter needs n_relations columns")
            bits = np.zeros((n_queries, mw * 32), dtype=bool)
            bits[:, :n_relations] = relation_filter
            words = np.packbits(bits, axis=1, bitorder="little").view(np.uint32)
        else:
            if relation_filter.shape[1] != mw:
                raise ValueError(f"relation mask words must have {mw} columns")
            words = relation_filter.astype(np.uint32)
            tail = mw * 32 - n_relations
            if tail and np.any(words[:, -1] >> np.uint32(32 - tail)):
                raise ValueError(f"relation id out of range (bound {n_relations})")
    elif isinstance(relation_filter, np.ndarray) or (
        len(relation_filter) == 0 or np.isscalar(next(iter(relation_filter)))
    ):
        words = np.tile(words_from_ids(relation_filter), (n_queries, 1))
    else:
        rows = list(relation_filter)
        if len(rows) != n_queries:
            raise ValueError("per-seed relation filter needs one entry per seed")
        lens = {np.size(r) for r in rows}
        if len(lens) == 1 and rows and next(iter(lens)) > 0:
            # equal-length id rows: one vectorised scatter + pack for the batch
            ids = np.asarray(rows, dtype=np.int64).reshape(n_queries, -1)
            if ids.min() < 0 or ids.max() >= n_relations:
                raise ValueError(f"relation id out of range (bound {n_relations})")
            bits = np.zeros((n_queries, mw * 32), dtype=bool)
            bits[np.arange(n_queries)[:, None], ids] = True
            words = np.packbits(bits, axis=1, bitorder="little").view(np.uint32)
        else:
            words = np.stack([words_from_ids(r) for r in rows]) if rows else np.zeros((0, mw), np.uint32)
    return np.ascontiguousarray(words, dtype=np.uint32).reshape(n_queries, mw)


class Retriever:
    """An engine session: device workspace + results on one CUDA stream."""

    def __init__(self, graph, stream=None):
        torch = _torch()
        self.graph = graph
        self.stream = stream if stream is not None else torch.cuda.current_stream(graph.device)
        lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(lib.th_session_create(ctypes.c_void_p(graph._handle),
                                         ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)))
        self._handle = h.value
        self._finalizer = weakref.finalize(self, lib.th_session_destroy, self._handle)
        self._keep = None

    # -- knobs / diagnostics -------------------------------------------------
    def set_pull_divisor(self, divisor: float) -> None:
        _lib.check(_lib.load().th_session_set_pull_divisor(self._handle, float(divisor)))

    def set_list_min_entities(self, n: int) -> None:
        """K4 strategy knob: list-driven materialisation for graphs with >= n entities."""
        _lib.check(_lib.load().th_session_set_list_min_entities(self._handle, int(n)))

    def set_k4_mode(self, mode: int) -> None:
        """K4 form for list-driven layers: 1 row-major (default), 0 transposes."""
        _lib.check(_lib.load().th_session_set_k4_mode(self._handle, int(mode)))

    def set_pull_screen(self, mode: int) -> None:
        """Pull item screening: -1 by graph shape (default), 0 off, 1 per lane in the pull kernel, 2 screen kernel + compacted pull."""
        _lib.check(_lib.load().th_session_set_pull_screen(self._handle, int(mode)))

    def set_knob(self, name: str, value: int) -> None:
        """Boolean strategy knobs: "paths_k2", "k4_cache", "list_first_hop", "priority",
        "k4_bucket", "pull_pair", "k4_cache_filtered" (th_b200.h)."""
        _lib.check(_lib.load().th_session_set_knob(self._handle, name.encode(), int(value)))

    def set_paths_k2(self, on: bool) -> None:
        self.set_knob("paths_k2", int(bool(on)))

    def set_overlap(self, on: bool) -> None:
        """Overlap hop h's K4 with hop h+1's expansion (frontier-only runs)."""
        _lib.check(_lib.load().th_session_set_overlap(self._handle, int(bool(on))))

    def set_dense_pull(self, divisor: float) -> None:
        """Pull hops gather unconditionally above 1/divisor active in-edges (<= 0: never)."""
        _lib.check(_lib.load().th_session_set_dense_pull(self._handle, float(divisor)))

    def set_graphs(self, on: bool) -> None:
        """Replay repeated batch shapes as one captured CUDA graph."""
        _lib.check(_lib.load().th_session_set_graphs(self._handle, int(bool(on))))

    def launch_count(self) -> int:
        return int(_lib.load().th_session_launch_count(self._handle))

    def set_profiling(self, on: bool) -> None:
        _lib.check(_lib.load().th_session_set_profiling(self._handle, int(bool(on))))

    def profile(self) -> dict:
        """{category: (ms, launches)} accumulated since the last call (syncs)."""
        n = len(_lib.PROF_CATEGORIES)
        ms = (ctypes.c_double * n)()
        ln = (ctypes.c_int64 * n)()
        _lib.check(_lib.load().th_session_profile(self._handle, ms, ln, n))
        return {c: (ms[i], int(ln[i])) for i, c in enumerate(_lib.PROF_CATEGORIES)}

    def profile_trace(self) -> list:
        """Timeline of the last profiled run: (category, stream, start ms,
        end ms) per kernel group; stream 0 = main, 1 / 2 = K4 side streams."""
        lib = _lib.load()
        n = int(lib.th_session_profile_trace(self._handle, None, 0))
        if n < 0:
            raise RuntimeError(lib.th_last_error().decode(errors="replace"))
        buf = (ctypes.c_double * max(4 * n, 1))()
        lib.th_session_profile_trace(self._handle, buf, n)
        return [(_lib.PROF_CATEGORIES[int(buf[4 * i])], int(buf[4 * i + 1]), buf[4 * i + 2], buf[4 * i + 3])
                for i in range(n)]

    def wave_lists(self, k: int) -> list[int]:
        """Entity-list lengths of the last wave: seeds, then rows set at each hop."""
        buf = (ctypes.c_int64 * (k + 1))()
        _lib.check(_lib.load().th_session_wave_lists(self._handle, buf, k + 1))
        return [int(x) for x in buf]

    def wave_modes(self, k: int) -> list[int]:
        """Direction of each hop of the last wave (index h = 1..k): 1 pull, 0 push."""
        buf = (ctypes.c_int32 * (k + 1))()
        _lib.check(_lib.load().th_session_wave_modes(self._handle, buf, k + 1))
        return [int(x) for x in buf]

    # -- raw device call ---------------------------------------------------
    def run(self, seed_offsets, seeds, k: int, semantics=HopSemantics.FRONTIER, masks=None,
            frontiers: bool = True, activated: bool = False, paths: bool = False,
            max_paths: int | None = DEFAULT_MAX_PATHS, singleton: bool = False,
            copy: bool = True, collect: bool = True) -> RetrievalResult:
        """One batched th_run over device tensors.

        seed_offsets: int32 [B+1], seeds: int32 (device); masks: uint32
        words [B, ceil(R/32)] (device) or None.  With copy=False the returned
        tensors alias session buffers, valid until the next run.
        """
        torch = _torch()
        sem = HopSemantics.parse(semantics)
        if k < 1:
            raise ValueError("hop count must be >= 1")
        if paths and max_paths is not None and max_paths < 0:
            raise ValueError("max_paths must be >= 0")
        B = int(seed_offsets.numel()) - 1
        q = _lib.Query()
        q.n_queries = B
        q.d_seed_offsets = seed_offsets.data_ptr()
        q.d_seeds = seeds.data_ptr() if seeds.numel() else seed_offsets.data_ptr()
        q.k = int(k)
        q.semantics = sem.code
        q.d_rel_masks = masks.data_ptr() if masks is not None else None
        q.mask_words = int(masks.shape[1]) if masks is not None else 0
        q.flags = ((_lib.TH_WANT_FRONTIERS if frontiers else 0)
                   | (_lib.TH_WANT_ACTIVATED if activated else 0)
                   | (_lib.TH_WANT_PATHS if paths else 0)
                   | (_lib.TH_SINGLETON_SEEDS if singleton else 0))
        q.max_paths = -1 if max_paths is None else int(max_paths)
        lib = _lib.load()
        res = _lib.Result()
        self._keep = (seed_offsets, seeds, masks)  # inputs must outlive the async run
        self._pending = (q, sem, frontiers, activated, paths)
        for _attempt in range(4):
            _lib.check(lib.th_run(self._handle, ctypes.byref(q)))
            if not collect:
                return None
            rc = lib.th_finish(self._handle, ctypes.byref(res))
            if rc != _lib.TH_ERR_OVERFLOW:
                _lib.check(rc)
                break
        else:
            _lib.check(rc)
        return self._wrap(res, sem, copy, frontiers, activated, paths)

    def collect(self, copy: bool = False) -> RetrievalResult:
        """Finish a run launched with ``collect=False`` (re-runs on overflow)."""
        lib = _lib.load()
        q, sem, frontiers, activated, paths = self._pending
        res = _lib.Result()
        rc = lib.th_finish(self._handle, ctypes.byref(res))
        for _attempt in range(3):
            if rc != _lib.TH_ERR_OVERFLOW:
                break
            _lib.check(lib.th_run(self._handle, ctypes.byref(q)))
            rc = lib.th_finish(self._handle, ctypes.byref(res))
        _lib.check(rc)
        return self._wrap(res, sem, copy, frontiers, activated, paths)

    def _wrap(self, res, sem, copy, frontiers, activated, paths) -> RetrievalResult:
        B, k = res.n_queries, res.k
        t = _lib.as_tensor
        out = RetrievalResult(B, k, sem, push_hops=res.push_hops, pull_hops=res.pull_hops,
                              _graph=self.graph)
        out.edges = t(res.edges, (k, B), "<i8", self)
        if frontiers:
            out.frontier_off = t(res.frontier_off, (k, B), "<i8", self)
            out.frontier_len = t(res.frontier_len, (k, B), "<i8", self)
            out.frontier_ids = t(res.frontier_ids, (res.frontier_total,), "<i4", self)
        if activated:
            out.act_off = t(res.act_off, (k, B), "<i8", self)
            out.act_len = t(res.act_len, (k, B), "<i8", self)
            out.act_ids = t(res.act_ids, (res.act_total,), "<i4", self)
        if paths:
            out.path_off = t(res.path_off, (B + 1,), "<i8", self)
            out.path_count = t(res.path_count, (B,), "<i8", self)
            out.path_truncated = t(res.path_truncated, (B,), "|u1", self).bool()
            out.path_tids = t(res.path_tids, (res.path_total, k), "<i4", self)
        if copy:
            for name in ("edges", "frontier_off", "frontier_len", "frontier_ids", "act_off", "act_len",
                         "act_ids", "path_off", "path_count", "path_tids"):
                v = getattr(out, name)
                if v is not None:
                    setattr(out, name, v.clone())
        return out

    # -- public API ---------------------------------------------------------
    def retrieve(self, seeds, k: int, relation_filter=None, semantics="frontier", paths: bool = False,
                 max_paths: int | None = DEFAULT_MAX_PATHS, activated: bool = False,
                 copy: bool = True) -> RetrievalResult:
        """Per-seed k-hop retrieval for a batch of seeds (one query per seed).

        relation_filter: None; an iterable of allowed relation ids shared by
        all seeds; per-seed iterables; a bool [B, R] matrix; or uint32 mask
        words [B, ceil(R/32)].
        """
        torch = _torch()
        g = self.graph
        dev = g.device
        if isinstance(seeds, torch.Tensor):
            if seeds.dtype != torch.int32 and seeds.numel():
                # a wider id would wrap in the int32 cast (possibly onto a
                # valid id): range-check before narrowing
                lo, hi = (int(x) for x in torch.aminmax(seeds.reshape(-1)))
                if lo < 0 or hi >= g.n_entities:
                    raise ValueError(f"id out of range for width {g.n_entities}")
            s = seeds.to(device=dev, dtype=torch.int32).reshape(-1)
        else:
            arr = np.asarray(seeds, dtype=np.int64).reshape(-1)
            if arr.size and (arr.min() < 0 or arr.max() >= g.n_entities):
                raise ValueError(f"id out of range for width {g.n_entities}")
            s = torch.from_numpy(arr.astype(np.int32)).to(dev)
        B = s.numel()
        offs = torch.arange(B + 1, dtype=torch.int32, device=dev)
        words = _relation_masks(relation_filter, B, g.n_relations)
        masks = None if words is None else torch.from_numpy(words.view(np.int32)).to(dev)
        return self.run(offs, s, k, semantics, masks, frontiers=True, activated=activated, paths=paths,
                        max_paths=max_paths, singleton=True, copy=copy)

    def k_hop(self, q0: EntityVector, k: int, semantics=HopSemantics.FRONTIER) -> HopTrace:
        g = self.graph
        if q0.width != g.n_entities:
            raise ValueError(f"query width {q0.width} != graph entity count {g.n_entities}")
        if k < 1:
            raise ValueError("hop count must be >= 1")
        torch = _torch()
        ids = torch.from_numpy(q0.ids.astype(np.int32)).to(g.device)
        offs = torch.tensor([0, ids.numel()], dtype=torch.int32, device=g.device)
        r = self.run(offs, ids, k, semantics, None, frontiers=True, activated=True, copy=False)
        return r.trace(0, q0.ids)

    def reconstruct_paths(self, q0: EntityVector, k: int,
                          max_paths: int | None = DEFAULT_MAX_PATHS) -> PathResult:
        g = self.graph
        if q0.width != g.n_entities:
            raise ValueError(f"query width {q0.width} != graph entity count {g.n_entities}")
        if k < 1:
            raise ValueError("hop count must be >= 1")
        if max_paths is not None and max_paths < 0:
            raise ValueError("max_paths must be >= 0")
        torch = _torch()
        ids = torch.from_numpy(q0.ids.astype(np.int32)).to(g.device)
        offs = torch.tensor([0, ids.numel()], dtype=torch.int32, device=g.device)
        r = self.run(offs, ids, k, HopSemantics.EXACT_WALK, None, frontiers=False, paths=True,
                     max_paths=max_paths, singleton=ids.numel() == 1, copy=False)
        return PathResult(r.paths(0), r.truncated(0))


# ---- module-level drop-ins (default retriever per graph) -------------------


def k_hop(q0: EntityVector, k: int, graph, semantics: HopSemantics = HopSemantics.FRONTIER) -> HopTrace:
    """k-hop retrieval on a single graph (incidence.py:319-330)."""
    return graph.retriever().k_hop(q0, k, semantics)


def one_hop(q: EntityVector, graph) -> tuple[TripleVector, EntityVector]:
    """Activate the triples whose subject is in q, then gather their objects."""
    if q.width != graph.n_entities:
        raise ValueError(f"query width {q.width} != graph entity count {graph.n_entities}")
    tr = graph.retriever().k_hop(q, 1, HopSemantics.EXACT_WALK)
    return tr.activated(1), tr.frontier(1)


def reconstruct_paths(q0: EntityVector, k: int, graph,
                      max_paths: int | None = DEFAULT_MAX_PATHS) -> PathResult:
    """All length-k walks from q0, lexicographic by triple ids, capped."""
    return graph.retriever().reconstruct_paths(q0, k, max_paths)


def retrieve(graph, seeds, k: int, relation_filter=None, semantics="frontier", paths: bool = False,
             max_paths: int | None = DEFAULT_MAX_PATHS, **kw) -> RetrievalResult:
    """North-star batch call: per-seed reachable sets (+ paths) on the device."""
    return graph.retriever().retrieve(seeds, k, relation_filter, semantics, paths, max_paths, **kw)
