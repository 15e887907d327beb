"""Store-backed partitioned retrieval: the reference's out-of-core mode
(SURVEY 8a rows a13-a16, 8f rows 2 and 4).

Reference (citations relative to /root/reference/pkg/src/triplehop):

* ``Subgraph`` / ``materialize_subgraphs`` ...... partition.py:100-154
* ``InMemoryStore`` / ``PartitionedGraph`` ....... engine.py:34-86
* ``_partitioned_expand`` / ``cross_graph_k_hop`` / ``cross_graph_paths``
  (Algorithm 1) ............................... engine.py:94-182
* ``save_partition_dir`` / ``load_partition_plan`` / ``DirectoryStore`` /
  ``open_partitioned`` ......................... archive.py:188-315
* label files ................................ archive.py:150-160

A ``PartitionedGraph(plan, store, cache)`` keeps the reference's contract:
partitions are loaded on demand through the LRU ``SubgraphCache`` (a miss
loads an LKG1 shard archive straight onto the device), a hop fetches only
the partitions its frontier routes to, in ascending order, so the cache
counters match the reference call for call.  The hop itself is B200-native:
each touched partition expands its local frontier with the engine's one-hop
kernels (one multi-seed query, activated triples on), and the routing,
global->local and local->global maps, the union of the partitions' results
and the FRONTIER/CUMULATIVE bookkeeping of ``run_hops``
(incidence.py:268-316) are device bitmaps over the entity and triple id
spaces (``csrc/idset.cu``).  Results are bit-identical to single-graph
retrieval (tests/test_gpu_store.py, against traces the reference wrote).
"""

from __future__ import annotations

import ctypes
import json
from pathlib import Path

import numpy as np

from . import _lib
from .cache import SubgraphCache
from .core_types import DEFAULT_MAX_PATHS, EntityVector, HopSemantics, HopStep, HopTrace, TripleVector
from .errors import IntegrityError
from .partition import PartitionedGraph, PartitionPlan

GRAPH_FILE = "graph.lkg"
ENTITIES_FILE = "entities.txt"
RELATIONS_FILE = "relations.txt"
MANIFEST_FILE = "manifest.json"
ASSIGNMENT_FILE = "assignment.u32"
ARCHIVE_VERSION = 1


# ------------------------------------------------------------ device helpers


def _torch():
    import torch

    return torch


def _stream_ptr(dev):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _bits(nbits: int, dev):
    """A zeroed device bitmap of nbits bits (int32 storage, uint32 words)."""
    torch = _torch()
    return torch.zeros(max((nbits + 31) // 32, 1), dtype=torch.int32, device=dev)


def _compact(bits, nbits: int, dev):
    """Ascending int32 ids of the set bits (device tensor): a counting call
    (capacity 0) sizes the output, the second call writes it."""
    torch = _torch()
    lib = _lib.load()
    n = ctypes.c_int64()
    rc = lib.th_bits_compact(bits.data_ptr(), nbits, None, 0, ctypes.byref(n), _stream_ptr(dev))
    if rc not in (0, _lib.TH_ERR_OVERFLOW):
        _lib.check(rc)
    out = torch.empty(max(n.value, 1), dtype=torch.int32, device=dev)
    if n.value:
        _lib.check(lib.th_bits_compact(bits.data_ptr(), nbits, out.data_ptr(), n.value, ctypes.byref(n),
                                       _stream_ptr(dev)))
    return out[: n.value]


def _scatter(bits, nbits: int, ids, dev, mapping=None) -> None:
    """bits[mapping[ids]] = 1 (or bits[ids] = 1)."""
    if ids.numel() == 0:
        return
    lib = _lib.load()
    _lib.check(lib.th_ids_map_scatter(None if mapping is None else mapping.data_ptr(),
                                      0 if mapping is None else mapping.numel(), ids.data_ptr(),
                                      ids.numel(), bits.data_ptr(), nbits, _stream_ptr(dev)))


def _host_ids(t) -> np.ndarray:
    return t.cpu().numpy().astype(np.int64)


# ------------------------------------------------------------ subgraphs


class Subgraph:
    """One partition's device incidence graph plus its global id maps
    (partition.py:100-122).  ``ent_to_global`` / ``tid_to_global`` are the
    reference's read-only ascending int64 arrays; device int32 copies back
    the hop kernels."""

    def __init__(self, index: int, graph, ent_to_global, tid_to_global):
        torch = _torch()
        self.index = int(index)
        self.graph = graph
        ents = np.asarray(ent_to_global, dtype=np.int64)
        tids = np.asarray(tid_to_global, dtype=np.int64)
        ents.setflags(write=False)
        tids.setflags(write=False)
        self.ent_to_global = ents
        self.tid_to_global = tids
        dev = graph.device
        self._d_ent = torch.from_numpy(ents.astype(np.int32)).to(dev)
        self._d_tid = torch.from_numpy(tids.astype(np.int32)).to(dev)
        self._retriever = None

    @property
    def retriever(self):
        if self._retriever is None:
            from .retriever import Retriever

            self._retriever = Retriever(self.graph)
        return self._retriever

    def _to_local_dev(self, global_ids):
        """Device: ascending local ids of the global ids present here."""
        dev = self.graph.device
        m = int(self._d_ent.numel())
        if global_ids.numel() == 0 or m == 0:
            return global_ids[:0]
        bits = _bits(m, dev)
        _lib.check(_lib.load().th_ids_to_local_bits(self._d_ent.data_ptr(), m, global_ids.data_ptr(),
                                                    global_ids.numel(), bits.data_ptr(),
                                                    _stream_ptr(dev)))
        return _compact(bits, m, dev)

    def entities_to_local(self, global_ids) -> np.ndarray:
        """Local ids of the (sorted) global ids present; absent ids dropped."""
        torch = _torch()
        g = np.asarray(global_ids, dtype=np.int64)
        if g.size == 0 or self.ent_to_global.size == 0:
            return np.empty(0, dtype=np.int64)
        if np.any(g[1:] < g[:-1]) or g.min() < 0 or g.max() > np.iinfo(np.int32).max:
            # reference order for unsorted input: position of each present id
            pos = np.minimum(np.searchsorted(self.ent_to_global, g), self.ent_to_global.size - 1)
            return pos[self.ent_to_global[pos] == g]
        d = torch.from_numpy(g.astype(np.int32)).to(self.graph.device)
        return _host_ids(self._to_local_dev(d))


def materialize_subgraphs(plan: PartitionPlan, triples) -> list:
    """Per-partition device subgraphs (partition.py:125-154).

    A triple belongs to its subject's partition; within a partition, local
    triple ids follow ascending global tids and local entity ids ascending
    global ids over the partition's subjects and objects.  One stable sort
    of the triples by partition yields every partition's tid run at once;
    ``np.unique(..., return_inverse=True)`` gives each run's entity map and
    local ids together.  ``triples``: (subj, rel, obj, n_entities,
    n_relations) or an object with ``arrays()``/``n_entities``/``n_relations``."""
    from .device_graph import build_incidence

    if hasattr(triples, "arrays"):
        subj, rel, obj = triples.arrays()
        n_entities, n_relations = triples.n_entities, triples.n_relations
    else:
        subj, rel, obj, n_entities, n_relations = triples
    subj, rel, obj = (np.asarray(c, dtype=np.int64) for c in (subj, rel, obj))
    owner = plan.assignment[subj]
    by_part = np.argsort(owner, kind="stable")  # ascending tids within a partition
    bounds = np.searchsorted(owner[by_part], np.arange(plan.m + 1))
    out = []
    for p in range(plan.m):
        tids = by_part[bounds[p]:bounds[p + 1]].astype(np.int64)
        n = tids.size
        ents, local = np.unique(np.concatenate([subj[tids], obj[tids]]), return_inverse=True)
        graph = build_incidence((local[:n], rel[tids], local[n:]), int(ents.size), n_relations)
        out.append(Subgraph(p, graph, ents, tids))
    return out


# ------------------------------------------------------------ stores


class InMemoryStore:
    """Store over prematerialised subgraphs (engine.py:45-60)."""

    def __init__(self, subgraphs, n_entities: int, n_relations: int):
        self._subgraphs = {sg.index: sg for sg in subgraphs}
        self.m = len(subgraphs)
        self.n_entities = int(n_entities)
        self.n_relations = int(n_relations)
        self.n_triples = sum(sg.graph.n_triples for sg in subgraphs)

    def load(self, index: int) -> Subgraph:
        try:
            return self._subgraphs[index]
        except KeyError:
            raise IntegrityError(f"store has no partition {index}") from None


class PartitionManifest:
    """The ``manifest.json`` of a partition directory (format of
    archive.py:188-237, checks of archive.py:240-255): partition count,
    strategy, entity / relation / triple counts, the assignment file and one
    entry per shard (archive, entity map, triple map, triple count)."""

    FORMAT = "LKG-partition"

    def __init__(self, fields: dict):
        self.fields = fields
        self.m = int(fields["m"])
        self.n_entities = int(fields["entity_count"])
        self.n_relations = int(fields["relation_count"])
        self.n_triples = int(fields["triple_count"])
        self.shards = {int(s["index"]): s for s in fields["partitions"]}

    @staticmethod
    def shard_stem(index: int) -> str:
        return f"shard-{index:04d}"

    @classmethod
    def read(cls, part_dir: Path) -> "PartitionManifest":
        path = part_dir / MANIFEST_FILE
        if not path.exists():
            raise IntegrityError(f"no partition manifest at {path}")
        try:
            fields = json.loads(path.read_text())
        except json.JSONDecodeError as exc:
            raise IntegrityError(f"unreadable manifest: {exc}") from exc
        problems = (
            (fields.get("format") != cls.FORMAT, "not a partition manifest"),
            (lambda: len(fields["partitions"]) != fields["m"], "manifest shard list disagrees with m"),
            (lambda: sum(s["triple_count"] for s in fields["partitions"]) != fields["triple_count"],
             "per-partition triple counts do not sum to the total"),
        )
        for bad, message in problems:
            if bad() if callable(bad) else bad:
                raise IntegrityError(message)
        return cls(fields)

    @classmethod
    def describe(cls, plan: PartitionPlan, subgraphs, n_relations: int) -> "PartitionManifest":
        entries = [{"index": sg.index, "shard_file": f"{cls.shard_stem(sg.index)}.lkg",
                    "entity_map_file": f"{cls.shard_stem(sg.index)}.ents.u64",
                    "triple_map_file": f"{cls.shard_stem(sg.index)}.tids.u64",
                    "triple_count": sg.graph.n_triples} for sg in subgraphs]
        return cls({"format": cls.FORMAT, "version": ARCHIVE_VERSION, "m": plan.m,
                    "strategy": plan.strategy, "entity_count": plan.n_entities,
                    "relation_count": n_relations, "triple_count": int(plan.loads.sum()),
                    "assignment_file": ASSIGNMENT_FILE, "partitions": entries})

    def write(self, part_dir: Path) -> None:
        (part_dir / MANIFEST_FILE).write_text(json.dumps(self.fields, indent=2, sort_keys=True) + "\n")


def _label_lines(labels) -> bytes:
    """Newline-terminated labels, line index = id (the label files of
    archive.py:150-160); ``labels`` is any sequence of strings or an object
    with ``labels()``."""
    seq = labels.labels() if hasattr(labels, "labels") else labels
    return "".join(f"{s}\n" for s in seq).encode("utf-8")


def _read_label_lines(path: Path) -> list:
    text = path.read_text(encoding="utf-8")
    return text.split("\n")[:-1] if text.endswith("\n") else text.split("\n") if text else []


def save_partition_dir(plan: PartitionPlan, subgraphs, entities, relations, n_relations: int,
                       out_dir) -> Path:
    """Write a partition directory the reference reads (archive.py:192-237):
    u32 assignment (UNASSIGNED as 0xFFFFFFFF), label files, and per shard an
    LKG1 archive plus little-endian u64 entity / triple maps."""
    from .archive import save_graph

    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    (out / ASSIGNMENT_FILE).write_bytes(plan.assignment.astype("<i4").view("<u4").tobytes())
    (out / ENTITIES_FILE).write_bytes(_label_lines(entities))
    (out / RELATIONS_FILE).write_bytes(_label_lines(relations))
    man = PartitionManifest.describe(plan, subgraphs, n_relations)
    for sg, entry in zip(subgraphs, man.fields["partitions"]):
        save_graph(sg.graph, out / entry["shard_file"])
        (out / entry["entity_map_file"]).write_bytes(sg.ent_to_global.astype("<u8").tobytes())
        (out / entry["triple_map_file"]).write_bytes(sg.tid_to_global.astype("<u8").tobytes())
    man.write(out)
    return out


def load_partition_plan(part_dir) -> PartitionPlan:
    """The plan a partition directory was written with (archive.py:258-272)."""
    d = Path(part_dir)
    man = PartitionManifest.read(d)
    raw = np.fromfile(d / man.fields["assignment_file"], dtype="<u4")
    if raw.size != man.n_entities:
        raise IntegrityError("assignment array length disagrees with entity count")
    assignment = raw.view("<i4").astype(np.int32)  # 0xFFFFFFFF reads back as -1 = UNASSIGNED
    loads = np.zeros(man.m, dtype=np.int64)
    idx = np.fromiter(man.shards.keys(), dtype=np.int64, count=len(man.shards))
    loads[idx] = [int(e["triple_count"]) for e in man.shards.values()]
    assignment.setflags(write=False)
    loads.setflags(write=False)
    return PartitionPlan(man.m, assignment, loads, man.fields.get("strategy", "lpt"))


class DirectoryStore:
    """Shard archives of a partition directory, loaded on demand straight
    onto the device (the role of archive.py:275-301)."""

    def __init__(self, part_dir):
        self.dir = Path(part_dir)
        self.manifest = PartitionManifest.read(self.dir)
        self.m = self.manifest.m
        self.n_entities = self.manifest.n_entities
        self.n_relations = self.manifest.n_relations
        self.n_triples = self.manifest.n_triples

    def load(self, index: int) -> Subgraph:
        from .archive import load_graph

        entry = self.manifest.shards.get(index)
        if entry is None:
            raise IntegrityError(f"manifest has no partition {index}")
        archive = self.dir / entry["shard_file"]
        if not archive.exists():
            raise IntegrityError(f"partition {index}: missing shard file {archive.name}")
        graph = load_graph(archive)
        ents, tids = (np.fromfile(self.dir / entry[key], dtype="<u8").astype(np.int64)
                      for key in ("entity_map_file", "triple_map_file"))
        if (ents.size, tids.size) != (graph.n_entities, graph.n_triples):
            raise IntegrityError(f"partition {index}: id map sizes disagree with shard")
        return Subgraph(index, graph, ents, tids)


def open_partitioned(part_dir, cache_capacity: int, record_trace: bool = False):
    """A partition directory as a queryable ``PartitionedGraph`` plus its
    entity and relation labels (lists, line index = id; archive.py:304-315)."""
    d = Path(part_dir)
    pg = PartitionedGraph(load_partition_plan(d), DirectoryStore(d),
                          SubgraphCache(cache_capacity, record_trace=record_trace))
    return pg, _read_label_lines(d / ENTITIES_FILE), _read_label_lines(d / RELATIONS_FILE)


# ------------------------------------------------------------ the graph


class StorePartitionedGraph(PartitionedGraph):
    """A partition plan, a subgraph store and the LRU tying them together
    (engine.py:62-86).  Built by ``PartitionedGraph(plan, store, cache)``."""

    def __init__(self, plan: PartitionPlan, store, cache: SubgraphCache):
        if plan.m != store.m:
            raise IntegrityError(f"plan has {plan.m} partitions, store has {store.m}")
        self.plan = plan
        self.store = store
        self.cache = cache
        self._d_assign = None

    @property
    def n_entities(self) -> int:
        return self.store.n_entities

    @property
    def n_relations(self) -> int:
        return self.store.n_relations

    @property
    def n_triples(self) -> int:
        return self.store.n_triples

    def fetch(self, index: int) -> Subgraph:
        return self.cache.get(index, self.store.load)

    @property
    def device(self):
        torch = _torch()
        return torch.device("cuda", torch.cuda.current_device())

    def _assign(self):
        if self._d_assign is None:
            self._d_assign = _torch().from_numpy(np.array(self.plan.assignment, np.int32)).to(self.device)
        return self._d_assign

    def _route_counts(self, frontier) -> np.ndarray:
        torch = _torch()
        dev = self.device
        m = self.plan.m
        counts = torch.zeros(max(m, 1), dtype=torch.int64, device=dev)
        _lib.check(_lib.load().th_ids_route_count(self._assign().data_ptr(), self.plan.n_entities,
                                                  frontier.data_ptr(), frontier.numel(), m,
                                                  counts.data_ptr(), _stream_ptr(dev)))
        return counts[:m].cpu().numpy()

    def expand(self, frontier, details: list | None = None):
        """One global hop (engine.py:94-135): device (activated tids, reached
        ids), both ascending and duplicate-free."""
        dev = self.device
        E, T = self.n_entities, self.n_triples
        reached, act = _bits(E, dev), _bits(T, dev)
        if frontier.numel():
            for p in np.flatnonzero(self._route_counts(frontier)).tolist():
                sg = self.fetch(int(p))
                local = sg._to_local_dev(frontier)
                if local.numel() == 0:
                    continue
                res = sg.retriever.run(_torch().tensor([0, local.numel()], dtype=_torch().int32, device=dev),
                                       local, 1, HopSemantics.EXACT_WALK, None, frontiers=True,
                                       activated=True, copy=False)
                fo, fl = int(res.frontier_off[0, 0]), int(res.frontier_len[0, 0])
                ao, al = int(res.act_off[0, 0]), int(res.act_len[0, 0])
                nxt, a_loc = res.frontier_ids[fo:fo + fl], res.act_ids[ao:ao + al]
                _scatter(reached, E, nxt, dev, sg._d_ent)
                _scatter(act, T, a_loc, dev, sg._d_tid)
                if details is not None and a_loc.numel():
                    g = sg.graph
                    a64 = a_loc.long()
                    details.append((sg._d_tid[a64], sg._d_ent[g.device_column("subj")[a64].long()],
                                    g.device_column("rel")[a64].int(), sg._d_ent[g.device_column("obj")[a64].long()]))
        return act, reached


def _check_query(q0: EntityVector, k: int, pg) -> None:
    if q0.width != pg.n_entities:
        raise ValueError(f"query width {q0.width} != graph entity count {pg.n_entities}")
    if k < 1:
        raise ValueError("hop count must be >= 1")


def store_k_hop(q0: EntityVector, k: int, pg: StorePartitionedGraph,
                semantics=HopSemantics.FRONTIER, details: list | None = None) -> HopTrace:
    """cross_graph_k_hop over a store (engine.py:138-154) with run_hops'
    semantics (incidence.py:268-316) on device bitmaps."""
    torch = _torch()
    _check_query(q0, k, pg)
    sem = HopSemantics.parse(semantics)
    dev = pg.device
    E, T = pg.n_entities, pg.n_triples
    cur = torch.from_numpy(q0.ids.astype(np.int32)).to(dev)
    visited = cum = None
    if sem is not HopSemantics.EXACT_WALK:
        visited = _bits(E, dev)
        _scatter(visited, E, cur, dev)
        if sem is HopSemantics.CUMULATIVE:
            cum = _bits(E, dev)
    lib = _lib.load()
    steps = []
    for _ in range(k):
        act, reached = pg.expand(cur, details)
        activated = _compact(act, T, dev)
        if sem is HopSemantics.EXACT_WALK:
            cur = _compact(reached, E, dev)
            out = cur
        else:
            _lib.check(lib.th_bits_andnot_update(reached.data_ptr(), visited.data_ptr(), E, _stream_ptr(dev)))
            cur = _compact(reached, E, dev)
            out = cur
            if cum is not None:
                _lib.check(lib.th_bits_or(cum.data_ptr(), reached.data_ptr(), E, _stream_ptr(dev)))
                out = _compact(cum, E, dev)
        steps.append(HopStep(EntityVector(_host_ids(out), E, _canonical=True),
                             TripleVector(_host_ids(activated), T, _canonical=True)))
    return HopTrace(sem, q0, steps)


def store_paths(q0: EntityVector, k: int, pg: StorePartitionedGraph,
                max_paths: int | None = DEFAULT_MAX_PATHS):
    """cross_graph_paths over a store (engine.py:157-182).

    Walks of the full graph are exactly the walks over the triples activated
    at their hop under exact-walk semantics; the exact-walk trace collects
    those triples (global tid, subject, relation, object) per partition, and
    the device path kernel (K5) enumerates their subgraph (local tids a
    monotone renumbering of the global ones) -- identical paths, order and
    truncation flag."""
    from .core_types import PathResult
    from .device_graph import build_incidence
    from .retriever import reconstruct_paths

    torch = _torch()
    _check_query(q0, k, pg)
    if max_paths is not None and max_paths < 0:
        raise ValueError("max_paths must be >= 0")
    details: list = []
    store_k_hop(q0, k, pg, HopSemantics.EXACT_WALK, details)
    dev = pg.device
    T = pg.n_triples
    if details:
        tid, s, r, o = (torch.cat(c) for c in zip(*details))
    else:
        tid = s = r = o = torch.empty(0, dtype=torch.int32, device=dev)
    bits = _bits(T, dev)
    _scatter(bits, T, tid, dev)
    order = _compact(bits, T, dev)  # distinct activated tids, ascending
    cols = []
    for c in (s, r, o):
        dense = torch.zeros(max(T, 1), dtype=torch.int32, device=dev)
        if tid.numel():
            dense[tid.long()] = c.int()
        cols.append(dense[order.long()])
    sub = build_incidence(tuple(cols), pg.n_entities, pg.n_relations)
    res = reconstruct_paths(q0, k, sub, max_paths)
    return PathResult(res.paths, res.truncated)
