"""Partitioned (multi-GPU) retrieval: SURVEY.md 8e, rows a12-a16 of 8a.

Reference (citations relative to /root/reference/pkg/src/triplehop):

* ``plan_partitions`` / ``PartitionPlan`` ... partition.py:28-98
* ``route`` / ``RouteResult`` ............... partition.py:157-181
* ``materialize_subgraphs`` ................ partition.py:125-154  -> th_shard_create
* ``_partitioned_expand`` (Algorithm 1) .... engine.py:94-135      -> run_wave
* ``cross_graph_k_hop`` .................... engine.py:138-154

The reference routes each frontier through subject-cohesive shards inside
one process and unions the shard results per hop.  Here every rank (one
process per GPU) owns a hash shard, ``own(v) = ((v * 0x9E3779B1) mod 2^32)
mod world`` (the reference's hash plan, applied to every entity), holding
the out-rows of its subjects and the per-query state of its entities.  The
top out-degree entities (hubs, default the top 0.01%) are edge-split over
all ranks instead -- the static form of the reference's shard cache for the
rows every query touches.  One wave of <= 1,024 queries runs hop by hop:

    expand (device)  -> all-to-all of (row, word, bits) records (NCCL)
    absorb (device)  -> sum of owned hub rows over ranks (NCCL all-reduce)
    hub merge, materialise owned frontier ids (device)

and the owners' sorted slices merge into the reference's per-query
results.  Results are bit-identical to the single-GPU engine and to the
reference's traces (tests/test_partition*.py, tests/test_gpu_partition.py).

The exchange is pluggable: ``DistExchange`` (torch.distributed -- NCCL on
B200s, gloo for the CPU tests) hosts one rank per process;
``LoopbackExchange`` hosts every rank of a small world in one process on
one device (GPU parity tests on a single B200).
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core_types import EntityVector, HopSemantics, HopStep, HopTrace, TripleVector
from .errors import IntegrityError, UsageError

UNASSIGNED = -1
STRATEGIES = ("lpt", "hash")
HASH_MULT = 0x9E3779B1
DEFAULT_HUB_FRACTION = 1e-4  # top 0.01% by out-degree (BASELINE configs[3])
MAX_WAVE = 1024


def hash_owner(ids, m: int) -> np.ndarray:
    """((id * 0x9E3779B1) mod 2^32) mod m  (partition.py:80-84)."""
    ids = np.asarray(ids, dtype=np.int64)
    return (((ids * HASH_MULT) & 0xFFFFFFFF) % m).astype(np.int32)


# --------------------------------------------------------------- plans


class PartitionPlan:
    """Subject -> partition assignment and per-partition triple loads
    (the reference's ``PartitionPlan``, partition.py:28-42): ``m``,
    ``assignment`` (int32 per entity, ``UNASSIGNED`` for entities that are
    never a subject), ``loads`` (int64 per partition) and ``strategy``."""

    __slots__ = ("m", "assignment", "loads", "strategy")

    def __init__(self, m: int, assignment: np.ndarray, loads: np.ndarray, strategy: str):
        object.__setattr__(self, "m", int(m))
        object.__setattr__(self, "assignment", assignment)
        object.__setattr__(self, "loads", loads)
        object.__setattr__(self, "strategy", strategy)

    def __setattr__(self, name, value):
        raise AttributeError("PartitionPlan is immutable")

    def __eq__(self, other) -> bool:
        return (isinstance(other, PartitionPlan) and self.m == other.m and self.strategy == other.strategy
                and np.array_equal(self.assignment, other.assignment)
                and np.array_equal(self.loads, other.loads))

    def __repr__(self) -> str:
        return f"PartitionPlan(m={self.m}, strategy={self.strategy!r}, loads={self.loads.tolist()})"

    @property
    def n_entities(self) -> int:
        return int(self.assignment.size)

    def partition_of(self, entity: int) -> int:
        return int(self.assignment[entity])


def _subject_columns(triples):
    """(subject column, entity count) from an IncidenceGraph or a pair."""
    if hasattr(triples, "subj") and hasattr(triples, "n_entities"):
        return triples.subj, int(triples.n_entities)
    subj, n_entities = triples
    return subj, int(n_entities)


def plan_partitions(triples, m: int, strategy: str = "lpt") -> PartitionPlan:
    """Place every subject on one of ``m`` partitions (partition.py:49-98).

    ``triples``: a (subject column, entity count) pair or an
    ``IncidenceGraph``.  The placement itself is native
    (``th_plan_subjects``, ``csrc/planner.cu``): ``"hash"`` is the
    reference's multiplicative hash, ``"lpt"`` its heaviest-first greedy
    (ties by smaller id onto the lightest, then lowest-index partition).
    Argument errors raise ``UsageError`` with the reference's messages.
    """
    subj, n_entities = _subject_columns(triples)
    degrees = np.bincount(np.asarray(subj, dtype=np.int64), minlength=n_entities).astype(np.int64)
    n_subjects = int(np.count_nonzero(degrees))
    if m < 1:
        raise UsageError("partition count must be >= 1")
    if m > n_subjects:
        raise UsageError(f"partition count {m} exceeds distinct subject count {n_subjects}")
    code = {"hash": _lib.TH_PLAN_HASH, "lpt": _lib.TH_PLAN_LPT}.get(strategy)
    if code is None:
        raise UsageError(f"unknown partition strategy {strategy!r}")
    assignment = np.empty(n_entities, dtype=np.int32)
    loads = np.empty(m, dtype=np.int64)
    _lib.check(_lib.load().th_plan_subjects(degrees.ctypes.data, n_entities, m, code,
                                             assignment.ctypes.data, loads.ctypes.data))
    assignment.setflags(write=False)
    loads.setflags(write=False)
    return PartitionPlan(m, assignment, loads, strategy)


class RouteResult:
    """Frontier ids grouped by partition (``buckets``: partition ->
    ``EntityVector``); ids that are never a subject go to ``sink``."""

    __slots__ = ("buckets", "sink")

    def __init__(self, buckets: dict, sink: EntityVector):
        self.buckets = buckets
        self.sink = sink


def route(q: EntityVector, plan: PartitionPlan) -> RouteResult:
    """Bucket the active entities of q by partition (partition.py:170-181).

    One stable sort by partition keeps each bucket ascending (q is), and the
    bucket boundaries split it; ``UNASSIGNED`` (-1) sorts first and is the
    sink.
    """
    if q.width != plan.n_entities:
        raise ValueError(f"query width {q.width} != plan entity count {plan.n_entities}")
    part = plan.assignment[q.ids]
    order = np.argsort(part, kind="stable")
    keys = part[order]
    cuts = np.flatnonzero(np.diff(keys)) + 1
    pieces = np.split(q.ids[order], cuts)
    heads = keys[np.concatenate([[0], cuts])] if keys.size else keys
    buckets, sink = {}, q.ids[:0]
    for p, ids in zip(heads.tolist(), pieces):
        if p == UNASSIGNED:
            sink = ids
        else:
            buckets[p] = EntityVector(ids, q.width, _canonical=True)
    return RouteResult(buckets, EntityVector(sink, q.width, _canonical=True))


@dataclass(frozen=True)
class ShardPlan:
    """Degree-aware owner plan shared by every rank.

    owner[v]  = hash_owner(v, world) for every entity
    lidx[v]   = row of v at its owner (rows number an owner's entities in
                ascending id order, so row order is id order)
    hub_ids   = hubs (top out-degree, ties by smaller id), edge-split
    hub_index = -1 or v's position in hub_ids
    """

    world: int
    n_entities: int
    owner: np.ndarray
    lidx: np.ndarray
    hub_ids: np.ndarray
    hub_index: np.ndarray
    n_local: np.ndarray  # int64 [world]

    def owned(self, rank: int) -> np.ndarray:
        return np.flatnonzero(self.owner == rank).astype(np.int32)

    @property
    def n_hubs(self) -> int:
        return int(self.hub_ids.size)


def select_hubs(subj, n_entities: int, n_hubs: int) -> np.ndarray:
    """The n_hubs highest out-degree subjects, ties by smaller id, ascending."""
    deg = np.bincount(np.asarray(subj, dtype=np.int64), minlength=n_entities)
    n_hubs = int(min(n_hubs, np.count_nonzero(deg)))
    if n_hubs <= 0:
        return np.empty(0, dtype=np.int32)
    kth = np.partition(deg, deg.size - n_hubs)[deg.size - n_hubs]  # n_hubs-th largest
    above = np.flatnonzero(deg > kth)
    at = np.flatnonzero(deg == kth)[: n_hubs - above.size]
    return np.sort(np.concatenate([above, at])).astype(np.int32)


def plan_sharding(subj, n_entities: int, world: int, hub_fraction: float = DEFAULT_HUB_FRACTION,
                  n_hubs: int | None = None) -> ShardPlan:
    if world < 1:
        raise UsageError("world size must be >= 1")
    owner = hash_owner(np.arange(n_entities, dtype=np.int64), world)
    lidx = np.empty(n_entities, dtype=np.int32)
    n_local = np.zeros(world, dtype=np.int64)
    for p in range(world):
        idx = np.flatnonzero(owner == p)
        lidx[idx] = np.arange(idx.size, dtype=np.int32)
        n_local[p] = idx.size
    if n_hubs is None:
        # (hubs only spread a row's edges over ranks: one rank needs none)
        n_hubs = int(round(n_entities * hub_fraction)) if world > 1 else 0
    hubs = select_hubs(subj, n_entities, n_hubs)
    hub_index = np.full(n_entities, -1, dtype=np.int32)
    hub_index[hubs] = np.arange(hubs.size, dtype=np.int32)
    for a in (owner, lidx, hubs, hub_index, n_local):
        a.setflags(write=False)
    return ShardPlan(world, n_entities, owner, lidx, hubs, hub_index, n_local)


# --------------------------------------------------------------- exchange


class Exchange:
    """What the partitioned wave needs from the transport between ranks.

    The data path itself is not here: shards write into each other's
    exchange regions from their kernels (k6_shard.cuh).  The exchange wires
    the regions together (``connect``), separates the phases of a hop
    (``barrier``: every peer's writes of the previous phase are complete),
    agrees on a flag (``any``) and gathers the owners' result slices at the
    end of a wave (``gather``).  It hosts ``ranks`` of a ``world``."""

    world: int
    ranks: list

    def connect(self, shards) -> None:
        raise NotImplementedError

    def barrier(self, shards) -> None:
        raise NotImplementedError

    def any(self, flags) -> bool:
        raise NotImplementedError

    def gather(self, parts) -> list:  # one dict of tensors per hosted rank -> every rank's, rank order
        raise NotImplementedError

    def sum_int(self, values) -> int:  # one int per hosted rank -> the sum over all ranks
        raise NotImplementedError


class LoopbackExchange(Exchange):
    """Every rank of the world in this process, on one device: the regions
    are plain device pointers, and the ranks' kernels run one after another
    on one stream, so stream order is the barrier."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def connect(self, shards) -> None:
        bases = [sh.region_handle(local=True) for sh in shards]
        for sh in shards:
            for p, base in enumerate(bases):
                sh.connect_peer(p, base, local=True)

    def barrier(self, shards) -> None:
        return None

    def any(self, flags) -> bool:
        return bool(any(flags))

    def gather(self, parts) -> list:
        return list(parts)

    def sum_int(self, values) -> int:
        return int(sum(int(v) for v in values))


class DistExchange(Exchange):
    """One rank per process over torch.distributed.  Peer regions are CUDA
    IPC mappings (handles shipped once with all_gather_object); the phase
    barrier is a stream synchronisation plus a process-group barrier, with
    no data read back (on NCCL the barrier is a 1-element all-reduce).
    ``gather`` moves the owners' result slices with all_gather (NCCL on
    B200s; gloo with host tensors in the CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]
        self.staged = dist.get_backend(group) != "nccl"

    def connect(self, shards) -> None:
        (sh,) = shards
        handles = [None] * self.world
        self.dist.all_gather_object(handles, sh.region_handle(local=False), group=self.group)
        for p, h in enumerate(handles):
            sh.connect_peer(p, h, local=False)
        self.dist.barrier(group=self.group)

    def barrier(self, shards) -> None:
        for sh in shards:
            sh.synchronize()
        self.dist.barrier(group=self.group)

    def any(self, flags) -> bool:
        import torch

        (f,) = flags
        t = torch.tensor([1 if f else 0], dtype=torch.int32, device="cpu" if self.staged else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def sum_int(self, values) -> int:
        import torch

        (v,) = values
        t = torch.tensor([int(v)], dtype=torch.int64, device="cpu" if self.staged else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return int(t.item())

    def gather(self, parts) -> list:
        """all_gather of every tensor of this rank's dict (sizes first, then
        padded payloads): one entry per rank, on this rank's device."""
        import torch

        (mine,) = parts
        names = sorted(k for k, v in mine.items() if v is not None)
        out = [dict() for _ in range(self.world)]
        for name in names:
            t = mine[name]
            dev = t.device
            src = t.reshape(-1).cpu() if self.staged else t.reshape(-1)
            n = torch.tensor([src.numel()], dtype=torch.int64, device=src.device)
            sizes = [torch.zeros_like(n) for _ in range(self.world)]
            self.dist.all_gather(sizes, n, group=self.group)
            sizes = [int(x.item()) for x in sizes]
            m = max(max(sizes), 1)
            pad = torch.zeros(m, dtype=src.dtype, device=src.device)
            pad[: src.numel()] = src
            bufs = [torch.empty_like(pad) for _ in range(self.world)]
            self.dist.all_gather(bufs, pad, group=self.group)
            for r in range(self.world):
                v = bufs[r][: sizes[r]].to(dev)
                out[r][name] = v.reshape(-1, *t.shape[1:]) if t.dim() > 1 else v
        return out


# --------------------------------------------------------------- device shard

DEFAULT_INBOX = 1 << 22  # records per exchange inbox; grown after an overflow


class GraphShard:
    """One rank's device shard (th_shard): owned out-rows + hub slices, and
    the exchange region its peers write into."""

    def __init__(self, cols, n_entities: int, n_relations: int, plan: ShardPlan, rank: int,
                 stream=None, inbox_records: int = DEFAULT_INBOX):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2604_18913_b200 needs a CUDA device (B200); no CPU fallback exists")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        self.plan = plan
        self.rank = rank
        self.n_entities = int(n_entities)
        self.n_relations = int(n_relations)
        s, r, o = (c if isinstance(c, torch.Tensor) and c.is_cuda else
                   torch.from_numpy(np.ascontiguousarray(np.asarray(c), dtype=np.int32)).to(dev)
                   for c in cols)
        s, r, o = (c.to(torch.int32).contiguous() for c in (s, r, o))
        self.n_triples = int(s.numel())
        up = lambda a: torch.from_numpy(np.array(a, dtype=np.int32)).to(dev)  # noqa: E731
        lidx, hidx, hubs = up(plan.lidx), up(plan.hub_index), up(plan.hub_ids)
        l2g = up(plan.owned(rank))
        lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(lib.th_shard_create(
            s.data_ptr(), r.data_ptr(), o.data_ptr(), self.n_triples, self.n_entities, self.n_relations,
            lidx.data_ptr(), hidx.data_ptr(), hubs.data_ptr() if hubs.numel() else None, hubs.numel(),
            l2g.data_ptr() if l2g.numel() else None, l2g.numel(), rank, plan.world, int(inbox_records),
            ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)))
        self._handle = h.value
        self._finalizer = weakref.finalize(self, lib.th_shard_destroy, self._handle)
        self.local_triples = int(lib.th_shard_local_triples(self._handle))
        self.can_pull = bool(lib.th_shard_can_pull(self._handle))
        self.inbox_records = int(inbox_records)

    def launch_count(self) -> int:
        return int(_lib.load().th_shard_launch_count(self._handle))

    def set_pull_divisor(self, divisor: float) -> None:
        _lib.check(_lib.load().th_shard_set_pull_divisor(self._handle, float(divisor)))

    # -- exchange wiring -----------------------------------------------------
    def region_handle(self, local: bool):
        """This shard's exchange region: its device address (same process)
        or its 64-byte CUDA IPC handle (other processes)."""
        lib = _lib.load()
        if local:
            base, nbytes, rec = ctypes.c_void_p(), ctypes.c_uint64(), ctypes.c_int64()
            _lib.check(lib.th_shard_region(self._handle, ctypes.byref(base), ctypes.byref(nbytes),
                                           ctypes.byref(rec)))
            return base.value
        buf = ctypes.create_string_buffer(64)
        _lib.check(lib.th_shard_ipc_handle(self._handle, buf))
        return bytes(buf.raw)

    def connect_peer(self, peer: int, handle, local: bool) -> None:
        lib = _lib.load()
        if local:
            _lib.check(lib.th_shard_connect(self._handle, peer, ctypes.c_void_p(handle)))
        elif peer == self.rank:
            _lib.check(lib.th_shard_connect(self._handle, peer, ctypes.c_void_p(self.region_handle(True))))
        else:
            _lib.check(lib.th_shard_ipc_open(self._handle, peer, ctypes.create_string_buffer(handle, 64)))

    def grow_inbox(self) -> None:
        self.inbox_records *= 4
        _lib.check(_lib.load().th_shard_grow_inbox(self._handle, self.inbox_records))

    def synchronize(self) -> None:
        self.stream.synchronize()

    def set_profiling(self, on: bool) -> None:
        _lib.check(_lib.load().th_shard_set_profiling(self._handle, int(bool(on))))

    def profile_trace(self) -> list:
        """Timeline of the last profiled wave: (category, stream, start ms,
        end ms) per kernel group (stream 0 main, 1 / 2 K4 side streams)."""
        lib = _lib.load()
        n = int(lib.th_shard_profile_trace(self._handle, None, 0))
        if n < 0:
            raise RuntimeError(lib.th_last_error().decode(errors="replace"))
        buf = (ctypes.c_double * max(4 * n, 1))()
        lib.th_shard_profile_trace(self._handle, buf, n)
        return [(_lib.PROF_CATEGORIES[int(buf[4 * i])], int(buf[4 * i + 1]), buf[4 * i + 2], buf[4 * i + 3])
                for i in range(n)]

    # -- K7 hub-adjacency cache ------------------------------------------------
    def enable_hub_cache(self, capacity_pages: int) -> None:
        """Page this shard's hub slices in on demand from a pinned host store
        into ``capacity_pages`` HBM pages, least recently used out first
        (csrc/hubcache.cu; the reference's LRU, cache.py:38-89)."""
        _lib.check(_lib.load().th_shard_hub_cache(self._handle, int(capacity_pages)))

    def hub_cache_stats(self) -> dict:
        """Counters (the reference's algebra) plus the cache geometry."""
        from .cache import CacheCounters

        out = (ctypes.c_int64 * 8)()
        _lib.check(_lib.load().th_shard_hub_cache_stats(self._handle, out))
        h, m, ld, ev, res, cap, pages, pe = (int(x) for x in out)
        return {"counters": CacheCounters(h, m, ld, ev, h / (h + m) if h + m else 0.0),
                "resident": res, "capacity": cap, "pages": pages, "page_edges": pe}

    def _cache_list(self, fn) -> list:
        lib = _lib.load()
        n = int(getattr(lib, fn)(self._handle, None, 0))
        if n < 0:
            raise RuntimeError("the shard has no hub cache (enable_hub_cache)")
        buf = (ctypes.c_int64 * max(n, 1))()
        getattr(lib, fn)(self._handle, buf, n)
        return [int(x) for x in buf[:n]]

    def hub_cache_trace(self) -> list:
        """Pages accessed since the last call, in access order (the log is
        cleared)."""
        return self._cache_list("th_shard_hub_cache_trace")

    def hub_cache_resident(self) -> list:
        """Resident pages, least recently used first."""
        return self._cache_list("th_shard_hub_cache_resident")

    # -- the wave ---------------------------------------------------------------
    def begin(self, query: "WaveQuery") -> None:
        _lib.check(_lib.load().th_shard_begin(self._handle, ctypes.byref(self.prepare(query))))

    def prepare(self, query: "WaveQuery"):
        """Upload the wave's query arrays; the th_query describing them."""
        q = _lib.Query()
        B = query.n_queries
        self._dev = {
            "offs": self._upload("offs", query.seed_offsets),
            "seeds": self._upload("seeds", query.seeds),
            "masks": None if query.masks is None else self._upload("masks", query.masks.view(np.int32)),
        }
        q.n_queries = B
        q.d_seed_offsets = self._dev["offs"].data_ptr()
        q.d_seeds = self._dev["seeds"].data_ptr() if self._dev["seeds"].numel() else q.d_seed_offsets
        q.k = query.k
        q.semantics = query.semantics.code
        q.d_rel_masks = None if self._dev["masks"] is None else self._dev["masks"].data_ptr()
        q.mask_words = 0 if query.masks is None else int(query.masks.shape[1])
        q.flags = _lib.TH_WANT_FRONTIERS | (_lib.TH_WANT_ACTIVATED if query.activated else 0)
        q.max_paths = 0
        self._q = q
        self._n_seeds = int(np.asarray(query.seeds).size)
        return q

    def _upload(self, name, arr):
        """Asynchronous H2D copy through a reused pinned staging buffer,
        ordered on the shard's stream before the wave's kernels (the buffer
        is rewritten only once its previous copy has finished)."""
        import torch

        a = np.ascontiguousarray(arr).reshape(-1)
        pins = self.__dict__.setdefault("_pins", {})
        buf, done = pins.get(name, (None, None))
        if buf is None or buf.numel() < a.size:
            buf = torch.empty(max(a.size, 1) * 2, dtype=torch.from_numpy(a[:0]).dtype).pin_memory()
            done = None
        if done is not None:
            done.synchronize()  # the previous copy out of this buffer has finished
        buf[: a.size].copy_(torch.from_numpy(a))
        dev = torch.empty(a.size, dtype=buf.dtype, device=self.device)
        with torch.cuda.stream(self.stream):
            dev.copy_(buf[: a.size], non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.stream)
        pins[name] = (buf, done)
        return dev.reshape(arr.shape)

    def hop(self, hop: int, phase: int) -> None:
        _lib.check(_lib.load().th_shard_hop(self._handle, hop, phase))

    def finish(self):
        """-> ("ok", ShardResult), ("overflow", None) or ("inbox", None)."""
        lib = _lib.load()
        res = _lib.Result()
        rc = lib.th_shard_finish(self._handle, ctypes.byref(res))
        if rc == _lib.TH_ERR_OVERFLOW:
            return ("inbox" if lib.th_shard_inbox_overflowed(self._handle) == 1 else "overflow"), None
        _lib.check(rc)
        return "ok", self._result(res)

    def sent_records(self, k: int) -> list:
        per = (ctypes.c_int64 * k)()
        _lib.check(_lib.load().th_shard_sent(self._handle, per, k))
        return [int(x) for x in per]

    def _result(self, res) -> "ShardResult":
        """Device views of the shard's results (valid until its next wave)."""
        B, k = res.n_queries, res.k
        t = _lib.as_tensor
        out = ShardResult(B, k)
        out.edges = t(res.edges, (k, B), "<i8", self)
        out.f_off = t(res.frontier_off, (k, B), "<i8", self)
        out.f_len = t(res.frontier_len, (k, B), "<i8", self)
        out.f_ids = t(res.frontier_ids, (res.frontier_total,), "<i4", self)
        if self._q.flags & _lib.TH_WANT_ACTIVATED:
            out.a_off = t(res.act_off, (k, B), "<i8", self)
            out.a_len = t(res.act_len, (k, B), "<i8", self)
            out.a_ids = t(res.act_ids, (res.act_total,), "<i4", self)
        return out

    def triples_of(self, tids):
        """(subject, relation, object) of this shard's triples with the given
        (sorted, global) tids, all global ids -- device tensors."""
        import torch

        cols = _lib.ShardCols()
        _lib.check(_lib.load().th_shard_columns(self._handle, ctypes.byref(cols)))
        t = _lib.as_tensor
        n = int(cols.n_triples)
        tid_l2g = t(cols.tid_l2g, (n,), "<i4", self)
        local = torch.searchsorted(tid_l2g, tids.to(torch.int32))
        row = t(cols.subj_row, (n,), "<i4", self)[local].long()
        rel = t(cols.rel, (n,), "<i2", self)[local].to(torch.int32) & 0xFFFF
        obj = t(cols.obj, (n,), "<i4", self)[local]
        # local rows: owned entities [0, n_local), then hub slices
        row_gid = torch.cat([t(cols.l2g, (int(cols.n_local),), "<i4", self),
                             t(cols.hub_ids, (int(cols.n_hubs),), "<i4", self)])
        return row_gid[row].int(), rel.int(), obj.int()


@dataclass
class WaveQuery:
    """One wave (<= 1,024 queries), identical on every rank."""

    seed_offsets: np.ndarray  # int32 [B+1]
    seeds: np.ndarray  # int32
    k: int
    semantics: HopSemantics
    masks: np.ndarray | None = None  # uint32 [B, words]
    activated: bool = False

    @property
    def n_queries(self) -> int:
        return int(self.seed_offsets.size) - 1


@dataclass
class ShardResult:
    """One rank's share of a wave: owned frontier ids, local activated tids,
    partial edge counts (CSR per (hop, query)); tensors."""

    n_queries: int
    k: int
    edges: object = None
    f_off: object = None
    f_len: object = None
    f_ids: object = None
    a_off: object = None
    a_len: object = None
    a_ids: object = None

    def tensors(self) -> dict:
        return {n: getattr(self, n) for n in ("edges", "f_off", "f_len", "f_ids", "a_off", "a_len", "a_ids")}


PULL_DIVISOR = 8.0  # pull when the frontier's out-edges exceed T / 8 (as K2/K3)


def run_wave(shards, xch: Exchange, query: WaveQuery, stats: dict | None = None):
    """Drive one wave through every hosted shard (Algorithm 1 per hop): three
    phases per hop, each followed by the exchange's barrier; the data moves
    between ranks inside the kernels.  Returns the hosted shards'
    ShardResults.  An output (or inbox) overflow on any rank makes every rank
    run the wave again with grown capacities."""
    for _attempt in range(6):
        if isinstance(xch, LoopbackExchange) and all(isinstance(sh, GraphShard) for sh in shards):
            # one process, one stream: begin and every phase in one native
            # call, replayed as a CUDA graph once the wave's shape repeats
            qs = (_lib.Query * len(shards))(*[sh.prepare(query) for sh in shards])
            handles = (ctypes.c_void_p * len(shards))(*[sh._handle for sh in shards])
            nseeds = (ctypes.c_int64 * len(shards))(*[sh._n_seeds for sh in shards])
            _lib.check(_lib.load().th_shards_run_wave(handles, len(shards), qs, nseeds))
        else:
            for sh in shards:
                sh.begin(query)
            xch.barrier(shards)
            for h in range(1, query.k + 1):
                for phase in (0, 1, 2):
                    for sh in shards:
                        sh.hop(h, phase)
                    xch.barrier(shards)
        done = [sh.finish() for sh in shards]
        inbox = xch.any([st == "inbox" for st, _ in done])
        if not xch.any([st != "ok" for st, _ in done]):
            if stats is not None:
                stats["sent_records"] = [sh.sent_records(query.k) for sh in shards]
            return [r for _, r in done]
        if inbox:
            for sh in shards:
                sh.grow_inbox()
            xch.connect(shards)
    raise RuntimeError("partitioned wave kept overflowing its buffers")


def merge_results(parts, n_queries: int, k: int, activated: bool, width_f: int, width_a: int):
    """The union of the owners' sorted slices per (hop, query), on the
    device of the parts: owners are disjoint, so one sort of (segment, id)
    keys gives every segment sorted and duplicate-free (the role of the
    reference's sort/unique of a concatenation, engine.py:121-127)."""
    import torch

    def merge(name_off, name_len, name_ids, width):
        keys = []
        for p in parts:
            off, ln, data = p[name_off], p[name_len], p[name_ids]
            dev = data.device
            flat_len = ln.reshape(-1).long()
            seg = torch.repeat_interleave(torch.arange(flat_len.numel(), device=dev), flat_len)
            start = torch.cumsum(flat_len, 0) - flat_len
            pos = off.reshape(-1).long()[seg] + (torch.arange(seg.numel(), device=dev) - start[seg])
            keys.append(seg * width + data[pos].long())
        key = torch.sort(torch.cat(keys)).values if keys else torch.empty(0, dtype=torch.int64)
        seg = key // width
        cnt = torch.bincount(seg, minlength=k * n_queries).reshape(k, n_queries)
        off = (torch.cumsum(cnt.reshape(-1), 0) - cnt.reshape(-1)).reshape(k, n_queries)
        return off, cnt, (key % width).to(torch.int32)

    if len(parts) == 1:
        # one rank owns everything: its segments are the answer already
        p = parts[0]
        out = {n: p[n] for n in ("edges", "f_off", "f_len", "f_ids")}
        if activated:
            out.update({n: p[n] for n in ("a_off", "a_len", "a_ids")})
        return out
    out = {"edges": sum(p["edges"].long() for p in parts)}
    out["f_off"], out["f_len"], out["f_ids"] = merge("f_off", "f_len", "f_ids", width_f)
    if activated:
        out["a_off"], out["a_len"], out["a_ids"] = merge("a_off", "a_len", "a_ids", width_a)
    return out


# --------------------------------------------------------------- user API


class PartitionedGraph:
    """Shards of one graph over ``exchange.world`` ranks; this process hosts
    ``exchange.ranks`` of them (engine.py:62-81's role).

    ``PartitionedGraph(plan, store, cache)`` -- the reference's constructor
    (engine.py:62-71) -- builds the store-backed, LRU-cached form instead
    (``store.StorePartitionedGraph``)."""

    def __new__(cls, *args, **kwargs):
        if cls is PartitionedGraph and args and isinstance(args[0], PartitionPlan):
            from .store import StorePartitionedGraph

            return super().__new__(StorePartitionedGraph)
        return super().__new__(cls)

    def __init__(self, triples, n_entities: int, n_relations: int, exchange: Exchange | None = None,
                 plan: ShardPlan | None = None, hub_fraction: float = DEFAULT_HUB_FRACTION,
                 n_hubs: int | None = None, shard_factory=None, hub_cache_pages: int | None = None):
        if exchange is None:
            exchange = LoopbackExchange(1)
        cols = triples if isinstance(triples, tuple) else tuple(np.asarray(list(triples)).reshape(-1, 3).T)
        subj = cols[0].cpu().numpy() if hasattr(cols[0], "cpu") else np.asarray(cols[0])
        for name, col, bound in (("subject", cols[0], n_entities), ("relation", cols[1], n_relations),
                                 ("object", cols[2], n_entities)):
            a = col.cpu().numpy() if hasattr(col, "cpu") else np.asarray(col)
            if a.size and (a.min() < 0 or a.max() >= bound):
                raise ValueError(f"{name} id out of range (bound {bound})")
        if plan is None:
            plan = plan_sharding(subj, n_entities, exchange.world, hub_fraction, n_hubs)
        if plan.world != exchange.world or plan.n_entities != n_entities:
            raise IntegrityError(f"plan is for {plan.world} ranks / {plan.n_entities} entities, "
                                 f"exchange has {exchange.world}")
        self.plan = plan
        self.exchange = exchange
        self.n_entities = int(n_entities)
        self.n_relations = int(n_relations)
        self.n_triples = int(len(subj))
        factory = shard_factory or GraphShard
        self.shards = [factory(cols, n_entities, n_relations, plan, r) for r in exchange.ranks]
        if hub_cache_pages is not None:
            # hub adjacency on demand (config 5): every hosted rank pages its
            # hub slices through its own HBM budget
            for sh in self.shards:
                sh.enable_hub_cache(hub_cache_pages)
        exchange.connect(self.shards)
        self.pull_divisor = PULL_DIVISOR

    @property
    def pull_divisor(self) -> float:
        return self._pull_divisor

    @pull_divisor.setter
    def pull_divisor(self, d: float) -> None:
        """Pull when the ranks' summed frontier out-edges exceed T / d (0 = push only)."""
        self._pull_divisor = float(d)
        for sh in self.shards:
            sh.set_pull_divisor(self._pull_divisor)

    def hub_cache_stats(self) -> list:
        """Per hosted rank: the hub cache's counters and geometry."""
        return [sh.hub_cache_stats() for sh in self.shards]

    def run(self, query: WaveQuery, stats: dict | None = None):
        """One wave; the hosted ranks' partial results (kept sharded)."""
        return run_wave(self.shards, self.exchange, query, stats)

    def merged(self, query: WaveQuery, stats: dict | None = None) -> dict:
        """One wave merged over all ranks (every rank gets the union), as
        device tensors: edges [k, B], f_off/f_len [k, B], f_ids, (+ a_*)."""
        parts = self.exchange.gather([r.tensors() for r in self.run(query, stats)])
        return merge_results(parts, query.n_queries, query.k, query.activated, self.n_entities,
                             self.n_triples)

    def retrieve(self, seeds, k: int, relation_filter=None, semantics="frontier",
                 activated: bool = False, copy: bool = True):
        """Per-seed retrieval (one query per seed), merged on every rank.

        Returns a ``RetrievalResult`` with the same accessors as the
        single-GPU engine (frontier(i, h), activated(i, h), edges): host
        tensors, or -- ``copy=False`` -- device tensors (the caller copies
        what it needs, e.g. into pinned buffers)."""
        import torch

        from .retriever import RetrievalResult, _relation_masks

        sem = HopSemantics.parse(semantics)
        if k < 1:
            raise ValueError("hop count must be >= 1")
        arr = np.asarray(seeds, dtype=np.int64).reshape(-1)
        if arr.size and (arr.min() < 0 or arr.max() >= self.n_entities):
            raise ValueError(f"id out of range for width {self.n_entities}")
        B = arr.size
        words = _relation_masks(relation_filter, B, self.n_relations)
        merged = {"edges": [], "f_off": [], "f_len": [], "f_ids": [], "a_off": [], "a_len": [], "a_ids": []}
        fbase = abase = 0
        for q0 in range(0, max(B, 1), MAX_WAVE):
            q1 = min(B, q0 + MAX_WAVE)
            nq = q1 - q0
            wq = WaveQuery(np.arange(nq + 1, dtype=np.int32), arr[q0:q1].astype(np.int32), k, sem,
                           None if words is None else words[q0:q1], activated)
            m = {n: (v.cpu() if copy and v is not None else v) for n, v in self.merged(wq).items()}
            merged["edges"].append(m["edges"])
            merged["f_off"].append(m["f_off"] + fbase)
            merged["f_len"].append(m["f_len"])
            merged["f_ids"].append(m["f_ids"])
            fbase += m["f_ids"].numel()
            if activated:
                merged["a_off"].append(m["a_off"] + abase)
                merged["a_len"].append(m["a_len"])
                merged["a_ids"].append(m["a_ids"])
                abase += m["a_ids"].numel()
            if B == 0:
                break
        cat = lambda xs, dim=1: xs[0] if len(xs) == 1 else torch.cat(xs, dim)  # noqa: E731
        out = RetrievalResult(B, k, sem, _graph=self)
        out.edges = cat(merged["edges"])
        out.frontier_off, out.frontier_len = cat(merged["f_off"]), cat(merged["f_len"])
        out.frontier_ids = cat(merged["f_ids"], 0)
        if activated:
            out.act_off, out.act_len = cat(merged["a_off"]), cat(merged["a_len"])
            out.act_ids = cat(merged["a_ids"], 0)
        return out


def cross_graph_k_hop(q0: EntityVector, k: int, pg: PartitionedGraph,
                      semantics: HopSemantics = HopSemantics.FRONTIER) -> HopTrace:
    """k-hop retrieval of one seed set across the partitions (engine.py:138-154);
    bit-identical to single-graph ``k_hop`` (frontier and activated sets)."""
    if getattr(pg, "store", None) is not None:
        from .store import store_k_hop

        return store_k_hop(q0, k, pg, semantics)
    if q0.width != pg.n_entities:
        raise ValueError(f"query width {q0.width} != graph entity count {pg.n_entities}")
    if k < 1:
        raise ValueError("hop count must be >= 1")
    sem = HopSemantics.parse(semantics)
    ids = q0.ids.astype(np.int32)
    wq = WaveQuery(np.array([0, ids.size], dtype=np.int32), ids, k, sem, None, True)
    m = {n: (v.cpu().numpy() if v is not None else None) for n, v in pg.merged(wq).items()}
    steps = []
    for h in range(k):
        fo, fl = int(m["f_off"][h, 0]), int(m["f_len"][h, 0])
        ao, al = int(m["a_off"][h, 0]), int(m["a_len"][h, 0])
        steps.append(HopStep(EntityVector(m["f_ids"][fo:fo + fl], pg.n_entities, _canonical=True),
                             TripleVector(m["a_ids"][ao:ao + al], pg.n_triples, _canonical=True)))
    return HopTrace(sem, q0, steps)


def cross_graph_paths(q0: EntityVector, k: int, pg: PartitionedGraph,
                      max_paths: int | None = 10_000):
    """All length-k walks from q0 across the partitions, lexicographic in the
    triple ids, capped (engine.py:157-182 -> assemble_paths).

    Rank-sharded graphs exchange walk counts and capped per-prefix offers
    between the ranks (``walks.sharded_paths``); the activated triples stay
    with their owners.  Store-backed graphs enumerate the walk subgraph of
    their exact-walk trace with the device path kernel (``store_paths``).
    Identical paths, order and truncation flag either way.
    """
    if getattr(pg, "store", None) is not None:
        from .store import store_paths

        return store_paths(q0, k, pg, max_paths)
    if q0.width != pg.n_entities:
        raise ValueError(f"query width {q0.width} != graph entity count {pg.n_entities}")
    if k < 1:
        raise ValueError("hop count must be >= 1")
    if max_paths is not None and max_paths < 0:
        raise ValueError("max_paths must be >= 0")
    from .walks import sharded_paths

    return sharded_paths(q0, k, pg, max_paths)


def walk_subgraph(q0: EntityVector, k: int, pg: PartitionedGraph):
    """(s, r, o) of every triple activated by q0's exact-walk trace, in
    ascending global tid order (the walk subgraph; every length-k walk is a
    walk of it -- a cross-check for ``sharded_paths``).  Every rank resolves the columns of ITS
    activated triples (it owns them) on its device and the owners' pieces
    are gathered -- no rank holds the full triple columns."""
    import torch

    ids = q0.ids.astype(np.int32)
    wq = WaveQuery(np.array([0, ids.size], dtype=np.int32), ids, k, HopSemantics.EXACT_WALK, None, True)
    mine = []
    for sh, r in zip(pg.shards, pg.run(wq)):
        a = r.a_ids.long() if r.a_ids is not None else torch.empty(0, dtype=torch.int64)
        tids = torch.unique(a)  # a triple may be activated at several hops
        s_, r_, o_ = sh.triples_of(tids)
        mine.append({"tid": tids.int(), "s": s_, "r": r_, "o": o_})
    parts = pg.exchange.gather(mine)
    tid = torch.cat([p["tid"].long().cpu() for p in parts])
    order = torch.argsort(tid)  # owners are disjoint: ascending global tids
    return tuple(torch.cat([p[c].cpu() for p in parts])[order].numpy() for c in ("s", "r", "o"))
