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
        n_hubs = int(round(n_entities * hub_fraction))
    hubs = select_hubs(subj, n_entities, n_hubs)
    hub_index = np.full(n_entities, -1, dtype=np.int32)
    hub_index[hubs] = np.arange(hubs.size, dtype=np.int32)
    for a in (owner, lidx, hubs, hub_index, n_local):
        a.setflags(write=False)
    return ShardPlan(world, n_entities, owner, lidx, hubs, hub_index, n_local)


# --------------------------------------------------------------- exchange


class Exchange:
    """Collectives of the partitioned hop; hosts ``ranks`` of a ``world``."""

    world: int
    ranks: list

    def all_to_all(self, sends):  # [(int64 tensor, counts[world])] -> [int64 tensor]
        raise NotImplementedError

    def sum_(self, tensors) -> None:  # in place, over ranks
        raise NotImplementedError

    def all_gather(self, sends):  # [(int64 tensor, counts)] -> [concat of all ranks' tensors]
        raise NotImplementedError

    def sum_int(self, values) -> int:  # sum of one int per hosted rank over all ranks
        raise NotImplementedError

    def any(self, flags) -> bool:
        raise NotImplementedError

    def gather(self, objs) -> list:  # one object per hosted rank -> all ranks', rank order
        raise NotImplementedError


class LoopbackExchange(Exchange):
    """Every rank of the world in this process (single-device testing)."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))
        self.bytes_sent = 0

    def all_to_all(self, sends):
        import torch

        G = self.world
        offs = [np.concatenate([[0], np.cumsum(c)]).astype(np.int64) for _, c in sends]
        out = []
        for d in range(G):
            parts = [t[int(o[d]): int(o[d + 1])] for (t, _), o in zip(sends, offs)]
            out.append(torch.cat(parts) if parts else sends[0][0][:0])
        self.bytes_sent += 8 * sum(int(sum(c)) for _, c in sends)
        return out

    def all_gather(self, sends):
        import torch

        parts = [t[: int(c[0])] if len(c) else t[:0] for t, c in sends]
        full = torch.cat(parts) if parts else sends[0][0][:0]
        self.bytes_sent += 8 * (self.world - 1) * sum(int(p.numel()) for p in parts)
        return [full for _ in sends]

    def sum_int(self, values):
        return int(sum(int(v) for v in values))

    def sum_(self, tensors):
        if len(tensors) <= 1:
            return
        total = tensors[0].clone()
        for t in tensors[1:]:
            total += t
        for t in tensors:
            t.copy_(total)

    def any(self, flags):
        return bool(any(flags))

    def gather(self, objs):
        return list(objs)


class DistExchange(Exchange):
    """One rank per process over torch.distributed.

    NCCL moves device buffers directly (the B200 path).  With gloo (CPU
    tests, or several ranks sharing one GPU in a functional test, where
    NCCL refuses duplicate devices) device tensors are staged through host
    memory, so no rank's kernels ever wait on another rank's.
    """

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]
        self.bytes_sent = 0
        self.staged = dist.get_backend(group) != "nccl"

    def _host(self, t):
        return t.cpu() if (self.staged and t.is_cuda) else t

    def all_to_all(self, sends):
        import torch

        (send, counts), = sends
        dev = send.device
        cdev = "cpu" if self.staged else dev
        cnt = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=cdev)
        rcnt = torch.empty_like(cnt)
        self.dist.all_to_all_single(rcnt, cnt, group=self.group)
        rc = [int(x) for x in rcnt.tolist()]
        n = int(sum(counts))
        src = self._host(send[:n].contiguous())
        recv = torch.empty(sum(rc), dtype=torch.int64, device=src.device)
        self.dist.all_to_all_single(recv, src, output_split_sizes=rc,
                                    input_split_sizes=[int(c) for c in counts], group=self.group)
        self.bytes_sent += 8 * (n - int(counts[self.ranks[0]]))
        return [recv.to(dev) if recv.device != dev else recv]

    def all_gather(self, sends):
        import torch

        (send, counts), = sends
        dev = send.device
        n = int(counts[0]) if len(counts) else 0
        cdev = "cpu" if self.staged else dev
        sizes = [torch.zeros(1, dtype=torch.int64, device=cdev) for _ in range(self.world)]
        self.dist.all_gather(sizes, torch.tensor([n], dtype=torch.int64, device=cdev), group=self.group)
        sizes = [int(x.item()) for x in sizes]
        m = max(sizes) if sizes else 0
        src = self._host(send[:n])
        padded = torch.zeros(max(m, 1), dtype=torch.int64, device=src.device)
        padded[:n] = src
        out = torch.empty(self.world * max(m, 1), dtype=torch.int64, device=src.device)
        self.dist.all_gather_into_tensor(out, padded, group=self.group)
        parts = [out[r * max(m, 1): r * max(m, 1) + sizes[r]] for r in range(self.world)]
        full = torch.cat(parts)
        self.bytes_sent += 8 * n * (self.world - 1)
        return [full.to(dev) if full.device != dev else full]

    def sum_int(self, values):
        import torch

        (v,) = values
        t = torch.tensor([int(v)], dtype=torch.int64, device="cpu" if self.staged else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return int(t.item())

    def sum_(self, tensors):
        (t,) = tensors
        h = self._host(t)
        self.dist.all_reduce(h, op=self.dist.ReduceOp.SUM, group=self.group)
        if h is not t:
            t.copy_(h)

    def any(self, flags):
        import torch

        (f,) = flags
        dev = "cpu" if self.staged else "cuda"
        t = torch.tensor([1 if f else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def gather(self, objs):
        (o,) = objs
        out = [None] * self.world
        self.dist.all_gather_object(out, o, group=self.group)
        return out


# --------------------------------------------------------------- device shard


class GraphShard:
    """One rank's device shard (th_shard): owned out-rows + hub slices."""

    def __init__(self, cols, n_entities: int, n_relations: int, plan: ShardPlan, rank: int,
                 stream=None):
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
            l2g.data_ptr() if l2g.numel() else None, l2g.numel(), rank, plan.world,
            ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)))
        self._handle = h.value
        self._finalizer = weakref.finalize(self, lib.th_shard_destroy, self._handle)
        self.local_triples = int(lib.th_shard_local_triples(self._handle))
        self.can_pull = bool(lib.th_shard_can_pull(self._handle))
        self._keep = None

    def launch_count(self) -> int:
        return int(_lib.load().th_shard_launch_count(self._handle))

    # -- the wave steps (ShardRunner protocol) ------------------------------
    def begin(self, query: "WaveQuery") -> None:
        import torch

        q = _lib.Query()
        B = query.n_queries
        self._dev = {
            "offs": torch.from_numpy(query.seed_offsets).to(self.device),
            "seeds": torch.from_numpy(query.seeds).to(self.device),
            "masks": None if query.masks is None else torch.from_numpy(query.masks.view(np.int32)).to(self.device),
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
        _lib.check(_lib.load().th_shard_begin(self._handle, ctypes.byref(q)))

    def frontier_cost(self, hop: int) -> int:
        """This rank's frontier out-edge total (direction choice)."""
        c = ctypes.c_int64()
        _lib.check(_lib.load().th_shard_plan(self._handle, hop, ctypes.byref(c)))
        return int(c.value)

    def expand(self, hop: int, mode: int = 0):
        counts = (ctypes.c_int64 * self.plan.world)()
        ptr = ctypes.c_void_p()
        _lib.check(_lib.load().th_shard_expand(self._handle, hop, mode, counts, ctypes.byref(ptr)))
        cnt = [int(c) for c in counts]
        n = sum(cnt)
        send = _lib.as_tensor(ptr.value, (n,), "<i8", owner=self)
        return send, cnt

    def absorb(self, hop: int, recv) -> None:
        self._keep = recv  # must outlive the asynchronous kernel
        _lib.check(_lib.load().th_shard_absorb(self._handle, hop, recv.data_ptr() if recv.numel() else None,
                                               int(recv.numel())))

    def hub_rows(self, hop: int):
        ptr = ctypes.c_void_p()
        words = ctypes.c_int64()
        _lib.check(_lib.load().th_shard_hub_rows(self._handle, hop, ctypes.byref(ptr), ctypes.byref(words)))
        return _lib.as_tensor(ptr.value, (int(words.value),), "<i4", owner=self)

    def hub_merge(self, hop: int) -> None:
        _lib.check(_lib.load().th_shard_hub_merge(self._handle, hop))

    def end_hop(self, hop: int) -> None:
        _lib.check(_lib.load().th_shard_end_hop(self._handle, hop))

    def finish(self):
        """-> ("ok", ShardResult) or ("overflow", None)."""
        res = _lib.Result()
        rc = _lib.load().th_shard_finish(self._handle, ctypes.byref(res))
        if rc == _lib.TH_ERR_OVERFLOW:
            return "overflow", None
        _lib.check(rc)
        return "ok", self._host_result(res)

    def _host_result(self, res) -> "ShardResult":
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

    def _to_host(self, r: "ShardResult") -> "ShardResult":
        return r.to_host()


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
    partial edge counts (CSR per (hop, query)); device tensors from a CUDA
    shard until ``to_host``."""

    n_queries: int
    k: int
    edges: np.ndarray = None
    f_off: np.ndarray = None
    f_len: np.ndarray = None
    f_ids: np.ndarray = None
    a_off: np.ndarray = None
    a_len: np.ndarray = None
    a_ids: np.ndarray = None

    def to_host(self) -> "ShardResult":
        conv = lambda x: x if x is None or isinstance(x, np.ndarray) else x.cpu().numpy()  # noqa: E731
        return ShardResult(self.n_queries, self.k, *(conv(getattr(self, f)) for f in
                                                      ("edges", "f_off", "f_len", "f_ids", "a_off", "a_len",
                                                       "a_ids")))


PULL_DIVISOR = 8.0  # pull when the frontier's out-edges exceed T / 8 (as K2/K3)


def run_wave(shards, xch: Exchange, query: WaveQuery, stats: dict | None = None,
             n_triples: int | None = None, pull_divisor: float = PULL_DIVISOR):
    """Drive one wave through every hosted shard (Algorithm 1 per hop).

    Per hop the ranks agree on a direction: push (candidate records to
    their owners, all-to-all) or, for dense frontiers, pull (every rank's
    owned frontier rows all-gathered, each owner pulls over its in-edges).
    Returns the hosted shards' ShardResults.  An output overflow on any
    rank makes every rank run the wave again with grown capacities.
    """
    can_pull = n_triples is not None and pull_divisor > 0 and all(
        getattr(sh, "can_pull", False) for sh in shards)
    for _attempt in range(4):
        for sh in shards:
            sh.begin(query)
        for h in range(1, query.k + 1):
            mode = 0
            if can_pull:
                cost = xch.sum_int([sh.frontier_cost(h) for sh in shards])
                mode = 1 if cost * pull_divisor > n_triples else 0
            sends = [sh.expand(h, mode) if mode else sh.expand(h) for sh in shards]
            if stats is not None:
                stats.setdefault("records", []).append(sum(sum(c) for _, c in sends))
                stats.setdefault("modes", []).append(mode)
            recvs = xch.all_gather(sends) if mode else xch.all_to_all(sends)
            for sh, rv in zip(shards, recvs):
                sh.absorb(h, rv)
            if h < query.k:  # the last layer is never expanded
                rows = [sh.hub_rows(h) for sh in shards]
                xch.sum_(rows)
                for sh in shards:
                    sh.hub_merge(h)
            for sh in shards:
                sh.end_hop(h)
        done = [sh.finish() for sh in shards]
        if not xch.any([st == "overflow" for st, _ in done]):
            return [r for _, r in done]
    raise RuntimeError("partitioned wave kept overflowing its result buffers")


def merge_results(parts, n_queries: int, k: int, activated: bool):
    """Per (hop, query): concatenate the ranks' sorted slices and sort.
    Owners are disjoint, so the union is duplicate-free."""

    def merge(name_off, name_len, name_ids):
        keys, ids = [], []
        for p in parts:
            off, ln, data = getattr(p, name_off), getattr(p, name_len), getattr(p, name_ids)
            flat_len = ln.reshape(-1)
            key = np.repeat(np.arange(flat_len.size, dtype=np.int64), flat_len)
            idx = np.concatenate([np.arange(o, o + n, dtype=np.int64)
                                  for o, n in zip(off.reshape(-1), flat_len)]) if key.size else \
                np.empty(0, np.int64)
            keys.append(key)
            ids.append(data[idx].astype(np.int64))
        key = np.concatenate(keys) if keys else np.empty(0, np.int64)
        val = np.concatenate(ids) if ids else np.empty(0, np.int64)
        order = np.lexsort((val, key))
        val = val[order]
        cnt = np.bincount(key, minlength=k * n_queries).reshape(k, n_queries)
        off = np.concatenate([[0], np.cumsum(cnt.reshape(-1))[:-1]]).reshape(k, n_queries)
        return off, cnt, val

    out = {"edges": sum(p.edges for p in parts)}
    out["f_off"], out["f_len"], out["f_ids"] = merge("f_off", "f_len", "f_ids")
    if activated:
        out["a_off"], out["a_len"], out["a_ids"] = merge("a_off", "a_len", "a_ids")
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
                 n_hubs: int | None = None, shard_factory=None):
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
        # host copy of the columns: cross_graph_paths gathers the (s, r, o)
        # of a query's activated triples from it (the reference keeps its
        # shards on disk and maps tids through tid_to_global the same way)
        self._cols = tuple(np.asarray(c.cpu().numpy() if hasattr(c, "cpu") else c, dtype=np.int32)
                           for c in cols)
        self.pull_divisor = PULL_DIVISOR  # 0 = push only
        factory = shard_factory or GraphShard
        self.shards = [factory(cols, n_entities, n_relations, plan, r) for r in exchange.ranks]

    def run(self, query: WaveQuery, stats: dict | None = None):
        """One wave; the hosted ranks' partial results (kept sharded)."""
        return run_wave(self.shards, self.exchange, query, stats, self.n_triples, self.pull_divisor)

    def retrieve(self, seeds, k: int, relation_filter=None, semantics="frontier",
                 activated: bool = False):
        """Per-seed retrieval (one query per seed), merged on every rank.

        Returns a host ``RetrievalResult`` with the same accessors as the
        single-GPU engine (frontier(i, h), activated(i, h), edges)."""
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
            parts = self.exchange.gather([r.to_host() for r in self.run(wq)])
            m = merge_results(parts, nq, k, activated)
            merged["edges"].append(m["edges"])
            merged["f_off"].append(m["f_off"] + fbase)
            merged["f_len"].append(m["f_len"])
            merged["f_ids"].append(m["f_ids"])
            fbase += m["f_ids"].size
            if activated:
                merged["a_off"].append(m["a_off"] + abase)
                merged["a_len"].append(m["a_len"])
                merged["a_ids"].append(m["a_ids"])
                abase += m["a_ids"].size
            if B == 0:
                break
        cat = lambda xs, axis=1: torch.from_numpy(np.concatenate(xs, axis=axis))  # noqa: E731
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
    parts = pg.exchange.gather([r.to_host() for r in pg.run(wq)])
    m = merge_results(parts, 1, k, True)
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

    Every step of a walk is a triple activated at its hop under exact-walk
    semantics, so the walks of the full graph are exactly the walks of the
    subgraph of activated triples.  The partitioned exact-walk trace
    supplies those triples; their subgraph (local tids a monotone renumbering
    of the global ones, the reference's tid_to_global idea,
    partition.py:145-153) is enumerated by the device path kernel (K5) and
    mapped back -- identical paths, order and truncation flag.
    """
    from .core_types import PathResult
    from .device_graph import build_incidence
    from .retriever import reconstruct_paths

    if getattr(pg, "store", None) is not None:
        from .store import store_paths

        return store_paths(q0, k, pg, max_paths)
    if q0.width != pg.n_entities:
        raise ValueError(f"query width {q0.width} != graph entity count {pg.n_entities}")
    if k < 1:
        raise ValueError("hop count must be >= 1")
    if max_paths is not None and max_paths < 0:
        raise ValueError("max_paths must be >= 0")
    tr = cross_graph_k_hop(q0, k, pg, HopSemantics.EXACT_WALK)
    act = [tr.activated(h).ids for h in range(1, k + 1)]
    tids = np.unique(np.concatenate(act)) if act else np.empty(0, np.int64)
    s, r, o = (c[tids] for c in pg._cols)
    sub = build_incidence((s, r, o), pg.n_entities, pg.n_relations)
    res = reconstruct_paths(q0, k, sub, max_paths)
    # entity and relation ids are global in the subgraph, so its Triples are
    # the full graph's
    return PathResult(res.paths, res.truncated)
