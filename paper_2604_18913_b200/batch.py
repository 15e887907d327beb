"""Batches of seed-set queries run in a cache-friendly order (SURVEY 8f row
4; the role of the reference's ``plan_batch`` / ``run_batch``,
engine.py:186-258, with the same observable order and error isolation).

* A query's signature is the sorted tuple of partitions its seeds route to
  (``route``; hop 0 only -- deeper footprints are unknown before running).
* ``plan_batch`` runs queries grouped by signature, the groups in ascending
  signature order and input order inside a group, so queries needing the
  same subgraphs run back to back and find them resident in the LRU.
* ``run_batch`` executes that order and reports in input order; a failing
  query is reported under its id and never aborts the others.

Store-backed graphs run query by query (the LRU's access sequence is the
point of the ordering).  On a rank-sharded ``PartitionedGraph`` the order
has no cache to serve, so queries of equal hop count are packed into device
waves of up to 1,024 seed sets (one bit lane per query, ``WaveQuery``) and
each wave's merged result is split into per-query traces.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core_types import EntityVector, HopSemantics, HopStep, HopTrace, TripleVector
from .partition import MAX_WAVE, PartitionPlan, WaveQuery, cross_graph_k_hop, route


@dataclass(frozen=True)
class BatchQuery:
    query_id: object
    q0: EntityVector
    k: int


@dataclass(frozen=True)
class QueryBatch:
    """The queries and the order they run in (a permutation of positions)."""

    queries: list
    execution_order: list = field(default_factory=list)

    @property
    def restore_order(self) -> list:
        """restore_order[pos] = the run step at which query pos executes."""
        inv = np.empty(len(self.execution_order), dtype=np.int64)
        inv[np.asarray(self.execution_order, dtype=np.int64)] = np.arange(len(self.execution_order))
        return inv.tolist()

    @classmethod
    def identity(cls, queries) -> "QueryBatch":
        return cls(list(queries), list(range(len(queries))))


@dataclass
class BatchResult:
    query_id: object
    trace: HopTrace | None
    error: str | None = None


def signature(q0: EntityVector, plan: PartitionPlan) -> tuple:
    """Partitions q0's seeds route to, ascending (the sink excluded)."""
    return tuple(sorted(route(q0, plan).buckets))


def plan_batch(queries, plan: PartitionPlan) -> QueryBatch:
    """Order queries by signature; Python's sort is stable, so queries with
    equal signatures keep their input order."""
    queries = list(queries)
    keys = [signature(q.q0, plan) for q in queries]
    return QueryBatch(queries, sorted(range(len(queries)), key=keys.__getitem__))


def _failure(exc: Exception) -> str:
    return f"{type(exc).__name__}: {exc}"


def run_batch(batch: QueryBatch, pg, semantics=HopSemantics.FRONTIER) -> list:
    """Run ``batch`` in its planned order; results come back in input order."""
    sem = HopSemantics.parse(semantics)
    results: list = [None] * len(batch.queries)
    if getattr(pg, "store", None) is not None:
        for pos in batch.execution_order:
            q = batch.queries[pos]
            try:
                results[pos] = BatchResult(q.query_id, cross_graph_k_hop(q.q0, q.k, pg, sem))
            except Exception as exc:  # noqa: BLE001 - one query's failure is its own
                results[pos] = BatchResult(q.query_id, None, _failure(exc))
        return results
    # rank-sharded graph: waves of equal-k queries, in planned order
    by_k: dict = {}
    for pos in batch.execution_order:
        q = batch.queries[pos]
        if q.q0.width != pg.n_entities:
            results[pos] = BatchResult(q.query_id, None, _failure(ValueError(
                f"query width {q.q0.width} != graph entity count {pg.n_entities}")))
        elif q.k < 1:
            results[pos] = BatchResult(q.query_id, None, _failure(ValueError("hop count must be >= 1")))
        else:
            by_k.setdefault(int(q.k), []).append(pos)
    for k, positions in by_k.items():
        for w0 in range(0, len(positions), MAX_WAVE):
            wave = positions[w0:w0 + MAX_WAVE]
            try:
                traces = _wave_traces(pg, [batch.queries[p].q0 for p in wave], k, sem)
            except Exception as exc:  # noqa: BLE001 - the wave's queries share the failure
                for p in wave:
                    results[p] = BatchResult(batch.queries[p].query_id, None, _failure(exc))
                continue
            for p, tr in zip(wave, traces):
                results[p] = BatchResult(batch.queries[p].query_id, tr)
    return results


def _wave_traces(pg, seed_sets, k: int, sem: HopSemantics) -> list:
    """One device wave over up to 1,024 seed sets -> one HopTrace each."""
    lens = np.array([q.ids.size for q in seed_sets], dtype=np.int64)
    offs = np.zeros(lens.size + 1, dtype=np.int32)
    np.cumsum(lens, out=offs[1:])
    ids = (np.concatenate([q.ids for q in seed_sets]) if lens.sum() else np.empty(0)).astype(np.int32)
    m = {n: (v.cpu().numpy() if v is not None else None)
         for n, v in pg.merged(WaveQuery(offs, ids, k, sem, None, True)).items()}
    out = []
    for i, q0 in enumerate(seed_sets):
        steps = []
        for h in range(k):
            fo, fl = int(m["f_off"][h, i]), int(m["f_len"][h, i])
            ao, al = int(m["a_off"][h, i]), int(m["a_len"][h, i])
            steps.append(HopStep(EntityVector(m["f_ids"][fo:fo + fl], pg.n_entities, _canonical=True),
                                 TripleVector(m["a_ids"][ao:ao + al], pg.n_triples, _canonical=True)))
        out.append(HopTrace(sem, q0, steps))
    return out
