"""CPU oracle for the k-hop retrieval hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
(``paper_2604_18913_b200``) never imports it and has no CPU fallback.

It restates, in numpy, the algorithm of the reference ``triplehop``
package (``/root/reference/pkg/src/triplehop``).  Citations are
``file:line`` relative to that directory:

* CSR build ............ ``incidence.py:154-196``  -> :func:`build_csr`
* row gather ........... ``incidence.py:199-211``  -> :func:`_concat_rows`
* one raw hop .......... ``incidence.py:214-221``  -> :func:`raw_hop`
* dense/sparse dedupe .. ``incidence.py:29-31,41-49`` -> :func:`_dedupe`
* semantics driver ..... ``incidence.py:268-316``  -> :func:`hop_trace`
* path enumeration ..... ``incidence.py:344-408``  -> :func:`walk_paths`
* relation filter ...... (absent in the reference; SURVEY.md section 8c
  restatement built from ``build_incidence`` + the ``tid_to_global``
  idea of ``partition.py:145-153``) -> :func:`filtered_view`
* partition plans ...... ``partition.py:49-98``    -> :func:`plan_owner`

The restatement keeps the reference's cost structure (numpy gathers,
``np.sort``, ``np.unique`` / dense mask switch, a fresh ``visited`` array
per query) so that timing it is a fair stand-in for the reference CPU
path.  Parity is pinned by ``tests/golden/`` (vectors produced by the real
reference through ``tests/golden/make_golden.py``).
"""

from __future__ import annotations

from dataclasses import dataclass
from itertools import islice
from typing import Iterator

import numpy as np

# Reference switch point: dense bitmask dedupe once ids >= width/32
# (incidence.py:29-31).
DENSE_SWITCH = 32
DEFAULT_MAX_PATHS = 10_000  # incidence.py:33

EXACT, FRONTIER, CUMULATIVE = "exact", "frontier", "cumulative"


@dataclass(frozen=True)
class OracleGraph:
    """Host CSR mirror of ``IncidenceGraph`` (incidence.py:121-151)."""

    indptr: np.ndarray  # int64[E+1]
    tids: np.ndarray  # int64[T], ascending inside each row
    subj: np.ndarray  # int64[T] in triple-id order
    rel: np.ndarray  # int64[T]
    obj: np.ndarray  # int64[T]
    n_entities: int
    n_relations: int

    @property
    def n_triples(self) -> int:
        return int(self.obj.size)

    def row(self, e: int) -> np.ndarray:
        return self.tids[self.indptr[e] : self.indptr[e + 1]]


def build_csr(subj, rel, obj, n_entities: int, n_relations: int) -> OracleGraph:
    """Counting-sort CSR build (incidence.py:154-196).

    Row lengths come from a bincount of subjects; a *stable* argsort by
    subject lays rows out in entity order while keeping triple ids
    ascending within a row.  Out-of-range ids raise ``ValueError``
    (incidence.py:175-179).
    """
    s = np.asarray(subj, dtype=np.int64).reshape(-1)
    r = np.asarray(rel, dtype=np.int64).reshape(-1)
    o = np.asarray(obj, dtype=np.int64).reshape(-1)
    if not (s.size == r.size == o.size):
        raise ValueError("subject/relation/object columns differ in length")
    for label, col, hi in (("subject", s, n_entities), ("relation", r, n_relations),
                           ("object", o, n_entities)):
        if col.size and (int(col.min()) < 0 or int(col.max()) >= hi):
            raise ValueError(f"{label} id out of range (bound {hi})")
    counts = np.bincount(s, minlength=n_entities) if s.size else np.zeros(n_entities, np.int64)
    indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    tids = np.argsort(s, kind="stable").astype(np.int64)
    return OracleGraph(indptr, tids, s.copy(), r.copy(), o.copy(), int(n_entities), int(n_relations))


def _dedupe(ids: np.ndarray, width: int) -> np.ndarray:
    """Sorted unique ids; dense mask path when len >= width/32 (incidence.py:41-49)."""
    if ids.size == 0:
        return np.empty(0, dtype=np.int64)
    if width > 0 and ids.size >= width // DENSE_SWITCH:
        hit = np.zeros(width, dtype=bool)
        hit[ids] = True
        return np.flatnonzero(hit).astype(np.int64)
    return np.unique(ids)


def _concat_rows(indptr: np.ndarray, data: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """All CSR rows of ``rows`` back to back (incidence.py:199-211)."""
    if rows.size == 0:
        return np.empty(0, dtype=data.dtype)
    lo = indptr[rows]
    n = indptr[rows + 1] - lo
    total = int(n.sum())
    if total == 0:
        return np.empty(0, dtype=data.dtype)
    seg_start = np.cumsum(n) - n
    idx = np.repeat(lo - seg_start, n) + np.arange(total, dtype=np.int64)
    return data[idx]


def raw_hop(g: OracleGraph, frontier: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """One boolean hop: (sorted activated tids, sorted unique objects).

    incidence.py:214-221.  Triple ids are unique across rows, so sorting
    the gathered ids canonicalises the activated set.
    """
    act = np.sort(_concat_rows(g.indptr, g.tids, np.asarray(frontier, dtype=np.int64)))
    return act, _dedupe(g.obj[act], g.n_entities)


def canonical_ids(ids, width: int) -> np.ndarray:
    """EntityVector canonical form: sorted, unique, range-checked (incidence.py:83-91)."""
    arr = np.asarray(ids if isinstance(ids, np.ndarray) else list(ids), dtype=np.int64).reshape(-1)
    # range check before the dense-mask dedupe (which would IndexError)
    if arr.size and (int(arr.min()) < 0 or int(arr.max()) >= width):
        raise ValueError(f"id out of range for width {width}")
    return _dedupe(arr, width)


def hop_trace(g: OracleGraph, seeds, k: int, semantics: str = FRONTIER):
    """k-hop trace: list of (frontier ids, activated tids) per hop.

    Semantics driver of incidence.py:268-316:
      exact      -- frontier_h = objects of rows(frontier_{h-1});
      frontier   -- new entities only; a per-query ``visited`` mask starts
                    with the seeds (seeds never reappear);
      cumulative -- sorted union of the frontier layers, still expanding
                    from the newest layer only (incidence.py:309-315).
    """
    if k < 1:
        raise ValueError("hop count must be >= 1")
    q0 = canonical_ids(seeds, g.n_entities)
    out = []
    if semantics == EXACT:
        cur = q0
        for _ in range(k):
            act, cur = raw_hop(g, cur)
            out.append((cur, act))
        return out
    if semantics not in (FRONTIER, CUMULATIVE):
        raise ValueError(f"unknown hop semantics {semantics!r}")
    seen = np.zeros(g.n_entities, dtype=bool)
    seen[q0] = True
    acc = np.empty(0, dtype=np.int64)
    cur = q0
    for _ in range(k):
        act, reached = raw_hop(g, cur)
        fresh = reached[~seen[reached]]
        seen[fresh] = True
        if semantics == CUMULATIVE:
            acc = np.sort(np.concatenate([acc, fresh]))
            out.append((acc, act))
        else:
            out.append((fresh, act))
        cur = fresh
    return out


# --- paths (incidence.py:333-408) ------------------------------------------


def walk_paths(g: OracleGraph, seeds, k: int, max_paths: int | None = DEFAULT_MAX_PATHS):
    """Length-k walks from the seed set, lexicographic in the tid sequence.

    Mirrors reconstruct_paths (incidence.py:391-408): run the exact-walk
    trace, group each hop's activated triples by subject in tid order
    (HopAdjacency, incidence.py:344-358), then a depth-first enumeration
    capped at ``max_paths`` with a truncation flag (incidence.py:361-388).
    Returns (list of tid tuples, truncated).
    """
    trace = hop_trace(g, seeds, k, EXACT)
    levels = []
    for _, act in trace:
        first = act.tolist()  # activated tids are sorted already
        by_subj: dict[int, list[int]] = {}
        for t, s in zip(first, g.subj[act].tolist()):
            by_subj.setdefault(s, []).append(t)
        levels.append((first, by_subj))
    obj = g.obj

    def dfs(depth: int, tail: int, prefix: list[int]) -> Iterator[tuple[int, ...]]:
        if depth == k:
            yield tuple(prefix)
            return
        first, by_subj = levels[depth]
        for t in (first if depth == 0 else by_subj.get(tail, ())):
            prefix.append(t)
            yield from dfs(depth + 1, int(obj[t]), prefix)
            prefix.pop()

    gen = dfs(0, -1, [])
    if max_paths is None:
        return list(gen), False
    if max_paths < 0:
        raise ValueError("max_paths must be >= 0")
    got = list(islice(gen, max_paths + 1))
    return got[:max_paths], len(got) > max_paths


def paths_as_triples(g: OracleGraph, paths):
    return [tuple((int(g.subj[t]), int(g.rel[t]), int(g.obj[t])) for t in p) for p in paths]


# --- relation filter restatement -----------------------------


def filtered_view(g: OracleGraph, allowed_relations) -> tuple[OracleGraph, np.ndarray]:
    """Graph over the triples whose relation is allowed, plus local->global tids.

    Entity and relation ids are unchanged and local tids are a monotone
    renumbering of the kept global tids, so sorted activated sets and the
    lexicographic path order carry over (same mechanism as the
    reference's ``tid_to_global``, partition.py:145-153).
    """
    allow = np.zeros(g.n_relations, dtype=bool)
    allow[np.asarray(list(allowed_relations), dtype=np.int64)] = True
    keep = allow[g.rel]
    local_to_global = np.flatnonzero(keep).astype(np.int64)
    sub = build_csr(g.subj[keep], g.rel[keep], g.obj[keep], g.n_entities, g.n_relations)
    return sub, local_to_global


def mask_words_to_relations(words, n_relations: int) -> np.ndarray:
    """Relation ids set in a little-endian u32 bitmask (bit r of word r//32)."""
    w = np.asarray(words, dtype=np.uint32).reshape(-1)
    bits = ((w[:, None] >> np.arange(32, dtype=np.uint32)[None, :]) & 1).astype(bool).reshape(-1)
    return np.flatnonzero(bits[:n_relations])


def retrieve_one(g: OracleGraph, seed: int, k: int, semantics: str = FRONTIER,
                 allowed_relations=None, paths: bool = False,
                 max_paths: int | None = DEFAULT_MAX_PATHS):
    """Per-seed retrieval contract of SURVEY.md section 8a (single seed).

    Returns dict(frontiers=[ids per hop], activated=[global tids per hop],
    edges=[|T_h| per hop], paths=[global tid tuples] | None, truncated).
    """
    view, l2g = (g, None) if allowed_relations is None else filtered_view(g, allowed_relations)
    trace = hop_trace(view, [seed], k, semantics)
    acts = [a if l2g is None else l2g[a] for _, a in trace]
    res = {
        "frontiers": [f for f, _ in trace],
        "activated": acts,
        "edges": [int(a.size) for a in acts],
        "paths": None,
        "truncated": False,
    }
    if paths:
        p, trunc = walk_paths(view, [seed], k, max_paths)
        if l2g is not None:
            p = [tuple(int(l2g[t]) for t in path) for path in p]
        res["paths"], res["truncated"] = p, trunc
    return res


# --- partition plans (partition.py:49-98) ------------------------------------


def plan_owner(subj: np.ndarray, n_entities: int, m: int, strategy: str = "lpt") -> np.ndarray:
    """Subject -> partition assignment; -1 for entities with no out-edges."""
    import heapq

    deg = np.bincount(np.asarray(subj, dtype=np.int64), minlength=n_entities)
    subjects = np.flatnonzero(deg)
    if m < 1 or m > subjects.size:
        raise ValueError("bad partition count")
    out = np.full(n_entities, -1, dtype=np.int64)
    if strategy == "hash":
        out[subjects] = ((subjects * 0x9E3779B1) & 0xFFFFFFFF) % m
        return out
    order = np.lexsort((subjects, -deg[subjects]))
    heap = [(0, p) for p in range(m)]
    for e in subjects[order].tolist():
        load, p = heapq.heappop(heap)
        out[e] = p
        heapq.heappush(heap, (load + int(deg[e]), p))
    return out
