"""Pack / unpack golden parity cases (graph + queries + reference results).

A case file (``*.npz``) holds one graph and a list of queries, each with
the results the *reference* ``triplehop`` produced for it (see
``make_golden.py``).  Ragged lists are stored as (offsets, values) pairs.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

SEM_CODES = {"exact": 0, "frontier": 1, "cumulative": 2}
SEM_NAMES = {v: k for k, v in SEM_CODES.items()}
HERE = Path(__file__).resolve().parent


@dataclass
class GoldenQuery:
    seeds: list[int]
    k: int
    semantics: str
    relations: list[int] | None  # allowed relation ids, None = no filter
    max_paths: int | None  # None = uncapped; -2 = paths not requested
    frontiers: list[np.ndarray] = field(default_factory=list)
    activated: list[np.ndarray] = field(default_factory=list)
    paths: list[tuple[int, ...]] | None = None
    truncated: bool = False

    @property
    def want_paths(self) -> bool:
        return self.max_paths != -2


@dataclass
class GoldenCase:
    name: str
    subj: np.ndarray
    rel: np.ndarray
    obj: np.ndarray
    n_entities: int
    n_relations: int
    queries: list[GoldenQuery]


def _ragged(lists):
    lists = [np.asarray(x, dtype=np.int64).reshape(-1) for x in lists]
    off = np.zeros(len(lists) + 1, dtype=np.int64)
    if lists:
        off[1:] = np.cumsum([x.size for x in lists])
    vals = np.concatenate(lists) if lists else np.empty(0, np.int64)
    return off, vals


def _unragged(off, vals):
    return [vals[off[i] : off[i + 1]] for i in range(off.size - 1)]


def save_case(path: Path, case: GoldenCase) -> None:
    qs = case.queries
    q_off, q_seeds = _ragged([q.seeds for q in qs])
    m_off, m_vals = _ragged([q.relations or [] for q in qs])
    f_off, f_vals = _ragged([f for q in qs for f in q.frontiers])
    a_off, a_vals = _ragged([a for q in qs for a in q.activated])
    flat_paths, path_counts = [], []
    for q in qs:
        ps = q.paths or []
        path_counts.append(len(ps))
        flat_paths.extend(ps)
    p_tids = np.asarray([t for p in flat_paths for t in p], dtype=np.int64)
    np.savez_compressed(
        path,
        name=np.array(case.name),
        subj=case.subj.astype(np.int32),
        rel=case.rel.astype(np.int32),
        obj=case.obj.astype(np.int32),
        dims=np.array([case.n_entities, case.n_relations], dtype=np.int64),
        q_off=q_off, q_seeds=q_seeds,
        q_k=np.array([q.k for q in qs], dtype=np.int64),
        q_sem=np.array([SEM_CODES[q.semantics] for q in qs], dtype=np.int64),
        q_hasmask=np.array([q.relations is not None for q in qs], dtype=bool),
        m_off=m_off, m_vals=m_vals,
        q_maxp=np.array([-1 if q.max_paths is None else q.max_paths for q in qs], dtype=np.int64),
        f_off=f_off, f_vals=f_vals, a_off=a_off, a_vals=a_vals,
        p_count=np.array(path_counts, dtype=np.int64), p_tids=p_tids,
        p_trunc=np.array([q.truncated for q in qs], dtype=bool),
    )


def load_case(path) -> GoldenCase:
    z = np.load(path)
    seeds = _unragged(z["q_off"], z["q_seeds"])
    masks = _unragged(z["m_off"], z["m_vals"])
    fr = _unragged(z["f_off"], z["f_vals"])
    ac = _unragged(z["a_off"], z["a_vals"])
    qs, hop_i, tid_i = [], 0, 0
    for i in range(seeds.__len__()):
        k = int(z["q_k"][i])
        maxp = int(z["q_maxp"][i])
        q = GoldenQuery(
            seeds=seeds[i].tolist(), k=k, semantics=SEM_NAMES[int(z["q_sem"][i])],
            relations=masks[i].tolist() if z["q_hasmask"][i] else None,
            max_paths=None if maxp == -1 else maxp,
        )
        q.frontiers = fr[hop_i : hop_i + k]
        q.activated = ac[hop_i : hop_i + k]
        hop_i += k
        n = int(z["p_count"][i])
        if q.want_paths:
            flat = z["p_tids"][tid_i : tid_i + n * k].reshape(n, k)
            q.paths = [tuple(int(t) for t in row) for row in flat]
            q.truncated = bool(z["p_trunc"][i])
        tid_i += n * k
        qs.append(q)
    d = z["dims"]
    return GoldenCase(str(z["name"]), z["subj"].astype(np.int64), z["rel"].astype(np.int64),
                      z["obj"].astype(np.int64), int(d[0]), int(d[1]), qs)


def all_cases():
    return sorted(HERE.glob("*.npz"))
