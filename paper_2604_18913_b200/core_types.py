"""Result and id-vector types of the retriever API.

Same names, fields and behaviour as the reference's public types so that a
caller of ``triplehop`` can switch imports:

* ``Triple``                      triples.py:19-22
* ``HopSemantics`` (+ ``parse``)  incidence.py:52-75
* ``EntityVector``/``TripleVector`` (sorted, unique, read-only int64,
  range-checked -> ``ValueError``)  incidence.py:78-118
* ``HopStep``/``HopTrace``        incidence.py:235-262
* ``PathResult``                  incidence.py:338-341
* ``jaccard``                     incidence.py:411-417

These are host-side containers for results the device produced; the only
arithmetic here is canonicalising caller-supplied seed ids.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Iterator, NamedTuple

import numpy as np

DEFAULT_MAX_PATHS = 10_000


class Triple(NamedTuple):
    subject: int
    relation: int
    object: int


class HopSemantics(enum.Enum):
    """EXACT_WALK: reachable by a walk of exactly h steps; FRONTIER: first
    reached at hop h (seeds excluded); CUMULATIVE: union of FRONTIER layers."""

    EXACT_WALK = "exact"
    FRONTIER = "frontier"
    CUMULATIVE = "cumulative"

    @classmethod
    def parse(cls, name) -> "HopSemantics":
        if isinstance(name, HopSemantics):
            return name
        key = str(name).strip().lower()
        if key in ("exact", "exact-walk", "exact_walk", "walk"):
            return cls.EXACT_WALK
        if key == "frontier":
            return cls.FRONTIER
        if key == "cumulative":
            return cls.CUMULATIVE
        raise ValueError(f"unknown hop semantics {name!r}")

    @property
    def code(self) -> int:
        return {"exact": 0, "frontier": 1, "cumulative": 2}[self.value]


def _canonicalise(ids, width: int) -> np.ndarray:
    if isinstance(ids, np.ndarray):
        arr = ids.astype(np.int64, copy=False).reshape(-1)
    else:
        try:
            import torch

            if isinstance(ids, torch.Tensor):
                ids = ids.detach().cpu().numpy()
        except ImportError:  # pragma: no cover
            pass
        arr = np.asarray(ids if isinstance(ids, np.ndarray) else list(ids), dtype=np.int64).reshape(-1)
    if arr.size and (int(arr.min()) < 0 or int(arr.max()) >= width):
        raise ValueError(f"id out of range for width {width}")
    return np.unique(arr)


class _IdVector:
    """Sorted duplicate-free id set over a fixed-width id space."""

    __slots__ = ("ids", "width")

    def __init__(self, ids, width: int, _canonical: bool = False):
        if _canonical:
            arr = np.asarray(ids, dtype=np.int64).reshape(-1)
            if arr.size and (arr[0] < 0 or arr[-1] >= width):
                raise ValueError(f"id out of range for width {width}")
        else:
            arr = _canonicalise(ids, width)
        arr.setflags(write=False)
        self.ids = arr
        self.width = int(width)

    def __len__(self) -> int:
        return int(self.ids.size)

    def __iter__(self) -> Iterator[int]:
        return iter(self.ids.tolist())

    def __eq__(self, other: object) -> bool:
        return (isinstance(other, _IdVector) and self.width == other.width
                and np.array_equal(self.ids, other.ids))

    def __repr__(self) -> str:
        return f"{type(self).__name__}({self.ids.tolist()}, width={self.width})"

    def to_set(self) -> set[int]:
        return set(self.ids.tolist())


class EntityVector(_IdVector):
    """Boolean row vector over the entity space (sparse form)."""


class TripleVector(_IdVector):
    """Boolean row vector over the triple space (sparse form)."""


@dataclass(frozen=True)
class HopStep:
    frontier: EntityVector
    activated: TripleVector


@dataclass(frozen=True)
class HopTrace:
    semantics: HopSemantics
    seeds: EntityVector
    steps: list

    @property
    def k(self) -> int:
        return len(self.steps)

    def frontier(self, hop: int) -> EntityVector:
        """Frontier after ``hop`` hops (1-based)."""
        return self.steps[hop - 1].frontier

    def activated(self, hop: int) -> TripleVector:
        return self.steps[hop - 1].activated

    @property
    def final_frontier(self) -> EntityVector:
        return self.steps[-1].frontier


@dataclass(frozen=True)
class PathResult:
    paths: list
    truncated: bool


def jaccard(a, b) -> float:
    """|a & b| / |a | b|; two empty sets count as identical."""
    sa = a.to_set() if isinstance(a, _IdVector) else set(a)
    sb = b.to_set() if isinstance(b, _IdVector) else set(b)
    if not sa and not sb:
        return 1.0
    return len(sa & sb) / len(sa | sb)
