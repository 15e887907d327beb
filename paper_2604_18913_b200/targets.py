"""Benchmark-target adapters.

The reference's harness drives any object with ``kind``, ``n_entities``,
``n_triples``, ``cache``, ``expand(frontier)`` and ``triples()``
(bench.py:98-137, ``SingleGraphTarget`` / ``PartitionedTarget``) through its
``ExpandFn`` seam (incidence.py:265).  These targets answer ``expand`` with
one device hop (exact-walk, k=1 -- the reference's ``_expand``,
incidence.py:214-221): (activated triple ids, reached entity ids), both
sorted int64.  A per-frontier callback costs a host round trip per hop;
the batched ``retrieve`` is the fast path.
"""

from __future__ import annotations

import numpy as np

from .core_types import EntityVector, HopSemantics, Triple


class GpuTarget:
    kind = "gpu"

    def __init__(self, graph):
        self.graph = graph
        self.n_entities = graph.n_entities
        self.n_triples = graph.n_triples
        self.cache = None

    def expand(self, frontier):
        ids = np.asarray(frontier, dtype=np.int64).reshape(-1)
        q = EntityVector(ids, self.n_entities)
        tr = self.graph.retriever().k_hop(q, 1, HopSemantics.EXACT_WALK)
        return tr.activated(1).ids, tr.frontier(1).ids

    def triples(self) -> list:
        g = self.graph
        return [Triple(*t) for t in zip(g.subj.tolist(), g.rel.tolist(), g.obj.tolist())]


class PartitionedGpuTarget:
    kind = "gpu-partitioned"

    def __init__(self, pg, triples_cols=None):
        self.pg = pg
        self.n_entities = pg.n_entities
        self.n_triples = pg.n_triples
        self.cache = None
        self._cols = triples_cols

    def expand(self, frontier):
        from .partition import cross_graph_k_hop

        q = EntityVector(np.asarray(frontier, dtype=np.int64).reshape(-1), self.n_entities)
        tr = cross_graph_k_hop(q, 1, self.pg, HopSemantics.EXACT_WALK)
        return tr.activated(1).ids, tr.frontier(1).ids

    def triples(self) -> list:
        if self._cols is None:
            raise ValueError("PartitionedGpuTarget was built without the triple columns")
        s, r, o = (np.asarray(c) for c in self._cols)
        return [Triple(*t) for t in zip(s.tolist(), r.tolist(), o.tolist())]
