"""GPU backend behind the reference's ``/query`` endpoint (SURVEY 8f row 3:
``GraphRegistry`` + ``query``, service/app.py:65-85,196-229; request and
response fields of service/models.py:40-76).

The registry keeps every graph it has loaded resident in HBM -- a graph
directory as a device ``IncidenceGraph`` (LKG1 archive decoded and built on
the device) with its label files, a partition directory as a store-backed
``PartitionedGraph`` per cache capacity, whose LRU of device subgraphs keeps
its state (and counters) between requests.  ``answer`` turns one request
into the reference's response body: labels -> ids (unknown labels reported,
never fatal), ``k_hop`` / ``reconstruct_paths`` (or their cross-partition
forms) on the device, ids -> labels.  ``create_app`` mounts it on FastAPI
with the reference's status codes and error payloads (400 usage, 422 data).

Only the query path is served; the reference's build / partition / bench /
verify endpoints are outside the hot path.
"""

from __future__ import annotations

import threading
from pathlib import Path
from typing import Literal, NamedTuple

import numpy as np
from pydantic import BaseModel, Field, model_validator

from .core_types import DEFAULT_MAX_PATHS, EntityVector, HopSemantics
from .errors import DataError, IntegrityError, UsageError

GRAPH_FILE = "graph.lkg"
ENTITIES_FILE = "entities.txt"
RELATIONS_FILE = "relations.txt"


class Labels:
    """Label <-> dense id, ids in first-occurrence order of the label file
    (the reference's dictionary files: line index = id); exported as
    ``Dictionary`` for the reference's name (triples.py:26-60)."""

    def __init__(self, labels=()):
        self._labels = list(dict.fromkeys(labels))
        self._ids = {lab: i for i, lab in enumerate(self._labels)}

    def add(self, label: str) -> int:
        """The id of ``label``, the next free id when it is new."""
        i = self._ids.get(label)
        if i is None:
            i = self._ids[label] = len(self._labels)
            self._labels.append(label)
        return i

    def __len__(self) -> int:
        return len(self._labels)

    def __contains__(self, label) -> bool:
        return label in self._ids

    def __eq__(self, other) -> bool:
        return isinstance(other, Labels) and self._labels == other._labels

    def id_of(self, label: str):
        return self._ids.get(label)

    def label_of(self, idx: int) -> str:
        return self._labels[idx]

    def labels(self) -> list:
        return list(self._labels)


def _labels_file(path: Path) -> Labels:
    from .store import _read_label_lines

    return Labels(_read_label_lines(path))


def load_graph_dir(graph_dir):
    """(device IncidenceGraph, entity Labels, relation Labels) of a graph
    directory the reference wrote (archive.py:175-185)."""
    from .archive import load_graph

    d = Path(graph_dir)
    g = load_graph(d / GRAPH_FILE)
    ents, rels = _labels_file(d / ENTITIES_FILE), _labels_file(d / RELATIONS_FILE)
    if len(ents) != g.n_entities or len(rels) != g.n_relations:
        raise IntegrityError("dictionary sizes disagree with the graph archive")
    return g, ents, rels


class DeviceGraphRegistry:
    """Loaded graphs, memoised by resolved directory (and cache capacity for
    partition directories); loads are serialised, queries are not."""

    def __init__(self):
        self._loaded: dict = {}
        self._lock = threading.Lock()

    def _memo(self, key, load):
        with self._lock:
            if key not in self._loaded:
                self._loaded[key] = load()
            return self._loaded[key]

    def graph(self, graph_dir):
        d = Path(graph_dir).resolve()
        return self._memo(("graph", d), lambda: load_graph_dir(d))

    def partitioned(self, part_dir, capacity: int):
        from .store import open_partitioned

        d = Path(part_dir).resolve()

        def load():
            pg, ents, rels = open_partitioned(d, capacity)
            return pg, Labels(ents), Labels(rels)

        return self._memo(("parts", d, int(capacity)), load)


class QueryRequest(BaseModel):
    """The /query body (field names, defaults and bounds of the reference)."""

    graph_dir: str | None = None
    partitioned_dir: str | None = None
    entities: list[str]
    hops: int = Field(ge=1)
    semantics: Literal["exact", "frontier", "cumulative"] = "frontier"
    cache_capacity: int = Field(default=16, ge=1)
    include_paths: bool = False
    max_paths: int = Field(default=DEFAULT_MAX_PATHS, ge=0)

    @model_validator(mode="after")
    def _one_target(self):
        if (self.graph_dir is None) == (self.partitioned_dir is None):
            raise ValueError("exactly one of graph_dir or partitioned_dir is required")
        return self


class LookupResult(NamedTuple):
    ids: list
    unknown: list


def lookup_entities(labels, entities: Labels) -> LookupResult:
    """(sorted distinct ids, unknown labels in request order); unknown
    labels are reported, never fatal."""
    ids, unknown = set(), []
    for lab in labels:
        i = entities.id_of(lab)
        if i is None:
            unknown.append(lab)
        else:
            ids.add(i)
    return LookupResult(sorted(ids), unknown)


def answer(registry: DeviceGraphRegistry, req: QueryRequest) -> dict:
    """One /query request -> the reference's response body."""
    from .partition import cross_graph_k_hop, cross_graph_paths
    from .retriever import k_hop, reconstruct_paths

    sem = HopSemantics.parse(req.semantics)
    cache = None
    if req.graph_dir is not None:
        g, ents, rels = registry.graph(req.graph_dir)
        ids, unknown = lookup_entities(req.entities, ents)
        q0 = EntityVector(np.asarray(ids, dtype=np.int64), g.n_entities)
        trace = k_hop(q0, req.hops, g, sem)
        paths = reconstruct_paths(q0, req.hops, g, req.max_paths) if req.include_paths else None
    else:
        pg, ents, rels = registry.partitioned(req.partitioned_dir, req.cache_capacity)
        ids, unknown = lookup_entities(req.entities, ents)
        q0 = EntityVector(np.asarray(ids, dtype=np.int64), pg.n_entities)
        trace = cross_graph_k_hop(q0, req.hops, pg, sem)
        paths = cross_graph_paths(q0, req.hops, pg, req.max_paths) if req.include_paths else None
        cache = pg.cache.snapshot_counters().as_dict()
    hops = [{"hop": h + 1, "entities": [ents.label_of(e) for e in step.frontier.ids.tolist()],
             "triple_count": int(step.activated.ids.size)} for h, step in enumerate(trace.steps)]
    return {
        "hops": hops,
        "unknown": unknown,
        "paths": None if paths is None else [
            [[ents.label_of(s), rels.label_of(r), ents.label_of(o)] for s, r, o in p] for p in paths.paths],
        "paths_truncated": None if paths is None else bool(paths.truncated),
        "cache": cache,
    }


def _problem(kind: str, message: str) -> dict:
    return {"detail": {"kind": kind, "message": message}}


def create_app(registry: DeviceGraphRegistry | None = None):
    """FastAPI app serving /query (and /healthz) from the device registry."""
    from fastapi import FastAPI
    from fastapi.exceptions import RequestValidationError
    from fastapi.responses import JSONResponse

    from . import __version__

    app = FastAPI(title="paper_2604_18913_b200", version=__version__)
    reg = registry if registry is not None else DeviceGraphRegistry()
    app.state.registry = reg

    def status(code: int, kind: str):
        async def handler(request, exc):
            if isinstance(exc, RequestValidationError):
                msg = "; ".join(".".join(str(p) for p in e["loc"] if p != "body") + ": " + e["msg"]
                                for e in exc.errors())
            else:
                msg = str(exc)
            return JSONResponse(status_code=code, content=_problem(kind, msg))

        return handler

    for exc_type, code, kind in ((RequestValidationError, 400, "usage"), (UsageError, 400, "usage"),
                                 (ValueError, 400, "usage"), (DataError, 422, "data"),
                                 (FileNotFoundError, 422, "data")):
        app.add_exception_handler(exc_type, status(code, kind))

    @app.get("/healthz")
    def healthz():
        return {"status": "ok", "version": __version__}

    @app.post("/query")
    def query(req: QueryRequest):
        return answer(reg, req)

    return app
