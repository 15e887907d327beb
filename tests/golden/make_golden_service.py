"""/query responses of the REAL reference service (build container only):

    python tests/golden/make_golden_service.py [/root/reference/pkg/src]

Writes graphdir/ (graph.lkg + entity/relation label files, written by the
reference's save_graph_dir for the store_graph.npy triples, labels e<i> /
r<i>) and service.json: a fixed request script POSTed to the reference's
FastAPI app (service/app.py:196-229) through its test client -- graph-dir
and partition-dir targets, unknown labels, every semantics, paths with caps,
the cache counters carried across requests, and rejected requests -- with
each status code and JSON body.  The device backend must answer the same
script identically (tests/test_gpu_service.py).
"""

import json
import sys
from pathlib import Path

import numpy as np

REF = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from fastapi.testclient import TestClient  # noqa: E402
from triplehop.archive import save_graph_dir  # noqa: E402
from triplehop.incidence import build_incidence  # noqa: E402
from triplehop.service.app import create_app  # noqa: E402
from triplehop.triples import Dictionary  # noqa: E402

OUT = Path(__file__).resolve().parent
E, R = 400, 6


def script(graph_dir: str, part_dir: str) -> list:
    reqs = []
    for ents in (["e0"], ["e5", "e17", "nope"], ["e123", "e399"], ["zz"], []):
        for sem in ("exact", "frontier", "cumulative"):
            for hops in (1, 2, 3):
                reqs.append({"graph_dir": graph_dir, "entities": ents, "hops": hops, "semantics": sem})
        reqs.append({"graph_dir": graph_dir, "entities": ents, "hops": 2, "include_paths": True})
        reqs.append({"graph_dir": graph_dir, "entities": ents, "hops": 3, "include_paths": True, "max_paths": 7})
    for ents in (["e0"], ["e2", "e3", "e250"], ["e399", "x"]):
        for cap in (2, 16):
            reqs.append({"partitioned_dir": part_dir, "entities": ents, "hops": 2, "cache_capacity": cap})
            reqs.append({"partitioned_dir": part_dir, "entities": ents, "hops": 2, "cache_capacity": cap,
                         "include_paths": True, "max_paths": 5, "semantics": "exact"})
    reqs += [
        {"graph_dir": graph_dir, "partitioned_dir": part_dir, "entities": ["e0"], "hops": 1},
        {"entities": ["e0"], "hops": 1},
        {"graph_dir": graph_dir, "entities": ["e0"], "hops": 0},
        {"graph_dir": graph_dir, "entities": ["e0"], "hops": 1, "semantics": "sideways"},
        {"graph_dir": graph_dir, "entities": ["e0"], "hops": 1, "max_paths": -1},
        {"partitioned_dir": part_dir, "entities": ["e0"], "hops": 1, "cache_capacity": 0},
    ]
    return reqs


def main():
    s, r, o = np.load(OUT / "store_graph.npy")
    g = build_incidence((s, r, o), E, R)
    save_graph_dir(g, Dictionary(f"e{i}" for i in range(E)), Dictionary(f"r{i}" for i in range(R)),
                   OUT / "graphdir")
    client = TestClient(create_app())
    out = []
    # paths relative to the golden directory; the client runs from there
    import os

    os.chdir(OUT)
    for req in script("graphdir", "partdir_hash"):
        resp = client.post("/query", json=req)
        out.append({"request": req, "status": resp.status_code, "body": resp.json()})
    (OUT / "service.json").write_text(json.dumps(out))
    print("wrote graphdir/ and service.json:", len(out), "requests")


if __name__ == "__main__":
    main()
