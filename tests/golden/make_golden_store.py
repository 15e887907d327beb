"""Partition directories and store-backed traces from the REAL reference
(build container only):

    python tests/golden/make_golden_store.py [/root/reference/pkg/src]

For the reference's own power-law generator (synth.py:34-49) at 400
entities / 2,400 triples, with an LPT plan (m=3) and a hash plan (m=4):

* partdir_<plan>/ -- written by triplehop.archive.save_partition_dir
  (archive.py:192-237): manifest, assignment, labels, shard LKG1 archives,
  entity/triple maps.  The device DirectoryStore must open these files.
* store_<plan>.json -- opened with open_partitioned(capacity 2, trace on),
  a fixed query script run through cross_graph_k_hop (every semantics,
  k = 1..3) and cross_graph_paths, recording each trace, each path list and
  the cache counters + access trace after every call; plus plan_batch's
  execution order and run_batch's per-query errors for a mixed batch.
"""

import json
import sys
from pathlib import Path

import numpy as np

REF = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from triplehop.archive import open_partitioned, save_partition_dir  # noqa: E402
from triplehop.engine import BatchQuery, cross_graph_k_hop, cross_graph_paths, plan_batch, run_batch  # noqa: E402
from triplehop.incidence import EntityVector, HopSemantics  # noqa: E402
from triplehop.partition import materialize_subgraphs, plan_partitions  # noqa: E402
from triplehop.synth import power_law  # noqa: E402
from triplehop.triples import Dictionary  # noqa: E402

OUT = Path(__file__).resolve().parent
E, T, R = 400, 2400, 6
PLANS = (("lpt", 3), ("hash", 4))
SEEDS = ([0], [5, 17], [123], [399], [2, 3, 250], [])


def _graph():
    ts = power_law(E, T, R, seed=7, alpha=1.1)
    s, r, o = ts.arrays()
    return ts, s, r, o


def main():
    ts, s, r, o = _graph()
    np.save(OUT / "store_graph.npy", np.stack([s, r, o]).astype(np.int32))  # (E, R) = (400, 6)
    ents = Dictionary(f"e{i}" for i in range(E))
    rels = Dictionary(f"r{i}" for i in range(R))
    for strategy, m in PLANS:
        plan = plan_partitions((s, E), m, strategy)
        sgs = materialize_subgraphs(plan, (s, r, o, E, R))
        d = OUT / f"partdir_{strategy}"
        save_partition_dir(plan, sgs, ents, rels, R, d)
        pg, _, _ = open_partitioned(d, 2, record_trace=True)
        calls = []
        for seeds in SEEDS:
            q0 = EntityVector(np.asarray(seeds, np.int64), E)
            for sem in ("exact", "frontier", "cumulative"):
                for k in (1, 2, 3):
                    tr = cross_graph_k_hop(q0, k, pg, HopSemantics.parse(sem))
                    c = pg.cache.snapshot_counters()
                    calls.append({
                        "kind": "k_hop", "seeds": seeds, "sem": sem, "k": k,
                        "frontiers": [tr.frontier(h).ids.tolist() for h in range(1, k + 1)],
                        "activated": [tr.activated(h).ids.tolist() for h in range(1, k + 1)],
                        "counters": [c.hits, c.misses, c.loads, c.evictions],
                        "trace_len": len(pg.cache.trace)})
            for k, cap in ((2, 10_000), (3, 25), (2, 0)):
                pr = cross_graph_paths(q0, k, pg, cap)
                c = pg.cache.snapshot_counters()
                calls.append({"kind": "paths", "seeds": seeds, "k": k, "max_paths": cap,
                              "paths": [[list(t) for t in p] for p in pr.paths],
                              "truncated": pr.truncated,
                              "counters": [c.hits, c.misses, c.loads, c.evictions],
                              "trace_len": len(pg.cache.trace)})
        # batch planning + per-query isolation (a k=0 query fails)
        qs = [BatchQuery(f"q{i}", EntityVector(np.asarray(sd, np.int64), E), 2)
              for i, sd in enumerate(SEEDS)]
        qs.append(BatchQuery("bad", EntityVector(np.asarray([1], np.int64), E), 0))
        batch = plan_batch(qs, pg.plan)
        res = run_batch(batch, pg)
        golden = {"strategy": strategy, "m": m, "calls": calls,
                  "cache_trace": list(pg.cache.trace),
                  "batch_order": batch.execution_order,
                  "batch": [{"id": br.query_id, "error": br.error,
                             "frontiers": None if br.trace is None else
                             [br.trace.frontier(h).ids.tolist() for h in (1, 2)]} for br in res]}
        (OUT / f"store_{strategy}.json").write_text(json.dumps(golden))
        print("wrote", d.name, f"store_{strategy}.json", len(calls), "calls")


if __name__ == "__main__":
    main()
