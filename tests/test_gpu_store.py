"""Store-backed partitioned retrieval on the device against the REAL
reference: the partition directories it wrote (tests/golden/partdir_*) are
opened with the device DirectoryStore and the reference's query script is
replayed -- traces, paths, truncation flags, cache counters and the cache's
access trace must all match (make_golden_store.py)."""

import json
import shutil

import numpy as np
import pytest

from golden_io import HERE as GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def th(cuda_device):
    import paper_2604_18913_b200 as th

    return th


def _golden(strategy):
    return json.loads((GOLDEN / f"store_{strategy}.json").read_text())


def _replay(th, pg, g):
    E = pg.n_entities
    for c in g["calls"]:
        q0 = th.EntityVector(np.asarray(c["seeds"], np.int64), E)
        if c["kind"] == "k_hop":
            tr = th.cross_graph_k_hop(q0, c["k"], pg, th.HopSemantics.parse(c["sem"]))
            for h in range(c["k"]):
                assert tr.frontier(h + 1).ids.tolist() == c["frontiers"][h], (c["seeds"], c["sem"], h)
                assert tr.activated(h + 1).ids.tolist() == c["activated"][h], (c["seeds"], c["sem"], h)
        else:
            pr = th.cross_graph_paths(q0, c["k"], pg, c["max_paths"])
            assert [[list(t) for t in p] for p in pr.paths] == c["paths"], (c["seeds"], c["k"])
            assert pr.truncated == c["truncated"]
        cnt = pg.cache.snapshot_counters()
        assert [cnt.hits, cnt.misses, cnt.loads, cnt.evictions] == c["counters"], c
        assert len(pg.cache.trace) == c["trace_len"]


@pytest.mark.parametrize("strategy", ["lpt", "hash"])
def test_directory_store_replays_reference(th, strategy):
    g = _golden(strategy)
    pg, ents, rels = th.open_partitioned(GOLDEN / f"partdir_{strategy}", 2, record_trace=True)
    assert len(ents) == 400 and len(rels) == 6
    _replay(th, pg, g)
    # the reference's script ends with a planned batch (plan_batch ->
    # run_batch): same order, same per-query isolation, and the cache sees the
    # same access sequence as the reference's LRU did
    E = pg.n_entities
    qs = [th.BatchQuery(f"q{i}", th.EntityVector(np.asarray(sd, np.int64), E), 2)
          for i, sd in enumerate(([0], [5, 17], [123], [399], [2, 3, 250], []))]
    qs.append(th.BatchQuery("bad", th.EntityVector(np.asarray([1], np.int64), E), 0))
    batch = th.plan_batch(qs, pg.plan)
    assert batch.execution_order == g["batch_order"]
    for br, want in zip(th.run_batch(batch, pg), g["batch"]):
        assert br.query_id == want["id"] and br.error == want["error"]
        if want["frontiers"] is not None:
            assert [br.trace.frontier(h).ids.tolist() for h in (1, 2)] == want["frontiers"]
    assert list(pg.cache.trace) == g["cache_trace"]


@pytest.mark.parametrize("strategy,m", [("lpt", 3), ("hash", 4)])
def test_materialize_and_save_match_reference_bytes(th, tmp_path, strategy, m):
    """Our device subgraphs written with save_partition_dir are byte-identical
    to the reference's directory, and an in-memory store over them replays
    the reference traces."""
    s, r, o = np.load(GOLDEN / "store_graph.npy")
    E, R = 400, 6
    plan = th.plan_partitions((s, E), m, strategy)
    sgs = th.materialize_subgraphs(plan, (s, r, o, E, R))
    ref_dir = GOLDEN / f"partdir_{strategy}"
    from paper_2604_18913_b200 import store

    ents = store._read_label_lines(ref_dir / "entities.txt")
    rels = store._read_label_lines(ref_dir / "relations.txt")
    out = th.save_partition_dir(plan, sgs, ents, rels, R, tmp_path / "p")
    for f in sorted(ref_dir.iterdir()):
        assert (out / f.name).read_bytes() == f.read_bytes(), f.name
    pg = th.PartitionedGraph(plan, th.InMemoryStore(sgs, E, R), th.SubgraphCache(2, record_trace=True))
    _replay(th, pg, _golden(strategy))
    sg = sgs[0]
    probe = np.array([0, 3, 17, 250, 399], np.int64)
    ref_pos = np.minimum(np.searchsorted(sg.ent_to_global, probe), sg.ent_to_global.size - 1)
    assert np.array_equal(sg.entities_to_local(probe), ref_pos[sg.ent_to_global[ref_pos] == probe])


def test_store_errors(th, tmp_path):
    d = tmp_path / "p"
    shutil.copytree(GOLDEN / "partdir_hash", d)
    pg, _, _ = th.open_partitioned(d, 1)
    q = th.EntityVector(np.asarray([0], np.int64), 400)
    with pytest.raises(ValueError):
        th.cross_graph_k_hop(th.EntityVector(np.asarray([0], np.int64), 401), 2, pg)
    with pytest.raises(ValueError):
        th.cross_graph_k_hop(q, 0, pg)
    with pytest.raises(ValueError):
        th.cross_graph_paths(q, 2, pg, -1)
    for f in d.glob("shard-*.lkg"):
        f.unlink()
    with pytest.raises(th.IntegrityError):
        th.cross_graph_k_hop(th.EntityVector(np.asarray([0, 1, 2, 3, 4], np.int64), 400), 1, pg)
    c = pg.cache.snapshot_counters()
    assert c.loads == 0 and len(pg.cache) == 0  # a failed load leaves the cache untouched
