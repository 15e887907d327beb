"""Store-backed partitioned retrieval, host side (no GPU): partition
directories written by the REAL reference (tests/golden/partdir_*, made by
make_golden_store.py), manifest validation, labels, batch planning."""

import json
import shutil

import numpy as np
import pytest

from golden_io import HERE as GOLDEN

import paper_2604_18913_b200 as th
from paper_2604_18913_b200 import store


def _golden(strategy):
    return json.loads((GOLDEN / f"store_{strategy}.json").read_text())


def _graph():
    s, r, o = np.load(GOLDEN / "store_graph.npy")
    return s, r, o, 400, 6


@pytest.mark.parametrize("strategy,m", [("lpt", 3), ("hash", 4)])
def test_plan_from_reference_dir_matches_our_planner(strategy, m):
    s, r, o, E, R = _graph()
    plan = store.load_partition_plan(GOLDEN / f"partdir_{strategy}")
    ours = th.plan_partitions((s, E), m, strategy)
    assert plan.m == m and plan.strategy == strategy
    assert np.array_equal(plan.assignment, ours.assignment)
    assert np.array_equal(plan.loads, ours.loads)
    assert not plan.assignment.flags.writeable


def test_manifest_errors(tmp_path):
    src = GOLDEN / "partdir_lpt"
    d = tmp_path / "p"
    shutil.copytree(src, d)
    st = store.DirectoryStore(d)
    assert st.m == 3 and st.n_entities == 400 and st.n_triples == len(_graph()[0])
    with pytest.raises(th.IntegrityError):
        st.load(7)
    (d / "shard-0001.lkg").unlink()
    with pytest.raises(th.IntegrityError, match="missing shard file"):
        st.load(1)
    man = json.loads((d / "manifest.json").read_text())
    man["triple_count"] += 1
    (d / "manifest.json").write_text(json.dumps(man))
    with pytest.raises(th.IntegrityError, match="do not sum"):
        store.DirectoryStore(d)
    (d / "manifest.json").write_text("{not json")
    with pytest.raises(th.IntegrityError, match="unreadable"):
        store.load_partition_plan(d)
    (d / "manifest.json").unlink()
    with pytest.raises(th.IntegrityError, match="no partition manifest"):
        store.DirectoryStore(d)


def test_label_files_round_trip(tmp_path):
    """Label files written by save_partition_dir are byte-identical to the
    reference's; open_partitioned reads them back as lists (line = id)."""
    ref = GOLDEN / "partdir_hash" / "entities.txt"
    labels = store._read_label_lines(ref)
    assert len(labels) == 400 and labels[17] == "e17" and labels[399] == "e399"
    assert store._label_lines(labels) == ref.read_bytes()
    (tmp_path / "x.txt").write_bytes(store._label_lines(labels))
    assert store._read_label_lines(tmp_path / "x.txt") == labels


def test_manifest_describe_round_trips(tmp_path):
    man = store.PartitionManifest.read(GOLDEN / "partdir_lpt")
    assert man.m == 3 and man.n_entities == 400 and man.n_relations == 6
    assert sorted(man.shards) == [0, 1, 2]
    assert store.PartitionManifest.shard_stem(7) == "shard-0007"


def test_store_constructor_dispatch_without_gpu():
    plan = store.load_partition_plan(GOLDEN / "partdir_lpt")
    st = store.DirectoryStore(GOLDEN / "partdir_lpt")
    pg = th.PartitionedGraph(plan, st, th.SubgraphCache(2))
    assert isinstance(pg, store.StorePartitionedGraph)
    assert pg.n_entities == 400 and pg.n_triples == len(_graph()[0]) and pg.n_relations == 6
    bad = th.PartitionPlan(2, plan.assignment, plan.loads[:2], "lpt")
    with pytest.raises(th.IntegrityError):
        th.PartitionedGraph(bad, st, th.SubgraphCache(2))


@pytest.mark.parametrize("strategy", ["lpt", "hash"])
def test_plan_batch_order_matches_reference(strategy):
    """plan_batch over the reference's own batch (make_golden_store.py)
    gives its execution order; restore_order inverts it."""
    import json

    import paper_2604_18913_b200 as th

    g = json.loads((GOLDEN / f"store_{strategy}.json").read_text())
    plan = th.load_partition_plan(GOLDEN / f"partdir_{strategy}")
    seeds = ([0], [5, 17], [123], [399], [2, 3, 250], [])
    qs = [th.BatchQuery(f"q{i}", th.EntityVector(np.asarray(sd, np.int64), 400), 2) for i, sd in enumerate(seeds)]
    qs.append(th.BatchQuery("bad", th.EntityVector(np.asarray([1], np.int64), 400), 0))
    b = th.plan_batch(qs, plan)
    assert b.execution_order == g["batch_order"]
    inv = b.restore_order
    assert [b.execution_order[inv[p]] for p in range(len(qs))] == list(range(len(qs)))
    assert th.QueryBatch.identity(qs).execution_order == list(range(len(qs)))
    sigs = [th.signature(qs[p].q0, plan) for p in b.execution_order]
    assert sigs == sorted(sigs)
