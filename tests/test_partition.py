"""CPU tests of the partitioned layer: plans, routing, and the multi-rank
exchange protocol (world_size 2 over gloo, one process per rank).

The per-rank arithmetic runs in tests/shard_ref.py (numpy stand-in with
the CUDA shard's layout and record format, exchange regions in host shared
memory); the wave protocol, region wiring, barriers, gathers and merging are
the product code of paper_2604_18913_b200.partition.  The CUDA shards
themselves are checked on the GPU (tests/test_gpu_partition.py)."""

import os
import socket

import numpy as np
import pytest
import torch

import paper_2604_18913_b200 as th
from paper_2604_18913_b200.partition import hash_owner
from oracle import khop_oracle as orc
from shard_ref import RefShard


def _graph(E, T, R, seed, alpha=1.2):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(E)
    w = np.cumsum(1.0 / np.arange(1, E + 1) ** alpha)
    w /= w[-1]
    s = perm[np.minimum(np.searchsorted(w, rng.random(T)), E - 1)]
    o = perm[np.minimum(np.searchsorted(w, rng.random(T)), E - 1)]
    r = rng.integers(0, R, T)
    key = np.unique((s.astype(np.int64) * R + r) * E + o)
    key = rng.permutation(key)
    return key // E // R, (key // E) % R, key % E


# ---------------------------------------------------------------- plans


def test_plan_partitions_matches_the_restated_planner():
    s, _, _ = _graph(400, 3000, 5, seed=1)
    for strategy in ("hash", "lpt"):
        for m in (1, 2, 3, 8):
            plan = th.plan_partitions((s, 400), m, strategy)
            assert np.array_equal(plan.assignment, orc.plan_owner(s, 400, m, strategy))
            deg = np.bincount(s, minlength=400)
            assert plan.loads.sum() == s.size
            for p in range(m):
                assert plan.loads[p] == deg[plan.assignment == p].sum()
            assert (plan.assignment[deg == 0] == th.UNASSIGNED).all()


def test_plan_partitions_errors():
    s = np.array([0, 0, 1])
    with pytest.raises(th.UsageError):
        th.plan_partitions((s, 5), 0)
    with pytest.raises(th.UsageError):
        th.plan_partitions((s, 5), 3)  # only 2 distinct subjects
    with pytest.raises(th.UsageError):
        th.plan_partitions((s, 5), 1, "round-robin")


def test_lpt_balances_heaviest_first():
    # degrees 5,4,3,3 over 2 partitions: LPT gives loads {8, 7}
    s = np.array([0] * 5 + [1] * 4 + [2] * 3 + [3] * 3)
    plan = th.plan_partitions((s, 4), 2, "lpt")
    assert sorted(plan.loads.tolist()) == [7, 8]
    assert plan.assignment[0] != plan.assignment[1]


def test_route_buckets_and_sink():
    s = np.array([0, 1, 2, 2])
    plan = th.plan_partitions((s, 6), 2, "hash")
    q = th.EntityVector([0, 1, 2, 4, 5], 6)
    rr = th.route(q, plan)
    assert rr.sink.ids.tolist() == [4, 5]
    got = sorted(i for v in rr.buckets.values() for i in v.ids.tolist())
    assert got == [0, 1, 2]
    for p, v in rr.buckets.items():
        assert (plan.assignment[v.ids] == p).all()
    with pytest.raises(ValueError):
        th.route(th.EntityVector([1], 7), plan)


def test_shard_plan_invariants():
    s, _, _ = _graph(1000, 8000, 3, seed=2)
    plan = th.plan_sharding(s, 1000, 3, n_hubs=10)
    assert np.array_equal(plan.owner, hash_owner(np.arange(1000), 3))
    for p in range(3):
        owned = plan.owned(p)
        assert np.array_equal(plan.lidx[owned], np.arange(owned.size))  # ascending-id rows
        assert plan.n_local[p] == owned.size
    deg = np.bincount(s, minlength=1000)
    hubs = plan.hub_ids
    assert hubs.size == 10 and (np.diff(hubs) > 0).all()
    assert deg[hubs].min() >= np.sort(deg)[-10]
    assert (plan.hub_index[hubs] == np.arange(10)).all()
    assert (plan.hub_index >= 0).sum() == 10


# ------------------------------------------------ in-process ranks (loopback)


@pytest.mark.parametrize("world,n_hubs", [(1, 0), (2, 3), (3, 8)])
@pytest.mark.parametrize("sem", ["exact", "frontier", "cumulative"])
def test_loopback_protocol_matches_oracle(world, n_hubs, sem):
    s, r, o = _graph(300, 2500, 6, seed=7)
    pg = th.PartitionedGraph((s, r, o), 300, 6, th.LoopbackExchange(world), n_hubs=n_hubs,
                             shard_factory=RefShard)
    og = orc.build_csr(s, r, o, 300, 6)
    seeds = np.random.default_rng(1).integers(0, 300, 40)
    res = pg.retrieve(seeds, 3, semantics=sem, activated=True)
    for i, sd in enumerate(seeds.tolist()):
        ref = orc.retrieve_one(og, sd, 3, sem)
        for h in range(3):
            assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h]), (i, h)
            assert np.array_equal(res.activated(i, h + 1), ref["activated"][h]), (i, h)
            assert int(res.edges[h, i]) == ref["edges"][h]


# ------------------------------------------------ two processes over gloo


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _dist_worker(rank, world, port, errfile):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, r, o = _graph(500, 5000, 8, seed=11)
        og = orc.build_csr(s, r, o, 500, 8)
        xch = th.DistExchange()
        pg = th.PartitionedGraph((s, r, o), 500, 8, xch, n_hubs=6, shard_factory=RefShard)
        rng = np.random.default_rng(3)
        seeds = rng.integers(0, 500, 60)
        filt = [sorted(rng.choice(8, 3, replace=False).tolist()) for _ in seeds]
        for sem in ("exact", "frontier", "cumulative"):
            res = pg.retrieve(seeds, 3, semantics=sem, activated=True)
            fres = pg.retrieve(seeds, 2, relation_filter=filt, semantics=sem)
            for i, sd in enumerate(seeds.tolist()):
                ref = orc.retrieve_one(og, sd, 3, sem)
                fref = orc.retrieve_one(og, sd, 2, sem, filt[i])
                for h in range(3):
                    assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h])
                    assert np.array_equal(res.activated(i, h + 1), ref["activated"][h])
                    assert int(res.edges[h, i]) == ref["edges"][h]
                for h in range(2):
                    assert np.array_equal(fres.frontier(i, h + 1), fref["frontiers"][h])
                    assert int(fres.edges[h, i]) == fref["edges"][h]
        tr = th.cross_graph_k_hop(th.EntityVector([1, 7, 42], 500), 2, pg)
        ref = orc.hop_trace(og, [1, 7, 42], 2, orc.FRONTIER)
        for h in range(2):
            assert np.array_equal(tr.frontier(h + 1).ids, ref[h][0])
            assert np.array_equal(tr.activated(h + 1).ids, ref[h][1])
        stats = {}
        q = th.partition.WaveQuery(np.arange(61, dtype=np.int32), seeds.astype(np.int32), 2,
                                   th.HopSemantics.FRONTIER)
        pg.run(q, stats)
        assert sum(stats["sent_records"][0]) > 0  # records really crossed ranks
        # paths across the two processes: walk counts and capped offers
        # exchanged over gloo (walks.sharded_paths) == the oracle's walks
        for seeds_p, k, cap in (([3], 2, 100), ([1, 7, 42], 3, 50), ([1, 7, 42], 2, None), ([9], 1, 0),
                                ([2, 3], 3, 1)):
            pr = th.cross_graph_paths(th.EntityVector(seeds_p, 500), k, pg, cap)
            ref_p, ref_t = orc.walk_paths(og, seeds_p, k, cap)
            assert [tuple(tuple(int(x) for x in t) for t in p) for p in pr.paths] == \
                orc.paths_as_triples(og, ref_p), (seeds_p, k, cap)
            assert pr.truncated == ref_t
        for seeds_p in ([3], [1, 7, 42]):
            s_, r_, o_ = th.partition.walk_subgraph(th.EntityVector(seeds_p, 500), 2, pg)
            act = np.unique(np.concatenate([a for _, a in orc.hop_trace(og, seeds_p, 2, orc.EXACT)]))
            assert np.array_equal(s_, og.subj[act]) and np.array_equal(r_, og.rel[act])
            assert np.array_equal(o_, og.obj[act])
    except BaseException as e:  # pragma: no cover - reported to the parent
        with open(errfile, "a") as f:
            f.write(f"rank {rank}: {type(e).__name__}: {e}\n")
        raise
    finally:
        dist.destroy_process_group()


def test_two_ranks_over_gloo_match_oracle(tmp_path):
    errfile = str(tmp_path / "err.txt")
    torch.multiprocessing.spawn(_dist_worker, args=(2, _free_port(), errfile), nprocs=2, join=True)
    assert not os.path.exists(errfile), open(errfile).read()


@pytest.mark.parametrize("world,n_hubs", [(1, 0), (2, 4), (3, 0), (4, 9)])
def test_sharded_paths_match_oracle(world, n_hubs):
    """Walk counts + capped offers exchanged between ranks (walks.py) give
    the reference's walks, order and truncation flag -- with hub rows split
    over the ranks, walks revisiting vertices, and every cap regime."""
    s, r, o = _graph(300, 4000, 5, seed=world)
    og = orc.build_csr(s, r, o, 300, 5)
    pg = th.PartitionedGraph((s, r, o), 300, 5, th.LoopbackExchange(world), n_hubs=n_hubs,
                             shard_factory=RefShard)
    rng = np.random.default_rng(world)
    for _ in range(12):
        seeds = sorted(set(rng.integers(0, 300, int(rng.integers(1, 4))).tolist()))
        k = int(rng.integers(1, 4))
        for cap in (0, 1, 5, 37, 1000, None):
            pr = th.cross_graph_paths(th.EntityVector(seeds, 300), k, pg, cap)
            ref_p, ref_t = orc.walk_paths(og, seeds, k, cap)
            got = [tuple(tuple(int(x) for x in t) for t in p) for p in pr.paths]
            assert got == orc.paths_as_triples(og, ref_p), (seeds, k, cap)
            assert pr.truncated == ref_t
