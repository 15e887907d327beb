"""GPU parity of the partitioned engine (K6, th_shard_*): every rank of a
small world hosted on one B200 through LoopbackExchange.  Bit-exact against
the single-graph engine, the oracle and the reference's golden traces --
frontier AND activated sets, mirroring test_engine.py:68-82 (cross-graph
traces bit-identical to single-graph ones)."""

import numpy as np
import pytest

from golden_io import HERE as GOLDEN
from golden_io import load_case
from oracle import khop_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def th(cuda_device):
    import paper_2604_18913_b200 as th

    return th


def _hub_graph(E, T, R, seed, alpha=1.2):
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


@pytest.mark.parametrize("direction", ["push", "auto", "pull"])
@pytest.mark.parametrize("world,n_hubs", [(1, 0), (2, 0), (2, 5), (3, 7), (4, 16)])
@pytest.mark.parametrize("sem", ["exact", "frontier", "cumulative"])
def test_partitioned_equals_single_and_oracle(th, world, n_hubs, sem, direction):
    s, r, o = _hub_graph(1500, 30000, 24, seed=21)
    E, R = 1500, 24
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(world), n_hubs=n_hubs)
    pg.pull_divisor = {"push": 0.0, "auto": 8.0, "pull": 1e18}[direction]
    assert sum(sh.local_triples for sh in pg.shards) == s.size  # each triple on one rank
    rng = np.random.default_rng(4)
    seeds = rng.integers(0, E, 300)
    part = pg.retrieve(seeds, 3, semantics=sem, activated=True)
    single = th.retrieve(g, seeds, 3, semantics=sem, activated=True)
    for i in range(seeds.size):
        for h in range(1, 4):
            assert np.array_equal(part.frontier(i, h), single.frontier(i, h)), (i, h)
            assert np.array_equal(part.activated(i, h), single.activated(i, h)), (i, h)
    assert np.array_equal(part.edges.numpy(), single.edges.cpu().numpy())
    for i in range(0, seeds.size, 23):
        ref = orc.retrieve_one(og, int(seeds[i]), 3, sem)
        for h in range(3):
            assert np.array_equal(part.frontier(i, h + 1), ref["frontiers"][h])
            assert int(part.edges[h, i]) == ref["edges"][h]


@pytest.mark.parametrize("world,n_hubs", [(1, 0), (2, 0), (3, 6)])
@pytest.mark.parametrize("sem", ["exact", "frontier"])
def test_partitioned_sparse_graph_two_phase_pull(th, world, n_hubs, sem):
    """A C4-shaped sparse graph (1.6 in-edges per entity): the shards' pull
    hops take the two-phase pull (edge screen + gather) by graph shape;
    forced pulls, against the single graph and the oracle."""
    E, R = 20000, 16
    s, r, o = _hub_graph(E, 32000, R, seed=61, alpha=1.3)
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(world), n_hubs=n_hubs)
    pg.pull_divisor = 1e18  # every hop after the first pulls
    rng = np.random.default_rng(9)
    seeds = rng.integers(0, E, 400)
    part = pg.retrieve(seeds, 3, semantics=sem)
    single = th.retrieve(g, seeds, 3, semantics=sem)
    for i in range(seeds.size):
        for h in range(1, 4):
            assert np.array_equal(part.frontier(i, h), single.frontier(i, h)), (i, h)
    assert np.array_equal(part.edges.numpy(), single.edges.cpu().numpy())
    for i in range(0, seeds.size, 37):
        ref = orc.retrieve_one(og, int(seeds[i]), 3, sem)
        for h in range(3):
            assert np.array_equal(part.frontier(i, h + 1), ref["frontiers"][h])


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_relation_filter(th, world):
    """Relation masks on push hops (world 2, auto) and on pull hops (world 4)."""
    s, r, o = _hub_graph(1200, 20000, 30, seed=8)
    E, R = 1200, 30
    og = orc.build_csr(s, r, o, E, R)
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(world), n_hubs=6)
    pg.pull_divisor = 1e18 if world == 4 else 8.0  # world 4: every hop pulls
    rng = np.random.default_rng(2)
    seeds = rng.integers(0, E, 200)
    filt = [sorted(rng.choice(R, 5, replace=False).tolist()) for _ in seeds]
    part = pg.retrieve(seeds, 2, relation_filter=filt, semantics="frontier", activated=True)
    for i in range(0, 200, 9):
        ref = orc.retrieve_one(og, int(seeds[i]), 2, "frontier", filt[i])
        for h in range(2):
            assert np.array_equal(part.frontier(i, h + 1), ref["frontiers"][h])
            assert np.array_equal(part.activated(i, h + 1), ref["activated"][h])
            assert int(part.edges[h, i]) == ref["edges"][h]


def test_two_waves_and_overflow_rerun(th):
    """1,300 seeds = two waves; the first run of each wave overflows the
    initial result capacity on every rank and is re-run transparently."""
    s, r, o = _hub_graph(3000, 90000, 16, seed=3)
    E, R = 3000, 16
    g = th.build_incidence((s, r, o), E, R)
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(3), n_hubs=10)
    seeds = np.random.default_rng(5).integers(0, E, 1300)
    part = pg.retrieve(seeds, 3)
    single = th.retrieve(g, seeds, 3)
    for i in range(0, 1300, 13):
        for h in range(1, 4):
            assert np.array_equal(part.frontier(i, h), single.frontier(i, h))


def test_inbox_overflow_grows_and_reconnects(th):
    """An exchange inbox far too small for a wave: the receivers flag the
    overflow, every rank grows its region, the ranks reconnect and the wave
    runs again -- results identical to the single-graph engine."""
    s, r, o = _hub_graph(2000, 40000, 8, seed=21)
    E, R = 2000, 8
    g = th.build_incidence((s, r, o), E, R)

    def small(cols, n_e, n_r, plan, rank):
        return th.partition.GraphShard(cols, n_e, n_r, plan, rank, inbox_records=1024)

    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(3), n_hubs=4, shard_factory=small)
    pg.pull_divisor = 0.0  # push only: every candidate becomes an inbox record
    seeds = np.random.default_rng(2).integers(0, E, 300)
    part = pg.retrieve(seeds, 3)
    assert all(sh.inbox_records > 1024 for sh in pg.shards)
    single = th.retrieve(g, seeds, 3)
    for i in range(0, 300, 11):
        for h in range(1, 4):
            assert np.array_equal(part.frontier(i, h), single.frontier(i, h))
            assert int(part.edges[h - 1, i]) == int(single.edges[h - 1, i])


@pytest.mark.parametrize("name", ["tiny", "er30_s0", "er60_s12", "pl500_hubs", "selfloop", "objonly"])
@pytest.mark.parametrize("world", [2, 3])
def test_cross_graph_k_hop_golden(th, name, world):
    """The reference's own traces (frontier and activated per hop) through
    cross_graph_k_hop on a partitioned graph."""
    case = load_case(GOLDEN / f"{name}.npz")
    pg = th.PartitionedGraph((case.subj, case.rel, case.obj), case.n_entities, case.n_relations,
                             th.LoopbackExchange(world), n_hubs=2)
    for q in case.queries:
        if q.relations is not None:
            continue
        tr = th.cross_graph_k_hop(th.EntityVector(q.seeds, case.n_entities), q.k, pg, q.semantics)
        for h in range(q.k):
            assert np.array_equal(tr.frontier(h + 1).ids, q.frontiers[h]), (name, q.seeds, h)
            assert np.array_equal(tr.activated(h + 1).ids, q.activated[h]), (name, q.seeds, h)


def test_bad_partition_inputs(th):
    s, r, o = _hub_graph(100, 500, 4, seed=1)
    with pytest.raises(ValueError):
        th.PartitionedGraph((s, r, o + 1000), 100, 4, th.LoopbackExchange(2))
    pg = th.PartitionedGraph((s, r, o), 100, 4, th.LoopbackExchange(2))
    with pytest.raises(ValueError):
        pg.retrieve([5, 100], 2)
    with pytest.raises(ValueError):
        pg.retrieve([5], 0)
    with pytest.raises(ValueError):
        th.cross_graph_k_hop(th.EntityVector([1], 99), 2, pg)


def test_bench_targets_expand_like_reference(th):
    """GpuTarget / PartitionedGpuTarget answer the reference harness's
    expand(frontier) (bench.py:98-137) with one device hop."""
    s, r, o = _hub_graph(400, 3000, 6, seed=12)
    E, R = 400, 6
    og = orc.build_csr(s, r, o, E, R)
    g = th.build_incidence((s, r, o), E, R)
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(2), n_hubs=3)
    for tgt in (th.GpuTarget(g), th.PartitionedGpuTarget(pg, (s, r, o))):
        assert (tgt.n_entities, tgt.n_triples) == (E, s.size)
        for f in ([0, 5, 17], [3], list(range(0, 400, 7))):
            act, nxt = tgt.expand(np.array(f))
            ref_act, ref_nxt = orc.raw_hop(og, np.array(f, dtype=np.int64))
            assert np.array_equal(act, ref_act) and np.array_equal(nxt, ref_nxt)
        assert len(tgt.triples()) == s.size


@pytest.mark.parametrize("name", ["tiny", "er30_s1", "pl500_hubs", "interleave", "selfloop"])
def test_cross_graph_paths_golden(th, name):
    """Paths across partitions == the reference's reconstruct_paths goldens
    (engine.py:157-182 / test_engine.py:99-123: cross paths == single paths)."""
    case = load_case(GOLDEN / f"{name}.npz")
    pg = th.PartitionedGraph((case.subj, case.rel, case.obj), case.n_entities, case.n_relations,
                             th.LoopbackExchange(3), n_hubs=2)
    n = 0
    for q in case.queries:
        if not q.want_paths or q.relations is not None:
            continue
        pr = th.cross_graph_paths(th.EntityVector(q.seeds, case.n_entities), q.k, pg, q.max_paths)
        want = [tuple(th.Triple(int(case.subj[t]), int(case.rel[t]), int(case.obj[t])) for t in p)
                for p in q.paths]
        assert pr.paths == want, (name, q.seeds, q.max_paths)
        assert pr.truncated == q.truncated
        n += 1
    assert n > 0


def _gpu_dist_worker(rank, world, port, errfile):
    """One rank per process with a REAL CUDA shard on the same device: the
    ranks' kernels write into each other's exchange regions through CUDA IPC
    mappings; gloo carries the phase barriers and the result gather (NCCL
    refuses two ranks on one device).  No kernel of one rank waits on
    another rank (the barriers are host-side)."""
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_18913_b200 as th

        s, r, o = _hub_graph(1500, 30000, 16, seed=33)
        E, R = 1500, 16
        og = orc.build_csr(s, r, o, E, R)
        xch = th.DistExchange()
        pg = th.PartitionedGraph((s, r, o), E, R, xch, n_hubs=8)
        assert isinstance(pg.shards[0], th.partition.GraphShard)
        seeds = np.random.default_rng(8).integers(0, E, 150)
        for sem in ("exact", "frontier", "cumulative"):
            res = pg.retrieve(seeds, 3, semantics=sem, activated=True)
            for i in range(0, 150, 7):
                ref = orc.retrieve_one(og, int(seeds[i]), 3, sem)
                for h in range(3):
                    assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h])
                    assert np.array_equal(res.activated(i, h + 1), ref["activated"][h])
                    assert int(res.edges[h, i]) == ref["edges"][h]
        stats = {}
        q = th.partition.WaveQuery(np.arange(151, dtype=np.int32), seeds.astype(np.int32), 2,
                                   th.HopSemantics.FRONTIER)
        pg.run(q, stats)
        assert sum(stats["sent_records"][0]) > 0  # records crossed processes
        pr = th.cross_graph_paths(th.EntityVector([int(seeds[0])], E), 2, pg, max_paths=100)
        ref_p, ref_t = orc.walk_paths(og, [int(seeds[0])], 2, 100)
        assert [tuple(tuple(int(x) for x in t) for t in p) for p in pr.paths] == orc.paths_as_triples(og, ref_p)
        assert pr.truncated == ref_t
        # the same world with each process paging its hub slices through a K7
        # hub cache (one page holds every slice here: hits after the first wave)
        del pg
        pc = th.PartitionedGraph((s, r, o), E, R, xch, n_hubs=8, hub_cache_pages=2)
        for sem in ("frontier", "exact"):
            res = pc.retrieve(seeds, 2, semantics=sem, activated=True)
            for i in range(0, 150, 11):
                ref = orc.retrieve_one(og, int(seeds[i]), 2, sem)
                for h in range(2):
                    assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h])
                    assert np.array_equal(res.activated(i, h + 1), ref["activated"][h])
        (st,) = pc.hub_cache_stats()
        c = st["counters"]
        assert c.hits > 0 and c.loads == c.misses <= st["pages"] and c.evictions == 0
    except BaseException as e:  # pragma: no cover - reported to the parent
        with open(errfile, "a") as f:
            f.write(f"rank {rank}: {type(e).__name__}: {e}\n")
        raise
    finally:
        dist.destroy_process_group()


def test_two_processes_with_cuda_shards(tmp_path):
    import socket

    import torch

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    errfile = str(tmp_path / "err.txt")
    torch.multiprocessing.spawn(_gpu_dist_worker, args=(2, port, errfile), nprocs=2, join=True)
    import os

    assert not os.path.exists(errfile), open(errfile).read()


def test_run_batch_on_sharded_graph(th):
    """run_batch packs equal-k queries into waves on a rank-sharded graph;
    every per-query trace equals single-graph k_hop, failures stay isolated."""
    s, r, o = _hub_graph(1500, 30000, 24, seed=21)
    E, R = 1500, 24
    g = th.build_incidence((s, r, o), E, R)
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(2), n_hubs=5)
    rng = np.random.default_rng(8)
    qs = [th.BatchQuery(i, th.EntityVector(rng.integers(0, E, int(rng.integers(0, 5))), E), int(rng.integers(1, 4)))
          for i in range(40)]
    qs.insert(7, th.BatchQuery("bad", th.EntityVector(np.array([1]), E), 0))
    plan = th.plan_partitions((s, E), 3)
    batch = th.plan_batch(qs, plan)
    # (a width mismatch fails planning already, as route does; run it unplanned)
    qs.append(th.BatchQuery("wide", th.EntityVector(np.array([1]), E + 1), 2))
    batch = th.QueryBatch(qs, batch.execution_order + [len(qs) - 1])
    for sem in ("frontier", "exact", "cumulative"):
        res = th.run_batch(batch, pg, sem)
        for q, br in zip(qs, res):
            assert br.query_id == q.query_id
            if q.k < 1 or q.q0.width != E:
                assert br.trace is None and br.error.startswith("ValueError")
                continue
            ref = th.k_hop(q.q0, q.k, g, th.HopSemantics.parse(sem))
            for h in range(1, q.k + 1):
                assert np.array_equal(br.trace.frontier(h).ids, ref.frontier(h).ids), (q.query_id, h)
                assert np.array_equal(br.trace.activated(h).ids, ref.activated(h).ids), (q.query_id, h)


@pytest.mark.parametrize("world,n_hubs", [(1, 0), (2, 12), (4, 40)])
def test_sharded_paths_equal_single_graph_k5(th, world, n_hubs):
    """Sharded walk enumeration (counts + capped offers between ranks) ==
    the single-graph K5 kernel on a hub-heavy graph: hub seeds whose walk
    counts dwarf the cap, multi-seed sets, uncapped small cases."""
    s, r, o = _hub_graph(20000, 400000, 32, seed=5)
    E, R = 20000, 32
    g = th.build_incidence((s, r, o), E, R)
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(world), n_hubs=n_hubs)
    deg = np.bincount(s, minlength=E)
    hubs = np.argsort(-deg)[:5]
    rng = np.random.default_rng(world)
    cases = [([int(hubs[0])], 3, 10_000), ([int(hubs[1]), int(hubs[2])], 2, 10_000), ([int(hubs[3])], 3, 7),
             (sorted(set(rng.integers(0, E, 6).tolist())), 3, 2_500), ([int(rng.integers(0, E))], 2, None),
             ([int(hubs[4])], 1, None), ([int(hubs[0])], 2, 0)]
    for seeds, k, cap in cases:
        q0 = th.EntityVector(seeds, E)
        a = th.cross_graph_paths(q0, k, pg, cap)
        b = th.reconstruct_paths(q0, k, g, cap)
        assert a.paths == b.paths, (seeds, k, cap)
        assert a.truncated == b.truncated
