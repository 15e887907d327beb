"""Randomised parity sweep over the engine's strategy switches: wave widths
(B from 1 to past one wave), k = 1..4, every semantics, relation filters,
K4 dense (mask cache) / list-driven (incl. the bit-sliced count pass and
the first-layer row list), push / pull / auto directions, CUDA-graph
replay -- each case against the oracle on sampled seeds."""

import numpy as np
import pytest

from oracle import khop_oracle as orc
from test_gpu_parity import _hub_graph

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(2026)
    out = []
    for i in range(60):
        out.append(dict(
            E=int(rng.integers(50, 1500)), T=int(rng.integers(200, 20000)), R=int(rng.integers(1, 40)),
            alpha=float(rng.choice([0.8, 1.1, 1.4])), B=int(rng.choice([1, 7, 32, 33, 200, 1024, 1100])),
            k=int(rng.integers(1, 5)), sem=str(rng.choice(["exact", "frontier", "cumulative"])),
            filt=bool(rng.random() < 0.35), list_mode=bool(rng.random() < 0.5),
            k4_mode=int(rng.integers(0, 3)), screen=int(rng.integers(-1, 3)),
            bucket=bool(rng.random() < 0.7),
            divisor=float(rng.choice([0.0, -1.0, 8.0])),
            paths=bool(rng.random() < 0.3), max_paths=[0, 5, 100, None][int(rng.integers(0, 4))], seed=i))
    return out


@pytest.mark.parametrize("c", _cases(), ids=lambda c: f"s{c['seed']}")
def test_random_configuration(th_mod, c):
    th = th_mod
    s, r, o = _hub_graph(c["E"], c["T"], c["R"], seed=c["seed"], alpha=c["alpha"])
    E, R = c["E"], c["R"]
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    rng = np.random.default_rng(c["seed"] + 100)
    ret = th.Retriever(g)
    ret.set_pull_divisor(c["divisor"])
    ret.set_list_min_entities(0 if c["list_mode"] else 1 << 40)
    ret.set_k4_mode(c["k4_mode"])
    ret.set_pull_screen(c["screen"])
    ret.set_knob("k4_bucket", int(c["bucket"]))
    for rep in range(3):  # eager run, graph capture, replay (new seeds each time)
        seeds = rng.integers(0, E, c["B"])
        filt = None
        if c["filt"]:
            filt = [sorted(rng.choice(R, max(1, R // 3), replace=False).tolist()) for _ in range(c["B"])]
        paths = c["paths"] and c["k"] <= 3
        res = ret.retrieve(seeds, c["k"], relation_filter=filt, semantics=c["sem"], paths=paths,
                           max_paths=c["max_paths"])
        for i in sorted(set([0, c["B"] - 1, c["B"] // 2])):
            ref = orc.retrieve_one(og, int(seeds[i]), c["k"], c["sem"], None if filt is None else filt[i],
                                   paths=paths, max_paths=c["max_paths"])
            for h in range(c["k"]):
                assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h]), (rep, i, h)
                assert int(res.edges[h, i]) == ref["edges"][h], (rep, i, h)
            if paths:
                assert res.path_tid_tuples(i) == ref["paths"], (rep, i)
                assert res.truncated(i) == ref["truncated"], (rep, i)


@pytest.fixture(scope="module")
def th_mod(cuda_device):
    import paper_2604_18913_b200 as th

    return th


@pytest.mark.parametrize("direction", [0.0, -1.0, 8.0], ids=["push", "pull", "auto"])
@pytest.mark.parametrize("list_mode", [False, True, 2], ids=["dense", "list", "list_t"])
def test_overlapped_layers_repeatedly(th_mod, direction, list_mode):
    """The overlapped K4s of consecutive layers (two streams) under many
    repeats: FRONTIER, frontiers only, k = 4, graphs replayed -- every
    segment checked against the oracle (races show up as wrong ids with the
    right counts)."""
    th = th_mod
    s, r, o = _hub_graph(1400, 15000, 3, seed=77, alpha=1.1)
    E, R = 1400, 3
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    ret = th.Retriever(g)
    ret.set_pull_divisor(direction)
    ret.set_list_min_entities(0 if list_mode else 1 << 40)
    ret.set_k4_mode(0 if list_mode == 2 else 1)
    rng = np.random.default_rng(5)
    refs = {}
    for rep in range(12):
        B = int(rng.choice([1, 3, 40]))
        seeds = rng.integers(0, E, B)
        res = ret.retrieve(seeds, 4)
        for i in range(B):
            sd = int(seeds[i])
            if sd not in refs:
                refs[sd] = orc.retrieve_one(og, sd, 4, "frontier")
            for h in range(4):
                assert np.array_equal(res.frontier(i, h + 1), refs[sd]["frontiers"][h]), (rep, i, h)


@pytest.mark.parametrize("seed", range(8))
def test_random_seed_sets_reference_api(th_mod, seed):
    """Multi-seed queries through the reference API (k_hop with activated
    sets, reconstruct_paths with caps): the non-singleton engine path."""
    th = th_mod
    rng = np.random.default_rng(seed)
    E, T, R = int(rng.integers(30, 600)), int(rng.integers(50, 5000)), int(rng.integers(1, 8))
    s, r, o = _hub_graph(E, T, R, seed=seed + 300, alpha=float(rng.choice([0.9, 1.2])))
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    for _ in range(3):
        ids = np.unique(rng.integers(0, E, int(rng.integers(1, 12))))
        k = int(rng.integers(1, 4))
        sem = str(rng.choice(["exact", "frontier", "cumulative"]))
        tr = th.k_hop(th.EntityVector(ids, E), k, g, th.HopSemantics.parse(sem))
        ref = orc.hop_trace(og, ids, k, sem)
        for h in range(k):
            assert np.array_equal(tr.frontier(h + 1).ids, ref[h][0]), (sem, h)
            assert np.array_equal(tr.activated(h + 1).ids, ref[h][1]), (sem, h)
        cap = [0, 3, 50, None][int(rng.integers(0, 4))]
        pr = th.reconstruct_paths(th.EntityVector(ids, E), k, g, max_paths=cap)
        want, trunc = orc.walk_paths(og, ids, k, cap)
        got = [tuple(tuple(int(x) for x in t) for t in p) for p in pr.paths]
        assert got == orc.paths_as_triples(og, want), (ids.tolist(), k, cap)
        assert pr.truncated == trunc


@pytest.mark.parametrize("seed", range(6))
def test_random_partitioned_graphs(th_mod, seed):
    """Random graphs on 1-4 loopback ranks (hash owners, edge-split hubs,
    push/pull/auto directions across partitions) against the single-graph
    engine: frontier and activated sets and edge counts per seed."""
    th = th_mod
    rng = np.random.default_rng(seed + 900)
    E, T, R = int(rng.integers(100, 1500)), int(rng.integers(300, 15000)), int(rng.integers(1, 10))
    s, r, o = _hub_graph(E, T, R, seed=seed + 500, alpha=float(rng.choice([0.9, 1.2, 1.4])))
    world = int(rng.integers(1, 5))
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(world), n_hubs=int(rng.integers(0, 12)))
    pg.pull_divisor = float(rng.choice([0.0, 8.0, 1e9]))
    g = th.build_incidence((s, r, o), E, R)
    seeds = rng.integers(0, E, int(rng.choice([1, 17, 300])))
    k = int(rng.integers(1, 4))
    sem = str(rng.choice(["exact", "frontier", "cumulative"]))
    filt = None
    if rng.random() < 0.3:
        filt = [sorted(rng.choice(R, max(1, R // 2), replace=False).tolist()) for _ in seeds]
    a = pg.retrieve(seeds, k, relation_filter=filt, semantics=sem, activated=True)
    b = th.Retriever(g).retrieve(seeds, k, relation_filter=filt, semantics=sem, activated=True)
    for i in range(len(seeds)):
        for h in range(k):
            assert np.array_equal(a.frontier(i, h + 1), b.frontier(i, h + 1)), (world, i, h)
            assert np.array_equal(a.activated(i, h + 1), b.activated(i, h + 1)), (world, i, h)
            assert int(a.edges[h, i]) == int(b.edges[h, i]), (world, i, h)


def test_duplicate_seeds_in_a_query(th_mod):
    """th_query allows duplicate seeds: a set query with repeats equals the
    deduplicated one (frontiers and hop-1 edge counts from seed init)."""
    import torch

    th = th_mod
    s, r, o = _hub_graph(300, 3000, 4, seed=3)
    g = th.build_incidence((s, r, o), 300, 4)
    ret = th.Retriever(g)
    dev = g.device
    dup = torch.tensor([5, 5, 7, 5, 7, 11], dtype=torch.int32, device=dev)
    uniq = torch.tensor([5, 7, 11], dtype=torch.int32, device=dev)
    for sem in ("exact", "frontier", "cumulative"):
        a = ret.run(torch.tensor([0, 6], dtype=torch.int32, device=dev), dup, 3, sem, copy=True)
        b = ret.run(torch.tensor([0, 3], dtype=torch.int32, device=dev), uniq, 3, sem, copy=True)
        assert bool((a.edges == b.edges).all()), sem
        for h in range(3):
            assert np.array_equal(a.frontier(0, h + 1), b.frontier(0, h + 1)), (sem, h)


@pytest.mark.parametrize("cache_filtered", [0, 1])
@pytest.mark.parametrize("k", [2, 3])
def test_filtered_waves_with_and_without_mask_cache(th_mod, cache_filtered, k):
    """Relation-filtered waves skip K4's tile-mask cache by default
    (k4_cache_filtered = 0); both forms against the oracle."""
    th = th_mod
    E, T, R = 1400, 24000, 30
    s, r, o = _hub_graph(E, T, R, seed=11 + k, alpha=1.1)
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    rng = np.random.default_rng(5 + k)
    ret = th.Retriever(g)
    ret.set_knob("k4_cache_filtered", cache_filtered)
    for rep in range(3):  # eager, capture, replay
        seeds = rng.integers(0, E, 1024)
        filt = [sorted(rng.choice(R, 10, replace=False).tolist()) for _ in range(1024)]
        res = ret.retrieve(seeds, k, relation_filter=filt)
        for i in (0, 1, 511, 1023):
            ref = orc.retrieve_one(og, int(seeds[i]), k, "frontier", filt[i])
            for h in range(k):
                assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h]), (rep, i, h)
                assert int(res.edges[h, i]) == ref["edges"][h]
