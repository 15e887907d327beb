"""K7 hub-adjacency cache (csrc/hubcache.cu): a shard's hub
slices paged through a budget of HBM pages on demand.

* results with the cache are bit-identical to the resident shard, the
  single-graph engine and the oracle (frontier, activated, edge counts);
* the access trace is exactly the pages of each hop's frontier hubs, resident
  ones first in recency order, then the misses ascending;
* the counters equal the independent LRU model over that trace
  (tests/lru_model.py; the reference's algebra, cache.py:38-117) and so does
  the final resident set;
* a hop whose hubs need more pages than the budget fails loudly and leaves
  the shard usable."""

import numpy as np
import pytest

from lru_model import simulate_lru
from oracle import khop_oracle as orc

pytestmark = pytest.mark.gpu

E, R, N_HUBS = 200_000, 40, 12


@pytest.fixture(scope="module")
def th(cuda_device):
    import paper_2604_18913_b200 as th

    return th


@pytest.fixture(scope="module")
def graph():
    """12 hubs of 0.3M-1.4M out-edges (~10M edges, several 1M-edge pages)
    into non-hub entities, a 1M-edge background among non-hubs, and one
    pointer entity per hub (pointer -> hub) so hubs also enter later hops."""
    rng = np.random.default_rng(11)
    hubs = rng.choice(E, N_HUBS, replace=False)
    is_hub = np.zeros(E, bool)
    is_hub[hubs] = True
    plain = np.flatnonzero(~is_hub)
    deg = rng.integers(300_000, 1_400_000, N_HUBS)
    s = [np.repeat(hubs, deg), rng.choice(plain, 1_000_000)]
    o = [rng.choice(plain, int(deg.sum())), rng.choice(plain, 1_000_000)]
    pointers = rng.choice(plain, N_HUBS, replace=False)
    s.append(pointers)
    o.append(hubs)
    s, o = np.concatenate(s), np.concatenate(o)
    r = rng.integers(0, R, s.size)
    key = np.unique((s.astype(np.int64) * R + r) * E + o)
    key = rng.permutation(key)
    s, r, o = (key // E // R).astype(np.int32), ((key // E) % R).astype(np.int32), (key % E).astype(np.int32)
    return s, r, o, hubs, pointers


def _pages_of_hubs(pg, graph, page_edges):
    """Page numbers of each hub row in a one-rank shard (hub rows follow the
    owned rows in hub-index order; the hub region starts on a page)."""
    s = graph[0]
    deg = np.bincount(s, minlength=E)[pg.plan.hub_ids]
    cum = np.concatenate([[0], np.cumsum(deg)])
    return {int(h): set(range(cum[i] // page_edges, (cum[i + 1] - 1) // page_edges + 1))
            for i, h in enumerate(pg.plan.hub_ids.tolist()) if deg[i]}


def _same(a, b, n, k):
    for i in range(n):
        for h in range(1, k + 1):
            assert np.array_equal(a.frontier(i, h), b.frontier(i, h)), (i, h)
            assert np.array_equal(a.activated(i, h), b.activated(i, h)), (i, h)
    assert np.array_equal(np.asarray(a.edges.cpu()), np.asarray(b.edges.cpu()))


def test_hub_cache_parity_trace_and_counters(th, graph):
    s, r, o, hubs, pointers = graph
    cap = 6
    plain = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(1), n_hubs=N_HUBS)
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(1), n_hubs=N_HUBS, hub_cache_pages=cap)
    assert set(pg.plan.hub_ids.tolist()) == set(hubs.tolist())
    (st,) = pg.hub_cache_stats()
    pe = st["page_edges"]
    assert st["capacity"] == cap and st["resident"] == 0
    assert st["pages"] == -(-int(np.isin(s, hubs).sum()) // pe) > cap  # evictions will happen
    pages = _pages_of_hubs(pg, graph, pe)
    shard = pg.shards[0]
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    rng = np.random.default_rng(5)
    plainids = np.setdiff1d(np.arange(E), hubs)
    model = []  # the LRU order (least recent first) the cache must follow
    trace = []
    for w in range(10):
        # hop 1: two hub seeds; k=2 waves add the pointers of two other hubs,
        # whose hubs are in hop 2's frontier
        hs = rng.choice(N_HUBS, 4, replace=False)
        seeds = np.concatenate([hubs[hs[:2]], rng.choice(plainids, 30)])
        k = 1 + (w % 2)
        if k == 2:
            seeds = np.concatenate([seeds, pointers[hs[2:]]])
        filt = None if w % 3 else [list(rng.choice(R, 12, replace=False)) for _ in seeds]
        got = pg.retrieve(seeds, k, relation_filter=filt, activated=True)
        _same(got, plain.retrieve(seeds, k, relation_filter=filt, activated=True), seeds.size, k)
        _same(got, th.retrieve(g, seeds, k, relation_filter=filt, activated=True), seeds.size, k)
        for i in (0, 1, seeds.size - 1):
            ref = orc.retrieve_one(og, int(seeds[i]), k, "frontier", None if filt is None else filt[i])
            for h in range(k):
                assert np.array_equal(got.frontier(i, h + 1), ref["frontiers"][h])
                assert np.array_equal(got.activated(i, h + 1), ref["activated"][h])
        # expected accesses: per hop the pages of the frontier's hubs (a wave
        # whose result buffers had to grow ran again: its accesses repeat)
        hop_sets, layer = [], set(seeds.tolist())
        for h in range(1, k + 1):
            hop_sets.append(set().union(*(pages[x] for x in layer if x in pages)))
            layer = set(np.concatenate([got.frontier(i, h) for i in range(seeds.size)]).tolist())
        dev = shard.hub_cache_trace()
        for runs in (1, 2, 3):
            m, t = list(model), []
            for want in hop_sets * runs:
                hit = [p for p in m if p in want]
                miss = sorted(want - set(hit))
                for p in hit:
                    m.remove(p)
                    m.append(p)
                for p in miss:
                    if len(m) == cap:
                        m.pop(0)
                    m.append(p)
                t += hit + miss
            if t == dev:
                break
        assert t == dev, (w, runs)
        model, trace = m, trace + t
    assert shard.hub_cache_trace() == []  # the log was handed over
    final = []
    (st,) = pg.hub_cache_stats()
    assert st["counters"] == simulate_lru(trace, cap, final)
    assert shard.hub_cache_resident() == final == model
    c = st["counters"]
    assert c.evictions > 0 and c.hits > 0 and c.loads == c.misses
    assert c.evictions == c.loads - st["resident"]


def test_hub_cache_budget_too_small_fails_loudly(th, graph):
    s, r, o, hubs, _ = graph
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(1), n_hubs=N_HUBS, hub_cache_pages=2)
    with pytest.raises(ValueError, match="pages"):
        pg.retrieve(hubs, 1)  # all twelve hubs span ~10 pages
    # the shard stays usable
    g = th.build_incidence((s, r, o), E, R)
    seeds = hubs[:1]
    got = pg.retrieve(seeds, 1, activated=True)
    _same(got, th.retrieve(g, seeds, 1, activated=True), 1, 1)


def test_hub_cache_two_ranks(th, graph):
    """World 2 on one device: each rank pages its half of every hub row."""
    s, r, o, hubs, pointers = graph
    plain = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(2), n_hubs=N_HUBS)
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(2), n_hubs=N_HUBS, hub_cache_pages=8)
    rng = np.random.default_rng(9)
    for w in range(4):
        seeds = np.concatenate([hubs[rng.choice(N_HUBS, 3, replace=False)],
                                pointers[rng.choice(N_HUBS, 2, replace=False)], rng.integers(0, E, 40)])
        for sem in ("frontier", "exact", "cumulative"):
            a = pg.retrieve(seeds, 2, semantics=sem, activated=True)
            b = plain.retrieve(seeds, 2, semantics=sem, activated=True)
            _same(a, b, seeds.size, 2)
    for sh, st in zip(pg.shards, pg.hub_cache_stats()):
        tr = sh.hub_cache_trace()
        assert st["counters"] == simulate_lru(tr, 8)
        assert st["counters"].hits + st["counters"].misses == len(tr) > 0
