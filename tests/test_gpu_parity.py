"""GPU parity: the CUDA path (through the C ABI) against the golden vectors
and the CPU oracle.  Integer/index work, so the bar is bit-exact."""

import numpy as np
import pytest

from golden_io import all_cases, load_case
from oracle import khop_oracle as orc

pytestmark = pytest.mark.gpu
CASES = all_cases()


@pytest.fixture(scope="module")
def th(cuda_device):
    import paper_2604_18913_b200 as th

    return th


def _masks_for(th, q, n_relations, device):
    import torch

    if q.relations is None:
        return None
    from paper_2604_18913_b200.retriever import _relation_masks

    w = _relation_masks(q.relations, 1, n_relations)
    return torch.from_numpy(w.view(np.int32)).to(device)


@pytest.mark.parametrize("path", CASES, ids=[p.stem for p in CASES])
def test_golden_case_query_by_query(th, path, cuda_device):
    """Every reference golden query (seed sets, filters, caps) through Retriever.run."""
    import torch

    case = load_case(path)
    g = th.build_incidence((case.subj, case.rel, case.obj), case.n_entities, case.n_relations)
    ret = th.Retriever(g)
    for q in case.queries:
        seeds = torch.tensor(sorted(set(q.seeds)), dtype=torch.int32, device=cuda_device)
        offs = torch.tensor([0, seeds.numel()], dtype=torch.int32, device=cuda_device)
        masks = _masks_for(th, q, case.n_relations, cuda_device)
        r = ret.run(offs, seeds, q.k, q.semantics, masks, activated=True, paths=q.want_paths,
                    max_paths=q.max_paths if q.want_paths else 0, singleton=seeds.numel() == 1)
        for h in range(q.k):
            assert np.array_equal(r.frontier(0, h + 1), q.frontiers[h]), (case.name, q.seeds, h)
            assert np.array_equal(r.activated(0, h + 1), q.activated[h]), (case.name, q.seeds, h)
            assert int(r.edges[h, 0]) == q.activated[h].size
        if q.want_paths:
            assert r.path_tid_tuples(0) == q.paths, (case.name, q.seeds, q.max_paths)
            assert r.truncated(0) == q.truncated


@pytest.mark.parametrize("path", CASES, ids=[p.stem for p in CASES])
def test_golden_case_batched_retrieve(th, path):
    """All single-seed golden queries of a case, batched by (k, semantics, filter)."""
    case = load_case(path)
    g = th.build_incidence((case.subj, case.rel, case.obj), case.n_entities, case.n_relations)
    groups = {}
    for q in case.queries:
        if len(q.seeds) == 1:
            key = (q.k, q.semantics, q.want_paths, q.max_paths)
            groups.setdefault(key, []).append(q)
    for (k, sem, want_p, maxp), qs in groups.items():
        seeds = [q.seeds[0] for q in qs]
        filt = [q.relations if q.relations is not None else list(range(case.n_relations)) for q in qs]
        r = th.retrieve(g, seeds, k, relation_filter=filt, semantics=sem, paths=want_p,
                        max_paths=maxp if want_p else 0, activated=True)
        for i, q in enumerate(qs):
            for h in range(k):
                assert np.array_equal(r.frontier(i, h + 1), q.frontiers[h])
                assert np.array_equal(r.activated(i, h + 1), q.activated[h])
            if want_p:
                assert r.path_tid_tuples(i) == q.paths
                assert r.truncated(i) == q.truncated


def test_reference_api_dropin_tiny(th):
    """The reference's own tiny-graph assertions (tests/test_incidence.py:54-221)."""
    A, B, C = 0, 1, 2
    tiny = [(A, 0, B), (B, 1, C), (A, 0, C), (C, 2, A)]
    g = th.build_incidence(tiny, 3, 3)
    assert g.sub_row(A).tolist() == [0, 2]
    assert g.sub_row(B).tolist() == [1]
    assert g.obj.tolist() == [B, C, C, A]
    assert g.rel.tolist() == [0, 1, 0, 2]
    ev = th.EntityVector
    act, nxt = th.one_hop(ev([A], 3), g)
    assert act.ids.tolist() == [0, 2] and nxt.ids.tolist() == [B, C]
    act, nxt = th.one_hop(ev([B, C], 3), g)
    assert act.ids.tolist() == [1, 3] and nxt.ids.tolist() == [A, C]
    tr = th.k_hop(ev([A], 3), 2, g, th.HopSemantics.EXACT_WALK)
    assert tr.frontier(1).ids.tolist() == [B, C] and tr.frontier(2).ids.tolist() == [A, C]
    tr = th.k_hop(ev([A], 3), 2, g, th.HopSemantics.FRONTIER)
    assert tr.frontier(2).ids.tolist() == []
    with pytest.raises(ValueError):
        th.k_hop(ev([A], 3), 0, g)
    with pytest.raises(ValueError):
        th.k_hop(ev([A], 4), 1, g)
    res = th.reconstruct_paths(ev([A], 3), 2, g)
    T = th.Triple
    assert res.paths == [(T(A, 0, B), T(B, 1, C)), (T(A, 0, C), T(C, 2, A))] and not res.truncated
    res = th.reconstruct_paths(ev([B], 3), 2, g, max_paths=1)
    assert res.paths == [(T(B, 1, C), T(C, 2, A))] and res.truncated is False
    res = th.reconstruct_paths(ev([A], 3), 2, g, max_paths=0)
    assert res.paths == [] and res.truncated is True
    with pytest.raises(ValueError):
        th.reconstruct_paths(ev([A], 3), 2, g, max_paths=-1)
    with pytest.raises(ValueError):
        th.build_incidence([(5, 0, 0)], 2, 1)
    with pytest.raises(ValueError):
        th.build_incidence([(0, 3, 0)], 2, 1)


def _hub_graph(E, T, R, seed, alpha=1.2):
    """Hub-to-hub power-law graph (same ranks for subjects and objects)."""
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


@pytest.mark.parametrize("k4", ["dense", "list", "list_nb", "list_t", "screen", "screen2"])
@pytest.mark.parametrize("divisor", [0.0, -1.0, 8.0], ids=["push", "pull", "auto"])
@pytest.mark.parametrize("sem", ["exact", "frontier", "cumulative"])
def test_hub_graph_two_waves_vs_oracle(th, sem, divisor, k4):
    """1,100 seeds (two waves), hub rows above the heavy thresholds, every
    direction policy, both K4 strategies; checked against the oracle seed by seed."""
    s, r, o = _hub_graph(3000, 100000, 64, seed=11)
    E, R = 3000, 64
    g = th.build_incidence((s, r, o), E, R)
    st = g.stats()
    assert st["max_out_degree"] > 4096 and st["max_in_degree"] > 4096
    og = orc.build_csr(s, r, o, E, R)
    rng = np.random.default_rng(3)
    seeds = rng.integers(0, E, 1100)
    ret = th.Retriever(g)
    ret.set_pull_divisor(divisor)
    ret.set_list_min_entities(0 if k4 != "dense" else 1 << 40)
    ret.set_k4_mode(0 if k4 == "list_t" else 1)  # list_t: the transposing list-driven K4
    ret.set_knob("k4_bucket", 0 if k4 == "list_nb" else 1)  # list: bucketed write; list_nb: transposing
    # screen: per-lane item screening in pulls; screen2: screen kernel + compacted pull
    ret.set_pull_screen({"screen": 1, "screen2": 2}.get(k4, 0))
    k = 3
    res = ret.retrieve(seeds, k, semantics=sem)
    if divisor == 0.0:
        assert res.pull_hops == 0
    if divisor < 0:
        assert res.push_hops == 0
    check = list(range(0, 1100, 37)) + [1099]
    for i in check:
        ref = orc.retrieve_one(og, int(seeds[i]), k, sem)
        for h in range(k):
            assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h]), (i, h)
            assert int(res.edges[h, i]) == ref["edges"][h]


@pytest.mark.parametrize("max_paths", [1, 7, 300, 5000])
@pytest.mark.parametrize("filtered", [False, True])
def test_k2_paths_cta_kernel_vs_dfs_and_oracle(th, max_paths, filtered):
    """k = 2 capped singleton path queries take the CTA-per-query kernel
    (paths_k2_kernel); it must equal the one-warp DFS and the oracle --
    paths in order, counts and truncation -- on hub seeds with rows longer
    than a 2,048-slot sweep step, with and without relation filters."""
    s, r, o = _hub_graph(3000, 120000, 40, seed=17)
    E, R = 3000, 40
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    deg = np.diff(og.indptr)
    rng = np.random.default_rng(4)
    seeds = np.concatenate([np.argsort(-deg)[:24], rng.integers(0, E, 40)])
    filt = [sorted(rng.choice(R, 5, replace=False).tolist()) for _ in seeds] if filtered else None
    out = {}
    for k2 in (1, 0):
        ret = th.Retriever(g)
        ret.set_paths_k2(bool(k2))
        out[k2] = ret.retrieve(seeds, 2, relation_filter=filt, paths=True, max_paths=max_paths)
    n_trunc = 0
    for i, sd in enumerate(seeds.tolist()):
        assert out[1].path_tid_tuples(i) == out[0].path_tid_tuples(i), (i, sd)
        assert out[1].truncated(i) == out[0].truncated(i), (i, sd)
        if i % 4 == 0:
            ref = orc.retrieve_one(og, sd, 2, "frontier", None if filt is None else filt[i], paths=True,
                                   max_paths=max_paths)
            assert out[1].path_tid_tuples(i) == ref["paths"], (i, sd)
            assert out[1].truncated(i) == ref["truncated"]
        n_trunc += out[1].truncated(i)
    assert n_trunc > 0


def test_filtered_hub_graph_vs_oracle(th):
    s, r, o = _hub_graph(2000, 40000, 40, seed=5)
    E, R = 2000, 40
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    rng = np.random.default_rng(9)
    seeds = rng.integers(0, E, 300)
    filt = [sorted(rng.choice(R, 6, replace=False).tolist()) for _ in seeds]
    for divisor, k4 in ((0.0, 1 << 40), (-1.0, 0)):
        ret = th.Retriever(g)
        ret.set_pull_divisor(divisor)
        ret.set_list_min_entities(k4)
        res = ret.retrieve(seeds, 2, relation_filter=filt, semantics="frontier", paths=True,
                           max_paths=300, activated=True)
        for i in range(0, 300, 7):
            ref = orc.retrieve_one(og, int(seeds[i]), 2, "frontier", filt[i], paths=True, max_paths=300)
            for h in range(2):
                assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h])
                assert np.array_equal(res.activated(i, h + 1), ref["activated"][h])
                assert int(res.edges[h, i]) == ref["edges"][h]
            assert res.path_tid_tuples(i) == ref["paths"]
            assert res.truncated(i) == ref["truncated"]


def test_bad_inputs(th):
    g = th.build_incidence([(0, 0, 1), (1, 0, 2)], 3, 1)
    with pytest.raises(ValueError):
        th.retrieve(g, [3], 1)
    with pytest.raises(ValueError):
        th.retrieve(g, [0], 0)
    with pytest.raises(ValueError):
        th.retrieve(g, [0], 1, relation_filter=[1])
    r = th.retrieve(g, [], 2)
    assert r.n_queries == 0
    import torch

    bad = torch.tensor([0, 7], dtype=torch.int32, device=g.device)
    with pytest.raises(ValueError):
        th.retrieve(g, bad, 2)
    # the session is still usable after a failed call
    r = th.retrieve(g, [0, 1, 2], 2, semantics="exact")
    assert r.frontier(0, 1).tolist() == [1] and r.frontier(0, 2).tolist() == [2]
    assert r.frontier(2, 1).tolist() == []


def test_empty_graph_and_isolated(th):
    g = th.build_incidence([], 4, 2)
    r = th.retrieve(g, [0, 3], 3, semantics="cumulative", paths=True)
    for i in range(2):
        for h in range(1, 4):
            assert r.frontier(i, h).size == 0
        assert r.path_tid_tuples(i) == [] and not r.truncated(i)


@pytest.mark.parametrize("filtered", [False, True])
def test_dense_pull_matches_flag_tested_pull(th, filtered):
    """Pull hops with and without the per-edge frontier test (dense_pull
    1e9 forces the unconditional gather, 0 disables it) agree with the oracle."""
    s, r, o = _hub_graph(2500, 50000, 24, seed=17)
    E, R = 2500, 24
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    rng = np.random.default_rng(2)
    seeds = rng.integers(0, E, 400)
    filt = [sorted(rng.choice(R, 10, replace=False).tolist()) for _ in seeds] if filtered else None
    out = []
    for dense in (0.0, 1e9):
        ret = th.Retriever(g)
        ret.set_pull_divisor(-1.0)
        ret.set_dense_pull(dense)
        out.append(ret.retrieve(seeds, 3, relation_filter=filt, semantics="frontier"))
    a, b = out
    assert bool((a.edges == b.edges).all())
    for i in range(400):  # (segment placement in the id array is not part of the contract)
        for h in range(3):
            assert np.array_equal(a.frontier(i, h + 1), b.frontier(i, h + 1))
    for i in range(0, 400, 23):
        ref = orc.retrieve_one(og, int(seeds[i]), 3, "frontier", None if filt is None else filt[i])
        for h in range(3):
            assert np.array_equal(b.frontier(i, h + 1), ref["frontiers"][h]), (i, h)


@pytest.mark.parametrize("pair", [0, 1])
@pytest.mark.parametrize("filtered", [False, True])
@pytest.mark.parametrize("sem", ["exact", "frontier", "cumulative"])
def test_two_phase_pull_every_hop_vs_oracle(th, sem, filtered, pair):
    """The two-phase pull (edge screen + gather over compacted frontier
    in-edges) forced on every hop and never dense, on a hub graph whose
    in-rows split over several pull items (merged with atomics) and whose
    whole rows straddle the screen's chunk and warp-range boundaries;
    with and without relation filters and two rows per lane group."""
    s, r, o = _hub_graph(3000, 100000, 64, seed=23)
    E, R = 3000, 64
    g = th.build_incidence((s, r, o), E, R)
    assert g.stats()["max_in_degree"] > 32  # split rows
    og = orc.build_csr(s, r, o, E, R)
    rng = np.random.default_rng(5)
    seeds = rng.integers(0, E, 700)
    filt = None
    if filtered:
        filt = [sorted(rng.choice(R, 20, replace=False).tolist()) for _ in seeds]
    ret = th.Retriever(g)
    ret.set_pull_divisor(-1.0)  # every hop pulls
    ret.set_dense_pull(0.0)  # never the dense (unscreened) form
    ret.set_pull_screen(2)
    ret.set_knob("pull_pair", pair)
    k = 3
    res = ret.retrieve(seeds, k, relation_filter=filt, semantics=sem)
    assert res.push_hops == 0
    for i in list(range(0, 700, 29)) + [699]:
        ref = orc.retrieve_one(og, int(seeds[i]), k, sem, None if filt is None else filt[i])
        for h in range(k):
            assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h]), (i, h)
            assert int(res.edges[h, i]) == ref["edges"][h], (i, h)
