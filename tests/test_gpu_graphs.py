"""CUDA-graph replay of repeated batch shapes (engine.cu run_graphed).

A session captures the second run of a shape and replays it from then on;
every replayed result must equal an eager session's, bit for bit, while the
seeds, masks and output capacities change underneath it."""

import numpy as np
import pytest

from oracle import khop_oracle as orc
from test_gpu_parity import _hub_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def th(cuda_device):
    import paper_2604_18913_b200 as th

    return th


def _segments(off, ln, ids):
    off, ln, ids = off.cpu().numpy(), ln.cpu().numpy(), ids.cpu().numpy()
    return [ids[o:o + n].tolist() for o, n in zip(off.ravel(), ln.ravel())]


def _same(a, b):
    """Same results.  Where the per-(hop, query) segments sit in the id
    arrays is not part of the contract (consecutive layers' K4s reserve
    their output ranges concurrently), so frontiers and activated sets are
    compared segment by segment; everything else exactly."""
    for name in ("edges", "frontier_len", "act_len", "path_off", "path_count", "path_tids",
                 "path_truncated"):
        x, y = getattr(a, name), getattr(b, name)
        assert (x is None) == (y is None), name
        if x is not None:
            assert x.shape == y.shape and bool((x == y).all()), name
    for pre in ("frontier", "act"):
        ids = "frontier_ids" if pre == "frontier" else "act_ids"
        if getattr(a, ids) is None:
            assert getattr(b, ids) is None
            continue
        sa = _segments(getattr(a, pre + "_off"), getattr(a, pre + "_len"), getattr(a, ids))
        sb = _segments(getattr(b, pre + "_off"), getattr(b, pre + "_len"), getattr(b, ids))
        assert sa == sb, pre


@pytest.mark.parametrize("paths", [False, True], ids=["frontier", "paths"])
@pytest.mark.parametrize("sem", ["exact", "frontier", "cumulative"])
def test_replay_matches_eager(th, sem, paths):
    s, r, o = _hub_graph(3000, 60000, 48, seed=21)
    E, R = 3000, 48
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    graphed, eager = th.Retriever(g), th.Retriever(g)
    eager.set_graphs(False)
    rng = np.random.default_rng(4)
    B, k = 700, 3 if not paths else 2
    for it in range(6):
        seeds = rng.integers(0, E, B)
        filt = None
        if it >= 3:  # three runs of each shape: eager, capture, replay
            filt = [sorted(rng.choice(R, 8, replace=False).tolist()) for _ in range(B)]
        kw = dict(relation_filter=filt, semantics=sem, paths=paths, max_paths=200, activated=paths)
        l0 = graphed.launch_count()
        a = graphed.retrieve(seeds, k, **kw)
        b = eager.retrieve(seeds, k, **kw)
        _same(a, b)
        assert graphed.launch_count() > l0
        for i in (0, B // 2, B - 1):
            ref = orc.retrieve_one(og, int(seeds[i]), k, sem, None if filt is None else filt[i],
                                   paths=paths, max_paths=200)
            for h in range(k):
                assert np.array_equal(a.frontier(i, h + 1), ref["frontiers"][h]), (it, i, h)
            if paths:
                assert a.path_tid_tuples(i) == ref["paths"]


def test_replay_grows_capacity_and_shape_changes(th):
    """Small outputs first (graph captured with small capacities), then a batch
    of hub seeds with the same shape overflows them: the run is redone
    eagerly and later replays use the grown buffers; a new B re-captures."""
    s, r, o = _hub_graph(4000, 120000, 16, seed=8)
    E, R = 4000, 16
    g = th.build_incidence((s, r, o), E, R)
    graphed, eager = th.Retriever(g), th.Retriever(g)
    eager.set_graphs(False)
    deg = np.bincount(s, minlength=E)
    leaves = np.flatnonzero(deg == 0)
    hubs = np.argsort(-deg)[:64]
    rng = np.random.default_rng(1)
    B = 1024
    batches = [rng.choice(leaves, B)] * 3 + [rng.choice(hubs, B)] * 3
    batches += [rng.integers(0, E, 300)] * 3 + [rng.integers(0, E, B)]
    for seeds in batches:
        _same(graphed.retrieve(seeds, 3), eager.retrieve(seeds, 3))


def test_profiling_under_replay(th):
    """Timing events are captured with the kernels: every replay reports the
    same launch counts per category as the eager run, with real times."""
    s, r, o = _hub_graph(1000, 10000, 8, seed=2)
    g = th.build_incidence((s, r, o), 1000, 8)
    ret = th.Retriever(g)
    ret.set_profiling(True)
    seeds = np.arange(200)
    first = ret.retrieve(seeds, 2)
    eager = ret.profile()
    assert sum(n for _ms, n in eager.values()) > 0
    for _ in range(3):
        _same(ret.retrieve(seeds, 2), first)
        prof = ret.profile()
        assert {c: n for c, (_ms, n) in prof.items()} == {c: n for c, (_ms, n) in eager.items()}
        assert sum(ms for ms, _n in prof.values()) > 0


def test_replay_two_waves_and_filters(th):
    """B = 1,500 (two waves of the bit-parallel engine) with per-seed filters:
    the captured graph covers both waves and the masks are staged."""
    s, r, o = _hub_graph(2500, 50000, 20, seed=13)
    E, R = 2500, 20
    g = th.build_incidence((s, r, o), E, R)
    graphed, eager = th.Retriever(g), th.Retriever(g)
    eager.set_graphs(False)
    rng = np.random.default_rng(6)
    for it in range(4):
        seeds = rng.integers(0, E, 1500)
        filt = [sorted(rng.choice(R, 5, replace=False).tolist()) for _ in range(1500)]
        a = graphed.retrieve(seeds, 3, relation_filter=filt, activated=True)
        b = eager.retrieve(seeds, 3, relation_filter=filt, activated=True)
        _same(a, b)


@pytest.mark.parametrize("B", [1, 2, 33, 100, 1025])
def test_replay_every_wave_width(th, B):
    """Word widths W = 1 .. 32 (and a second wave): replayed graphs equal
    eager runs for each width, with seeds that change between replays."""
    s, r, o = _hub_graph(1200, 20000, 12, seed=31)
    E, R = 1200, 12
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    graphed, eager = th.Retriever(g), th.Retriever(g)
    eager.set_graphs(False)
    rng = np.random.default_rng(B)
    for it in range(6):  # per semantics: eager run, capture, replay
        seeds = rng.integers(0, E, B)
        sem = "frontier" if it < 3 else "cumulative"
        a = graphed.retrieve(seeds, 3, semantics=sem)
        b = eager.retrieve(seeds, 3, semantics=sem)
        _same(a, b)
    i = B - 1
    ref = orc.retrieve_one(og, int(seeds[i]), 3, "cumulative")
    for h in range(3):
        assert np.array_equal(a.frontier(i, h + 1), ref["frontiers"][h])
