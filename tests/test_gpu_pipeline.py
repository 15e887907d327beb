"""RetrievalPipeline (pipeline.py): streamed batches with host results are
identical to one-at-a-time Retriever.retrieve and to the oracle, across
batch sizes that change between batches (graph re-capture per session),
filters, and pipeline depths 1-3."""

import numpy as np
import pytest

from oracle import khop_oracle as orc
from test_gpu_parity import _hub_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def th_mod(cuda_device):
    import paper_2604_18913_b200 as th

    return th


@pytest.mark.parametrize("depth", [1, 2, 3])
@pytest.mark.parametrize("filtered", [False, True])
def test_pipeline_matches_retrieve_and_oracle(th_mod, depth, filtered):
    import torch

    th = th_mod
    E, T, R, k = 1200, 16000, 24, 3
    s, r, o = _hub_graph(E, T, R, seed=7 + depth, alpha=1.1)
    g = th.build_incidence((s, r, o), E, R)
    og = orc.build_csr(s, r, o, E, R)
    rng = np.random.default_rng(depth)
    sizes = [256, 256, 1024, 1024, 1024, 33, 1024, 1]
    batches = [rng.integers(0, E, n).astype(np.int32) for n in sizes]
    filt = sorted(rng.choice(R, 9, replace=False).tolist()) if filtered else None
    pinned = [torch.from_numpy(b).pin_memory() for b in batches]
    pipe = th.RetrievalPipeline(g, depth=depth)
    ret = th.Retriever(g)
    got = 0
    for hb in pipe.run(pinned, k, relation_filter=filt):
        b = batches[hb.index]
        assert hb.n_queries == b.size and hb.k == k
        ref = ret.retrieve(b, k, relation_filter=filt)
        for h in range(k):
            assert np.array_equal(hb.edges[h], ref.edges[h].cpu().numpy())
        for q in range(b.size):
            for h in range(k):
                assert np.array_equal(hb.frontier(q, h + 1), ref.frontier(q, h + 1)), (hb.index, q, h)
        for q in sorted({0, b.size // 2, b.size - 1}):
            want = orc.retrieve_one(og, int(b[q]), k, "frontier", filt)
            for h in range(k):
                assert np.array_equal(hb.frontier(q, h + 1), want["frontiers"][h])
                assert int(hb.edges[h, q]) == want["edges"][h]
        got += 1
    assert got == len(batches)


def test_pipeline_host_copy_outlives_the_stream(th_mod):
    import torch

    th = th_mod
    E, T, R = 600, 5000, 8
    s, r, o = _hub_graph(E, T, R, seed=3, alpha=1.1)
    g = th.build_incidence((s, r, o), E, R)
    rng = np.random.default_rng(1)
    batches = [torch.from_numpy(rng.integers(0, E, 128).astype(np.int32)).pin_memory() for _ in range(5)]
    kept = [hb.copy() for hb in th.RetrievalPipeline(g).run(batches, 2)]
    ret = th.Retriever(g)
    for hb, b in zip(kept, batches):
        ref = ret.retrieve(b.numpy(), 2)
        for q in range(128):
            assert np.array_equal(hb.frontier(q, 2), ref.frontier(q, 2))
