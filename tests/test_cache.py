"""SubgraphCache: the reference's LRU counter algebra (cache.py:38-117),
checked against the independent list model; device units on the GPU."""

import numpy as np
import pytest

from lru_model import simulate_lru

from paper_2604_18913_b200.cache import SubgraphCache


def test_lru_golden_sequence():
    c = SubgraphCache(2, record_trace=True)
    load = lambda i: f"g{i}"  # noqa: E731
    for i in (0, 1, 0, 2, 1, 1, 3):
        c.get(i, load)
    k = c.snapshot_counters()
    assert (k.hits, k.misses, k.loads, k.evictions) == (2, 5, 5, 3)
    assert c.resident_indices() == [1, 3]
    assert c.trace == [0, 1, 0, 2, 1, 1, 3]


def test_loader_failure_leaves_state_untouched():
    c = SubgraphCache(2)
    c.get(0, lambda i: i)
    before = (c.hits, c.misses, c.loads, c.evictions, c.resident_indices())

    def boom(i):
        raise OSError("disk")

    with pytest.raises(OSError):
        c.get(5, boom)
    assert (c.hits, c.misses, c.loads, c.evictions, c.resident_indices()) == before


@pytest.mark.parametrize("seed", range(20))
def test_counters_equal_independent_model(seed):
    rng = np.random.default_rng(seed)
    cap = int(rng.integers(1, 6))
    trace = rng.integers(0, 9, 200).tolist()
    c = SubgraphCache(cap)
    for i in trace:
        c.get(i, lambda j: j)
    assert c.snapshot_counters() == simulate_lru(trace, cap)
    k = c.snapshot_counters()
    assert k.hits + k.misses == len(trace) and k.loads == k.misses
    assert k.evictions == k.loads - len(c)  # every load beyond residency evicted one


def test_stack_property_more_capacity_never_fewer_hits():
    rng = np.random.default_rng(3)
    trace = rng.integers(0, 12, 300).tolist()
    hits = [simulate_lru(trace, c).hits for c in range(1, 10)]
    assert hits == sorted(hits)


def test_bad_capacity():
    with pytest.raises(ValueError):
        SubgraphCache(0)
    with pytest.raises(ValueError):
        simulate_lru([1], 0)


@pytest.mark.gpu
def test_device_units_load_and_evict(cuda_device):
    """Units are device graphs loaded from LKG1 bytes; eviction frees them."""
    import paper_2604_18913_b200 as th
    from pathlib import Path

    data = (Path(__file__).resolve().parent / "golden" / "tiny.lkg").read_bytes()
    c = SubgraphCache(1)
    g0 = c.get(0, lambda i: th.graph_from_bytes(data))
    assert c.get(0, lambda i: None) is g0
    g1 = c.get(1, lambda i: th.graph_from_bytes(data))
    assert 0 not in c and 1 in c and g1 is not g0
    res = th.retrieve(g1, [0], 2)
    assert res.frontier(0, 1).tolist() == [1, 2]


@pytest.mark.parametrize("seed", range(5))
def test_public_simulate_lru_matches_independent_model(seed):
    """th.simulate_lru (the reference's public entry point, cache.py:92-117)
    against the test suite's independent list model."""
    import paper_2604_18913_b200 as th

    rng = np.random.default_rng(100 + seed)
    cap = int(rng.integers(1, 7))
    trace = rng.integers(0, 11, 300).tolist()
    assert th.simulate_lru(trace, cap) == simulate_lru(trace, cap)
