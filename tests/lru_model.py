"""Independent LRU model for the cache tests (test infrastructure only):
replays an access trace over a recency-ordered list and returns the counters
the reference's cache reports (its own model: cache.py:92-117)."""

from paper_2604_18913_b200.cache import CacheCounters


def simulate_lru(trace, capacity: int, resident: list | None = None) -> CacheCounters:
    """Counters of an LRU of ``capacity`` over ``trace``; ``resident``, when
    given, receives the final residents (least recent first)."""
    if capacity < 1:
        raise ValueError("cache capacity must be >= 1")
    recent = []  # least recent first
    hits = misses = evictions = 0
    for idx in trace:
        if idx in recent:
            hits += 1
            recent.remove(idx)
        else:
            misses += 1
            if len(recent) == capacity:
                recent.pop(0)
                evictions += 1
        recent.append(idx)
    if resident is not None:
        resident[:] = recent
    n = hits + misses
    return CacheCounters(hits, misses, misses, evictions, hits / n if n else 0.0)
