"""Seeded synthetic workloads standing in for the reference's datasets.

BASELINE.json's configs quote UMLS-/PKG-shaped graphs that
are not in this container; these generators reproduce their sizes and degree
shapes.  Every generator is deterministic in its seed.

C1  the reference's own ``synth.power_law(10_000, 50_000, 16, seed=0,
    alpha=1.1)`` (synth.py:34-49).  Its triples are shipped verbatim in
    tests/golden/c1.npz (made by the reference itself), so no re-derivation.
C2  407,000 entities / exactly 3,400,000 distinct triples / 400 relations.
    Subjects and objects are drawn from ONE rank^-1.2 Zipf law over a random
    permutation of ids (hubs are both prolific subjects and popular objects,
    as in UMLS; hubs are scattered over the id space), relations from
    rank^-1.0 over 400; duplicates are resampled until exactly T distinct
    triples remain; triple order is shuffled so tids are not row-sorted.
    Achieved: top-40 (0.01%) subjects average ~33.4k out-edges -- the
    config's "hubs average ~33k 1-hop neighbours" (0.1% is arithmetically
    impossible at T=3.4M).
C3  C2's graph; 2,048 uniform + 2,048 top-1%-degree seeds; per-seed 32-of-400
    relation masks.
C4  54.4M entities / exactly 86.5M distinct triples / 1,000 uniform
    relations, PKG-shaped.  Chung-Lu style power law:
    exactly 1% of entities are isolated; every other entity gets one
    incident "base" edge (as subject or object, coin flip) so nothing else
    is isolated; the remaining endpoints are drawn with weights whose tail
    is P(w >= x) ~ x^-1.3 (the config's "Zipf 1.3"), sampled in closed form
    by inverse CDF over rank (rank = N * U^(1/(1-1/1.3))).  One random
    rank->id permutation serves both sides, so prolific subjects are also
    popular objects (a hub core, as in C2; independent permutations leave
    the hubs unreachable, with k=3 frontiers of a few entities per seed).
    Duplicates are topped up to exactly T; triple order is shuffled.
C5  200M entities / exactly 1e9 distinct triples / 2,000 uniform relations,
    R-MAT(a=.57, b=.19, c=.19, d=.05) at scale 2^28 with ids >= 2e8
    rejected, then one random id permutation; 16,384 seeds with per-seed
    64-of-2,000 relation masks.  Generated on the GPU with torch (numpy
    would need ~60 GB and minutes); deterministic for a given seed on a
    given device and software stack.
"""


from __future__ import annotations

from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent


def _unique_sorted(k: np.ndarray) -> np.ndarray:
    k = np.sort(k)
    if k.size == 0:
        return k
    keep = np.empty(k.size, dtype=bool)
    keep[0] = True
    np.not_equal(k[1:], k[:-1], out=keep[1:])
    return k[keep]


def zipf_graph(n_entities: int, n_triples: int, n_relations: int, seed: int, alpha: float = 1.2,
               rel_alpha: float = 1.0, shared_ranks: bool = True):
    """Exactly ``n_triples`` distinct (s, r, o) with Zipf subjects/objects."""
    rng = np.random.default_rng(seed)
    E, T, R = n_entities, n_triples, n_relations
    perm_s = rng.permutation(E)
    perm_o = perm_s if shared_ranks else rng.permutation(E)
    cw = np.cumsum(1.0 / np.arange(1, E + 1, dtype=np.float64) ** alpha)
    cw /= cw[-1]
    cr = np.cumsum(1.0 / np.arange(1, R + 1, dtype=np.float64) ** rel_alpha)
    cr /= cr[-1]
    keys = np.empty(0, dtype=np.int64)
    while keys.size < T:
        n = int((T - keys.size) * 1.3) + 1024
        s = perm_s[np.minimum(np.searchsorted(cw, rng.random(n)), E - 1)].astype(np.int64)
        o = perm_o[np.minimum(np.searchsorted(cw, rng.random(n)), E - 1)].astype(np.int64)
        r = np.minimum(np.searchsorted(cr, rng.random(n)), R - 1).astype(np.int64)
        keys = _unique_sorted(np.concatenate([keys, (s * R + r) * E + o]))
    keys = keys[np.sort(rng.choice(keys.size, T, replace=False))] if keys.size > T else keys
    keys = rng.permutation(keys)
    o = (keys % E).astype(np.int32)
    r = ((keys // E) % R).astype(np.int32)
    s = (keys // E // R).astype(np.int32)
    return s, r, o


def c1_graph():
    z = np.load(ROOT / "tests" / "golden" / "c1.npz")
    return z["subj"], z["rel"], z["obj"], 10_000, 16


def c1_seeds():
    return np.random.default_rng(1).choice(10_000, 64, replace=False)


C2_DIMS = (407_000, 3_400_000, 400)


def c2_graph(seed: int = 2):
    E, T, R = C2_DIMS
    s, r, o = zipf_graph(E, T, R, seed)
    return s, r, o, E, R


def seed_batches(n_entities: int, batch: int, count: int, seed: int) -> np.ndarray:
    """``count`` batches of ``batch`` distinct uniform seeds, int32 [count, batch]."""
    rng = np.random.default_rng(seed)
    return np.stack([rng.choice(n_entities, batch, replace=False) for _ in range(count)]).astype(np.int32)


def c3_queries(s: np.ndarray, n_entities: int, n_relations: int, seed: int = 3, n: int = 4096,
               mask_size: int = 32):
    """Half uniform seeds, half from the top-1% out-degree hubs; per-seed masks."""
    rng = np.random.default_rng(seed)
    deg = np.bincount(s, minlength=n_entities)
    top = np.argsort(-deg, kind="stable")[: max(1, n_entities // 100)]
    hubs = rng.choice(top, n // 2, replace=False)
    rest = np.setdiff1d(np.arange(n_entities), hubs)
    uni = rng.choice(rest, n - n // 2, replace=False)
    seeds = np.concatenate([uni, hubs]).astype(np.int32)
    masks = np.stack([rng.choice(n_relations, mask_size, replace=False) for _ in range(n)])
    return seeds, masks


def graph_stats(s, o, n_entities: int) -> dict:
    deg = np.bincount(s, minlength=n_entities)
    ind = np.bincount(o, minlength=n_entities)
    top = np.sort(deg)[::-1]
    k001 = max(1, n_entities // 10_000)
    return {
        "n_triples": int(s.size), "max_out_degree": int(top[0]), "max_in_degree": int(ind.max()),
        "top_0.01pct_mean_out": float(top[:k001].mean()),
        "zero_out_frac": float((deg == 0).mean()),
        "isolated_frac": float(((deg == 0) & (ind == 0)).mean()),
    }


C4_DIMS = (54_400_000, 86_500_000, 1_000)


def _sorted_unique(keys: np.ndarray) -> np.ndarray:
    # np.sort + neighbour mask (numpy 2.3's np.unique is ~80x slower here)
    return _unique_sorted(keys)


def powerlaw_graph(n_entities: int, n_triples: int, n_relations: int, seed: int,
                   alpha: float = 1.3, isolated: float = 0.01, shared_ranks: bool = True):
    """Exactly ``n_triples`` distinct (s, r, o); ``isolated`` of entities untouched."""
    rng = np.random.default_rng(seed)
    E, T, R = n_entities, n_triples, n_relations
    perm = rng.permutation(E).astype(np.int64)
    act = perm[int(round(E * isolated)):]
    N = act.size
    by_rank_out = act
    by_rank_in = act if shared_ranks else act[rng.permutation(N)]
    ex = 1.0 / (1.0 - 1.0 / alpha)

    def draw(by_rank, n):
        k = (N * rng.random(n) ** ex).astype(np.int64)
        return by_rank[np.minimum(k, N - 1)]

    side = rng.random(N) < 0.5
    s = np.where(side, act, draw(by_rank_out, N))
    o = np.where(side, draw(by_rank_in, N), act)
    extra = max(0, T - N)
    s = np.concatenate([s, draw(by_rank_out, extra)])
    o = np.concatenate([o, draw(by_rank_in, extra)])
    r = rng.integers(0, R, s.size)
    keys = _sorted_unique((s * R + r) * E + o)
    del s, o, r
    while keys.size < T:
        n = 2 * (T - keys.size) + 1024
        add = _sorted_unique((draw(by_rank_out, n) * R + rng.integers(0, R, n)) * E
                             + draw(by_rank_in, n))
        pos = np.minimum(np.searchsorted(keys, add), keys.size - 1)
        add = add[keys[pos] != add][: T - keys.size]
        keys = np.sort(np.concatenate([keys, add]))
    if keys.size > T:
        keys = keys[np.sort(rng.choice(keys.size, T, replace=False))]
    keys = keys[rng.permutation(T)]
    o = (keys % E).astype(np.int32)
    r = ((keys // E) % R).astype(np.int32)
    s = (keys // E // R).astype(np.int32)
    return s, r, o


def c4_graph(seed: int = 4):
    E, T, R = C4_DIMS
    s, r, o = powerlaw_graph(E, T, R, seed)
    return s, r, o, E, R


C5_DIMS = (200_000_000, 1_000_000_000, 2_000)


def rmat_graph_gpu(n_entities: int, n_triples: int, n_relations: int, seed: int = 5,
                   abcd=(0.57, 0.19, 0.19, 0.05), chunk: int = 1 << 27, device="cuda"):
    """Exactly ``n_triples`` distinct R-MAT triples as int32 CUDA tensors."""
    import torch

    E, T, R = n_entities, n_triples, n_relations
    scale = max(1, (E - 1).bit_length())
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    a, b, c, _ = abcd
    cut = torch.tensor([a, a + b, a + b + c], device=device, dtype=torch.float32)

    def draw(n):
        s = torch.zeros(n, dtype=torch.int64, device=device)
        o = torch.zeros(n, dtype=torch.int64, device=device)
        for _ in range(scale):
            u = torch.rand(n, generator=gen, device=device)
            q = torch.bucketize(u, cut)  # 0..3 = quadrant (a, b, c, d)
            s = (s << 1) | (q >> 1)
            o = (o << 1) | (q & 1)
        keep = (s < E) & (o < E)
        return s[keep], o[keep]

    perm = torch.randperm(E, generator=gen, device=device)
    parts_s, parts_o, parts_r, got = [], [], [], 0
    target = int(T * 1.05)
    while True:
        while got < target:
            s, o = draw(chunk)
            parts_s.append(perm[s].to(torch.int32))
            parts_o.append(perm[o].to(torch.int32))
            parts_r.append(torch.randint(0, R, (s.numel(),), generator=gen, device=device,
                                         dtype=torch.int32))
            got += s.numel()
        s = torch.cat(parts_s)
        o = torch.cat(parts_o)
        r = torch.cat(parts_r)
        parts_s, parts_o, parts_r = [s], [o], [r]
        # distinct (s, r, o): stable sort by r, then by (s, o) -> lexicographic
        key = (s.to(torch.int64) << 28) | o.to(torch.int64)
        order = torch.sort(r, stable=True).indices
        order = order[torch.sort(key[order], stable=True).indices]
        ks, rs = key[order], r[order]
        first = torch.ones(ks.numel(), dtype=torch.bool, device=device)
        first[1:] = (ks[1:] != ks[:-1]) | (rs[1:] != rs[:-1])
        idx = order[first]
        del key, order, ks, rs, first
        if idx.numel() >= T:
            break
        target = got + int((T - idx.numel()) * 1.5) + chunk // 4  # top up and re-deduplicate
        del idx
    # exactly T: a random subset, in random triple order
    pick = torch.randperm(idx.numel(), generator=gen, device=device)[:T]
    idx = idx[pick]
    return s[idx].contiguous(), r[idx].contiguous(), o[idx].contiguous()


def c5_graph_gpu(seed: int = 5):
    E, T, R = C5_DIMS
    s, r, o = rmat_graph_gpu(E, T, R, seed)
    return s, r, o, E, R


def c5_queries(n_entities: int, n_relations: int, seed: int = 6, n: int = 16_384, mask_size: int = 64):
    rng = np.random.default_rng(seed)
    seeds = rng.choice(n_entities, n, replace=False).astype(np.int32)
    masks = np.argsort(rng.random((n, n_relations)), axis=1)[:, :mask_size]
    return seeds, masks
