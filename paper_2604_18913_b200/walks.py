"""Capped lexicographic walk enumeration across shards (the
reference's ``cross_graph_paths`` -> ``assemble_paths``, engine.py:157-182,
incidence.py:344-408) with walk counts exchanged between ranks instead of
the walk subgraph.

A length-k walk from the seed set is t1..tk with subj(t1) a seed and
subj(t[i+1]) = obj(t[i]); under exact-walk semantics every t[h] is a triple
activated at hop h, and the triples of hop h live on the rank that owns
their subject (or their slice of a hub row).  Walks are ordered
lexicographically by their tids and the first ``max_paths`` are returned.

1. Counts, last hop first.  c_k(t) = 1; W_h(v) = sum of c_h over the hop-h
   triples of subject v (each rank sums its own, the ranks' partial sums
   are gathered and added); c_h(t) = W_{h+1}(obj t).  Counts saturate at
   max_paths + 1 (only "more than the cap" matters), so int64 never
   overflows.  The total over hop 1 decides ``truncated``.
2. Selection, first hop first.  A selected prefix p carries its last
   vertex, its rank offset (walks before it) and its budget (walks of it
   still inside the cap).  Every rank offers, per prefix, its triples of
   that vertex at the next hop in tid order while its OWN running count is
   below the budget -- the global running count at a tid is at least the
   rank's, so nothing inside the cap is held back -- at most budget
   entries per prefix and rank.  The offers are gathered and merged by
   (prefix, tid); an offer is selected while the global running count
   stays below the budget.

So each hop moves at most world x max_paths offers plus the counts' partial
sums, never the activated triples themselves.  Results equal the
reference's (tests: the reference goldens, its restatement, single-graph K5).
"""

from __future__ import annotations

import numpy as np

from .core_types import PathResult, Triple

_UNCAPPED_LIMIT = 1 << 31  # an uncapped request enumerating more walks cannot be held


def _seg_sum(keys, vals, sat):
    """(distinct keys ascending, saturated sums of vals per key)."""
    import torch

    uk, inv = torch.unique(keys, return_inverse=True)
    s = torch.zeros(uk.numel(), dtype=torch.int64, device=keys.device).index_add_(0, inv, vals)
    return uk, s.clamp_(max=sat)


def _lookup(keys, vals, q):
    """vals[keys == q] or 0 (keys ascending)."""
    import torch

    if keys.numel() == 0:
        return torch.zeros(q.numel(), dtype=torch.int64, device=q.device)
    pos = torch.searchsorted(keys, q).clamp_(max=keys.numel() - 1)
    return torch.where(keys[pos] == q, vals[pos], torch.zeros_like(pos))


def _ragged(lo, n):
    """Concatenated ranges [lo[i], lo[i] + n[i]) and their owner i."""
    import torch

    owner = torch.repeat_interleave(torch.arange(n.numel(), device=n.device), n)
    start = torch.cumsum(n, 0) - n
    return lo[owner] + torch.arange(owner.numel(), device=n.device) - start[owner], owner


def sharded_paths(q0, k: int, pg, max_paths):
    """PathResult of q0's length-k walks over a rank-sharded graph."""
    import torch

    from .core_types import HopSemantics
    from .partition import WaveQuery

    xch = pg.exchange
    ids = q0.ids.astype(np.int32)
    wq = WaveQuery(np.array([0, ids.size], dtype=np.int32), ids, k, HopSemantics.EXACT_WALK, None, True)
    # this process's ranks: per hop the owned activated triples (tid order)
    mine = []
    for sh, res in zip(pg.shards, pg.run(wq)):
        a_off, a_len = res.a_off.cpu().numpy(), res.a_len.cpu().numpy()
        hops = []
        for h in range(k):
            t = res.a_ids[int(a_off[h, 0]):int(a_off[h, 0] + a_len[h, 0])].long()
            s_, r_, o_ = sh.triples_of(t)
            hops.append({"t": t, "s": s_.long(), "r": r_.long(), "o": o_.long()})
        mine.append(hops)
    dev = mine[0][0]["t"].device
    cap = None if max_paths is None else int(max_paths)
    sat = _UNCAPPED_LIMIT if cap is None else min(cap + 1, _UNCAPPED_LIMIT)

    # 1. counts, last hop first
    for hops in mine:
        hops[k - 1]["c"] = torch.ones_like(hops[k - 1]["t"])
    for h in range(k - 2, -1, -1):
        parts = []
        for hops in mine:
            v, w = _seg_sum(hops[h + 1]["s"], hops[h + 1]["c"], sat)
            parts.append({"v": v, "w": w})
        allp = xch.gather(parts)
        gv, gw = _seg_sum(torch.cat([p["v"].to(dev) for p in allp]),
                          torch.cat([p["w"].to(dev) for p in allp]), sat)
        for hops in mine:
            hops[h]["c"] = _lookup(gv.to(hops[h]["o"].device), gw.to(hops[h]["o"].device), hops[h]["o"])
    total = xch.sum_int([int(hops[0]["c"].sum()) for hops in mine])
    if cap is None:
        if total >= _UNCAPPED_LIMIT:
            raise OverflowError(f"more than {_UNCAPPED_LIMIT - 1} walks; pass max_paths")
        cap = total
    truncated = total > cap
    if cap == 0 or total == 0:
        return PathResult([], truncated)

    # 2. selection, first hop first.  Level 0 = one virtual prefix holding
    # the seeds: every hop-1 triple is its child.
    levels = []  # per hop: dict of selected offers (parent, t, s, r, o, offset)
    parent_v = None  # last vertex per selected prefix (None: the seed prefix)
    budget = torch.tensor([cap], dtype=torch.int64, device=dev)
    offset = torch.zeros(1, dtype=torch.int64, device=dev)
    for h in range(k):
        offers = []
        for hops in mine:
            a = hops[h]
            keep = a["c"] > 0
            s_, t_, c_ = a["s"][keep], a["t"][keep], a["c"][keep]
            r_, o_ = a["r"][keep], a["o"][keep]
            if parent_v is not None:
                # (subject, tid) order: t_ ascends already, the sort is stable
                order = torch.argsort(s_, stable=True)
                s_, t_, c_, r_, o_ = s_[order], t_[order], c_[order], r_[order], o_[order]
            run = torch.cumsum(c_, 0)
            excl = run - c_
            run = torch.cat([torch.zeros(1, dtype=torch.int64, device=run.device), run])
            loc_dev = s_.device
            if parent_v is None:  # hop 1: every triple is a child, in tid order
                lo = torch.zeros(1, dtype=torch.int64, device=loc_dev)
                hi = torch.full((1,), s_.numel(), dtype=torch.int64, device=loc_dev)
            else:
                pv = parent_v.to(loc_dev)
                lo = torch.searchsorted(s_, pv)
                hi = torch.searchsorted(s_, pv, right=True)
            base = run[lo]  # walks of this rank's entries before the prefix's group
            # this rank's running count below the budget
            end = torch.searchsorted(excl, base + budget.to(loc_dev))
            n = (torch.minimum(end, hi) - lo).clamp_(min=0)
            idx, owner = _ragged(lo, n)
            offers.append({"p": owner, "t": t_[idx], "s": s_[idx], "r": r_[idx], "o": o_[idx], "c": c_[idx]})
        allo = xch.gather(offers)
        cat = {f: torch.cat([o[f].to(dev) for o in allo]) for f in ("p", "t", "s", "r", "o", "c")}
        # merge by (prefix, tid); owners are disjoint, so tids never repeat
        key = cat["p"] * (int(pg.n_triples) + 1) + cat["t"]
        order = torch.argsort(key)
        cat = {f: v[order] for f, v in cat.items()}
        p, c = cat["p"], cat["c"]
        run = torch.cumsum(c, 0) - c
        first = torch.searchsorted(p, p)  # start of each prefix's group
        within = run - run[first]
        sel = within < budget[p]
        cat = {f: v[sel] for f, v in cat.items()}
        p, within = cat["p"], within[sel]
        offset = offset[p] + within
        budget = torch.minimum(cat["c"], budget[p] - within)
        parent_v = cat["o"]
        levels.append({"p": p, "s": cat["s"], "r": cat["r"], "o": cat["o"]})
    # the last hop's selections are complete walks, ranked by offset
    order = torch.argsort(offset)
    idx = order
    steps = [None] * k
    for h in range(k - 1, -1, -1):
        lv = levels[h]
        steps[h] = torch.stack([lv["s"][idx], lv["r"][idx], lv["o"][idx]], 1).cpu().numpy()
        idx = lv["p"][idx]
    paths = [tuple(Triple(*(int(x) for x in steps[h][i])) for h in range(k)) for i in range(order.numel())]
    return PathResult(paths, truncated)
