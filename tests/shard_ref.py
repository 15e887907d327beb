"""Numpy stand-in for one rank's device shard -- TEST INFRASTRUCTURE ONLY.

It implements the wave-step protocol of ``paper_2604_18913_b200.partition``
(begin / expand / absorb / hub_rows / hub_merge / end_hop / finish) with
the same shard layout and the same exchange record format as the CUDA
shard (csrc/k6_shard.cuh), but with boolean [row, query] matrices on the
host.  It lets the multi-process exchange path (DistExchange over gloo,
world_size 2) run on a CPU-only box: the collectives, the record routing,
the hub all-reduce and the owners' merge are the product code; only the
per-rank arithmetic is replaced.
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2604_18913_b200.partition import ShardResult, hash_owner


def _pick_words(nq: int) -> int:
    w = 1
    while 32 * w < nq:
        w <<= 1
    return w


class RefShard:
    def __init__(self, cols, n_entities, n_relations, plan, rank):
        s, r, o = (np.asarray(c.cpu().numpy() if hasattr(c, "cpu") else c, dtype=np.int64) for c in cols)
        self.E, self.R, self.plan, self.rank, self.world = n_entities, n_relations, plan, rank, plan.world
        self.n_local = int(plan.n_local[rank])
        self.H = plan.n_hubs
        T = s.size
        hub = plan.hub_index[s] >= 0
        keep = np.where(hub, hash_owner(np.arange(T), self.world) == rank, plan.owner[s] == rank)
        tids = np.flatnonzero(keep)
        row = np.where(hub[tids], self.n_local + plan.hub_index[s[tids]], plan.lidx[s[tids]])
        self.t_row, self.t_rel, self.t_obj, self.t_gid = row, r[tids], o[tids], tids
        self.local_triples = int(tids.size)
        self.l2g = plan.owned(rank).astype(np.int64)

    # -- wave --------------------------------------------------------------
    def begin(self, query):
        B = query.n_queries
        self.q = query
        self.B, self.W = B, _pick_words(max(B, 1))
        rows = self.n_local + self.H
        self.X = np.zeros((rows, B), bool)
        self.N = np.zeros((rows, B), bool)
        self.V = np.zeros((rows, B), bool)
        self.S = np.zeros((rows, B), bool)
        if query.masks is None:
            self.allow = np.ones((B, self.R), bool)
        else:
            bits = np.unpackbits(query.masks.view(np.uint8), axis=1, bitorder="little")
            self.allow = bits[:, : self.R].astype(bool)
        for q in range(B):
            for e in query.seeds[query.seed_offsets[q]: query.seed_offsets[q + 1]].tolist():
                if self.plan.owner[e] == self.rank:
                    rr = self.plan.lidx[e]
                    self.X[rr, q] = True
                    if query.semantics.value != "exact":
                        self.V[rr, q] = True
                    if query.semantics.value == "cumulative":
                        self.S[rr, q] = True
                if self.plan.hub_index[e] >= 0:
                    self.X[self.n_local + self.plan.hub_index[e], q] = True
        k = query.k
        self.edges = np.zeros((k, B), np.int64)
        self.frontiers = [[None] * B for _ in range(k)]
        self.acts = [[None] * B for _ in range(k)]

    def _local_set(self, row, q):
        """Apply (row, query) candidates to the owned state."""
        if self.q.semantics.value == "exact":
            self.N[row, q] = True
            return
        new = ~self.V[row, q]
        self.V[row[new], q[new]] = True
        self.N[row[new], q[new]] = True

    def expand(self, hop):
        act = self.X[self.t_row] & self.allow[:, self.t_rel].T  # [local triples, B]
        self.edges[hop - 1] = act.sum(0)
        for q in range(self.B):
            self.acts[hop - 1][q] = self.t_gid[act[:, q]]
        t, q = np.nonzero(act)
        v = self.t_obj[t]
        own = self.plan.owner[v] == self.rank
        self._local_set(self.plan.lidx[v[own]], q[own])
        v, q = v[~own], q[~own]
        dest = self.plan.owner[v].astype(np.int64)
        key = self.plan.lidx[v].astype(np.int64) * self.W + q // 32
        bit = np.left_shift(np.uint64(1), (q % 32).astype(np.uint64))
        order = np.lexsort((key, dest))
        dest, key, bit = dest[order], key[order], bit[order]
        if key.size:
            first = np.ones(key.size, bool)
            first[1:] = (key[1:] != key[:-1]) | (dest[1:] != dest[:-1])
            grp = np.cumsum(first) - 1
            words = np.zeros(grp[-1] + 1, np.uint64)
            np.bitwise_or.at(words, grp, bit)
            rec = (key[first].astype(np.uint64) << np.uint64(32)) | words
            dest = dest[first]
        else:
            rec = np.empty(0, np.uint64)
        counts = np.bincount(dest, minlength=self.world).tolist()
        return torch.from_numpy(rec.view(np.int64).copy()), counts

    def absorb(self, hop, recv):
        rec = recv.cpu().numpy().view(np.uint64)
        key = (rec >> np.uint64(32)).astype(np.int64)
        word = (rec & np.uint64(0xFFFFFFFF)).astype(np.uint64)
        row, j = key // self.W, key % self.W
        assert (row < self.n_local).all(), "record for a row this rank does not own"
        bits = ((word[:, None] >> np.arange(32, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(bool)
        r_idx, b_idx = np.nonzero(bits)
        q = j[r_idx] * 32 + b_idx
        self._local_set(row[r_idx], q)

    def _pack(self, m):  # bool [n, B] -> uint32 [n, W]
        out = np.zeros((m.shape[0], self.W * 32), bool)
        out[:, : self.B] = m
        return np.packbits(out, axis=1, bitorder="little").view(np.uint32)

    def hub_rows(self, hop):
        rows = np.zeros((self.H, self.W), np.uint32)
        for h, v in enumerate(self.plan.hub_ids.tolist()):
            if self.plan.owner[v] == self.rank:
                rows[h] = self._pack(self.N[self.plan.lidx[v]][None, :])[0]
        self._hub = torch.from_numpy(rows.reshape(-1).view(np.int32).copy())
        return self._hub

    def hub_merge(self, hop):
        rows = self._hub.numpy().view(np.uint32).reshape(self.H, self.W)
        bits = np.unpackbits(rows.view(np.uint8), axis=1, bitorder="little")[:, : self.B].astype(bool)
        self.N[self.n_local: self.n_local + self.H] = bits

    def end_hop(self, hop):
        own = slice(0, self.n_local)
        layer = (self.V[own] & ~self.S[own]) if self.q.semantics.value == "cumulative" else self.N[own]
        for q in range(self.B):
            self.frontiers[hop - 1][q] = self.l2g[layer[:, q]]
        self.X = self.N
        self.N = np.zeros_like(self.X)

    def finish(self):
        k, B = self.q.k, self.B
        res = ShardResult(B, k, edges=self.edges)

        def csr(lists):
            ln = np.array([[lists[h][q].size for q in range(B)] for h in range(k)], np.int64).reshape(k, B)
            off = np.concatenate([[0], np.cumsum(ln.reshape(-1))[:-1]]).reshape(k, B)
            ids = np.concatenate([lists[h][q] for h in range(k) for q in range(B)]) if B else np.empty(0)
            return off, ln, ids.astype(np.int32)

        res.f_off, res.f_len, res.f_ids = csr(self.frontiers)
        if self.q.activated:
            res.a_off, res.a_len, res.a_ids = csr(self.acts)
        return "ok", res
