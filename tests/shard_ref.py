"""Numpy stand-in for one rank's device shard -- TEST INFRASTRUCTURE ONLY.

It implements the wave protocol of ``paper_2604_18913_b200.partition``
(begin / hop(h, phase) / finish, with exchange regions its peers write
into) with the same shard layout and record format as the CUDA shard
(csrc/k6_shard.cuh), but with boolean [row, query] matrices on the host and
exchange regions in host shared memory.  It lets the multi-process path
(DistExchange over gloo, world_size 2: region handles shipped between
processes, the phase barriers, the owners' gathered slices and the merge)
run on a CPU-only box; only the per-rank arithmetic is replaced.

Differences that do not change results: records go to a per-sender segment
of the receiver's inbox (numpy has no atomic fetch-add on shared memory;
the device reserves from one cursor), and the stand-in only pushes.
"""

from __future__ import annotations

from multiprocessing import shared_memory

import numpy as np
import torch

from paper_2604_18913_b200.partition import ShardResult, hash_owner

SEG = 1 << 16  # records per sender segment


def _pick_words(nq: int) -> int:
    w = 1
    while 32 * w < nq:
        w <<= 1
    return w


class _Region:
    """An exchange region: [world] sender cursors, [world] published costs,
    [world][SEG] record keys and bits, and the [H][32] hub board."""

    def __init__(self, world, H, name=None):
        self.world, self.H = world, H
        sizes = [("cursor", np.int64, world), ("cost", np.int64, world),
                 ("keys", np.int64, world * SEG), ("bits", np.uint32, world * SEG),
                 ("hubs", np.uint32, max(H, 1) * 32)]
        nbytes = sum(np.dtype(t).itemsize * n for _, t, n in sizes)
        if name is None:
            self.shm = shared_memory.SharedMemory(create=True, size=nbytes)
            self.owner = True
        else:
            self.shm = shared_memory.SharedMemory(name=name)
            self.owner = False
        off = 0
        for f, t, n in sizes:
            setattr(self, f, np.ndarray((n,), dtype=t, buffer=self.shm.buf, offset=off))
            off += np.dtype(t).itemsize * n
        if self.owner:
            self.cursor[:] = 0
            self.cost[:] = 0
        self.keys = self.keys.reshape(world, SEG)
        self.bits = self.bits.reshape(world, SEG)

    def close(self):
        for f in ("cursor", "cost", "keys", "bits", "hubs"):
            setattr(self, f, None)
        self.shm.close()
        if self.owner:
            self.shm.unlink()


class RefShard:
    can_pull = False

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
        self.t_subj = s[tids]
        self.local_triples = int(tids.size)
        self.l2g = plan.owned(rank).astype(np.int64)
        self.deg = np.bincount(row, minlength=self.n_local + self.H)
        self.region = _Region(self.world, self.H)
        self.peers = [None] * self.world

    def __del__(self):
        try:
            for p, reg in enumerate(self.peers):
                if reg is not None and reg is not self.region and not reg.owner:
                    reg.close()
            self.region.close()
        except Exception:  # pragma: no cover
            pass

    # -- exchange wiring -----------------------------------------------------
    def region_handle(self, local):
        return self.region if local else self.region.shm.name

    def connect_peer(self, p, handle, local):
        if p == self.rank:
            self.peers[p] = self.region
        elif local:
            self.peers[p] = handle
        else:
            self.peers[p] = _Region(self.world, self.H, name=handle)

    def set_pull_divisor(self, d):
        self.pull_divisor = d

    def synchronize(self):
        pass

    def grow_inbox(self):  # pragma: no cover - segments are sized for the tests
        raise RuntimeError("stand-in inbox overflowed")

    def launch_count(self):
        return 0

    # -- wave ------------------------------------------------------------------
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
        self.sent = np.zeros(k, np.int64)
        self.region.cursor[:] = 0
        self._publish_cost(self.X)

    def _publish_cost(self, layer):
        cost = int(self.deg[layer.any(1)].sum())
        for reg in self.peers:
            reg.cost[self.rank] = cost

    def _local_set(self, row, q):
        """Apply (row, query) candidates to the owned state."""
        if self.q.semantics.value == "exact":
            self.N[row, q] = True
            return
        new = ~self.V[row, q]
        self.V[row[new], q[new]] = True
        self.N[row[new], q[new]] = True

    def hop(self, h, phase):
        getattr(self, ("_send", "_receive", "_end")[phase])(h)

    def _send(self, h):
        act = self.X[self.t_row] & self.allow[:, self.t_rel].T  # [local triples, B]
        self.edges[h - 1] = act.sum(0)
        for q in range(self.B):
            self.acts[h - 1][q] = self.t_gid[act[:, q]]
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
            key, dest = key[first], dest[first]
        else:
            words = np.empty(0, np.uint64)
        for d in range(self.world):
            sel = dest == d
            n = int(sel.sum())
            reg = self.peers[d]
            c = int(reg.cursor[self.rank])
            assert c + n <= SEG, "stand-in inbox segment overflow"
            reg.keys[self.rank, c: c + n] = key[sel]
            reg.bits[self.rank, c: c + n] = words[sel].astype(np.uint32)
            reg.cursor[self.rank] = c + n
            if d != self.rank:
                self.sent[h - 1] += n

    def _receive(self, h):
        reg = self.region
        for src in range(self.world):
            n = int(reg.cursor[src])
            key = reg.keys[src, :n].copy()
            word = reg.bits[src, :n].astype(np.uint64)
            row, j = key // self.W, key % self.W
            assert (row < self.n_local).all(), "record for a row this rank does not own"
            bits = ((word[:, None] >> np.arange(32, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(bool)
            r_idx, b_idx = np.nonzero(bits)
            self._local_set(row[r_idx], j[r_idx] * 32 + b_idx)
        reg.cursor[:] = 0
        if h < self.q.k:
            for hh, v in enumerate(self.plan.hub_ids.tolist()):
                if self.plan.owner[v] == self.rank:
                    row = self._pack(self.N[self.plan.lidx[v]][None, :])[0]
                    for peer in self.peers:
                        peer.hubs[hh * 32: hh * 32 + self.W] = row

    def _pack(self, m):  # bool [n, B] -> uint32 [n, W]
        out = np.zeros((m.shape[0], self.W * 32), bool)
        out[:, : self.B] = m
        return np.packbits(out, axis=1, bitorder="little").view(np.uint32)

    def _end(self, h):
        if h < self.q.k and self.H:
            rows = self.region.hubs.reshape(-1, 32)[: self.H, : self.W].copy()
            bits = np.unpackbits(rows.view(np.uint8), axis=1, bitorder="little")[:, : self.B].astype(bool)
            self.N[self.n_local: self.n_local + self.H] = bits
        own = slice(0, self.n_local)
        layer = (self.V[own] & ~self.S[own]) if self.q.semantics.value == "cumulative" else self.N[own]
        for q in range(self.B):
            self.frontiers[h - 1][q] = self.l2g[layer[:, q]]
        if h < self.q.k:
            self._publish_cost(self.N)
        self.X = self.N
        self.N = np.zeros_like(self.X)

    def finish(self):
        k, B = self.q.k, self.B
        res = ShardResult(B, k, edges=torch.from_numpy(self.edges))

        def csr(lists):
            ln = np.array([[lists[h][q].size for q in range(B)] for h in range(k)], np.int64).reshape(k, B)
            off = np.concatenate([[0], np.cumsum(ln.reshape(-1))[:-1]]).reshape(k, B)
            ids = np.concatenate([lists[h][q] for h in range(k) for q in range(B)]) if B else np.empty(0)
            return torch.from_numpy(off), torch.from_numpy(ln), torch.from_numpy(ids.astype(np.int32))

        res.f_off, res.f_len, res.f_ids = csr(self.frontiers)
        if self.q.activated:
            res.a_off, res.a_len, res.a_ids = csr(self.acts)
        return "ok", res

    def sent_records(self, k):
        return self.sent[:k].tolist()

    def triples_of(self, tids):
        t = tids.cpu().numpy().astype(np.int64)
        local = np.searchsorted(self.t_gid, t)
        return (torch.from_numpy(self.t_subj[local].astype(np.int32)),
                torch.from_numpy(self.t_rel[local].astype(np.int32)),
                torch.from_numpy(self.t_obj[local].astype(np.int32)))
