"""Streaming retrieval: batch i+1 runs on the device while batch i's results
cross PCIe into pinned host memory.

A serving loop that returns every seed's frontiers to the host is bound by
the device-to-host link (C2: ~378 MB of ids per 1,024-seed batch, ~7 ms at
PCIe Gen5 rates, against ~0.56 ms of device work).  Calling
:meth:`Retriever.retrieve` and copying its results serialises the two; this
pipeline keeps ``depth`` engine sessions (one stream each) and a copy
stream, so a batch's hops overlap the previous batch's copy-out and the
steady-state cost per batch is the larger of the two, not their sum.

Role in the reference: the batch loop of its service / bench
(``service/app.py:196-229``, ``bench.py`` query loop) that calls
``k_hop`` once per seed and hands the arrays back to the caller; results are
the same per-seed sorted frontiers (canonical ``EntityVector`` ids,
``incidence.py:83-91``) and per-hop ``triple_count`` (``service/app.py:97``).
"""

from __future__ import annotations

import numpy as np

from .retriever import Retriever

_FIELDS = ("frontier_off", "frontier_len", "frontier_ids", "edges")


class HostBatch:
    """Host (pinned) results of one batch; arrays alias the pipeline's
    buffers and stay valid until the next batch is requested from
    :meth:`RetrievalPipeline.run` (call :meth:`copy` to keep them longer)."""

    def __init__(self, index: int, n_queries: int, k: int, arrays: dict):
        self.index = index
        self.n_queries = n_queries
        self.k = k
        self.frontier_off = arrays["frontier_off"]  # int64 [k, B]
        self.frontier_len = arrays["frontier_len"]  # int64 [k, B]
        self.frontier_ids = arrays["frontier_ids"]  # int32 [total]
        self.edges = arrays["edges"]  # int64 [k, B]

    def frontier(self, q: int, hop: int) -> np.ndarray:
        """Sorted frontier ids of query ``q`` after hop ``hop`` (1-based)."""
        o = int(self.frontier_off[hop - 1, q])
        return self.frontier_ids[o : o + int(self.frontier_len[hop - 1, q])]

    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.frontier_off, self.frontier_len, self.frontier_ids, self.edges))

    def copy(self) -> "HostBatch":
        return HostBatch(self.index, self.n_queries, self.k,
                         {f: getattr(self, f).copy() for f in _FIELDS})


class RetrievalPipeline:
    """Double-buffered batch retrieval with host results (frontier semantics
    chosen per call, as :meth:`Retriever.retrieve`)."""

    def __init__(self, graph, depth: int = 2):
        import torch

        if depth < 1:
            raise ValueError("pipeline depth must be >= 1")
        self.graph = graph
        self.depth = depth
        dev = graph.device
        self.sessions = [Retriever(graph, stream=torch.cuda.Stream(dev)) for _ in range(depth)]
        self.copy_stream = torch.cuda.Stream(dev)
        self._pinned = [{} for _ in range(depth)]
        self._copied = [None] * depth  # event: slot's copy-out finished

    def _buffer(self, slot: int, name: str, t):
        import torch

        buf = self._pinned[slot].get(name)
        if buf is None or buf.numel() < t.numel() or buf.dtype != t.dtype:
            buf = torch.empty(int(t.numel() * 1.25) + 16, dtype=t.dtype).pin_memory()
            self._pinned[slot][name] = buf
        return buf

    def run(self, batches, k: int, relation_filter=None, semantics="frontier"):
        """Yield one :class:`HostBatch` per input seed batch, in order.

        ``batches``: an iterable of seed batches (host arrays / pinned host
        tensors; one query per seed, as ``Retriever.retrieve``).
        """
        import torch

        pending = []  # (index, slot, B, host views) awaiting their copy-out
        for i, seeds in enumerate(batches):
            slot = i % self.depth
            ses = self.sessions[slot]
            if self._copied[slot] is not None:
                # the slot's session buffers are still being read by its copy
                ses.stream.wait_event(self._copied[slot])
            if len(pending) == self.depth:
                # the slot's pinned buffers are about to be overwritten: its
                # previous batch must have been handed out (and copied) first
                yield self._finish(pending.pop(0))
            with torch.cuda.stream(ses.stream):
                res = ses.retrieve(seeds, k, relation_filter=relation_filter, semantics=semantics,
                                   copy=False)
            self.copy_stream.wait_stream(ses.stream)
            views = {}
            with torch.cuda.stream(self.copy_stream):
                for name in _FIELDS:
                    t = getattr(res, name)
                    buf = self._buffer(slot, name, t)
                    buf[: t.numel()].copy_(t.reshape(-1), non_blocking=True)
                    views[name] = (buf, tuple(t.shape))
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            self._copied[slot] = ev
            pending.append((i, slot, res.n_queries, res.k, views, ev))
            if len(pending) > 1:
                # hand out the previous batch once its copy is done (this
                # batch's hops were launched before the wait)
                yield self._finish(pending.pop(0))
        while pending:
            yield self._finish(pending.pop(0))

    @staticmethod
    def _finish(p) -> HostBatch:
        i, slot, B, k, views, ev = p
        ev.synchronize()
        arrays = {}
        for name, (buf, shape) in views.items():
            n = int(np.prod(shape)) if shape else 1
            arrays[name] = buf[:n].numpy().reshape(shape)
        return HostBatch(i, B, k, arrays)
