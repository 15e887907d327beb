"""Partitioned path reconstruction on the C2 graph (world 2 on one device):
walk counts + capped offers between ranks (walks.sharded_paths, the
product path) against gathering the walk subgraph and running K5 on it
(the round-1 form), per seed set; results must agree."""

import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402
from paper_2604_18913_b200.partition import walk_subgraph  # noqa: E402


def gathered(q0, k, pg, cap):
    s, r, o = walk_subgraph(q0, k, pg)
    sub = th.build_incidence((s, r, o), pg.n_entities, pg.n_relations)
    return th.reconstruct_paths(q0, k, sub, cap)


def main():
    s, r, o, E, R = workloads.c2_graph()
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(2))
    deg = np.bincount(s, minlength=E)
    hubs = np.argsort(-deg)[:8]
    rng = np.random.default_rng(1)
    cases = [([int(h)], k, 10_000) for h in hubs[:4] for k in (2, 3)]
    cases += [(sorted(rng.integers(0, E, 4).tolist()), 3, 10_000) for _ in range(4)]
    for fn in (th.cross_graph_paths, gathered):  # warm-up
        fn(th.EntityVector(cases[0][0], E), 2, pg, 100)
    tot = {"sharded": 0.0, "gathered": 0.0}
    for seeds, k, cap in cases:
        q0 = th.EntityVector(seeds, E)
        out = {}
        for name, fn in (("sharded", th.cross_graph_paths), ("gathered", gathered)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out[name] = fn(q0, k, pg, cap)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            tot[name] += dt
            out[name + "_ms"] = dt * 1e3
        assert out["sharded"].paths == out["gathered"].paths and out["sharded"].truncated == out["gathered"].truncated
        walk = sum(int(x.numel()) for x in [torch.as_tensor(walk_subgraph(q0, k, pg)[0])])
        print(f"seeds={seeds} k={k} cap={cap}: paths={len(out['sharded'].paths)} trunc={out['sharded'].truncated} "
              f"walk_subgraph={walk} triples  sharded {out['sharded_ms']:.1f} ms  gathered {out['gathered_ms']:.1f} ms",
              flush=True)
    print(f"total: sharded {tot['sharded'] * 1e3:.0f} ms, gathered+K5 {tot['gathered'] * 1e3:.0f} ms")


if __name__ == "__main__":
    main()
