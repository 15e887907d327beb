"""Kernel-group timelines of one C4 wave (k from argv, default 2): the
single-graph engine and the partitioned path on one rank, side by side
(CUDA events per group on its stream; 0 = main, 1/2 = K4 side streams)."""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402


def show(name, tr):
    end = max(t1 for _, _, _, t1 in tr)
    print(f"== {name}: {end:.3f} ms from the first scope to the last")
    for cat, st, t0, t1 in sorted(tr, key=lambda x: x[2]):
        bar = " " * int(t0 * 40) + "#" * max(1, int((t1 - t0) * 40))
        print(f"{cat:9s} s{st} {t0:7.3f} {t1:7.3f} {(t1 - t0):6.3f}  {bar[:160]}")


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    s, r, o, E, R = workloads.c4_graph()
    seeds = workloads.seed_batches(E, 1024, 4, seed=400)
    g = th.build_incidence((s, r, o), E, R)
    ret = th.Retriever(g)
    offs = torch.arange(1025, dtype=torch.int32, device="cuda")
    ret.set_profiling(True)
    for b in seeds:
        ret.run(offs, torch.from_numpy(b).cuda(), k, "frontier", None, singleton=True, copy=False)
    show(f"single graph k={k}", ret.profile_trace())
    del ret, g
    torch.cuda.empty_cache()
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(1))
    sh = pg.shards[0]
    sh.set_profiling(True)
    for b in seeds:
        q = th.partition.WaveQuery(np.arange(1025, dtype=np.int32), b, k, th.HopSemantics.FRONTIER)
        pg.run(q)
    show(f"partitioned, one rank, k={k}", sh.profile_trace())


if __name__ == "__main__":
    main()
