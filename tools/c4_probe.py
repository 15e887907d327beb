"""C4 (54.4M entities / 86.5M triples) single-GPU probe: build, k=2/3 waves,
result sizes, per-category device time, and oracle parity on a few seeds."""

import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402
from oracle import khop_oracle as orc  # noqa: E402


def main():
    t0 = time.time()
    s, r, o, E, R = workloads.c4_graph()
    print("gen", round(time.time() - t0, 1), workloads.graph_stats(s, o, E), flush=True)
    torch.cuda.synchronize()
    t0 = time.time()
    g = th.build_incidence((s, r, o), E, R)
    torch.cuda.synchronize()
    print("build", round(time.time() - t0, 2), g.stats(), flush=True)
    ret = th.Retriever(g)
    seeds = torch.from_numpy(workloads.seed_batches(E, 1024, 1, seed=400)[0]).cuda()
    for k in (2, 3):
        for rep in range(3):
            ret.set_profiling(True)
            ret.profile()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            res = ret.retrieve(seeds, k, copy=False)
            b.record()
            torch.cuda.synchronize()
            prof = ret.profile()
            fl = res.frontier_len.sum(1).tolist()
            print(f"k={k} rep={rep} ms={a.elapsed_time(b):.2f} ids/hop={fl} edges={int(res.edges.sum())} "
                  f"push/pull={res.push_hops}/{res.pull_hops} "
                  f"prof={ {c: round(v[0], 3) for c, v in prof.items() if v[0]} }", flush=True)
    print("mem GB", torch.cuda.max_memory_allocated() / 1e9, flush=True)
    og = orc.build_csr(s, r, o, E, R)
    res = ret.retrieve(seeds[:64], 3, copy=False)
    print("k3 ids per seed (first 64):", res.frontier_len.sum(0).tolist(), flush=True)
    sd = seeds[:64].cpu().numpy()
    checked = 0
    t0 = time.time()
    for i in range(64):
        if time.time() - t0 > 120:
            break
        ref = orc.retrieve_one(og, int(sd[i]), 3, "frontier", None)
        for h in range(3):
            assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h]), (i, h)
            assert int(res.edges[h, i]) == ref["edges"][h]
        checked += 1
    print("oracle parity ok on", checked, "seeds (k=3)", flush=True)


if __name__ == "__main__":
    main()
