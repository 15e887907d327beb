"""C3 probe: C2 graph, 4,096 seeds (2,048 uniform + 2,048 top-1% hubs), per-seed
32-of-400 relation masks, k=2, paths capped at 10,000 per seed."""

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
    s, r, o, E, R = workloads.c2_graph()
    g = th.build_incidence((s, r, o), E, R)
    seeds, masks = workloads.c3_queries(s, E, R)
    ret = th.Retriever(g)
    for rep in range(3):
        ret.set_profiling(True)
        ret.profile()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = ret.retrieve(seeds, 2, relation_filter=list(masks), paths=True, max_paths=10_000, copy=False)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        prof = ret.profile()
        print(f"rep={rep} wall_ms={1e3 * dt:.2f} paths={int(res.path_count.sum())} "
              f"trunc={int(res.path_truncated.sum())} ids={res.frontier_len.sum(1).tolist()} "
              f"edges={int(res.edges.sum())} prof={ {c: round(v[0], 3) for c, v in prof.items() if v[0]} }",
              flush=True)
    og = orc.build_csr(s, r, o, E, R)
    t0 = time.time()
    checked = 0
    for i in list(range(0, 2048, 97)) + list(range(2048, 4096, 97)):
        if time.time() - t0 > 240:
            break
        ref = orc.retrieve_one(og, int(seeds[i]), 2, "frontier", masks[i], paths=True, max_paths=10_000)
        for h in range(2):
            assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h]), (i, h)
            assert int(res.edges[h, i]) == ref["edges"][h]
        assert res.path_tid_tuples(i) == ref["paths"], i
        assert res.truncated(i) == ref["truncated"]
        checked += 1
    print("oracle parity ok on", checked, "seeds", round(time.time() - t0, 1), "s", flush=True)


if __name__ == "__main__":
    main()
