"""Short C3 run for ncu captures: two batches of the C3 query set
(4,096 seeds, per-seed 32-of-400 masks, k=2, paths capped at 10,000)."""

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402


def main():
    s, r, o, E, R = workloads.c2_graph()
    g = th.build_incidence((s, r, o), E, R)
    seeds, masks = workloads.c3_queries(s, E, R)
    ret = th.Retriever(g)
    for _ in range(2):
        res = ret.retrieve(seeds, 2, relation_filter=list(masks), paths=True, max_paths=10_000, copy=False)
    torch.cuda.synchronize()
    print("paths", int(res.path_count.sum()), "edges", int(res.edges.sum()))


if __name__ == "__main__":
    main()
