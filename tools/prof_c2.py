"""Short C2 run for ncu captures: 2 warm-up batches, then one timed batch.

    python tools/prof_c2.py [--k 3] [--filter] [--paths]

Each batch launches, per hop, one pull_kernel, one mat_kernel count pass
and one mat_kernel write pass, so `-k regex:"mat_kernel|pull_kernel"
-s 18 -c 9` captures the last (k=3) batch.
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=3)
    ap.add_argument("--batches", type=int, default=3)
    ap.add_argument("--filter", action="store_true")
    ap.add_argument("--paths", action="store_true")
    args = ap.parse_args()
    s, r, o, E, R = workloads.c2_graph()
    g = th.build_incidence((s, r, o), E, R)
    ret = th.Retriever(g)
    seeds = torch.from_numpy(workloads.seed_batches(E, 1024, 1, seed=100)[0]).cuda()
    flt = None
    if args.filter:
        rng = np.random.default_rng(5)
        flt = [rng.choice(R, 32, replace=False) for _ in range(seeds.numel())]
    for b in range(args.batches):
        if b == args.batches - 1:  # ncu --profile-from-start off: only the last batch
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        res = ret.retrieve(seeds, args.k, relation_filter=flt, paths=args.paths, copy=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ids", int(res.frontier_len.sum()), "edges", int(res.edges.sum()))


if __name__ == "__main__":
    main()
