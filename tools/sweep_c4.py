"""C4 (k=3, 1,024 seeds) pull-divisor sweep; device ms per batch."""

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402


def main():
    s, r, o, E, R = workloads.c4_graph()
    g = th.build_incidence((s, r, o), E, R)
    del s, r, o
    ret = th.Retriever(g)
    seeds = torch.from_numpy(workloads.seed_batches(E, 1024, 2, seed=400)).cuda()
    offs = torch.arange(1025, dtype=torch.int32, device="cuda")
    for div in [8.0, 4.0, 2.0, 1.0, 0.5, 0.25, 0.0]:
        ret.set_pull_divisor(div)
        ret.run(offs, seeds[0], 3, "frontier", None, singleton=True, copy=False)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        res = ret.run(offs, seeds[1], 3, "frontier", None, singleton=True, copy=False)
        b.record()
        torch.cuda.synchronize()
        print(f"div={div:5} ms={a.elapsed_time(b):.2f} push/pull={res.push_hops}/{res.pull_hops}", flush=True)


if __name__ == "__main__":
    main()
