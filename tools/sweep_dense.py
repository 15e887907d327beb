"""Dense-pull threshold sweep on C2 (k=3, 1,024 seeds): device ms per batch
(graphs on, L2 flushed)."""

import statistics
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
    seeds = torch.from_numpy(workloads.seed_batches(E, 1024, 8, seed=100)).cuda()
    offs = torch.arange(1025, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for rep in range(2):
        for div in (0.0, 1.25, 2.0, 4.0, 16.0):
            ret = th.Retriever(g)
            ret.set_dense_pull(div)
            for i in range(3):
                ret.run(offs, seeds[i], 3, "frontier", None, singleton=True, copy=False)
            ts = []
            for i in range(16):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ret.run(offs, seeds[i % 8], 3, "frontier", None, singleton=True, copy=False, collect=False)
                b.record()
                ret.collect()
                ts.append(a.elapsed_time(b))
            print(f"rep={rep} dense_pull={div} median={statistics.median(ts):.4f} ms", flush=True)


if __name__ == "__main__":
    main()
