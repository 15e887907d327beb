"""A/B of CUDA-graph replay on C2 (k=3, 1,024 seeds): device ms per batch,
with and without profiling events, flushed L2 and back-to-back."""

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
        for graphs in (False, True):
            for prof in (False, True):
                ret = th.Retriever(g)
                ret.set_graphs(graphs)
                ret.set_profiling(prof)
                for i in range(4):
                    ret.run(offs, seeds[i], 3, "frontier", None, singleton=True, copy=False)
                ret.profile()
                ts = []
                for i in range(20):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    ret.run(offs, seeds[i % 8], 3, "frontier", None, singleton=True, copy=False,
                            collect=False)
                    b.record()
                    ret.collect()
                    ts.append(a.elapsed_time(b))
                # back-to-back: 20 runs, one finish each (host syncs in between)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                for i in range(20):
                    ret.run(offs, seeds[i % 8], 3, "frontier", None, singleton=True, copy=False,
                            collect=False)
                b.record()
                torch.cuda.synchronize()
                ret.collect()
                print(f"rep={rep} graphs={graphs} prof={prof} flushed median={statistics.median(ts):.4f} "
                      f"min={min(ts):.4f} back2back={a.elapsed_time(b) / 20:.4f} ms", flush=True)


if __name__ == "__main__":
    main()
