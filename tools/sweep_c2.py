"""Knob sweep on C2 (k=3, 1,024 seeds): pull divisor x overlap; device ms per batch."""

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
    ret = th.Retriever(g)
    seeds = torch.from_numpy(workloads.seed_batches(E, 1024, 4, seed=100)).cuda()
    offs = torch.arange(1025, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for div in [0.0, 2.0, 4.0, 8.0, 16.0, 64.0, -1.0]:
        for ov in (True, False):
            ret.set_pull_divisor(div)
            ret.set_overlap(ov)
            for i in range(2):
                ret.run(offs, seeds[i], 3, "frontier", None, singleton=True, copy=False)
            ts = []
            for i in range(4):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                res = ret.run(offs, seeds[i], 3, "frontier", None, singleton=True, copy=False)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            print(f"div={div:5} overlap={ov} ms={sorted(ts)[1]:.3f} push/pull={res.push_hops}/{res.pull_hops}",
                  flush=True)


if __name__ == "__main__":
    main()
