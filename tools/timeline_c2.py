"""Per-kernel-group timeline of one C2 k=3 batch (CUDA events on the stream
each group runs on; 0 = main stream, 1/2 = K4 side streams), after warm-up,
L2 flushed before the batch as in bench.py."""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402


def main():
    s, r, o, E, R = workloads.c2_graph()
    g = th.build_incidence((s, r, o), E, R)
    ret = th.Retriever(g)
    batches = workloads.seed_batches(E, 1024, 8, seed=7)
    offs = torch.arange(1025, dtype=torch.int32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    ret.set_profiling(True)
    for b in batches[:4]:
        ret.run(offs, torch.from_numpy(b).cuda(), 3, "frontier", None, singleton=True, copy=False)
    for b in batches[4:]:
        seeds = torch.from_numpy(b).cuda()
        flush.fill_(1)
        torch.cuda.synchronize()
        ret.profile()
        ret.run(offs, seeds, 3, "frontier", None, singleton=True, copy=False)
        tr = ret.profile_trace()
    end = max(t1 for _, _, _, t1 in tr)
    print(f"batch: {end * 1e3:.0f} us from the first scope to the last")
    for cat, st, t0, t1 in sorted(tr, key=lambda x: x[2]):
        bar = " " * int(t0 * 1e3 / 8) + "#" * max(1, int((t1 - t0) * 1e3 / 8))
        print(f"{cat:9s} s{st} {t0 * 1e3:7.1f} {t1 * 1e3:7.1f} {(t1 - t0) * 1e3:6.1f}  {bar}")


if __name__ == "__main__":
    main()
