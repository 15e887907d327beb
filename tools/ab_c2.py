"""A/B of session knobs on C2 (k=3, 1,024 seeds, L2 flushed before every
batch): device ms per batch, CUDA graphs on, no profiling.

    python tools/ab_c2.py "{'k4_mode': 0}" "{'k4_mode': 1}"
"""

import ast
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402


def main():
    configs = [ast.literal_eval(a) for a in sys.argv[1:]] or [{}]
    s, r, o, E, R = workloads.c2_graph()
    g = th.build_incidence((s, r, o), E, R)
    seeds = torch.from_numpy(workloads.seed_batches(E, 1024, 8, seed=100)).cuda()
    offs = torch.arange(1025, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for rep in range(3):
        for cfg in configs:
            ret = th.Retriever(g)
            for name, v in cfg.items():
                (getattr(ret, "set_" + name)(v) if hasattr(ret, "set_" + name) else ret.set_knob(name, v))
            for i in range(4):
                ret.run(offs, seeds[i], 3, "frontier", None, singleton=True, copy=False)
            ts = []
            for i in range(24):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ret.run(offs, seeds[i % 8], 3, "frontier", None, singleton=True, copy=False, collect=False)
                b.record()
                ret.collect()
                ts.append(a.elapsed_time(b))
            print(f"rep={rep} {cfg} median={statistics.median(ts):.4f} min={min(ts):.4f} ms", flush=True)
            del ret


if __name__ == "__main__":
    main()
