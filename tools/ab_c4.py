"""A/B of knobs on C4 k=2/3 (1,024 seeds per wave): device ms per wave,
graphs on, no profiling.  Knob sets are given as python dict literals:

    TH_EXP=<bits> python tools/ab_c4.py "{'dense_pull': 0}" "{'dense_pull': 2}"
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
    s, r, o, E, R = workloads.c4_graph()
    g = th.build_incidence((s, r, o), E, R)
    del s, r, o
    seeds = torch.from_numpy(workloads.seed_batches(E, 1024, 6, seed=400)).cuda()
    offs = torch.arange(1025, dtype=torch.int32, device="cuda")
    for rep in range(2):
        for cfg in configs:
            ret = th.Retriever(g)
            for name, v in cfg.items():
                (getattr(ret, "set_" + name)(v) if hasattr(ret, "set_" + name) else ret.set_knob(name, v))
            for k in (2, 3):
                for i in range(2):
                    ret.run(offs, seeds[i], k, "frontier", None, singleton=True, copy=False)
                ts = []
                for i in range(2, 6):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    ret.run(offs, seeds[i], k, "frontier", None, singleton=True, copy=False, collect=False)
                    b.record()
                    ret.collect()
                    ts.append(a.elapsed_time(b))
                print(f"rep={rep} {cfg} k={k} median={statistics.median(ts):.3f} min={min(ts):.3f} ms",
                      flush=True)
            del ret


if __name__ == "__main__":
    main()
