"""Per-batch times of the bench's C4 leg shape (run + th_finish inside the
events, 8 batches after 2 untimed), for knob settings given as dicts."""

import ast
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
    batches = torch.from_numpy(workloads.seed_batches(E, 1024, 8, seed=400)).cuda()
    offs = torch.arange(1025, dtype=torch.int32, device="cuda")
    for cfg in configs:
        ret = th.Retriever(g)
        for name, v in cfg.items():
            (getattr(ret, "set_" + name)(v) if hasattr(ret, "set_" + name) else ret.set_knob(name, v))
        for k in (2, 3):
            step = lambda i: ret.run(offs, batches[i], k, "frontier", None, singleton=True, copy=False)  # noqa
            step(0)
            step(1)
            ts = []
            for i in range(8):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                step(i)
                b.record()
                torch.cuda.synchronize()
                ts.append(round(a.elapsed_time(b), 3))
            print(cfg, f"k={k}", ts, flush=True)
        del ret


if __name__ == "__main__":
    main()
