"""A/B of session knobs on C3 (C2 graph, 4,096 filtered seeds, k=2, paths
<= 10,000): device ms per batch with the per-category breakdown.

    python tools/ab_c3.py "{'paths_k2': 0}" "{'paths_k2': 1}"
"""

import ast
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402
from paper_2604_18913_b200.retriever import _relation_masks  # noqa: E402


def main():
    configs = [ast.literal_eval(a) for a in sys.argv[1:]] or [{}]
    s, r, o, E, R = workloads.c2_graph()
    g = th.build_incidence((s, r, o), E, R)
    seeds, rel = workloads.c3_queries(s, E, R)
    B = seeds.size
    words = _relation_masks(list(rel), B, R)
    d_seeds = torch.from_numpy(seeds).cuda()
    d_masks = torch.from_numpy(words.view(np.int32)).cuda()
    offs = torch.arange(B + 1, dtype=torch.int32, device="cuda")
    for rep in range(2):
        for cfg in configs:
            ret = th.Retriever(g)
            for name, v in cfg.items():
                ret.set_knob(name, v) if name in ("paths_k2", "k4_cache", "list_first_hop") else \
                    (getattr(ret, "set_" + name)(v) if hasattr(ret, "set_" + name) else ret.set_knob(name, v))
            for _ in range(2):
                ret.run(offs, d_seeds, 2, "frontier", d_masks, paths=True, max_paths=10_000, singleton=True,
                        copy=False)
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                res = ret.run(offs, d_seeds, 2, "frontier", d_masks, paths=True, max_paths=10_000,
                              singleton=True, copy=False)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ret.set_profiling(True)
            for _ in range(2):
                ret.run(offs, d_seeds, 2, "frontier", d_masks, paths=True, max_paths=10_000, singleton=True,
                        copy=False)
            ret.profile()
            ret.run(offs, d_seeds, 2, "frontier", d_masks, paths=True, max_paths=10_000, singleton=True,
                    copy=False)
            prof = ret.profile()
            print(f"rep={rep} {cfg} median={statistics.median(ts):.3f} ms paths={int(res.path_count.sum())} "
                  f"paths_ms={prof['paths'][0]:.3f}", flush=True)
            del ret


if __name__ == "__main__":
    main()
