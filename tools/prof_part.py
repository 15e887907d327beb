"""Host-side profile of partitioned waves at world=1 (NCCL): where the wall
time goes beyond the device kernels."""

import cProfile
import os
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0), rank=0, world_size=1)
    s, r, o, E, R = workloads.c4_graph()
    pg = th.PartitionedGraph((s, r, o), E, R, th.DistExchange())
    batches = workloads.seed_batches(E, 1024, 6, seed=400)

    def wave(i):
        q = th.partition.WaveQuery(np.arange(1025, dtype=np.int32), batches[i], 2, th.HopSemantics.FRONTIER)
        parts = pg.run(q)
        torch.cuda.synchronize()
        return parts

    for i in range(2):
        wave(i)
    t0 = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    for i in range(2, 6):
        wave(i)
    pr.disable()
    print("ms per wave", (time.perf_counter() - t0) / 4 * 1e3)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
