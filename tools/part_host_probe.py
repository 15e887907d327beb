"""Host-side split of a partitioned C4 wave on one rank (loopback): issue
(th_shards_run_wave: begin + hops, a CUDA graph once the shape repeats)
and finish (waits for the device), with CUDA events around both."""

import ctypes
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18913_b200 as th  # noqa: E402
import workloads  # noqa: E402
from paper_2604_18913_b200 import _lib  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    s, r, o, E, R = workloads.c4_graph()
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(1))
    sh = pg.shards[0]
    batches = workloads.seed_batches(E, 1024, 4, seed=400)

    def wq(i):
        return th.partition.WaveQuery(np.arange(1025, dtype=np.int32), batches[i % 4], k, th.HopSemantics.FRONTIER)

    for i in range(6):
        pg.run(wq(i))
    torch.cuda.synchronize()
    for rep in range(4):
        q = wq(rep)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        qs = (_lib.Query * 1)(sh.prepare(q))
        h = (ctypes.c_void_p * 1)(sh._handle)
        n = (ctypes.c_int64 * 1)(sh._n_seeds)
        _lib.check(_lib.load().th_shards_run_wave(h, 1, qs, n))
        t1 = time.perf_counter()
        st, res = sh.finish()
        t2 = time.perf_counter()
        b.record()
        torch.cuda.synchronize()
        print(f"k={k} issue {1e3 * (t1 - t0):.3f} finish {1e3 * (t2 - t1):.3f} events {a.elapsed_time(b):.3f} ms "
              f"launches {sh.launch_count()}", flush=True)


if __name__ == "__main__":
    main()
