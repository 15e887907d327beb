import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2604_18913_b200 as th, workloads
from paper_2604_18913_b200 import _lib
import ctypes
s, r, o, E, R = workloads.c4_graph()
pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(1))
sh = pg.shards[0]
batches = workloads.seed_batches(E, 1024, 4, seed=400)
def wq(i, k=2): return th.partition.WaveQuery(np.arange(1025, dtype=np.int32), batches[i % 4], k, th.HopSemantics.FRONTIER)
for i in range(6): pg.run(wq(i))
torch.cuda.synchronize()
for rep in range(3):
    q = wq(rep)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); a.record()
    sh.begin(q); t1 = time.perf_counter()
    h = (ctypes.c_void_p * 1)(sh._handle)
    _lib.check(_lib.load().th_shards_run_hops(h, 1, q.k)); t2 = time.perf_counter()
    st, res = sh.finish(); t3 = time.perf_counter(); b.record()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"begin {1e3*(t1-t0):.3f} hops {1e3*(t2-t1):.3f} finish {1e3*(t3-t2):.3f} total_host {1e3*(t4-t0):.3f} events {a.elapsed_time(b):.3f} ms")
