import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch, torch.distributed as dist
import paper_2604_18913_b200 as th, workloads
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29611")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0), rank=0, world_size=1)
s, r, o, E, R = workloads.c4_graph()
pg = th.PartitionedGraph((s, r, o), E, R, th.DistExchange())
for nb, seed in ((3, 400), (6, 400)):
    batches = workloads.seed_batches(E, 1024, nb, seed=seed)
    def wave(i):
        q = th.partition.WaveQuery(np.arange(1025, dtype=np.int32), batches[i % nb], 2, th.HopSemantics.FRONTIER)
        return pg.run(q)
    for i in range(3): wave(i)
    if os.environ.get("BARRIER"): dist.barrier()
    torch.cuda.synchronize()
    for i in range(6):
        t0 = time.perf_counter()
        parts = wave(3 + i)
        e = int(parts[0].edges.sum())
        if not os.environ.get("NOSYNC"): torch.cuda.synchronize()
        print(nb, "batch", (3 + i) % nb, "ms", round((time.perf_counter() - t0) * 1e3, 2), "edges", e, flush=True)
dist.destroy_process_group()
