import statistics, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2604_18913_b200 as th, workloads
s, r, o, E, R = workloads.c2_graph()
g = th.build_incidence((s, r, o), E, R)
seeds = torch.from_numpy(workloads.seed_batches(E, 1024, 8, seed=100)).cuda()
offs = torch.arange(1025, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for ov in (True, False, True, False):
    ret = th.Retriever(g); ret.set_overlap(ov)
    for i in range(3): ret.run(offs, seeds[i], 3, "frontier", None, singleton=True, copy=False)
    ts = []
    for i in range(16):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ret.run(offs, seeds[i % 8], 3, "frontier", None, singleton=True, copy=False, collect=False); b.record(); ret.collect()
        ts.append(a.elapsed_time(b))
    print("overlap", ov, round(statistics.median(ts), 4))
