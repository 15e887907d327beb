import cProfile, pstats, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2604_18913_b200 as th, workloads
s, r, o, E, R = workloads.c2_graph()
g = th.build_incidence((s, r, o), E, R)
seeds, rel_ids = workloads.c3_queries(s, E, R)
ret = th.Retriever(g)
def once():
    rr = ret.retrieve(seeds, 2, relation_filter=list(rel_ids), paths=True, max_paths=10_000, copy=False)
    host = [x.cpu() for x in (rr.frontier_off, rr.frontier_len, rr.frontier_ids, rr.edges, rr.path_off, rr.path_count, rr.path_tids, rr.path_truncated)]
    return host
once(); once()
torch.cuda.synchronize()
t0 = time.perf_counter(); once(); torch.cuda.synchronize(); print("e2e s", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable(); once(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
