import sys; sys.path.insert(0, '.')
import torch, numpy as np
import paper_2604_18913_b200 as th, workloads
s, r, o, E, R = workloads.c4_graph()
g = th.build_incidence((s, r, o), E, R)
seeds = torch.from_numpy(workloads.seed_batches(E, 1024, 2, seed=400)).cuda()
offs = torch.arange(1025, dtype=torch.int32, device="cuda")
ret = th.Retriever(g)
res = ret.run(offs, seeds[0], 3, "frontier", None, singleton=True, copy=False)
print("E", E, "T", s.size, "wave_lists", ret.wave_lists(3), "ids per layer", res.frontier_len.sum(1).tolist(), "modes", ret.wave_modes(3))
