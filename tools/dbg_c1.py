"""Debug helper: replay golden queries one by one with progress output."""
import sys, os
import numpy as np, torch
sys.path.insert(0, 'tests/golden'); sys.path.insert(0, '.')
from golden_io import load_case
import paper_2604_18913_b200 as th
from paper_2604_18913_b200.retriever import _relation_masks

case = load_case(sys.argv[1] if len(sys.argv) > 1 else 'tests/golden/c1.npz')
start = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = th.build_incidence((case.subj, case.rel, case.obj), case.n_entities, case.n_relations)
ret = th.Retriever(g)
for qi, q in enumerate(case.queries):
    if qi < start:
        continue
    print("query", qi, q.seeds[:4], q.k, q.semantics, q.relations, q.max_paths, flush=True)
    seeds = torch.tensor(sorted(set(q.seeds)), dtype=torch.int32, device='cuda')
    offs = torch.tensor([0, seeds.numel()], dtype=torch.int32, device='cuda')
    masks = None
    if q.relations is not None:
        masks = torch.from_numpy(_relation_masks(q.relations, 1, case.n_relations).view(np.int32)).cuda()
    r = ret.run(offs, seeds, q.k, q.semantics, masks, activated=True, paths=q.want_paths,
                max_paths=q.max_paths if q.want_paths else 0, singleton=seeds.numel() == 1)
    ok = all(np.array_equal(r.frontier(0, h + 1), q.frontiers[h]) for h in range(q.k))
    print("ok" if ok else "MISMATCH", r.pull_hops, r.push_hops, flush=True)
