import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/tests/golden")
import numpy as np
import paper_2604_18913_b200 as th
from oracle import khop_oracle as orc
from test_gpu_fuzz import _cases
from test_gpu_parity import _hub_graph

idx = int(sys.argv[1])
c = _cases()[idx]
print(c)
s, r, o = _hub_graph(c["E"], c["T"], c["R"], seed=c["seed"], alpha=c["alpha"])
E, R = c["E"], c["R"]
g = th.build_incidence((s, r, o), E, R)
og = orc.build_csr(s, r, o, E, R)
import itertools
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["default", "nographs", "nooverlap", "push", "pull"]
for variant in variants * int(sys.argv[3] if len(sys.argv) > 3 else 1):
    rng = np.random.default_rng(c["seed"] + 100)
    ret = th.Retriever(g)
    ret.set_pull_divisor(c["divisor"])
    ret.set_list_min_entities(0 if c["list_mode"] else 1 << 40)
    if variant == "nographs": ret.set_graphs(False)
    if variant == "nooverlap": ret.set_overlap(False)
    if "push" in variant: ret.set_pull_divisor(0.0)
    if "nog" in variant: ret.set_graphs(False)
    if "noov" in variant: ret.set_overlap(False)
    if variant == "pull": ret.set_pull_divisor(-1.0)
    bad = []
    for rep in range(3):
        seeds = rng.integers(0, E, c["B"])
        res = ret.retrieve(seeds, c["k"], semantics=c["sem"])
        for i in sorted(set([0, c["B"] - 1, c["B"] // 2])):
            ref = orc.retrieve_one(og, int(seeds[i]), c["k"], c["sem"], None)
            for h in range(c["k"]):
                a = res.frontier(i, h + 1); b = ref["frontiers"][h]
                if not np.array_equal(a, b):
                    bad.append((rep, i, h, len(a), len(b), res.push_hops, res.pull_hops))
    print(variant, "bad:", bad[:6])
