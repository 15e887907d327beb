"""C5 (200M entities / 1e9 triples / 2,000 relations, R-MAT) on ONE B200:
16,384 seeds in waves of 1,024, k=2, per-seed 64-of-2,000 relation masks.
Optional sampled oracle parity (--oracle N; builds the numpy CSR at 1e9)."""

import argparse
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--oracle", type=int, default=0)
    ap.add_argument("--waves", type=int, default=16)
    ap.add_argument("--partitioned", action="store_true",
                    help="run through PartitionedGraph (one rank, the device-side exchange protocol)")
    ap.add_argument("--hubs", type=int, default=0,
                    help="partitioned: hub rows (top out-degree; 0.01%% of E = 20000 for config 5)")
    ap.add_argument("--hub-cache", type=int, default=0,
                    help="partitioned: page the hub rows through this many HBM pages (K7)")
    args = ap.parse_args()
    t0 = time.time()
    s, r, o, E, R = workloads.c5_graph_gpu()
    torch.cuda.synchronize()
    print(f"gen {time.time() - t0:.1f}s T={s.numel()} mem={torch.cuda.max_memory_allocated() / 1e9:.1f}GB",
          flush=True)
    host = None
    if args.oracle:
        host = (s.cpu().numpy(), r.cpu().numpy(), o.cpu().numpy())
    if args.partitioned:
        return partitioned(args, s, r, o, E, R, host)
    t0 = time.time()
    g = th.build_incidence((s, r, o), E, R)
    del s, r, o
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    print(f"build {time.time() - t0:.1f}s {g.stats()}", flush=True)
    seeds, rel = workloads.c5_queries(E, R)
    from paper_2604_18913_b200.retriever import _relation_masks

    words = _relation_masks(list(rel), seeds.size, R)
    d_seeds = torch.from_numpy(seeds).cuda()
    d_masks = torch.from_numpy(words.view(np.int32)).cuda()
    ret = th.Retriever(g)
    offs = torch.arange(1025, dtype=torch.int32, device="cuda")
    ret.run(offs, d_seeds[:1024], 2, "frontier", d_masks[:1024], singleton=True, copy=False)
    ret.set_profiling(True)
    ret.profile()
    tot_ms, edges, ids = 0.0, 0, 0
    for w in range(args.waves):
        sl = slice(1024 * w, 1024 * (w + 1))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        res = ret.run(offs, d_seeds[sl], 2, "frontier", d_masks[sl], singleton=True, copy=False)
        b.record()
        torch.cuda.synchronize()
        tot_ms += a.elapsed_time(b)
        edges += int(res.edges.sum())
        ids += int(res.frontier_len.sum())
    prof = ret.profile()
    n = 1024 * args.waves
    print(f"C5 k=2 filtered: {n} seeds in {tot_ms:.1f} ms -> {n / tot_ms * 1e3:.0f} seeds/s, "
          f"{edges / tot_ms * 1e3 / 1e9:.2f} G edges/s, ids/wave={ids / args.waves:.0f}, "
          f"prof={ {c: round(v[0] / args.waves, 3) for c, v in prof.items() if v[0]} } "
          f"peak_mem={torch.cuda.max_memory_allocated() / 1e9:.1f}GB", flush=True)
    if args.oracle:
        from oracle import khop_oracle as orc

        t0 = time.time()
        og = orc.build_csr(*host, E, R)
        print(f"oracle csr {time.time() - t0:.1f}s", flush=True)
        sl = slice(1024 * (args.waves - 1), 1024 * args.waves)
        base = 1024 * (args.waves - 1)
        for i in range(0, 1024, 1024 // args.oracle):
            ref = orc.retrieve_one(og, int(seeds[base + i]), 2, "frontier", rel[base + i])
            for h in range(2):
                assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h]), (i, h)
                assert int(res.edges[h, i]) == ref["edges"][h]
        print(f"oracle parity ok on {args.oracle} seeds ({time.time() - t0:.1f}s)", flush=True)


def partitioned(args, s, r, o, E, R, host):
    """C5 through the partitioned path on one rank: 64-bit exchange keys make
    200M entities x 32 words addressable (round 1's 32-bit keys refused C5)."""
    from paper_2604_18913_b200.retriever import _relation_masks

    torch.cuda.empty_cache()  # (the generator's cached blocks: the shard allocates outside torch)
    t0 = time.time()
    pg = th.PartitionedGraph((s, r, o), E, R, th.LoopbackExchange(1), n_hubs=args.hubs or None,
                             hub_cache_pages=args.hub_cache or None)
    del s, r, o
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    print(f"partitioned build {time.time() - t0:.1f}s local_triples={pg.shards[0].local_triples} "
          f"hubs={pg.plan.n_hubs} mem={torch.cuda.max_memory_allocated() / 1e9:.1f}GB", flush=True)
    if args.hub_cache:
        st = pg.hub_cache_stats()[0]
        print(f"hub cache: {st['pages']} pages of {st['page_edges']} edges, capacity {st['capacity']}",
              flush=True)
    seeds, rel = workloads.c5_queries(E, R)
    words = _relation_masks(list(rel), seeds.size, R)
    sem = th.HopSemantics.FRONTIER

    def wave(w, stats=None):
        sl = slice(1024 * w, 1024 * (w + 1))
        q = th.partition.WaveQuery(np.arange(1025, dtype=np.int32), seeds[sl], 2, sem, words[sl])
        return pg.run(q, stats)

    wave(0)
    wave(1)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for w in range(args.waves):
        wave(w)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    edges = ids = 0
    for w in range(args.waves):
        (part,) = wave(w)
        edges += int(part.edges.sum())
        ids += int(part.f_len.sum())
    n = 1024 * args.waves
    print(f"C5 partitioned (1 rank, {pg.plan.n_hubs} hubs, hub cache {args.hub_cache or 'off'}) k=2 filtered: "
          f"{n} seeds in {ms:.1f} ms -> {n / ms * 1e3:.0f} seeds/s, "
          f"{edges / ms * 1e3 / 1e9:.2f} G edges/s, ids/wave={ids / args.waves:.0f} "
          f"peak_mem={torch.cuda.max_memory_allocated() / 1e9:.1f}GB", flush=True)
    if args.hub_cache:
        st = pg.hub_cache_stats()[0]
        print(f"hub cache after {2 * args.waves + 2} waves: {st['counters']._asdict()} resident={st['resident']}",
              flush=True)
    if args.oracle:
        from oracle import khop_oracle as orc

        og = orc.build_csr(*host, E, R)
        base = 1024 * (args.waves - 1)
        res = pg.retrieve(seeds[base:base + 1024], 2, relation_filter=list(rel[base:base + 1024]))
        for i in range(0, 1024, 1024 // args.oracle):
            ref = orc.retrieve_one(og, int(seeds[base + i]), 2, "frontier", rel[base + i])
            for h in range(2):
                assert np.array_equal(res.frontier(i, h + 1), ref["frontiers"][h]), (i, h)
                assert int(res.edges[h, i]) == ref["edges"][h]
        print(f"oracle parity ok on {args.oracle} seeds", flush=True)


if __name__ == "__main__":
    main()
