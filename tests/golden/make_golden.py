"""Generate the golden parity fixtures by running the REAL reference.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py [/root/reference/pkg/src]

Every number in ``tests/golden/*.npz`` comes from the unmodified
reference ``triplehop`` package: ``build_incidence``, ``k_hop`` and
``reconstruct_paths`` (incidence.py:154,319,391) on its own seeded
generators (synth.py:22-49) and the tiny graph of tests/conftest.py:6-8.
Relation-filtered cases follow the SURVEY.md 8c restatement using only
reference functions: build_incidence over the kept triples, local tids
mapped back through ``np.flatnonzero(keep)``.  Nothing here is imported at
test time; the fixtures travel, the reference does not.
"""

from __future__ import annotations

import random
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import triplehop as th  # noqa: E402
from triplehop.synth import erdos_renyi, power_law  # noqa: E402

from golden_io import GoldenCase, GoldenQuery, save_case  # noqa: E402

OUT = Path(__file__).resolve().parent
SEMS = {"exact": th.HopSemantics.EXACT_WALK, "frontier": th.HopSemantics.FRONTIER,
        "cumulative": th.HopSemantics.CUMULATIVE}
NO_PATHS = -2


def arrays_of(ts):
    a = np.asarray(ts.triples, dtype=np.int64).reshape(-1, 3)
    return a[:, 0], a[:, 1], a[:, 2]


def run_query(s, r, o, E, R, seeds, k, sem, relations=None, max_paths=NO_PATHS):
    if relations is None:
        keep = np.ones(s.size, dtype=bool)
    else:
        allow = np.zeros(R, dtype=bool)
        allow[list(relations)] = True
        keep = allow[r]
    l2g = np.flatnonzero(keep).astype(np.int64)
    g = th.build_incidence((s[keep], r[keep], o[keep]), E, R)
    q0 = th.EntityVector(seeds, E)
    trace = th.k_hop(q0, k, g, SEMS[sem])
    q = GoldenQuery(list(map(int, seeds)), k, sem,
                    None if relations is None else sorted(map(int, relations)), max_paths)
    q.frontiers = [trace.frontier(h).ids.copy() for h in range(1, k + 1)]
    q.activated = [l2g[trace.activated(h).ids] for h in range(1, k + 1)]
    if max_paths != NO_PATHS:
        res = th.reconstruct_paths(q0, k, g, max_paths)
        tid_of = {}
        for t in range(g.n_triples):
            tid_of.setdefault(tuple(int(x) for x in g.triple(t)), t)
        q.paths = [tuple(int(l2g[tid_of[tuple(int(x) for x in step)]]) for step in p)
                   for p in res.paths]
        q.truncated = bool(res.truncated)
    return q


def case(name, s, r, o, E, R, specs):
    qs = [run_query(s, r, o, E, R, *spec) for spec in specs]
    save_case(OUT / f"{name}.npz", GoldenCase(name, s, r, o, E, R, qs))
    print(f"{name}: T={s.size} queries={len(qs)}")


def main():
    # 1. the reference's tiny graph (tests/conftest.py:6-8)
    tiny = th.ingest_triples(["A\tr1\tB", "B\tr2\tC", "A\tr1\tC", "C\tr3\tA"])
    s, r, o = arrays_of(tiny)
    specs = []
    for seeds in ([0], [1], [2], [1, 2], [0, 1, 2], []):
        for k in (1, 2, 3):
            for sem in SEMS:
                specs.append((seeds, k, sem, None, NO_PATHS))
            for cap in (None, 0, 1, 2, 10_000):
                specs.append((seeds, k, "exact", None, cap))
    case("tiny", s, r, o, 3, 3, specs)

    # 2. degenerate graphs: self loop, object-only entity, empty graph
    case("selfloop", np.array([0]), np.array([0]), np.array([0]), 1, 1,
         [([0], k, sem, None, 10) for k in (1, 2, 3) for sem in SEMS])
    case("objonly", np.array([0]), np.array([0]), np.array([1]), 2, 1,
         [([e], k, sem, None, 10) for e in (0, 1) for k in (1, 2) for sem in SEMS])
    empty = np.empty(0, dtype=np.int64)
    case("empty", empty, empty, empty, 5, 2,
         [([e], 2, sem, None, 10) for e in (0, 4) for sem in SEMS])

    # 3. set-query path interleaving example of SURVEY.md 8a
    case("interleave", np.array([1, 0, 1, 2]), np.array([0, 0, 1, 0]), np.array([2, 2, 0, 1]), 3, 2,
         [([0, 1], 2, "exact", None, None), ([0], 2, "exact", None, None),
          ([1], 2, "exact", None, None), ([0, 1], 3, "frontier", None, 3)])

    # 4. ER graphs of tests/test_incidence.py:133-155 (matrix power / BFS layers)
    for seed in range(5):
        ts = erdos_renyi(30, 90, 3, seed=seed)
        s, r, o = arrays_of(ts)
        seeds = np.random.default_rng(seed).choice(30, size=3, replace=False).tolist()
        specs = [(seeds, 4, sem, None, None if sem == "exact" else NO_PATHS) for sem in SEMS]
        specs += [([e], 3, "frontier", None, NO_PATHS) for e in range(30)]
        case(f"er30_s{seed}", s, r, o, 30, 3, specs)
    for seed in range(5):
        ts = erdos_renyi(60, 200, 3, seed=seed + 10)
        s, r, o = arrays_of(ts)
        seeds = [seed % 60, (seed * 7) % 60]
        case(f"er60_s{seed + 10}", s, r, o, 60, 3,
             [(seeds, 4, sem, None, NO_PATHS) for sem in SEMS])

    # 5. every entity as a single seed, all modes, capped paths
    ts = erdos_renyi(80, 400, 3, seed=3)
    s, r, o = arrays_of(ts)
    specs = []
    for e in range(80):
        specs.append(([e], 3, "exact", None, 50))
        specs.append(([e], 3, "frontier", None, NO_PATHS))
        specs.append(([e], 3, "cumulative", None, NO_PATHS))
    specs.append(([0, 5, 9], 3, "exact", None, 200))
    case("er80_perseed", s, r, o, 80, 3, specs)

    # 6. relation filter restatement on the SURVEY 8c probe graph
    ts = power_law(200, 800, 4, seed=3)
    s, r, o = arrays_of(ts)
    rng = np.random.default_rng(42)
    specs = [([e], 3, sem, [1, 3], 100 if sem == "exact" else NO_PATHS)
             for e in range(0, 200, 7) for sem in SEMS]
    for e in range(0, 200, 5):
        rel = sorted(rng.choice(4, size=int(rng.integers(1, 4)), replace=False).tolist())
        specs.append(([e], 2, "frontier", rel, 25))
    specs.append(([0, 1, 2], 3, "exact", [0, 2], 64))
    specs.append(([3], 2, "frontier", [], 5))  # empty mask: nothing passes
    case("pl200_filter", s, r, o, 200, 4, specs)

    # 7. hub-heavy graph: deep walks, truncation at several caps
    ts = power_law(500, 5000, 4, seed=7, alpha=1.5)
    s, r, o = arrays_of(ts)
    deg = np.bincount(s, minlength=500)
    hubs = np.argsort(-deg, kind="stable")[:6].tolist()
    specs = []
    for h in hubs:
        for k, cap in ((1, 3), (2, 100), (2, 1000), (3, 257)):
            specs.append(([h], k, "exact", None, cap))
        specs.append(([h], 3, "frontier", None, NO_PATHS))
        specs.append(([h], 3, "cumulative", None, NO_PATHS))
    specs.append((hubs[:3], 2, "exact", None, 500))
    specs.append((hubs[:2], 2, "exact", [1, 2], 300))
    case("pl500_hubs", s, r, o, 500, 4, specs)

    # 8. acceptance-grid subset (tests/test_acceptance.py:45-53, 81-116)
    sizes = np.geomspace(100, 10_000, 50).astype(int)
    for i in (0, 7, 19, 33, 49):
        t = int(sizes[i])
        n = max(50, min(1000, t // 8))
        gen = erdos_renyi if i % 2 == 0 else power_law
        ts = gen(n, t, 4, seed=1000 + i)
        s, r, o = arrays_of(ts)
        prng = random.Random(i)
        queries = [sorted(prng.sample(range(n), prng.randint(1, min(5, n)))) for _ in range(3)]
        case(f"grid{i:02d}", s, r, o, n, 4,
             [(q, 5, sem, None, NO_PATHS) for q in queries for sem in SEMS])

    # 9. configs[0] (C1): the reference's own power_law(10k, 50k, 16, 1.1)
    ts = power_law(10_000, 50_000, 16, seed=0, alpha=1.1)
    s, r, o = arrays_of(ts)
    seeds = np.random.default_rng(1).choice(10_000, 64, replace=False).tolist()
    specs = [([e], 2, "frontier", None, 10_000) for e in seeds]
    specs += [([e], 2, sem, None, NO_PATHS) for e in seeds for sem in ("exact", "cumulative")]
    specs += [([e], 3, "frontier", None, NO_PATHS) for e in seeds[:16]]
    mrng = np.random.default_rng(5)
    specs += [([e], 2, "frontier", sorted(mrng.choice(16, 4, replace=False).tolist()), 10_000)
              for e in seeds[:32]]
    specs += [([0], 2, "exact", None, 10_000), ([0], 1, "frontier", None, NO_PATHS)]
    case("c1", s, r, o, 10_000, 16, specs)


if __name__ == "__main__":
    main()
