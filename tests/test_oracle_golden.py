"""Pin the CPU oracle against vectors produced by the real reference.

Every golden case (tests/golden/*.npz, made by make_golden.py from the
unmodified triplehop package) is replayed through oracle/khop_oracle.py.
The oracle is the checker for the GPU parity tests, so it must agree with
the reference bit for bit before it is trusted.
"""

import numpy as np
import pytest

from golden_io import all_cases, load_case
from oracle import khop_oracle as orc

CASES = all_cases()


@pytest.mark.parametrize("path", CASES, ids=[p.stem for p in CASES])
def test_oracle_matches_reference_golden(path):
    case = load_case(path)
    g = orc.build_csr(case.subj, case.rel, case.obj, case.n_entities, case.n_relations)
    for q in case.queries:
        view, l2g = (g, None) if q.relations is None else orc.filtered_view(g, q.relations)
        trace = orc.hop_trace(view, q.seeds, q.k, q.semantics)
        assert len(trace) == q.k
        for h, (fr, act) in enumerate(trace):
            assert np.array_equal(fr, q.frontiers[h]), (case.name, q.seeds, h)
            glob = act if l2g is None else l2g[act]
            assert np.array_equal(glob, q.activated[h]), (case.name, q.seeds, h)
        if q.want_paths:
            paths, trunc = orc.walk_paths(view, q.seeds, q.k, q.max_paths)
            if l2g is not None:
                paths = [tuple(int(l2g[t]) for t in p) for p in paths]
            assert paths == q.paths
            assert trunc == q.truncated


def test_golden_set_is_complete():
    names = {p.stem for p in CASES}
    for required in ("tiny", "c1", "pl200_filter", "pl500_hubs", "interleave", "empty"):
        assert required in names


def test_oracle_contract_errors():
    g = orc.build_csr([0, 1], [0, 0], [1, 0], 2, 1)
    with pytest.raises(ValueError):
        orc.hop_trace(g, [0], 0)
    with pytest.raises(ValueError):
        orc.hop_trace(g, [5], 1)
    with pytest.raises(ValueError):
        orc.walk_paths(g, [0], 1, -1)
    with pytest.raises(ValueError):
        orc.build_csr([3], [0], [0], 2, 1)
    with pytest.raises(ValueError):
        orc.build_csr([0], [2], [0], 2, 1)


def test_csr_layout_tiny():
    # tests/test_incidence.py:55-61 of the reference
    g = orc.build_csr([0, 1, 0, 2], [0, 1, 0, 2], [1, 2, 2, 0], 3, 3)
    assert g.row(0).tolist() == [0, 2]
    assert g.row(1).tolist() == [1]
    assert g.row(2).tolist() == [3]


def test_retrieve_one_filter_matches_bruteforce():
    rng = np.random.default_rng(0)
    E, R, T = 40, 5, 300
    s, r, o = rng.integers(0, E, T), rng.integers(0, R, T), rng.integers(0, E, T)
    g = orc.build_csr(s, r, o, E, R)
    allowed = [1, 4]
    for seed in range(0, E, 3):
        res = orc.retrieve_one(g, seed, 3, "exact", allowed, paths=True, max_paths=None)
        cur = {seed}
        for h in range(3):
            act = sorted(t for t in range(T) if s[t] in cur and r[t] in allowed)
            assert res["activated"][h].tolist() == act
            cur = {int(o[t]) for t in act}
            assert res["frontiers"][h].tolist() == sorted(cur)
        for p in res["paths"]:
            assert s[p[0]] == seed and all(r[t] in allowed for t in p)
            assert all(o[a] == s[b] for a, b in zip(p, p[1:]))
        assert res["paths"] == sorted(res["paths"])
