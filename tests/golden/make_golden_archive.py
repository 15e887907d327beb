"""Write LKG1 archives with the REAL reference (build container only):

    python tests/golden/make_golden_archive.py [/root/reference/pkg/src]

tiny.lkg: the tiny graph of the reference's tests/conftest.py:6-18;
c1.lkg: the C1 graph (synth.power_law(10_000, 50_000, 16, seed=0, alpha=1.1)).
Both come from triplehop.archive.graph_to_bytes (archive.py:66-81), so the
device loader is pinned to files the reference itself produced.
"""

import sys
from pathlib import Path

import numpy as np

REF = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from triplehop.archive import graph_to_bytes  # noqa: E402
from triplehop.incidence import build_incidence  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    for name, E, R in (("tiny", 3, 3), ("c1", 10_000, 16)):
        z = np.load(OUT / f"{name}.npz")
        cols = tuple(z[c].astype(np.int64) for c in ("subj", "rel", "obj"))
        (OUT / f"{name}.lkg").write_bytes(graph_to_bytes(build_incidence(cols, E, R)))
    print("wrote tiny.lkg, c1.lkg")


if __name__ == "__main__":
    main()
