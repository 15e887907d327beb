"""A pure C caller (examples/c_abi_khop.c: no Python, no torch) drives the
engine through include/th_b200.h; its printed frontiers, edge counts and
paths must equal the oracle's."""

import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import khop_oracle as orc
from test_gpu_parity import _hub_graph

ROOT = Path(__file__).resolve().parent.parent


def compile_example(tmp_path) -> Path:
    exe = tmp_path / "c_abi_khop"
    lib = ROOT / "paper_2604_18913_b200" / "lib"
    subprocess.run(["gcc", str(ROOT / "examples" / "c_abi_khop.c"), f"-I{ROOT / 'include'}",
                    "-I/usr/local/cuda/include", f"-L{lib}", "-lth_b200", "-L/usr/local/cuda/lib64",
                    "-lcudart", f"-Wl,-rpath,{lib}", "-Wall", "-Werror", "-o", str(exe)], check=True)
    return exe


def test_c_example_compiles(tmp_path):
    """The header is plain C and the library links from C (no GPU needed)."""
    assert compile_example(tmp_path).exists()


@pytest.mark.gpu
def test_c_caller_matches_oracle(tmp_path, cuda_device):
    exe = compile_example(tmp_path)
    s, r, o = _hub_graph(500, 3000, 8, seed=23)
    E, R, k = 500, 8, 2
    rng = np.random.default_rng(4)
    seeds = rng.integers(0, E, 40)
    text = "".join(f"{a} {b} {c}\n" for a, b, c in zip(s, r, o)) + "--\n" + " ".join(map(str, seeds)) + "\n"
    out = subprocess.run([str(exe), str(E), str(R), str(k)], input=text, capture_output=True,
                         text=True, check=True, timeout=120).stdout.splitlines()
    og = orc.build_csr(s, r, o, E, R)
    it = iter(out)
    for sd in seeds:
        assert next(it) == f"seed {sd}"
        ref = orc.retrieve_one(og, int(sd), k, "frontier", None, paths=True, max_paths=10_000)
        for h in range(k):
            parts = next(it).split()
            assert parts[:2] == ["hop", str(h + 1)] and int(parts[3]) == ref["edges"][h]
            assert [int(x) for x in parts[5:]] == ref["frontiers"][h].tolist()
        parts = next(it).split()
        n = int(parts[1])
        assert bool(int(parts[3])) == ref["truncated"]
        paths = [tuple(int(x) for x in next(it).split()[1:]) for _ in range(n)]
        assert paths == ref["paths"]
