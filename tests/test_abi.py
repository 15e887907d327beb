"""CPU-side checks of the C ABI library and the host logic (no kernel runs)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "th_b200.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(th_[a-z_0-9]+)\s*\(", text, re.M)))


def test_header_declares_the_binding_list():
    from paper_2604_18913_b200 import _lib

    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    from paper_2604_18913_b200 import _lib

    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.th_abi_version() == _lib.ABI_VERSION


def test_sm100a_code_in_library():
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    from paper_2604_18913_b200 import _lib

    out = subprocess.run([tool, "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_null_handles_are_rejected_without_a_gpu():
    from paper_2604_18913_b200 import _lib

    lib = _lib.load()
    res = _lib.Result()
    assert lib.th_finish(None, ctypes.byref(res)) == _lib.TH_ERR_INVALID
    assert b"NULL" in lib.th_last_error()
    with pytest.raises(ValueError):
        _lib.check(_lib.TH_ERR_INVALID)
    assert lib.th_session_launch_count(None) == -1


def test_semantics_parse_matches_reference_spellings():
    from paper_2604_18913_b200 import HopSemantics

    for name in ("exact", "exact-walk", "exact_walk", "walk", " EXACT "):
        assert HopSemantics.parse(name) is HopSemantics.EXACT_WALK
    assert HopSemantics.parse("frontier") is HopSemantics.FRONTIER
    assert HopSemantics.parse("cumulative") is HopSemantics.CUMULATIVE
    with pytest.raises(ValueError):
        HopSemantics.parse("bfs")


def test_entity_vector_canonical_form():
    from paper_2604_18913_b200 import EntityVector, jaccard

    v = EntityVector([5, 1, 5, 3], 10)
    assert v.ids.tolist() == [1, 3, 5]
    assert not v.ids.flags.writeable
    with pytest.raises(ValueError):
        EntityVector([10], 10)
    with pytest.raises(ValueError):
        EntityVector([-1], 10)
    assert jaccard(EntityVector([1, 2], 5), EntityVector([2, 1], 5)) == 1.0
    assert jaccard(set(), set()) == 1.0


def test_relation_mask_normalisation():
    from paper_2604_18913_b200.retriever import _relation_masks

    shared = _relation_masks([0, 33, 39], 3, 40)
    assert shared.shape == (3, 2)
    assert shared[0, 0] == 1 and shared[0, 1] == (1 << 1) | (1 << 7)
    per = _relation_masks([[1], [], [2, 3]], 3, 4)
    assert per[:, 0].tolist() == [2, 0, 12]
    boolm = np.zeros((2, 4), dtype=bool)
    boolm[1, 3] = True
    assert _relation_masks(boolm, 2, 4)[:, 0].tolist() == [0, 8]
    with pytest.raises(ValueError):
        _relation_masks([4], 1, 4)
    with pytest.raises(ValueError):
        _relation_masks(np.array([[1 << 5]], dtype=np.uint32), 1, 4)


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2604_18913_b200 as th

    with pytest.raises(RuntimeError, match="CUDA"):
        th.build_incidence([(0, 0, 1)], 2, 1)


def test_product_never_imports_the_oracle():
    pkg = ROOT / "paper_2604_18913_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in f.read_text().replace("oracle/", ""), f


def test_pipeline_rejects_bad_depth():
    """RetrievalPipeline validates its depth before touching the device."""
    import paper_2604_18913_b200 as th

    with pytest.raises(ValueError):
        th.RetrievalPipeline(None, depth=0)
