"""The /query service layer without a GPU: request validation and error
payloads against the REAL reference's answers (tests/golden/service.json,
make_golden_service.py), label lookup."""

import json

import pytest

from golden_io import HERE as GOLDEN


def _golden():
    return json.loads((GOLDEN / "service.json").read_text())


def _local(req):
    out = dict(req)
    for key in ("graph_dir", "partitioned_dir"):
        if key in out:
            out[key] = str(GOLDEN / out[key])
    return out


def test_rejected_requests_match_reference():
    """Requests the reference rejects are rejected before any device work,
    with its status codes and messages."""
    from fastapi.testclient import TestClient

    from paper_2604_18913_b200.service import create_app

    client = TestClient(create_app())
    bad = [c for c in _golden() if c["status"] != 200]
    assert len(bad) == 6
    for c in bad:
        resp = client.post("/query", json=_local(c["request"]))
        assert resp.status_code == c["status"]
        assert resp.json() == c["body"], c["request"]
    assert client.get("/healthz").json()["status"] == "ok"


def test_labels_and_lookup():
    from paper_2604_18913_b200.service import Labels, lookup_entities

    lab = Labels(["a", "b", "a", "c"])  # duplicates keep their first id
    assert len(lab) == 3 and lab.id_of("c") == 2 and lab.label_of(1) == "b" and lab.id_of("zz") is None
    assert lookup_entities(["c", "x", "a", "c", "y"], lab) == ([0, 2], ["x", "y"])


def test_graph_dir_label_mismatch_is_integrity_error(tmp_path):
    import shutil

    from paper_2604_18913_b200.errors import IntegrityError
    from paper_2604_18913_b200.service import load_graph_dir

    d = tmp_path / "g"
    shutil.copytree(GOLDEN / "graphdir", d)
    (d / "relations.txt").write_text("r0\n")
    with pytest.raises((IntegrityError, RuntimeError)):  # (RuntimeError: no device to build on)
        load_graph_dir(d)


def test_dictionary_export():
    import paper_2604_18913_b200 as th

    d = th.Dictionary()
    assert [d.add(x) for x in ("p", "q", "p")] == [0, 1, 0]
    assert "q" in d and len(d) == 2 and d == th.Dictionary(["p", "q"])
    assert th.lookup_entities(["q", "zz"], d) == th.LookupResult([1], ["zz"])
