"""The GPU /query backend answers the REAL reference service's request
script identically (tests/golden/service.json, make_golden_service.py):
graph directories and partition directories kept resident in the device
registry, unknown labels, every semantics, capped paths, and the LRU
counters carried from request to request."""

import json

import pytest

from golden_io import HERE as GOLDEN

pytestmark = pytest.mark.gpu


def test_query_script_matches_reference(cuda_device):
    from fastapi.testclient import TestClient

    from paper_2604_18913_b200.service import DeviceGraphRegistry, create_app

    reg = DeviceGraphRegistry()
    client = TestClient(create_app(reg))
    calls = json.loads((GOLDEN / "service.json").read_text())
    for c in calls:
        req = dict(c["request"])
        for key in ("graph_dir", "partitioned_dir"):
            if key in req:
                req[key] = str(GOLDEN / req[key])
        resp = client.post("/query", json=req)
        assert resp.status_code == c["status"], (c["request"], resp.json())
        assert resp.json() == c["body"], c["request"]
    # one device graph and two partitioned graphs (capacities 2 and 16) stayed resident
    assert len(reg._loaded) == 3
