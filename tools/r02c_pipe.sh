#!/bin/bash
# streaming e2e: pipeline parity tests, PCIe probe, quick bench (no CPU leg)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest -q tests/test_gpu_pipeline.py > gpurun_out/pipe_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/pipe_tests.log
timeout 300 python tools/d2h_probe.py > gpurun_out/d2h_probe.txt 2>&1; echo probe=$?; cat gpurun_out/d2h_probe.txt
timeout 900 python bench.py --no-cpu > gpurun_out/pipe_bench.log 2>&1; echo bench=$?
python - <<'PY'
import json
for l in open("gpurun_out/pipe_bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        e = d["e2e"]
        print("C2", round(d["value"]), round(d["ms_per_step"], 4), "e2e pipe", round(e["value"]), round(e["link_GBps"], 1), "blocking", round(e["blocking"]["value"]), round(e["blocking"]["link_GBps"], 1))
PY
tail -3 gpurun_out/pipe_bench.log | grep -v '^{' | cut -c1-400
