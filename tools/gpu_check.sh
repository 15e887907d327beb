#!/bin/bash
# Quick GPU iteration: parity suite + short bench (no CPU leg).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu "$@" > gpurun_out/bench_quick.log 2>&1; echo bench=$?
python - <<'PY'
import json
for l in open("gpurun_out/bench_quick.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value", round(d["value"]), "ms/step", round(d["ms_per_step"], 4), "roofline", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3))
        print("per_k", {k: round(v["ms_per_batch"], 4) for k, v in d["per_k"].items()})
        print("kernels", {k: round(v, 4) for k, v in d["kernel_ms_per_step"].items()})
        print("e2e", round(d["e2e"]["value"]))
PY
tail -5 gpurun_out/bench_quick.log | grep -v '^{' | cut -c1-300
