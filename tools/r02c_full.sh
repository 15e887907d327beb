#!/bin/bash
# Round-2 (third session) check: full GPU suite, smoke, default bench line (saved as JSON)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1500 python -m pytest -q tests -m gpu > gpurun_out/full_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/full_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/r02c_bench_full.log 2>&1; echo bench=$?
grep '^{' gpurun_out/r02c_bench_full.log | tail -1 > gpurun_out/r02c_bench_full.json
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02c_bench_full.json"))
print("C2", round(d["value"]), d["ms_per_step"], "roofline", round(d["roofline"]["frac"], 3), "pull", round(d["roofline_pull"]["frac"], 3), "e2e", round(d["e2e"]["value"]))
print("C4", {k: round(d["c4"][k]["ms_per_batch"], 3) for k in ("k2", "k3")}, "part", {k: round(d["partitioned"][k]["ms_per_wave"], 3) for k in ("k2", "k3")})
print("c3", round(d["c3"]["ms_per_batch"], 3), "cpu", d["cpu_baseline"]["value"])
PY
