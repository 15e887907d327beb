#!/bin/bash
# bench line with the C5 single-GPU leg (no CPU leg)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
SECONDS=0; timeout 1500 python bench.py --no-cpu > gpurun_out/c5_bench.log 2> gpurun_out/c5_bench.err; echo bench=$?
echo elapsed=${SECONDS}s
python - <<'PY'
import json
for l in open("gpurun_out/c5_bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("C2", round(d["value"]), "C4 k3", round(d["c4"]["k3"]["ms_per_batch"], 3))
        print("C5", d["c5"])
PY
tail -5 gpurun_out/c5_bench.err | cut -c1-300
