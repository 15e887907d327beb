#!/bin/bash
# bench line with the C4 streamed e2e (no CPU leg)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1200 python bench.py --no-cpu > gpurun_out/c4e2e_bench.log 2>&1; echo bench=$?
python - <<'PY'
import json
for l in open("gpurun_out/c4e2e_bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("C2", round(d["value"]), "e2e", round(d["e2e"]["value"]), round(d["e2e"]["link_GBps"], 1))
        for k in ("k2", "k3"):
            c = d["c4"][k]
            print("C4", k, round(c["ms_per_batch"], 3), "e2e", c.get("e2e"))
PY
tail -4 gpurun_out/c4e2e_bench.log | grep -v '^{' | cut -c1-300
