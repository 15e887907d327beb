cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python tools/ab_c2.py "{}" "{'k4_mode': 0}" "{'pull_screen': 1}" "{'list_min_entities': 1099511627776}" > gpurun_out/abc2.log 2>&1; echo ab=$?
cat gpurun_out/abc2.log
