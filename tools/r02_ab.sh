cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/ab_tests.log
timeout 600 python tools/ab_c4.py "{'k4_mode': 0}" "{'k4_mode': 1}" > gpurun_out/ab.log 2>&1; echo ab=$?
tail -8 gpurun_out/ab.log
