cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/ab_tests.log
timeout 600 python tools/ab_c2.py ${AB:-"{}" "{'k4_mode': 2}"} 2>&1 | tail -6
timeout 600 python tools/ab_c4.py ${AB:-"{}" "{'k4_mode': 2}"} 2>&1 | tail -8
