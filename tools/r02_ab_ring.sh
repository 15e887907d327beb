cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_scale.py > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/ab_tests.log
timeout 900 python tools/ab_c4.py "{\"k4_ring\": 0}" "{\"k4_ring\": 1}" 2>&1 | tail -8
timeout 600 python tools/ab_c2.py "{\"k4_ring\": 0}" "{\"k4_ring\": 1}" 2>&1 | tail -4
