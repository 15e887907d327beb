cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_graphs.py tests/test_gpu_c_abi.py > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/ab_tests.log
timeout 900 python -m pytest -q -x tests/test_gpu_scale.py -k "c3" > gpurun_out/ab_tests2.log 2>&1; echo tests2=$?; tail -3 gpurun_out/ab_tests2.log
timeout 600 python tools/ab_c3.py "{'paths_k2': 0}" "{'paths_k2': 1}" 2>&1 | tail -4
