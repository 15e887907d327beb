# A/B of the current library against lib_prev (C4 k=2/3 and C2), tests first
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_scale.py > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/ab_tests.log
for L in lib lib_prev lib lib_prev; do
  echo "== $L"
  TH_B200_LIB=paper_2604_18913_b200/$L/libth_b200.so timeout 600 python tools/ab_c4.py "{}" 2>&1 | tail -2
done
