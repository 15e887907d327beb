cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 1500 python tools/c5_probe.py --waves 16 --partitioned > gpurun_out/c5_part.log 2>&1; echo c5part=$?; tail -4 gpurun_out/c5_part.log
