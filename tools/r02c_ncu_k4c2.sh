#!/bin/bash
# ncu --set full with source of one C2 k=3 batch's K4 kernels (the last
# layer's cached write pass is the step's tail)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"mat_kernel" -f -o gpurun_out/r02c_k4c2 python tools/prof_c2.py > gpurun_out/r02c_ncu_k4c2.log 2>&1; echo ncu=$?
python tools/ncu_summary.py gpurun_out/r02c_k4c2.ncu-rep > gpurun_out/r02c_k4c2.txt; echo sum=$?
