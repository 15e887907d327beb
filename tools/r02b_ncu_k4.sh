#!/bin/bash
# ncu --set full with source of the C4 k=3 last-layer K4 write pass (5th mat_kernel launch of the wave)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"mat_kernel|rs_count" -f -o gpurun_out/r02b_k4 python tools/prof_c4.py 3 > gpurun_out/r02b_ncu_k4.log 2>&1; echo ncu=$?
python tools/ncu_summary.py gpurun_out/r02b_k4.ncu-rep > gpurun_out/r02b_k4.txt; echo sum=$?
