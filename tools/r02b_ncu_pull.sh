#!/bin/bash
# ncu --set full of the C4 k=3 pull kernels (screen + compacted pull) of one wave
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"pull" -f -o gpurun_out/r02b_pull python tools/prof_c4.py ${K:-3} > gpurun_out/r02b_ncu_pull.log 2>&1; echo ncu=$?
tail -3 gpurun_out/r02b_ncu_pull.log
python tools/ncu_summary.py gpurun_out/r02b_pull.ncu-rep > gpurun_out/r02b_pull.txt; echo sum=$?
