#!/bin/bash
# launch list (ncu gpu__time_duration, cold-cache, serialised) of a short C2 bench run
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file /tmp/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-c4 --no-c5 \
  > gpurun_out/r02c_ncu_launches.log 2>&1; echo launches=$?
python tools/summarize_launches.py /tmp/launches.csv > gpurun_out/r02c_launches.txt; echo sum=$?
head -30 gpurun_out/r02c_launches.txt
