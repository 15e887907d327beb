#!/bin/bash
# One GPU call that refreshes the committed evidence for the current code:
#   gpurun_out/bench_full.json      default bench line (CPU leg included)
#   gpurun_out/launches.csv         ncu launch list of a short bench run
#   gpurun_out/step.ncu-rep         ncu --set full of one C2 k=3 step
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
grep '^{' gpurun_out/bench_full.log | tail -1 > gpurun_out/bench_full.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-c4 \
  > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"mat_kernel|pull_kernel|push_|clear_rows|mat_scan" -s 42 -c 21 \
  -o gpurun_out/step python tools/prof_c2.py > gpurun_out/ncu_step.log 2>&1; echo step=$?
