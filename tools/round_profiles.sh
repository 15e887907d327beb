#!/bin/bash
# One GPU call that refreshes the committed evidence for the current code:
#   gpurun_out/bench_full.json       default bench line (CPU leg included)
#   gpurun_out/launches.txt          ncu launch list of a short bench run (summarised)
#   gpurun_out/step_summary.txt      ncu --set full of one C2 k=3 step (summarised)
#   gpurun_out/step_traffic.json     its DRAM bytes per kernel group
# (the raw .ncu-rep stays on the box: gpurun_out travels back only under 64 MiB)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
grep '^{' gpurun_out/bench_full.log | tail -1 > gpurun_out/bench_full.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file /tmp/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-c4 \
  > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
python tools/summarize_launches.py /tmp/launches.csv > gpurun_out/launches.txt
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"mat_kernel|pull_kernel|push_|clear_rows|mat_scan" -s 52 -c 26 \
  -f -o /tmp/step python tools/prof_c2.py > gpurun_out/ncu_step.log 2>&1; echo step=$?
python tools/ncu_summary.py /tmp/step.ncu-rep > gpurun_out/step_summary.txt
python tools/ncu_traffic.py /tmp/step.ncu-rep gpurun_out/step_traffic.json
