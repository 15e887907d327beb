#!/bin/bash
# Round-2 baseline on a fresh box: GPU tests, bench line, C4 k=3 ncu capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo bench=$?
grep '^{' gpurun_out/r02_bench.log | tail -1 > gpurun_out/r02_bench.json
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"mat_kernel|pull_kernel|flag_|push_" -s 14 -c 14 \
  -f -o /tmp/c4 python tools/prof_c4.py 3 > gpurun_out/r02_ncu_c4.log 2>&1; echo c4=$?
python tools/ncu_summary.py /tmp/c4.ncu-rep > gpurun_out/r02_ncu_c4.txt
python tools/ncu_traffic.py /tmp/c4.ncu-rep gpurun_out/r02_c4_traffic.json > /dev/null
cp /tmp/c4.ncu-rep gpurun_out/r02_c4.ncu-rep 2>/dev/null
ls -la gpurun_out/r02_c4.ncu-rep
