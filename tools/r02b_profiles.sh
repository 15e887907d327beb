#!/bin/bash
# Round-2 (second session) evidence for the current code (one GPU call):
#   gpurun_out/r02b_ncu_c2_step.txt / r02b_c2_traffic.json   ncu --set full, one C2 k=3 batch
#   gpurun_out/r02b_ncu_c4.txt / r02b_c4_traffic.json        ncu --set full, one C4 k=3 wave
#   gpurun_out/r02b_launches.txt                            launch list of a short bench run
#   gpurun_out/r02b_bench_full.json                         default bench line (after the traffic files)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -f -o /tmp/c2step python tools/prof_c2.py > gpurun_out/r02b_ncu_c2.log 2>&1; echo c2=$?
python tools/ncu_summary.py /tmp/c2step.ncu-rep > gpurun_out/r02b_ncu_c2_step.txt
python tools/ncu_traffic.py /tmp/c2step.ncu-rep gpurun_out/r02b_c2_traffic.json > /dev/null
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -f -o /tmp/c4wave python tools/prof_c4.py 3 > gpurun_out/r02b_ncu_c4.log 2>&1; echo c4=$?
python tools/ncu_summary.py /tmp/c4wave.ncu-rep > gpurun_out/r02b_ncu_c4.txt
python tools/ncu_traffic.py /tmp/c4wave.ncu-rep gpurun_out/r02b_c4_traffic.json > /dev/null
cp gpurun_out/r02b_c2_traffic.json gpurun_out/r02b_c4_traffic.json profiles/
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file /tmp/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-c4 \
  > gpurun_out/r02b_ncu_launches.log 2>&1; echo launches=$?
python tools/summarize_launches.py /tmp/launches.csv > gpurun_out/r02b_launches.txt
timeout 900 python bench.py > gpurun_out/r02b_bench_full.log 2>&1; echo bench=$?
grep '^{' gpurun_out/r02b_bench_full.log | tail -1 > gpurun_out/r02b_bench_full.json
