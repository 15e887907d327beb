cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file /tmp/c4l.csv python tools/prof_c4.py 3 > /dev/null 2>&1; echo c4l=$?
python tools/summarize_launches.py /tmp/c4l.csv > gpurun_out/l_c4.txt
cp /tmp/c4l.csv gpurun_out/l_c4.csv
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"mat_kernel|pull_kernel|rs_count|clear_rows|push_" -c 40 \
  -f -o /tmp/c4f python tools/prof_c4.py 3 > gpurun_out/c4f.log 2>&1; echo c4f=$?
python tools/ncu_summary.py /tmp/c4f.ncu-rep > gpurun_out/c4f.txt
ls -la /tmp/c4f.ncu-rep
