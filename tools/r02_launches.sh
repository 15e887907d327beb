# per-kernel launch lists (ncu gpu__time_duration) of one C2 and one C4 k=3 batch
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file /tmp/c2l.csv python tools/prof_c2.py --batches 2 > /dev/null 2>&1; echo c2=$?
python tools/summarize_launches.py /tmp/c2l.csv > gpurun_out/l_c2.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file /tmp/c4l.csv python tools/prof_c4.py 3 > /dev/null 2>&1; echo c4=$?
python tools/summarize_launches.py /tmp/c4l.csv > gpurun_out/l_c4.txt
cp /tmp/c4l.csv gpurun_out/l_c4.csv
