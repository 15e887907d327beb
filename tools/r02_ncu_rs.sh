cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"rs_count_kernel|rs_write_kernel" -s 8 -c 4 \
  -f -o /tmp/rs python tools/prof_c4.py 3 > gpurun_out/rs_ncu.log 2>&1; echo c4=$?
python tools/ncu_summary.py /tmp/rs.ncu-rep > gpurun_out/rs_ncu.txt
cp /tmp/rs.ncu-rep gpurun_out/rs.ncu-rep
