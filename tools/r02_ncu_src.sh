cd "${GRAFT_REPO_ROOT:-/root/repo}"
# the last-layer K4 write pass of a C4 k=3 batch: 3 list-write launches per batch
export CUDA_MODULE_LOADING=EAGER
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k regex:"pull_kernel" -s 8 -c 1 \
  -f -o /tmp/w python tools/prof_c4.py 3 > gpurun_out/w.log 2>&1; echo w=$?
python tools/ncu_summary.py /tmp/w.ncu-rep > gpurun_out/w.txt
ncu -i /tmp/w.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/w_src.csv 2>/dev/null; echo src=$?
ncu -i /tmp/w.ncu-rep --page source --csv > gpurun_out/w_src_cuda.csv 2>/dev/null; echo src2=$?
ls -la gpurun_out/w_src*.csv
