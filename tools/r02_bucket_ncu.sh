# ncu of the bucketed K4 write pass on one C4 k=3 wave (kernel times + DRAM)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 900 ncu --clock-control none --profile-from-start off -k regex:"bucket|rs_count|mat_kernel" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --csv python tools/prof_c4.py 3 > gpurun_out/bucket_ncu.csv 2> gpurun_out/bucket_ncu.err; echo ncu=$?
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/bucket_ncu.csv")))
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        print(d["Kernel Name"][:60], d["Metric Name"], d["Metric Value"], d["Metric Unit"])
PY
