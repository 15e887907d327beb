# kernel times of one C4 k=2 wave (ncu, serialised, cold-ish caches)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
timeout 900 ncu --clock-control none --profile-from-start off \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
  --csv python tools/prof_c4.py 2 > gpurun_out/c4k2_ncu.csv 2> gpurun_out/c4k2_ncu.err; echo ncu=$?
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/c4k2_ncu.csv")))
hdr = None; k = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"][:70])
        k.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"]
for (i, name), m in k.items():
    print(f"{i:>4} {name:70s} us={float(m['gpu__time_duration.sum'])/1e3:8.1f} rd={float(m['dram__bytes_read.sum'])/1e6:8.1f}MB wr={float(m['dram__bytes_write.sum'])/1e6:8.1f}MB inst={float(m['smsp__inst_executed.sum'])/1e6:8.1f}M")
PY
