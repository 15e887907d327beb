"""Sum dram__bytes_read + dram__bytes_write per kernel group of an ncu report
(one captured k=3 batch) into a JSON file bench.py reads for roofline.traffic.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep profiles/r01_c2_traffic.json
"""

import csv
import io
import json
import re
import subprocess
import sys

GROUPS = {"frontier": r"mat_kernel<.*(DenseSrc|ListSrc)|mat_scan|flag_|rs_count|bucket_", "pull": r"pull_(kernel|screen|edges)",
          "push": r"push_(light|heavy)", "clear": r"clear_rows"}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {g: {"bytes": 0.0, "launches": 0, "us": 0.0} for g in GROUPS}
    for d in data:
        name = d[hdr.index("Kernel Name")]
        for g, pat in GROUPS.items():
            if re.search(pat, name):
                b = 0.0
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    i = hdr.index(m)
                    b += float(d[i]) * scale[units[i]]
                i = hdr.index("gpu__time_duration.sum")
                res[g]["bytes"] += b
                res[g]["us"] += float(d[i]) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                                               "msecond": 1e3, "ms": 1e3}.get(units[i], 1.0)
                res[g]["launches"] += 1
    res["source"] = rep
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
