"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel.

    python tools/summarize_launches.py gpurun_out/launches.csv > profiles/rNN_launches.txt

ncu times are cold-cache and serialised: compare each kernel's SHARE of the
step with the CUDA-event breakdown bench.py prints, not the absolutes.
"""

import collections
import csv
import sys


def main(path: str) -> None:
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                data.append(d)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        name = name.replace("th::<unnamed>::", "").replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"# {path}: {len(data)} launches, {tot / 1e3:.1f} us total (ncu cold-cache, serialised)")
    print(f"{'us':>10} {'share':>6} {'n':>5}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1] / 1e3:10.1f} {100 * v[1] / tot:5.1f}% {v[0]:5d}  {k[:110]}")


if __name__ == "__main__":
    main(sys.argv[1])
