"""Per-CUDA-line instructions and stall samples from an ncu source export.

    ncu -i rep --page source --csv --print-source cuda,sass -k regex:K \
        --launch-skip S --launch-count 1 > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    lines = []
    for r in rows:
        if r and r[0].isdigit():
            f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
            try:
                lines.append((int(r[0]), f(r[ii]), f(r[si]), r[1][:90]))
            except (ValueError, IndexError):
                continue
    ti = sum(x[1] for x in lines) or 1
    ts = sum(x[2] for x in lines) or 1
    print(f"total inst {ti:.3e} samples {ts:.0f}")
    for ln, i, s, src in sorted(lines, key=lambda x: -x[2])[:top]:
        print(f"{ln:5d} inst {100 * i / ti:5.1f}% stall {100 * s / ts:5.1f}%  {src}")


if __name__ == "__main__":
    main()
