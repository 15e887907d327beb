"""Key metrics per captured launch of an ncu report (read here, no GPU).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [regex]
"""

import csv
import io
import re
import subprocess
import sys

WANT = [
    ("Kernel Name", "kernel"), ("Grid Size", "grid"), ("Block Size", "block"),
    ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"), ("lts__t_bytes.sum", "l2_bytes"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("smsp__inst_executed.sum", "inst"), ("launch__registers_per_thread", "regs"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_lsb"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall_lgthr"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall_mio"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall_ssb"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall_math"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_bar"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "stall_membar"),
    ("smsp__average_warps_issue_stalled_drain_per_issue_active.ratio", "stall_drain"),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "stall_noinst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
]


def main(path, pattern=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for d in data:
        name = d[hdr.index("Kernel Name")]
        if pattern and not re.search(pattern, name):
            continue
        out = []
        for key, short in WANT:
            if key not in hdr:
                continue
            i = hdr.index(key)
            v = d[i]
            if short == "kernel":
                v = re.sub(r"\(.*", "", v.replace("(anonymous namespace)::", ""))[:70]
            out.append(f"{short}={v}{'' if short in ('kernel', 'grid', 'block') else units[i] and ' ' + units[i]}")
        print(" | ".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
