#!/bin/bash
# A/B of two builds of the library (TH_B200_LIB): C2 and C4 k=3, interleaved
cd "${GRAFT_REPO_ROOT:-/root/repo}"
A=${A:-gpurun_out/ab/lib_base.so}
B=${B:-paper_2604_18913_b200/lib/libth_b200.so}
for r in 1 2; do
  for L in $A $B; do
    echo "== $L C2"; TH_B200_LIB=$L timeout 300 python tools/ab_c2.py "{}" 2>&1 | tail -2
  done
done
for L in $A $B $A $B; do
  echo "== $L C4"; TH_B200_LIB=$L timeout 600 python tools/ab_c4.py "{}" 2>&1 | tail -3
done
