#!/bin/bash
# ncu --set full of one iteration's kernels on C4, C2 and C1, summarised on the box
# (shared-memory excess wavefronts, LSU pipe); the reports stay in /tmp
set -u
mkdir -p gpurun_out
for C in C4 C2 C1; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'dst_|conv_|rows_|cols_|tdt' -s 12 -c 8 -o /tmp/r04e_${C}_full -f \
    python tools/config_probe.py $C 0 1 1 > gpurun_out/r04e_${C}.log 2>&1
  echo "ncu $C exit $?"
  python tools/ncu_excess.py /tmp/r04e_${C}_full.ncu-rep 6 > gpurun_out/r04e_${C}_excess.txt 2>&1
done
