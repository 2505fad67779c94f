#!/bin/bash
# ncu --set full of one C5 Rader DST row pass (in-place CT core) and one C4 Bluestein pass
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'dst_rows' -s 4 -c 1 -o gpurun_out/r02l_c5 -f \
  python tools/config_probe.py C5 0 1 1 > gpurun_out/r02l_c5.log 2>&1
echo "ncu c5 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'dst_rows' -s 4 -c 1 -o gpurun_out/r02l_c4 -f \
  python tools/config_probe.py C4 0 1 1 > gpurun_out/r02l_c4.log 2>&1
echo "ncu c4 exit $?"
