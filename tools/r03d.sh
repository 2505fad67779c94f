#!/bin/bash
# ncu --set full of the C4 separate-pass kernels (dst_rows PFA 2047, conv FFT 2160, transpose)
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'dst_rows|conv_col|conv_row|transpose' \
  -s 20 -c 7 -o gpurun_out/r03d_c4_full -f python tools/config_probe.py C4 > gpurun_out/r03d_ncu.log 2>&1
echo "ncu exit $?"
tail -3 gpurun_out/r03d_ncu.log
