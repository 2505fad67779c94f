#!/bin/bash
# C5 separate-pass kernels: launch list of the first iterations and ncu --set full of the transform kernels
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r04c_c5_launches.csv \
  python tools/config_probe.py C5 0 1 1 > gpurun_out/r04c_launch.log 2>&1
echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'dst_rows|dst_cols|tdt' -s 3 -c 4 -o gpurun_out/r04c_c5_full -f \
  python tools/config_probe.py C5 0 1 1 > gpurun_out/r04c_full.log 2>&1
echo "ncu full exit $?"
