#!/bin/bash
# launch lists of one C4 and one C2 run (graph path, config_probe): which kernels dominate the side configs
set -u
mkdir -p gpurun_out
for c in C4 C2 C1; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02t_$c.csv \
  python tools/config_probe.py $c 0 1 1 > gpurun_out/r02t_$c.log 2>&1
echo "$c exit $?"
done
