#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'dst_tcols' -s 2 -c 1 -o gpurun_out/r02h_w -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/r02h_w.log 2>&1
echo "ncu exit $?"
