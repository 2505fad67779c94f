#!/bin/bash
# ncu --set full of one dst_tcols_w launch and one dst_tcols launch (C3, 64 images)
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'dst_tcols' -s 2 -c 1 -o gpurun_out/r02f_w -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/r02f_w.log 2>&1
echo "ncu w exit $?"
DBX_WDST=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'dst_tcols' -s 2 -c 1 -o gpurun_out/r02f_old -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/r02f_old.log 2>&1
echo "ncu old exit $?"
