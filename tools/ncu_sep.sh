#!/bin/bash
# ncu --set full of one separable-pipeline iteration (six kernels) of the C3 bench
TAG=${1:-sep}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'cols_sep|rows_|dst_tcols' \
  -s 7 -c 6 -o gpurun_out/${TAG}_full -f python bench.py --images 8 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs \
  > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?"
