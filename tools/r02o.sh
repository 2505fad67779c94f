#!/bin/bash
# Measurement pass: bench line (N=1, C3 headline + side configs), C5 through the C++ slab loop,
# ncu launch list, and the six C3 kernels under ncu --set full at the benched 64 images.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err
echo "bench exit $?"; cat gpurun_out/r02o_bench.json | head -c 600; echo
timeout 600 python bench.py --config C5 --slab --steps 3 --warmup 1 > gpurun_out/r02o_slab.json 2> gpurun_out/r02o_slab.err
echo "slab exit $?"; cat gpurun_out/r02o_slab.json | head -c 400; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02o_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/r02o_ncu_list.log 2>&1
echo "ncu list exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'cols_sep|rows_|dst_tcols' \
  -s 7 -c 6 -o gpurun_out/r02o_full64 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs \
  > gpurun_out/r02o_ncu_full.log 2>&1
echo "ncu full exit $?"
