#!/bin/bash
# Round-2 measurement call B: FP64 DMMA/DFMA concurrency probe, per-class
# kernel times of the side configs, and the C3 six-kernel ncu --set full
# capture at the benched 64 images (DRAM traffic with arrays far above L2).
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/r02b_fp64.json 2>&1
cat gpurun_out/r02b_fp64.json
for c in C1 C2 C4 C5; do timeout 300 python tools/config_probe.py $c >> gpurun_out/r02b_probe.jsonl 2>>gpurun_out/r02b_probe.err; done
cat gpurun_out/r02b_probe.jsonl
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'cols_sep|rows_|dst_tcols' \
  -s 7 -c 6 -o gpurun_out/r02b_full64 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs \
  > gpurun_out/r02b_ncu_full.log 2>&1
echo "ncu full exit $?"; tail -3 gpurun_out/r02b_ncu_full.log
