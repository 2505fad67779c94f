#!/bin/bash
# Batch-size sweep of the C3 fused pipeline: per-image kernel times when the
# per-iteration working set fits in L2 (B small) vs not (B = 64).
set -u
mkdir -p gpurun_out
for B in 1 2 4 8 16 64; do
  timeout 300 python bench.py --images $B --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other-configs 2>>gpurun_out/r03b.err \
   | python -c "
import json,sys
d=json.loads(sys.stdin.read()); B=$B
ks=d['roofline']['kernels']
print(B, round(d['value'],1), round(d['ms_per_step'],3), [(k['kernel'], round(k['avg_launch_ms']*64/B,3)) for k in ks])" | tee -a gpurun_out/r03b_sweep.txt
done
