#!/bin/bash
# e2e chunk-split sweep at v56 kernel speeds (bench e2e leg; value printed alongside)
set -u
mkdir -p gpurun_out
for depth in 2 3; do
for sp in 8,24,24,8 8,24,16,16 8,16,16,16,8 4,12,16,16,12,4 8,20,20,12,4 16,24,16,8; do
  r=$(DBX_CHUNK_DEPTH=$depth DBX_E2E_SPLIT=$sp timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs 2>>gpurun_out/r02w.err | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["e2e"]["value"],1))')
  echo "depth=$depth split=$sp $r" | tee -a gpurun_out/r02w_e2e.txt
done
done
