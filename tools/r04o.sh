#!/bin/bash
# e2e chunk-split A/B, three interleaved repeats
set -u
mkdir -p gpurun_out
run() {
  v=$(DBX_E2E_SPLIT=$1 DBX_CHUNK_DEPTH=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs 2>>gpurun_out/r04o.err \
      | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["e2e"]["value"],1))')
  echo "split=$1 depth=$2 value/e2e $v" | tee -a gpurun_out/r04o_sweep.txt
}
for rep in 1 2 3; do
  run 8,24,24,8 2
  run 9,46,9 2
  run 9,23,23,9 2
  run 12,40,12 2
  run 6,52,6 2
done
