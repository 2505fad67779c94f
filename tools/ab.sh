#!/bin/bash
# A/B throughput of library variants on the headline workload (interleaved,
# two rounds): tools/ab.sh TAG LIB1 [LIB2 ...]   (LIB = path to a libdbx*.so)
TAG=$1; shift
mkdir -p gpurun_out
for round in 1 2; do
  for lib in "$@"; do
    v=$(DBX_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other-configs 2>>gpurun_out/${TAG}_ab.err \
        | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]["class_ms_per_step"]; print(round(d["value"],1), {k: round(v,2) for k,v in r.items()})')
    echo "$round $(basename $lib) $v" | tee -a gpurun_out/${TAG}_ab.txt
  done
done
