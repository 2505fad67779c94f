#!/bin/bash
# Launch lists of the small configs: per-kernel durations vs the graph's
# per-iteration time (is C1/C2 launch-gap bound or kernel-latency bound?)
set -u
mkdir -p gpurun_out
for C in C1 C2 C4; do
  timeout 300 python tools/config_probe.py $C > gpurun_out/r03c_${C}_probe.json 2>>gpurun_out/r03c.err
  cat gpurun_out/r03c_${C}_probe.json
  timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread --clock-control none -s 400 -c 120 --csv \
    --log-file gpurun_out/r03c_${C}_launches.csv python tools/config_probe.py $C > /dev/null 2>>gpurun_out/r03c.err
  echo "ncu $C exit $?"
done
