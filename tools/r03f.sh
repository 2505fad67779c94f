#!/bin/bash
# TMA-staged DST fill: GPU suite, then A/B (staged vs not) on C4 and C5
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r03f_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r03f_pytest.log; tail -3 gpurun_out/r03f_pytest.log
for round in 1 2; do for C in C4 C5; do for lib in libdbx libdbx_ns; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py $C 2>>gpurun_out/r03f.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r03f_ab.txt
done; done; done
