#!/bin/bash
set -u
mkdir -p gpurun_out
for round in 1 2; do for lib in libdbx libdbx_w2; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py C1 2>>gpurun_out/r02ah.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r02ah_ab.txt
done; done
