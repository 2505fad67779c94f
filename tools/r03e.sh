#!/bin/bash
# A/B of the C4 FFT row kernels at 3 CTAs/SM (register cap) vs the default 2
set -u
mkdir -p gpurun_out
for round in 1 2 3; do for lib in libdbx libdbx_cm3; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py C4 2>>gpurun_out/r03e.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r03e_ab.txt
done; done
