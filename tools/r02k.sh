#!/bin/bash
# A/B of the CT core variants on C4/C5 (config_probe, graph path)
set -u
mkdir -p gpurun_out
for round in 1 2; do
for lib in libdbx libdbx_ct8 libdbx_stock libdbx_t1024; do
  for c in C4 C5; do
    r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py $c 2>>gpurun_out/r02k.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'])")
    echo "$round $lib $r" | tee -a gpurun_out/r02k_ab.txt
  done
done
done
