#!/bin/bash
# warp-owned kernels for C1's 256-point lines (W255) + templated W1023: parity, C1 probe, C3 A/B
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -m gpu -x -q -k "C1 or c1 or fused or separable or batch or C3" > gpurun_out/r02ag_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02ag_pytest.log; tail -3 gpurun_out/r02ag_pytest.log
for round in 1 2; do for lib in libdbx libdbx_prev; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py C1 2>>gpurun_out/r02ag.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r02ag_ab.txt
done; done
bash tools/ab.sh r02ag paper_1211_0393_b200/libdbx.so paper_1211_0393_b200/libdbx_prev.so
