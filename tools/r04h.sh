#!/bin/bash
# Radix-6 last level of the in-place CT core (8190 = 13.7.15.6): C5 parity + goldens, A/B on C5
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_golden.py tests/test_fullsize_parity.py tests/test_gpu_parity.py -m gpu -x -q -k "golden or c5 or rader or 8190 or ct_core or core" > gpurun_out/r04h_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r04h_pytest.log; tail -3 gpurun_out/r04h_pytest.log
for round in 1 2; do for lib in libdbx libdbx_r6off; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py C5 2>>gpurun_out/r04h.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r04h_ab.txt
done; done
