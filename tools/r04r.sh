#!/bin/bash
# Element-major kernel spectrum for the 8190-point CT product pass (DBX_CT_KT): C5 parity + goldens, A/B on C5
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_golden.py tests/test_fullsize_parity.py -m gpu -x -q -k "golden or c5" > gpurun_out/r04r_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r04r_pytest.log; tail -3 gpurun_out/r04r_pytest.log
for round in 1 2; do for lib in libdbx libdbx_ktoff; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py C5 2>>gpurun_out/r04r.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r04r_ab.txt
done; done
