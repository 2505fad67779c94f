#!/bin/bash
# cols_sep_real residual mode with hoisted g loads (C5 separate passes): parity subset + C5 probe
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_slab.py -m gpu -x -q -k "separable or C5 or slab or cpp" > gpurun_out/r02af_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02af_pytest.log; tail -2 gpurun_out/r02af_pytest.log
for round in 1 2; do
  r=$(timeout 300 python tools/config_probe.py C5 2>>gpurun_out/r02af.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), d['class_ms'])")
  echo "$round $r" | tee -a gpurun_out/r02af_probe.txt
done
