#!/bin/bash
# prime-factor core (C4 2047 = 23 x 89): parity, then C4 A/B vs Bluestein
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -x -q -k "pfa or golden or dst_engines or rader or C4" > gpurun_out/r02y_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02y_pytest.log; tail -15 gpurun_out/r02y_pytest.log
for round in 1 2; do for e in 1 0; do
  r=$(DBX_DST_PFA=$e timeout 300 python tools/config_probe.py C4 2>>gpurun_out/r02y.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'], d['best'])")
  echo "$round PFA=$e $r" | tee -a gpurun_out/r02y_ab.txt
done; done
