#!/bin/bash
# Transposed-store epilogue of D's row passes (DBX_DST_TOUT=1): GPU suite, A/B on C4/C5
set -u
mkdir -p gpurun_out
DBX_DST_TOUT=1 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r03g_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r03g_pytest.log; tail -3 gpurun_out/r03g_pytest.log
for round in 1 2; do for C in C4 C5; do for to in 1 0; do
  r=$(DBX_DST_TOUT=$to timeout 300 python tools/config_probe.py $C 2>>gpurun_out/r03g.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'])")
  echo "$round tout=$to $r" | tee -a gpurun_out/r03g_ab.txt
done; done; done
