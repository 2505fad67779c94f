#!/bin/bash
# fused T~ d T row pass + L2 prefetch: GPU parity, then C4/C5 A/B
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02m_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02m_pytest.log; tail -3 gpurun_out/r02m_pytest.log
for round in 1 2; do
for env in "DBX_DST_TDT=1 DBX_DST_PF=0" "DBX_DST_TDT=1 DBX_DST_PF=1" "DBX_DST_TDT=0 DBX_DST_PF=0"; do
  for c in C4 C5; do
    r=$(env $env timeout 300 python tools/config_probe.py $c 2>>gpurun_out/r02m.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'])")
    echo "$round $env $r" | tee -a gpurun_out/r02m_ab.txt
  done
done
done
