#!/bin/bash
# prime-factor lines in the fused pipeline (C2: 511 = 7 x 73): parity, then C2 A/B vs Bluestein 1024
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py tests/test_golden.py -m gpu -x -q -k "C2 or c2 or pfa or golden or fused or dst_engines" > gpurun_out/r02aa_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02aa_pytest.log; tail -15 gpurun_out/r02aa_pytest.log
for round in 1 2; do for e in 1 0; do
  r=$(DBX_DST_PFA=$e timeout 300 python tools/config_probe.py C2 2>>gpurun_out/r02aa.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), d['fused'], d['class_ms'], d['best'])")
  echo "$round PFA=$e $r" | tee -a gpurun_out/r02aa_ab.txt
done; done
