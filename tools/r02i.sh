#!/bin/bash
# PDL: full GPU suite with programmatic dependent launches, then A/B on/off
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02i_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02i_pytest.log; tail -3 gpurun_out/r02i_pytest.log
for pdl in 1 0; do
  for c in C1 C2 C4 C5; do DBX_PDL=$pdl timeout 300 python tools/config_probe.py $c 2>>gpurun_out/r02i_probe.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$pdl', d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3))" | tee -a gpurun_out/r02i_ab.txt; done
  r=$(DBX_PDL=$pdl timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other-configs 2>>gpurun_out/r02i_ab.err | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],2))')
  echo "pdl=$pdl C3 $r" | tee -a gpurun_out/r02i_ab.txt
done
