#!/bin/bash
# last-block finalize in the fused residual kernels: GPU parity (fused + full-size C1-C3), A/B on C1/C2/C3
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py tests/test_experiment.py -m gpu -x -q -k "not c4 and not c5 and not C4 and not C5" > gpurun_out/r02x_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02x_pytest.log; tail -3 gpurun_out/r02x_pytest.log
for round in 1 2; do for e in 1 0; do
  for c in C1 C2; do
    r=$(DBX_FIN_FUSED=$e timeout 300 python tools/config_probe.py $c 2>>gpurun_out/r02x.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1))")
    echo "$round FIN_FUSED=$e $r" | tee -a gpurun_out/r02x_ab.txt
  done
  r=$(DBX_FIN_FUSED=$e timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other-configs 2>>gpurun_out/r02x.err | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))')
  echo "$round FIN_FUSED=$e C3 $r" | tee -a gpurun_out/r02x_ab.txt
done; done
