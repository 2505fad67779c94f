#!/bin/bash
# rows_sep_seg: all staging loads in flight before the stores — parity (separate-pass separable blur users), A/B on C5
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_slab.py tests/test_fullsize_parity.py tests/test_reflective.py -m gpu -x -q -k "not c3 and not c2 and not c4" > gpurun_out/r04u_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r04u_pytest.log; tail -3 gpurun_out/r04u_pytest.log
for round in 1 2; do for lib in libdbx libdbx_prev; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py C5 2>>gpurun_out/r04u.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r04u_ab.txt
done; done
