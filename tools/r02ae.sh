#!/bin/bash
# batched epilogue operand loads (dst_rows, conv_row_inv): parity subset, C4/C5 A/B
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_slab.py tests/test_cgls.py -m gpu -x -q > gpurun_out/r02ae_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02ae_pytest.log; tail -3 gpurun_out/r02ae_pytest.log
for round in 1 2; do for lib in libdbx libdbx_prev; do for c in C4 C5; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py $c 2>>gpurun_out/r02ae.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r02ae_ab.txt
done; done; done
