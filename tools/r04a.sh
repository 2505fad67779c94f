#!/bin/bash
# Transposed level-1 twiddle table (DBX_TW1T) for the warp-owned DFTs: parity subset, A/B on C3 and C1
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -x -q > gpurun_out/r04a_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r04a_pytest.log; tail -3 gpurun_out/r04a_pytest.log
bash tools/ab.sh r04a paper_1211_0393_b200/libdbx.so paper_1211_0393_b200/libdbx_notw1t.so
for round in 1 2; do for lib in libdbx libdbx_notw1t; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py C1 2>>gpurun_out/r04a.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), round(d['ms_per_run'],3), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r04a_c1.txt
done; done
