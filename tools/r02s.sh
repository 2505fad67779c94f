#!/bin/bash
# dst_tcols_w CTA-staged 64-byte row stores vs per-warp 16-byte stores (C3 A/B, interleaved)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C3 or fused or separable or batch" > gpurun_out/r02s_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02s_pytest.log; tail -2 gpurun_out/r02s_pytest.log
bash tools/ab.sh r02s paper_1211_0393_b200/libdbx.so paper_1211_0393_b200/libdbx_nocs.so
for lib in libdbx libdbx_nocs; do for c in C1 C2; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py $c 2>>gpurun_out/r02s.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), d['class_ms'])")
  echo "$lib $r" | tee -a gpurun_out/r02s_probe.txt
done; done
