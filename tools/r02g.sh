#!/bin/bash
# A/B of wdst variants on the C3 headline (interleaved, 2 rounds)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fullsize_parity.py -m gpu -x -q -k "c3 or C3" > gpurun_out/r02g_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02g_pytest.log; tail -2 gpurun_out/r02g_pytest.log
for round in 1 2; do
  for v in "libdbx.so 1" "libdbx_ri0.so 1" "libdbx_ri2.so 1" "libdbx.so 0"; do
    set -- $v
    r=$(DBX_WDST=$2 DBX_LIB=paper_1211_0393_b200/$1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other-configs 2>>gpurun_out/r02g_ab.err \
        | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k={e["kernel"]: round(e["avg_launch_ms"],4) for e in d["roofline"]["kernels"]}; print(round(d["value"],1), k.get("dst_tcols#2"))')
    echo "$round $1 wdst=$2 $r" | tee -a gpurun_out/r02g_ab.txt
  done
done
