#!/bin/bash
# warp-owned separable row kernels (rows_tt_w, rows_t_axpy_w): GPU parity, then C3 A/B (DBX_WROWS=1/0)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C3 or fused or separable or batch or chunk" > gpurun_out/r02q_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02q_pytest.log; tail -3 gpurun_out/r02q_pytest.log
for round in 1 2; do
for e in 1 2 3 0; do
  r=$(DBX_WROWS=$e timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other-configs 2>>gpurun_out/r02q.err | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"],1), [(k["kernel"], round(k["avg_launch_ms"],4)) for k in r["kernels"][:6]])')
  echo "$round WROWS=$e $r" | tee -a gpurun_out/r02q_ab.txt
done
done
