#!/bin/bash
# Final measurement pass v62: GPU suite, smoke, bench line, ncu launch list
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v62_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v62_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/v62_pytest.log; tail -3 gpurun_out/v62_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v62_smoke.log 2>&1; tail -1 gpurun_out/v62_smoke.log
timeout 900 python bench.py > gpurun_out/v62_bench.json 2> gpurun_out/v62_bench.err
echo "bench exit $?"; head -c 400 gpurun_out/v62_bench.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v62_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/v62_ncu_list.log 2>&1
echo "ncu list exit $?"
