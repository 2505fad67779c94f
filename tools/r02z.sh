#!/bin/bash
# v57: full GPU suite (PFA core for C4) + bench line
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02z_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02z_pytest.log; tail -3 gpurun_out/r02z_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err
echo "bench exit $?"; head -c 300 gpurun_out/r02z_bench.json; echo
