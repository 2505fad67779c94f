#!/bin/bash
# Session re-entry check: GPU suite + default bench line at HEAD.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v58_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v58_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/v58_pytest.log
tail -3 gpurun_out/v58_pytest.log
timeout 900 python bench.py > gpurun_out/v58_bench.json 2> gpurun_out/v58_bench.err
echo "bench exit $?"; head -c 600 gpurun_out/v58_bench.json
