#!/bin/bash
# Round-2 call D: full GPU suite (new: device synthesis, oracle-checked sweep
# with reflective cells + PGMs, semiconvergence) and the default bench line.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02d_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02d_pytest.log; tail -22 gpurun_out/r02d_pytest.log
timeout 900 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
echo "bench exit $?"; python -c "
import json; d=json.load(open('gpurun_out/r02d_bench.json')); print(d['value'], d['e2e']['value']); print(json.dumps(d['other_configs']))"
