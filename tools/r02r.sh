#!/bin/bash
# full GPU suite after the warp-owned row kernels + C++ face changes
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02r_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02r_pytest.log; tail -22 gpurun_out/r02r_pytest.log
