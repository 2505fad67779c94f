#!/bin/bash
# Split 33rd level-2 row (DBX_WROW33_SPLIT): parity subset, A/B on C3
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -x -q > gpurun_out/r04q_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r04q_pytest.log; tail -3 gpurun_out/r04q_pytest.log
bash tools/ab.sh r04q paper_1211_0393_b200/libdbx.so paper_1211_0393_b200/libdbx_r33off.so
