#!/bin/bash
# padded per-warp line stride (bank-conflict-free CTA-cooperative reads) A/B on C3 + parity subset
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C3 or fused or separable or batch" > gpurun_out/r02ab_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02ab_pytest.log; tail -2 gpurun_out/r02ab_pytest.log
bash tools/ab.sh r02ab paper_1211_0393_b200/libdbx.so paper_1211_0393_b200/libdbx_nopad.so
