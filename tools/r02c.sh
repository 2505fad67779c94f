#!/bin/bash
# Round-2 call C: parity of the DMMA radix-31 stage and the DMMA dense GEMM,
# then A/B against the SIMT stage on the headline, and the C1/C2 dense probe.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -x -q > gpurun_out/r02c_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02c_pytest.log; tail -3 gpurun_out/r02c_pytest.log
bash tools/ab.sh r02c paper_1211_0393_b200/libdbx.so paper_1211_0393_b200/libdbx_nodmma.so
for c in C1 C2; do for dst in 0 1; do timeout 300 python tools/config_probe.py $c 0 1 3 $dst >> gpurun_out/r02c_probe.jsonl 2>>gpurun_out/r02c_probe.err; done; done
cat gpurun_out/r02c_probe.jsonl
