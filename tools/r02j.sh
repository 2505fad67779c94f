#!/bin/bash
# in-place Cooley-Tukey convolution core for the Rader/Bluestein DST lines: parity + C4/C5 probes
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02j_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02j_pytest.log; tail -3 gpurun_out/r02j_pytest.log
for c in C4 C5 C2 C1; do timeout 300 python tools/config_probe.py $c 2>>gpurun_out/r02j_probe.err | tee -a gpurun_out/r02j_probe.jsonl; done
