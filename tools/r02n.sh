#!/bin/bash
# C++ row-slab loop: GPU tests (slab + full-size C5 slab parity), then C5 slab-run throughput at P=1 vs the single-image path
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_slab.py -m gpu -x -q > gpurun_out/r02n_slab.log 2>&1
echo "slab exit $?" >> gpurun_out/r02n_slab.log; tail -5 gpurun_out/r02n_slab.log
timeout 1200 python -m pytest tests/test_fullsize_parity.py -m gpu -x -q -k "c5" > gpurun_out/r02n_full.log 2>&1
echo "full exit $?" >> gpurun_out/r02n_full.log; tail -5 gpurun_out/r02n_full.log
timeout 600 python tools/slab_probe.py 1 > gpurun_out/r02n_probe.txt 2>&1; cat gpurun_out/r02n_probe.txt
timeout 600 python tools/slab_probe.py 2 >> gpurun_out/r02n_probe.txt 2>&1; tail -2 gpurun_out/r02n_probe.txt
