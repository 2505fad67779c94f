#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_slab.py -m gpu -x -q > gpurun_out/r04l_slab.log 2>&1
echo "slab file exit $?"; tail -3 gpurun_out/r04l_slab.log
timeout 900 python -m pytest tests/test_reflective.py tests/test_semiconvergence.py tests/test_slab.py -m gpu -x -q > gpurun_out/r04l_slab3.log 2>&1
echo "3 files exit $?"; tail -3 gpurun_out/r04l_slab3.log
bash tools/r04j.sh
