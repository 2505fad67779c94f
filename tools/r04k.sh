#!/bin/bash
set -u
mkdir -p gpurun_out
for lib in libdbx libdbx_padon libdbx_r6off; do
  DBX_LIB=paper_1211_0393_b200/$lib.so timeout 600 python -m pytest "tests/test_slab.py::test_slab_landweber_matches_single_image" -m gpu -x -q -k "8192" > gpurun_out/r04k_$lib.log 2>&1
  echo "$lib exit $?"; grep -n "assert\|passed\|failed" gpurun_out/r04k_$lib.log | head -5
done
