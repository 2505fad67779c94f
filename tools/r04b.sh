#!/bin/bash
# Per-warp line stride pad 2 (DBX_WSTRIDE_PAD=2): A/B on C3
set -u
mkdir -p gpurun_out
bash tools/ab.sh r04b paper_1211_0393_b200/libdbx.so paper_1211_0393_b200/libdbx_pad2.so
