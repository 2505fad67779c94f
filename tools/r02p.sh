#!/bin/bash
# parity floor report: GPU vs FP64 oracle vs long-double oracle, best vs runner-up RRE margins
set -u
mkdir -p gpurun_out
timeout 2700 python tools/parity_report.py --ld-iters C5:3,C4:10 --out gpurun_out/r02p_parity_report.json > gpurun_out/r02p.log 2>&1
echo "report exit $?"; tail -8 gpurun_out/r02p.log
