#!/bin/bash
# GPU suite twice more (order-dependent race check after the slab.py / _ptr fix) + refreshed traffic capture
set -u
mkdir -p gpurun_out
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04p_pytest$i.log 2>&1
  echo "pytest $i exit $?"; tail -1 gpurun_out/r04p_pytest$i.log
done
timeout 1500 ncu --set full --clock-control none -k regex:'cols_sep|rows_|dst_tcols' \
  -s 7 -c 6 -o /tmp/v60b_full64 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs \
  > gpurun_out/r04p_ncu_full.log 2>&1
echo "ncu full exit $?"
python tools/ncu_traffic.py /tmp/v60b_full64.ncu-rep 64 gpurun_out/r04p_ncu_traffic.json > gpurun_out/r04p_traffic.log 2>&1; tail -8 gpurun_out/r04p_traffic.log
