#!/bin/bash
# One GPU-box pass: parity tests, the default bench line, the ncu launch list of
# the same command, and one `--set full` capture of the fused iteration's six
# kernels.  Usage (from the repo root, under gpurun): tools/gpu_round.sh TAG [skip-tests]
set -u
TAG=${1:-v}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "${2:-}" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
  tail -3 gpurun_out/${TAG}_pytest.log
fi
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?"; cat gpurun_out/${TAG}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs \
  > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'conv_col|cols_sep|rows_|dst_tcols' \
  -s 7 -c 6 -o gpurun_out/${TAG}_full -f python bench.py --images 8 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?"
