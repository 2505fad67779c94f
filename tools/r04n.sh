#!/bin/bash
# Final measurement pass v60: GPU suite, smoke, bench line, reference arm, ncu launch list,
# six C3 kernels under ncu --set full at the benched 64 images (summarised on the box)
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v60_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v60_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/v60_pytest.log; tail -3 gpurun_out/v60_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v60_smoke.log 2>&1; tail -1 gpurun_out/v60_smoke.log
timeout 900 python bench.py > gpurun_out/v60_bench.json 2> gpurun_out/v60_bench.err
echo "bench exit $?"; head -c 400 gpurun_out/v60_bench.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/v60_bench_ref.json 2> gpurun_out/v60_bench_ref.err
echo "reference arm exit $?"; head -c 600 gpurun_out/v60_bench_ref.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v60_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/v60_ncu_list.log 2>&1
echo "ncu list exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'cols_sep|rows_|dst_tcols' \
  -s 7 -c 6 -o /tmp/v60_full64 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs \
  > gpurun_out/v60_ncu_full.log 2>&1
echo "ncu full exit $?"
python tools/ncu_traffic.py /tmp/v60_full64.ncu-rep 64 gpurun_out/v60_ncu_traffic.json > gpurun_out/v60_traffic.log 2>&1
python tools/ncu_summary.py /tmp/v60_full64.ncu-rep gpurun_out/v60_launches.csv > gpurun_out/v60_ncu_summary.md 2>gpurun_out/v60_summary.err
python tools/ncu_excess.py /tmp/v60_full64.ncu-rep 6 > gpurun_out/v60_c3_excess.txt 2>&1
