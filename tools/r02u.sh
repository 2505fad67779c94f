#!/bin/bash
# measurement pass v55: fused-Bluestein CT A/B on C2, bench line, ncu launch list, six C3 kernels under ncu --set full
set -u
mkdir -p gpurun_out
for round in 1 2; do for lib in libdbx libdbx_fct; do
  r=$(DBX_LIB=paper_1211_0393_b200/$lib.so timeout 300 python tools/config_probe.py C2 2>>gpurun_out/r02u.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['mpx_it_s'],1), d['class_ms'])")
  echo "$round $lib $r" | tee -a gpurun_out/r02u_fct.txt
done; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02u_bench.json 2> gpurun_out/r02u_bench.err
echo "bench exit $?"; head -c 300 gpurun_out/r02u_bench.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02u_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/r02u_ncu_list.log 2>&1
echo "ncu list exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'cols_sep|rows_|dst_tcols' \
  -s 7 -c 6 -o gpurun_out/r02u_full64 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs \
  > gpurun_out/r02u_ncu_full.log 2>&1
echo "ncu full exit $?"
