#!/bin/bash
# full GPU suite at HEAD + fresh C5 kernel profile summarised on the box
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04i_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r04i_pytest.log; tail -3 gpurun_out/r04i_pytest.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'dst_rows' -s 3 -c 3 -o /tmp/r04i_c5_full -f \
  python tools/config_probe.py C5 0 1 1 > gpurun_out/r04i_full.log 2>&1
echo "ncu full exit $?"
python tools/ncu_excess.py /tmp/r04i_c5_full.ncu-rep 14 > gpurun_out/r04i_c5_excess.txt 2>&1
python tools/ncu_lines.py /tmp/r04i_c5_full.ncu-rep dst_rows 30 > gpurun_out/r04i_c5_lines.txt 2>&1
