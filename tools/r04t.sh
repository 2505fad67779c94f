#!/bin/bash
# C5 blur kernels (rows_sep_seg, cols_sep_real) under ncu --set full, summarised on the box
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'rows_sep_seg|cols_sep_real' -s 2 -c 4 -o /tmp/r04t_c5_blur -f \
  python tools/config_probe.py C5 0 1 1 > gpurun_out/r04t_full.log 2>&1
echo "ncu full exit $?"
python tools/ncu_excess.py /tmp/r04t_c5_blur.ncu-rep 10 > gpurun_out/r04t_c5_blur_excess.txt 2>&1
python tools/ncu_lines.py /tmp/r04t_c5_blur.ncu-rep rows_sep_seg 25 > gpurun_out/r04t_rows_sep_lines.txt 2>&1
ncu -i /tmp/r04t_c5_blur.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sectors_op_write.sum','lts__t_sectors_op_read.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum','l1tex__t_requests_pipe_lsu_mem_global_op_st.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum','launch__grid_size','launch__block_size','launch__shared_mem_per_block_dynamic','launch__occupancy_limit_shared_mem','launch__occupancy_limit_registers','sm__warps_active.avg.pct_of_peak_sustained_active']
for r in rows[2:]:
    print(r[h.index('Kernel Name')][:60])
    for w in want:
        if w in h: print('   ',w,r[h.index(w)], rows[1][h.index(w)])
" > gpurun_out/r04t_raw.txt 2>&1
