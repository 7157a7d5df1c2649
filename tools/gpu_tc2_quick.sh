#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-tc2q}
timeout 300 python tools/fluct_time.py > gpurun_out/${T}_fluct.log 2>&1
cat gpurun_out/${T}_fluct.log
timeout 600 ncu --nvtx --nvtx-include "steady/" --section SpeedOfLight --section MemoryWorkloadAnalysis --metrics smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:k_conv_tc" -c 1 -o gpurun_out/${T}_full -f python tools/c3_steady.py --events 1 > gpurun_out/${T}_prof.log 2>&1
ncu -i gpurun_out/${T}_full.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
for k,x in zip(h,v):
    if k in ('gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__inst_executed.sum','sm__warps_active.avg.pct_of_peak_sustained_active','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'): print(k,x)
"
