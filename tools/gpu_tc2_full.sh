#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-tc2f}
timeout 900 ncu --nvtx --nvtx-include "steady/" --set full --import-source on --clock-control none -k "regex:k_conv_tc" -c 1 -o gpurun_out/${T}_full -f python tools/c3_steady.py --events 1 > gpurun_out/${T}_prof.log 2>&1
tail -1 gpurun_out/${T}_prof.log
