#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-tc2}
timeout 600 python -m pytest tests/test_gpu_conv_tc.py -x -q -p no:cacheprovider -k "past_2_11" > gpurun_out/${T}_tests.log 2>&1
tail -3 gpurun_out/${T}_tests.log
timeout 900 ncu --nvtx --nvtx-include "steady/" --set full --import-source on --clock-control none -k "regex:k_conv_tc" -c 1 -o gpurun_out/${T}_full -f python tools/c3_steady.py --events 1 > gpurun_out/${T}_prof.log 2>&1
tail -2 gpurun_out/${T}_prof.log
