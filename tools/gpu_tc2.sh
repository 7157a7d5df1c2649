#!/bin/bash
# k_conv_tc2 bring-up: its parity tests (both kernels), the C3 full-size tests, C3 timing
mkdir -p gpurun_out
T=${TAG:-tc2}
timeout 600 python -m pytest tests/test_gpu_conv_tc.py -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
tail -15 gpurun_out/${T}_tests.log
timeout 300 python tools/fluct_time.py > gpurun_out/${T}_fluct.log 2>&1
WS_CONV_TC2=0 timeout 300 python tools/fluct_time.py >> gpurun_out/${T}_fluct.log 2>&1
cat gpurun_out/${T}_fluct.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "c3 or C3" > gpurun_out/${T}_full.log 2>&1
tail -3 gpurun_out/${T}_full.log
