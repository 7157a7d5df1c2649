#!/bin/bash
# k_direct_mma vs the round-1 kernel: direct-path parity tests and bench lines for both
mkdir -p gpurun_out
T=${TAG:-mma}
timeout 600 python -m pytest tests/test_gpu_direct.py tests/test_gpu_parity.py -q -p no:cacheprovider -x --timeout 600 > gpurun_out/${T}_tests.log 2>&1; tail -15 gpurun_out/${T}_tests.log
WS_DIRECT_MMA=0 timeout 300 python bench.py --no-e2e --no-cpu-baseline | cut -c 1-700
timeout 300 python bench.py --no-e2e --no-cpu-baseline | cut -c 1-700
