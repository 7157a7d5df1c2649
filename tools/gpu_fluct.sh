#!/bin/bash
# Fluctuation iteration: the fluctuation parity tests, the C3 bench line, a
# launch list and a full capture of the walk kernels.
mkdir -p gpurun_out
T=${TAG:-fl}
timeout 900 python -m pytest tests/test_gpu_fluct_walk.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_overflow.py tests/test_gpu_configs.py tests/test_gpu_impacts.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
tail -3 gpurun_out/${T}_tests.log
timeout 600 python bench.py --workload c3 --steps 5 --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
tail -c 600 gpurun_out/${T}_bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${T}_launches_c3.csv \
  python bench.py --workload c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_fluct_prep|k_fluct_walk" -c 2 \
  -o gpurun_out/${T}_full_c3 -f python bench.py --workload c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full_c3.log 2>&1
ls gpurun_out | grep ${T}
