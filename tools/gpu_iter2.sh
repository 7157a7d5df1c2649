#!/bin/bash
# Iteration on the GPU box: the given test files, one bench workload, a launch
# list of it and a full capture of the kernels matching $K.
#   TAG=x TESTS="tests/a.py tests/b.py" W=c3 K="k_conv_tc" bash tools/gpu_iter2.sh
mkdir -p gpurun_out
T=${TAG:-it}; W=${W:-c3}; K=${K:-k_conv_tc}
timeout 900 python -m pytest ${TESTS:-tests} -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
tail -3 gpurun_out/${T}_tests.log
timeout 600 python bench.py --workload $W --steps 5 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --workload $W --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -c 2 \
  -o gpurun_out/${T}_full -f python bench.py --workload $W --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full.log 2>&1
ls gpurun_out | grep ${T}_
