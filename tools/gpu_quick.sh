#!/bin/bash
# Quick GPU iteration: gpu tests (optionally a subset) + bench + kappa sweep + launch list.
mkdir -p gpurun_out
T=${1:-tests}
timeout 1200 python -m pytest $T -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for k in 0 16 48 1000000; do WS_DIRECT_KAPPA=$k timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_k$k.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
tail -n 5 gpurun_out/pytest_gpu.log
