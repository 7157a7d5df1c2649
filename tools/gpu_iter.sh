#!/bin/bash
# iteration: gpu tests + bench (direct / fft) + launch list + ncu full of the prep + conv kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
WS_DIRECT_KAPPA=0 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_k0.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
bash tools/ncu_capture.sh "${1:-k_direct|k_gprof|k_sample|k_fill}" ${2:-4} iter
