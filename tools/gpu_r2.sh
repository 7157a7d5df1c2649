#!/bin/bash
# round-2 validation on the GPU box: tests, default bench, configs[3]/[4] workloads
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r2_tests.log 2>&1
tail -5 gpurun_out/r2_tests.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 3000 gpurun_out/r2_bench.json
for w in c4 c5; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err
  tail -c 1500 gpurun_out/r2_bench_$w.json; tail -3 gpurun_out/r2_bench_$w.err
done
