#!/bin/bash
# Round-2 profile set (run on the GPU box): the GPU test suite, bench lines
# (event with CPU baseline, c1, c3, c4, c5), ncu launch lists (event, steady-state
# c3) and --set full captures of the hot kernels (k_direct / k_gprof_umma2 /
# k_sample_off; the fluctuation walk, its record pass and k_conv_tc2).
mkdir -p gpurun_out
T=${TAG:-r2d}
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/${T}_tests.log 2>&1
tail -3 gpurun_out/${T}_tests.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --workload c1 --steps 10 > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
timeout 900 python bench.py --workload c3 --steps 5 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 900 python bench.py --workload c4 --steps 5 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
for n in 1000 10000 100000 1000000; do
  timeout 900 python bench.py --workload c5 --depos $n --steps 3 --no-cpu-baseline > gpurun_out/${T}_bench_c5_$n.json 2> gpurun_out/${T}_bench_c5_$n.err
done
timeout 600 python bench.py --workload sigproc > gpurun_out/${T}_bench_sigproc.json 2> gpurun_out/${T}_bench_sigproc.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_b.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "steady/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv \
  python tools/c3_steady.py --events 2 > gpurun_out/${T}_ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_direct|k_gprof|k_sample" -c 3 \
  -o gpurun_out/${T}_full_direct -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full_direct.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "steady/" --set full --import-source on --clock-control none -k "regex:k_fluct_walk|k_fluct_prep|k_conv_tc2" -c 3 \
  -o gpurun_out/${T}_full_c3 -f python tools/c3_steady.py --events 1 > gpurun_out/${T}_full_c3.log 2>&1
ls -la gpurun_out/ | grep ${T} | wc -l
