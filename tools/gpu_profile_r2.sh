#!/bin/bash
# Round-2 profile set (run on the GPU box): full-size parity tests, bench
# lines (event, c3), ncu launch lists (event, c3) and --set full captures of
# the hot kernels of both (k_direct / k_gprof_umma / k_sample_off; the
# fluctuation-on walk and the mode-1 row FFT).
mkdir -p gpurun_out
T=${TAG:-r2a}
python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout 1200 > gpurun_out/${T}_fullsize.log 2>&1
tail -3 gpurun_out/${T}_fullsize.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --workload c3 --steps 5 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_b.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${T}_launches_c3.csv \
  python bench.py --workload c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_direct|k_gprof|k_sample" -c 3 \
  -o gpurun_out/${T}_full_direct -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full_direct.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:k_fluctuate_exact|k_conv" -c 2 \
  -o gpurun_out/${T}_full_c3 -f python bench.py --workload c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full_c3.log 2>&1
tail -2 gpurun_out/${T}_*.log
cat gpurun_out/${T}_bench.json gpurun_out/${T}_bench_c3.json | cut -c 1-600
