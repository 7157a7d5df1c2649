#!/bin/bash
# Round profile set: bench line, ncu launch list of the bench, ncu --set full of
# each hot kernel (direct path; plus k_conv on the forced row-FFT path).
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_direct|k_gprof|k_sample|k_fill|k_scan" -c 5 \
  -o gpurun_out/full_direct -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/full_direct.log 2>&1
WS_DIRECT_KAPPA=0 timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_conv" -c 1 \
  -o gpurun_out/full_fft -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/full_fft.log 2>&1
tail -2 gpurun_out/*.log
