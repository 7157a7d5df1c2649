#!/bin/bash
# C3 subset of the round's profile set (after a fluctuation-only change): GPU
# suite, the C3 bench line, the steady-state C3 launch list and --set full
# capture of the walk, its record pass and k_conv_tc2.
mkdir -p gpurun_out
T=${TAG:-r2i}
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/${T}_tests.log 2>&1
tail -3 gpurun_out/${T}_tests.log
timeout 900 python bench.py --workload c3 --steps 5 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 600 ncu --nvtx --nvtx-include "steady/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv \
  python tools/c3_steady.py --events 2 > gpurun_out/${T}_ncu_c3.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "steady/" --set full --import-source on --clock-control none -k "regex:k_fluct_walk|k_fluct_prep|k_conv_tc2" -c 3 \
  -o gpurun_out/${T}_full_c3 -f python tools/c3_steady.py --events 1 > gpurun_out/${T}_full_c3.log 2>&1
ls gpurun_out/ | grep ${T} | wc -l
