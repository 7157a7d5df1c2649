mkdir -p gpurun_out
timeout 600 ncu --nvtx --nvtx-include "steady/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_c3_steady.csv python tools/c3_steady.py --events 2 > gpurun_out/r2c_c3s.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "steady/" --set full --import-source on --clock-control none -k "regex:k_fluct_walk|k_fluct_prep|k_fluctuate_exact" -c 3 -o gpurun_out/r2c_full_walk -f python tools/c3_steady.py --events 1 > gpurun_out/r2c_fw.log 2>&1
tail -3 gpurun_out/r2c_c3s.log gpurun_out/r2c_fw.log
