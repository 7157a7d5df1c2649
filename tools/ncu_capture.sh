#!/bin/bash
# ncu --set full of selected kernels in one bench step: tools/ncu_capture.sh <regex> <count> <name>
mkdir -p gpurun_out
K=${1:-k_conv}; C=${2:-1}; NAME=${3:-prof}
shift 3
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -c $C -o gpurun_out/$NAME -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/$NAME.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$NAME.log
