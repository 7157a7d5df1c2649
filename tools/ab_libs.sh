#!/bin/bash
# A/B timing of library builds on one bench workload: tools/ab_libs.sh <workload> <lib>... (path or "base")
mkdir -p gpurun_out
W=$1; shift
for lib in "$@"; do
  for r in 1 2; do
    if [ "$lib" = base ]; then L=""; else L="WS_GPU_LIB=$PWD/$lib"; fi
    env $L timeout 300 python bench.py --workload $W --steps ${STEPS:-20} --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), 'conv', round(d['roofline']['kernel_ms'],4), d['config']['stage_ms'])"
  done
done
