#!/bin/bash
# A/B timing of alternative builds of libwsgpu.so (tools/bin/libwsgpu_<tag>.so) on one workload.
mkdir -p gpurun_out
W=${W:-c3}
cp paper_2104_08265_b200/libwsgpu.so /tmp/libwsgpu_orig.so
for f in tools/bin/libwsgpu_*.so; do
  t=$(basename $f .so); cp $f paper_2104_08265_b200/libwsgpu.so
  for r in 1 2; do
    timeout 300 python bench.py --workload $W --steps ${STEPS:-5} --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', d['ms_per_step'])"
  done
done > gpurun_out/variants_$W.txt 2>&1
cp /tmp/libwsgpu_orig.so paper_2104_08265_b200/libwsgpu.so
cat gpurun_out/variants_$W.txt
