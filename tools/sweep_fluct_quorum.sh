mkdir -p gpurun_out
for q in 2 4 6 8 11; do
  WS_FLUCT_QUORUM=$q timeout 300 python bench.py --workload c3 --steps 5 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('q=$q', d['ms_per_step'])"
done > gpurun_out/sweep_q.txt 2>&1
cat gpurun_out/sweep_q.txt
