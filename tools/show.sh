#!/bin/bash
# summarize gpurun_out after gpu_iter.sh
cd "$(dirname "$0")/.."
grep -E "Error|assert |passed|failed" gpurun_out/pytest_gpu.log | head -5
for f in gpurun_out/bench.log gpurun_out/bench_k0.log; do echo $f; python -c "
import json
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],4), d['config'].get('stage_ms'), round(d['roofline']['frac'],3), d.get('e2e') and d['e2e']['ms_per_step'])
"; done
python - <<'PY'
import csv,collections
rows=[r for r in csv.reader(open('gpurun_out/launches.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki].split('(')[0].split('<')[0].replace('void ','')].append(float(r[vi]))
print(' | '.join(f"{k} {sum(v)/len(v)/1000:.1f}us" for k,v in agg.items()))
PY
[ -f gpurun_out/iter.ncu-rep ] && python tools/ncu_summary.py gpurun_out/iter.ncu-rep
