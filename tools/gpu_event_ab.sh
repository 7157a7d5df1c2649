#!/bin/bash
# A/B of library builds on the headline event's kernels (ncu launch times): tools/gpu_event_ab.sh <lib>... ("base" = in-tree)
for lib in "$@"; do
  if [ "$lib" = base ]; then L=""; else L="WS_GPU_LIB=$PWD/$lib"; fi
  env $L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 18 --csv --log-file /tmp/ab_ev.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python - "$lib" <<'PY'
import csv, io, sys
lines = [l for l in open('/tmp/ab_ev.csv').read().splitlines() if l.startswith('"')]
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines))) if r["Metric Name"] == "gpu__time_duration.sum"]
tot, cnt = {}, {}
for r in rows:
    k = r["Kernel Name"].split("(")[0].replace("void ", "").replace("wsb::", "")[:24]
    tot[k] = tot.get(k, 0) + float(r["Metric Value"].replace(",", ""))
    cnt[k] = cnt.get(k, 0) + 1
print(sys.argv[1], {k: round(v / cnt[k] / 1e3, 1) for k, v in tot.items()})
PY
done
