#!/bin/bash
# A/B of library builds on the steady-state C3 kernels: tools/gpu_c3_ab.sh <lib>... ("base" = in-tree)
for lib in "$@"; do
  if [ "$lib" = base ]; then L=""; else L="WS_GPU_LIB=$PWD/$lib"; fi
  env $L timeout 600 ncu --nvtx --nvtx-include "steady/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/ab_c3.csv python tools/c3_steady.py --events 1 > /dev/null 2>&1
  python - "$lib" <<'PY'
import csv, io, sys
lines = [l for l in open('/tmp/ab_c3.csv').read().splitlines() if l.startswith('"')]
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines))) if r["Metric Name"] == "gpu__time_duration.sum"]
tot = {}
for r in rows:
    k = r["Kernel Name"].split("(")[0].replace("void ", "").replace("wsb::", "")[:28]
    tot[k] = tot.get(k, 0) + float(r["Metric Value"].replace(",", ""))
print(sys.argv[1], "total %.1f us" % (sum(tot.values()) / 1e3), {k: round(v / 1e3, 1) for k, v in tot.items() if v > 20000})
PY
done
