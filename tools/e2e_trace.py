"""Timeline of the end-to-end call (ws_run_events) for a workload: kernels and
copies from CUPTI via torch.profiler, to see what overlaps."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2104_08265_b200 import Context, Plane, RngConfig, SimConfig, run_events
from paper_2104_08265_b200.workloads import microboone_event, microboone_grids

fl = len(sys.argv) > 1 and sys.argv[1] == "c3"
ctx = Context(0)
grids, resps = microboone_grids()
planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
evs = []
for k in range(2):
    row = []
    for d in microboone_event(100_000, seed=1 + k):
        t = torch.empty(d.nbytes, dtype=torch.uint8).pin_memory()
        t.numpy()[:] = d.view(np.uint8)
        row.append(t.numpy().view(d.dtype))
    evs.append(row)
cfg = SimConfig(fluctuate=fl, rng=RngConfig(mode="philox", seed=12345))
bufs = [[torch.empty(p.shape, dtype=torch.uint16).pin_memory().numpy() for p in planes] for _ in range(2)]
batch = [evs[i % 2] for i in range(4)]
adcs = [bufs[i % 2] for i in range(4)]
run_events(ctx, planes, batch[:2], cfg, adc_type="u16", adcs=adcs[:2])
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run_events(ctx, planes, batch, cfg, adc_type="u16", adcs=adcs)
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev)
for e in sorted(ev, key=lambda e: e.time_range.start):
    d = e.time_range.end - e.time_range.start
    if d > 50 or "fluct" in e.name or "emset" in e.name or "Sort" in e.name or "noise" in e.name:
        print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms +{d / 1e3:7.3f}  {e.name[:60]}")
