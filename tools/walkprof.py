"""Setup vs walk cycles and lane occupancy of k_fluct_walk: build with
  bash tools/build_variant_all.sh wprof -DWS_WALK_PROF
and run with WS_GPU_LIB=$PWD/tools/bin/libwsgpu_wprof.so (prints per-event totals over all warps)."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2104_08265_b200 import Context, Plane, RngConfig, SimConfig, simulate_event_device, _lib
from paper_2104_08265_b200.workloads import microboone_event, microboone_grids

ctx = Context(0)
grids, resps = microboone_grids()
planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
ev = microboone_event(100_000, seed=1)
dev = [torch.from_numpy(d.view(np.uint8)).cuda() for d in ev]
n = [len(d) for d in ev]
frames = [torch.empty(p.shape, dtype=torch.float32, device="cuda") for p in planes]
cfg = SimConfig(fluctuate=True, rng=RngConfig(mode="philox", seed=12345))
for _ in range(2):
    simulate_event_device(ctx, planes, dev, n, cfg, frames)
    ctx.synchronize()
lib = _lib.load()
lib.wsb_walk_prof_dump()
simulate_event_device(ctx, planes, dev, n, cfg, frames)
ctx.synchronize()
lib.wsb_walk_prof_dump()
