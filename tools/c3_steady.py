"""Steady-state C3 event (fluctuation on, Philox, shaper on) for launch lists:
warm-up events + synchronize (workspace sized), then --events events inside an
NVTX range "steady" (ncu --nvtx --nvtx-include steady/)."""
import argparse, sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2104_08265_b200 import Context, Plane, RngConfig, SimConfig, simulate_event_device
from paper_2104_08265_b200.workloads import microboone_event, microboone_grids

ap = argparse.ArgumentParser()
ap.add_argument("--events", type=int, default=2)
ap.add_argument("--approx", action="store_true")
a = ap.parse_args()
ctx = Context(0)
grids, resps = microboone_grids()
planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
ev = microboone_event(100_000, seed=1)
dev = [torch.from_numpy(d.view(np.uint8)).cuda() for d in ev]
n = [len(d) for d in ev]
frames = [torch.empty(p.shape, dtype=torch.float32, device="cuda") for p in planes]
cfg = SimConfig(fluctuate=True, approx=a.approx, rng=RngConfig(mode="philox", seed=12345))
for _ in range(3):
    simulate_event_device(ctx, planes, dev, n, cfg, frames)
    ctx.synchronize()
torch.cuda.nvtx.range_push("steady")
for _ in range(a.events):
    simulate_event_device(ctx, planes, dev, n, cfg, frames)
ctx.synchronize()
torch.cuda.nvtx.range_pop()
print("ok")
