"""Device time of the MicroBooNE event with fluctuation on (C3: Philox, shaper on)."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2104_08265_b200 import Context, Plane, RngConfig, SimConfig, simulate_event_device
from paper_2104_08265_b200._lib import TimingC
from paper_2104_08265_b200.workloads import microboone_event, microboone_grids

ctx = Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
grids, resps = microboone_grids()
planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
ev = microboone_event(100_000, seed=1)
dev = [torch.from_numpy(d.view(np.uint8)).cuda() for d in ev]
n = [len(d) for d in ev]
frames = [torch.empty(p.shape, dtype=torch.float32, device="cuda") for p in planes]
for approx in (False, True):
    cfg = SimConfig(fluctuate=True, approx=approx, rng=RngConfig(mode="philox", seed=12345))
    for _ in range(3):
        simulate_event_device(ctx, planes, dev, n, cfg, frames)
    ctx.synchronize()
    t = TimingC()
    simulate_event_device(ctx, planes, dev, n, cfg, frames, timing=t)
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        simulate_event_device(ctx, planes, dev, n, cfg, frames)
    e1.record(stream)
    ctx.synchronize()
    print(f"fluct on (approx={approx}): {e0.elapsed_time(e1) / 10:.3f} ms/event; stages prepare {t.prepare_ms:.3f} "
          f"fluct {t.fluctuate_ms:.3f} bin {t.bin_ms:.3f} conv {t.convolve_ms:.3f}")
