"""Time-domain vs row-FFT path on dense events (C5 1M depos): device time per
event after the workspace has grown (a host call re-runs on overflow)."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2104_08265_b200 import Context, Plane, SimConfig, simulate_event_device, simulate_events
from paper_2104_08265_b200.workloads import microboone_event, microboone_grids

for n in [int(a) for a in sys.argv[1:]] or [300_000, 1_000_000]:
    for path in ("direct", "fft", "auto"):
        ctx = Context(0)
        ctx.set_conv_path(path)
        grids, resps = microboone_grids()
        planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
        ev = microboone_event(n, seed=3)
        outs = [[np.empty(p.shape, np.float32) for p in planes]]
        simulate_events(ctx, planes, [ev], SimConfig(), frames=outs)  # grows the workspace
        dev = [torch.from_numpy(d.view(np.uint8)).cuda() for d in ev]
        frames = [torch.empty(p.shape, dtype=torch.float32, device="cuda") for p in planes]
        nn = [len(d) for d in ev]
        for _ in range(2):
            simulate_event_device(ctx, planes, dev, nn, SimConfig(), frames)
        ctx.synchronize()
        s = torch.cuda.ExternalStream(ctx.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            simulate_event_device(ctx, planes, dev, nn, SimConfig(), frames)
        e1.record(s)
        ctx.synchronize()
        print(f"{n} depos/plane, path {path}: {e0.elapsed_time(e1) / 5:.3f} ms/event")
        ctx.close()
